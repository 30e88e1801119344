"""Step-by-step GPU diagnostics: MMA self test, then K1 / K2 / K3 against the oracle.
Prints a line per check; exits non-zero on the first hard failure."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2602_01077_b200 as P  # noqa: E402


def bf(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).cuda()


def main():
    torch.manual_seed(0)
    print("device", torch.cuda.get_device_name(0), flush=True)
    # ---- MMA self test
    a = (torch.randn(128, 128) * 0.5).to(torch.bfloat16)
    b = (torch.randn(128, 128) * 0.5).to(torch.bfloat16)
    out = P.selftest_mma(a.cuda(), b.cuda()).cpu()
    torch.cuda.synchronize()
    A, B = a.float(), b.float()
    refs = [A @ B[:64].T, A[:64].T @ B[:64], A[:, :64] @ B[:64], A @ B]
    cols = [64, 128, 128, 128]
    names = ["SS K-major (QK^T)", "SS MN-major (K^T V)", "TS (P V)", "SS K/MN (Q Hbar)"]
    ok_all = True
    for i in range(4):
        got = out[i, :, :cols[i]]
        err = (got - refs[i]).abs().max().item()
        ok = err < 1e-2
        ok_all &= ok
        print(f"selftest {names[i]}: max err {err:.3e} {'OK' if ok else 'FAIL'}", flush=True)
        if not ok:
            print("  got[0,:8]", got[0, :8].tolist())
            print("  ref[0,:8]", refs[i][0, :8].tolist())
            # look for a transposition
            print("  err vs transposed ref", (got - refs[i][:, :cols[i]].T[:got.shape[0], :got.shape[1]]).abs().max().item() if refs[i].shape[0] == refs[i].shape[1] else "n/a")
    if not ok_all:
        print("SELFTEST FAILED")
    # ---- K1 / K2 / K3 per shape
    for (kind, H, L, d, r) in [("gaussian", 2, 1024, 128, 0.75), ("clustered", 2, 1024, 64, 0.75),
                               ("gaussian", 1, 1000, 128, 0.5), ("clustered", 2, 2048, 128, 0.875)]:
        q, k, v = O.gen(kind, 0, H, L, d)
        qt, kt, vt = bf(q), bf(k), bf(v)
        t0 = time.time()
        st = P.compute_prepare(qt, kt, vt)
        torch.cuda.synchronize()
        kb = st.k_bar[0].cpu().numpy(); vh = st.v_hat[0].cpu().numpy()
        qb = st.q_bar[0].cpu().numpy(); hb = st.h_bar[0].cpu().numpy()
        e = {"kbar": 0, "vhat": 0, "qbar": 0, "hbar": 0}
        for h in range(H):
            okb, ovh, ohb, _ = O.block_stats(k[h], v[h])
            oqb = O.query_means(q[h])
            e["kbar"] = max(e["kbar"], np.abs(kb[h] - okb).max())
            e["vhat"] = max(e["vhat"], np.abs(vh[h] - ovh).max())
            e["qbar"] = max(e["qbar"], np.abs(qb[h] - oqb).max())
            e["hbar"] = max(e["hbar"], np.abs(hb[h] - ohb).max() / max(1e-30, np.abs(ohb).max()))
        print(f"[{kind} H={H} L={L} d={d}] K1 errs " + " ".join(f"{n}={x:.2e}" for n, x in e.items()),
              f"({time.time()-t0:.2f}s)", flush=True)
        N = (L + 63) // 64
        kk, _ = O.sparsity_to_k(r, N)
        scale = 1 / np.sqrt(d)
        sel = P.select_topk_plain(st.q_bar[0], st.k_bar[0], kk, scale).cpu().numpy()
        mism = 0
        for h in range(H):
            okb, ovh, ohb, okg = O.block_stats(k[h], v[h])
            oqb = O.query_means(q[h])
            osel = O.select_plain(oqb, okb, kk, scale)
            mism += int((np.sort(sel[h], 1) != osel).any(1).sum())
        print(f"   K2 rows with index-set mismatch: {mism} / {H*N}", flush=True)
        for variant in ["hybrid", "zeroth", "sparse_only"]:
            o, ex = P.fwd(qt.unsqueeze(0), kt.unsqueeze(0), vt.unsqueeze(0), sparsity=r,
                          variant=P.PisaVariant[{"hybrid": "Hybrid", "zeroth": "Zeroth", "sparse_only": "SparseOnly"}[variant]],
                          out_dtype=torch.float32, diagnostics=True, return_plan=True)
            torch.cuda.synchronize()
            og = o[0].cpu().numpy()
            gsel = ex["selected"][0].cpu().numpy()
            worst = 0; cosmin = 1
            for h in range(H):
                stt = O.block_stats(k[h], v[h])
                ref, rm, ell, et = O.pisa_attention(q[h], k[h], v[h], gsel[h], stt, scale, variant)
                err = np.abs(og[h] - ref).max()
                cos = (og[h] * ref).sum() / np.sqrt((og[h] ** 2).sum() * (ref ** 2).sum())
                worst = max(worst, err); cosmin = min(cosmin, cos)
            print(f"   K3 {variant}: max abs {worst:.3e} cos {cosmin:.6f} "
                  f"{'OK' if worst < 2e-2 and cosmin > 0.999 else 'FAIL'}", flush=True)
    print("DONE")


if __name__ == "__main__":
    main()
