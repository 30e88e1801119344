"""Generates tests/golden/*.npz from the UNMODIFIED reference library
(oracle/_ref/libpisa_ref.so, compiled from /root/reference by oracle/Makefile).

Run in the dev container (where /root/reference exists):
    python tests/golden/make_golden.py
The fixtures travel with the repo, so the GPU box can pin the oracle without
/root/reference. Each case stores the bf16-rounded inputs, the reference plan,
prepare products and outputs of pisa_multihead (Hybrid / Zeroth / SparseOnly /
GlobalCentroid, streaming where the reference offers it), and the covariance-aware
router's norms M_j, plan and Hybrid output.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402

CASES = [
    # name, kind, seed, H, L, d, r, force_diagonal
    ("clustered_h2_l512_d64", "clustered", 0, 2, 512, 64, 0.75, False),
    ("gaussian_h1_l1024_d64", "gaussian", 1, 1, 1024, 64, 0.875, False),
    ("clustered_h1_l768_d128_diag", "clustered", 2, 1, 768, 128, 0.5, True),
]


def main():
    for name, kind, seed, H, L, d, r, fd in CASES:
        q, k, v = O.ref_gen(kind, seed, H, L, d)
        q, k, v = (O.round_bf16(x) for x in (q, k, v))
        rec = dict(q=q, k=k, v=v, r=np.float64(r), force_diagonal=np.int32(fd))
        for variant in ("hybrid", "zeroth", "sparse_only", "global_centroid"):
            res = O.ref_multihead(q, k, v, r=r, variant=variant, force_diagonal=fd,
                                  accum_f64=True, streaming=(variant == "hybrid"))
            rec[f"out_{variant}"] = res["out"]
            rec[f"denom_{variant}"] = res["denom"]
            rec[f"ell_tail_{variant}"] = res["ell_tail"]
            rec["selected"] = res["selected"]
            rec["topk"] = np.int64(res["k"])
        # covariance-aware router (select_topk_covariance + spectral norms)
        res = O.ref_multihead(q, k, v, r=r, variant="hybrid", force_diagonal=fd, accum_f64=True,
                              streaming=True, router="covariance")
        rec["out_hybrid_cov"] = res["out"]
        rec["selected_cov"] = res["selected"]
        rec["m_norms"] = np.stack([O.ref_block_norms(k[h], v[h]) for h in range(H)])
        stats = [O.ref_block_stats(q[h], k[h], v[h]) for h in range(H)]
        rec["k_bar"] = np.stack([s[0] for s in stats])
        rec["v_hat"] = np.stack([s[1] for s in stats])
        rec["h_bar"] = np.stack([s[2] for s in stats])
        rec["q_bar"] = np.stack([s[3] for s in stats])
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **rec)
        print("wrote", name)
    # RNG golden sequence and sparsity_to_k table straight from the reference
    u = np.empty(8, np.uint64)
    O.ref().ref_rng_u64(42, u, 8)
    g = np.empty(8)
    O.ref().ref_rng_gaussian(0, g, 8)
    np.savez(os.path.join(HERE, "rng.npz"), u64_seed42=u, gauss_seed0=g)
    print("wrote rng")


if __name__ == "__main__":
    main()
