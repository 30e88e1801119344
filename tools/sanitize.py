"""Every kernel of the library at small shapes, for compute-sanitizer:

    compute-sanitizer --tool memcheck  python tools/sanitize.py
    compute-sanitizer --tool racecheck python tools/sanitize.py --quick
    compute-sanitizer --tool synccheck python tools/sanitize.py --quick
    compute-sanitizer --tool initcheck python tools/sanitize.py --quick

Covers K1 block statistics, K1c block norms (d 128 and the paired d 64
kernel), K2a/K2b routing (tile, streamed and one-launch select from N = 516),
K2c/K2d pairing (forced on), K3 in every variant,
ragged lengths, the query-range entry point and the chunked host path. The
outputs are only checked for finiteness here; parity lives in tests/."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_01077_b200 as P  # noqa: E402


def rnd(shape, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(shape, generator=g, device="cuda", dtype=torch.bfloat16)


def main():
    quick = "--quick" in sys.argv
    ctx = P.Context.get(0)
    shapes = [(1, 2, 1000, 128), (1, 2, 777, 64)] if quick else \
        [(1, 2, 1000, 128), (2, 3, 1601, 128), (1, 2, 777, 64), (1, 1, 64, 128), (1, 1, 65, 64)]
    variants = [P.PisaVariant.Hybrid] if quick else list(P.PisaVariant)
    n = 0
    for si, (B, H, L, d) in enumerate(shapes):
        q, k, v = (rnd((B, H, L, d), 3 * si + i) for i in range(3))
        for pairing in (0, 2):
            ctx.set_pairing(pairing)
            for router in (P.RouterStrategy.Plain, P.RouterStrategy.CovarianceAware):
                for var in variants:
                    try:
                        out = P.fwd(q, k, v, sparsity=0.75, variant=var, router=router, ctx=ctx,
                                    out_dtype=torch.float32)
                    except P.Unsupported:  # BlockFirst has no CUDA path
                        continue
                    assert torch.isfinite(out).all(), (B, H, L, d, pairing, router, var)
                    n += 1
        Nq = (L + 63) // 64
        if Nq >= 3:
            out = torch.zeros((B, H, L, d), device="cuda", dtype=torch.bfloat16)
            P.fwd(q, k, v, out, sparsity=0.75, ctx=ctx, q_blocks=(1, Nq))
            n += 1
    ctx.set_pairing(1)
    # N >= 512 key blocks: K1's k_bar split, the streamed select (pipelined
    # scoring + top-k) and the one-launch select (sparsity 0.98 keeps K3 short)
    for si, d in enumerate((128, 64)):
        q, k, v = (rnd((1, 1, 33000, d), 50 + 3 * si + i) for i in range(3))
        for mode in ("stream", "1"):
            if mode == "1":
                os.environ["PISA_B200_FUSED_SELECT"] = "1"
            for router in (P.RouterStrategy.Plain, P.RouterStrategy.CovarianceAware):
                out = P.fwd(q, k, v, sparsity=0.98, router=router, ctx=ctx, out_dtype=torch.float32)
                assert torch.isfinite(out).all(), (d, mode, router)
                n += 1
            os.environ.pop("PISA_B200_FUSED_SELECT", None)
    B, H, L, d = 1, 5, 1000, 128
    hq, hk, hv = (rnd((B, H, L, d), 100 + i).cpu().pin_memory() for i in range(3))
    ho = torch.empty((B, H, L, d), dtype=torch.bfloat16).pin_memory()
    P.fwd_host(hq, hk, hv, ho, ctx=ctx, sparsity=0.75)
    assert torch.isfinite(ho.float()).all()
    n += 1
    torch.cuda.synchronize()
    print(f"sanitize driver: {n} calls ok")


if __name__ == "__main__":
    main()
