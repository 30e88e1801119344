"""Per-kernel device time of the fused forward at a BASELINE workload for the
plain and covariance-aware routers (CUDA events through the C ABI).
Usage: python tools/time_router.py [H] [L] [d]"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_01077_b200 as P  # noqa: E402


def main():
    H = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 75600
    d = int(sys.argv[3]) if len(sys.argv) > 3 else 128
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v = (torch.randn((1, H, L, d), generator=g, device=dev, dtype=torch.bfloat16) for _ in range(3))
    ctx = P.Context.get(0)
    names = P.kernel_names()
    for router in (P.RouterStrategy.Plain, P.RouterStrategy.CovarianceAware):
        kw = dict(sparsity=0.875, router=router, epsilon=1e-6)
        for _ in range(2):
            P.fwd(q, k, v, **kw)
        torch.cuda.synchronize()
        ctx.lib.pisa_b200_set_profiling(ctx.handle, 1)
        steps = 5
        for _ in range(steps):
            P.fwd(q, k, v, **kw)
        ms = (C.c_double * 8)()
        n = (C.c_int64 * 8)()
        ctx.lib.pisa_b200_read_profile(ctx.handle, ms, n)
        ctx.lib.pisa_b200_set_profiling(ctx.handle, 0)
        per = {names[i]: round(ms[i] / steps, 3) for i in range(len(names)) if n[i]}
        print(router.name, f"total {sum(per.values()):.3f} ms", per)


if __name__ == "__main__":
    main()
