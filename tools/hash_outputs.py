"""Prints a hash of the forward's outputs (and the fused kernel's tile count)
for a few shapes with overlap-aware pairing forced on: run it against two
builds (PISA_B200_LIB=...) to show that a change only moved time, not bits."""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_01077_b200 as P  # noqa: E402


def main():
    ctx = P.Context.get(0)
    ctx.set_pairing(2)
    for (H, L, d, r, kind) in [(4, 75600, 128, 0.85, "gaussian"), (2, 118800, 128, 0.875, "clustered"),
                               (3, 33000, 64, 0.75, "clustered"), (24, 4608, 128, 0.85, "gaussian")]:
        gen = P.gen_gaussian if kind == "gaussian" else P.gen_clustered
        q, k, v = (x.reshape(1, H, L, d).cuda() for x in gen(11, H, L, d))
        ctx.set_profiling(True)
        ctx.fused_tiles()
        o = P.fwd(q, k, v, sparsity=r)
        torch.cuda.synchronize()
        tiles = ctx.fused_tiles()
        ctx.set_profiling(False)
        h = hashlib.sha256(o.view(torch.int16).cpu().numpy().tobytes()).hexdigest()[:16]
        print(f"H={H} L={L} d={d} r={r} {kind}: tiles={tiles} out={h}")
        del q, k, v, o
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
