"""Pipeline timeline of one fused-kernel CTA (needs the PISA_TRACE build:
PISA_B200_LIB=.../libpisa_b200_trace.so). Prints per-role timestamps (cycles).

    python tools/trace_timeline.py [H] [gaussian|clustered]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PISA_B200_LIB", os.path.join(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__))), "paper_2602_01077_b200", "lib", "libpisa_b200_trace.so"))
import ctypes as C  # noqa: E402

import paper_2602_01077_b200 as P  # noqa: E402

ROLES = ["K issued", "V issued", "S issued", "PV issued", "smA got S", "smB got S",
         "smA P done", "smB P done", "mma K rdy", "mma P rdy", "mma V rdy", "mma wait K"]


def main():
    H, L, d = int(sys.argv[1]) if len(sys.argv) > 1 else 40, 75600, 128
    tile = 100
    dev = torch.device("cuda", 0)
    kind = sys.argv[2] if len(sys.argv) > 2 else "gaussian"
    if kind == "clustered":
        q, k, v = (x.reshape(1, H, L, d).to(dev) for x in P.gen_clustered(0, H, L, d))
    else:
        q, k, v = (torch.randn((1, H, L, d), device=dev, dtype=torch.bfloat16) for _ in range(3))
    ctx = P.Context.get(0)
    buf = torch.zeros(32 * 1024, dtype=torch.int64, device=dev)
    for _ in range(2):
        P.fwd(q, k, v, sparsity=0.875)
    ctx.lib.pisa_b200_debug_trace(ctx.handle, C.c_void_p(buf.data_ptr()), tile)
    P.fwd(q, k, v, sparsity=0.875)
    torch.cuda.synchronize()
    tr = buf.view(32, 1024).cpu().tolist()
    n = max(i for i in range(1024) if tr[2][i] or i == 0) + 1
    print("t  " + " ".join(f"{r:>11s}" for r in ROLES))
    for t in range(n):
        print(f"{t:3d} " + " ".join(f"{tr[r][t]:11d}" for r in range(len(ROLES))))
    # per-tile deltas in steady state
    ds = [tr[2][t + 1] - tr[2][t] for t in range(20, n - 30)]
    print("median S-issue period (cycles):", sorted(ds)[len(ds) // 2] if ds else None)
    print(f"prologue (cycles from CTA start): TMEM alloc {tr[12][0]}, masks {tr[13][0]}, "
          f"CTA barrier {tr[14][0]}, Q landed {tr[15][0]}, first K issued {tr[0][0]}, first S issued {tr[2][0]}; "
          f"K producer: loop entry {tr[12][1]}, rows {tr[13][1]}, expect_tx {tr[14][1]}")
    last = max(t for t in range(1024) if tr[3][t])
    print(f"tail: last PV issued {tr[3][last]} (t={last}), QH issued {tr[12][2]}, O+QH complete {tr[13][2]}, "
          f"epilogue stored {tr[14][2]}")
    # per-warp P publish (roles 16..23: warpgroup A warps q4 = 0..3, then B) and
    # rescales (roles 24..31), relative to the warpgroup's q4 = 0 warp
    print("\nper-warp P publish - q4=0 warp (A: q4=1..3 | B: q4=1..3), rescale marks R")
    for t in range(n):
        row = []
        for hh in range(2):
            base = tr[16 + hh * 4][t]
            row.append(" ".join(f"{tr[16 + hh * 4 + w][t] - base:6d}" for w in range(1, 4)))
            row.append("".join("R" if tr[24 + hh * 4 + w][t] else "." for w in range(4)))
        print(f"{t:3d}  A {row[0]} {row[1]}   B {row[2]} {row[3]}   mmaP-lastP {tr[9][t] - max(tr[16 + i][t] for i in range(8)):6d}")


if __name__ == "__main__":
    main()
