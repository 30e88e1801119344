"""Head-chunk pipelining probe: does running a small head chunk's fused kernel
(K3) beside the rest of the heads' prologue (K1 / K2 / pairing) shorten the
Wan2.1-14B step?

Times, on the device with CUDA events:
  base            one pisa_b200_fwd over all heads
  split a / prio  fwd(heads [0, a)) on stream s0 and fwd(heads [a, H)) on s1
                  (s1 high priority when prio=1), both forked from and joined
                  into the current stream
and checks the split outputs are bit-identical to the base output (heads are
independent: every kernel of the path works per head).

  python tools/head_pipe.py [--L 75600] [--H 40] [--reps 6]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2602_01077_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=75600)
    ap.add_argument("--H", type=int, default=40)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--reps", type=int, default=6)
    ap.add_argument("--splits", default="1,2,4,8")
    args = ap.parse_args()
    torch.manual_seed(0)
    dev = torch.device("cuda:0")
    H, L, d = args.H, args.L, args.d
    q, k, v = (torch.randn(1, H, L, d, device=dev).to(torch.bfloat16) for _ in range(3))
    out = torch.empty_like(q)
    kw = dict(sparsity=0.875, variant=P.PisaVariant.Hybrid)
    P.fwd(q, k, v, out, **kw)
    torch.cuda.synchronize()
    ref = out.clone()

    cur = torch.cuda.current_stream()
    lo, hi = torch.cuda.Stream.priority_range()
    streams = {0: (torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=0)),
               1: (torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=hi))}

    def run(split, prio):
        if split == 0:
            P.fwd(q, k, v, out, **kw)
            return
        s0, s1 = streams[prio]
        e = torch.cuda.Event()
        e.record(cur)
        s0.wait_event(e)
        s1.wait_event(e)
        with torch.cuda.stream(s0):
            P.fwd(q[:, :split], k[:, :split], v[:, :split], out[:, :split], **kw)
        with torch.cuda.stream(s1):
            P.fwd(q[:, split:], k[:, split:], v[:, split:], out[:, split:], **kw)
        cur.wait_stream(s0)
        cur.wait_stream(s1)

    cases = [(0, 0)] + [(int(s), p) for s in args.splits.split(",") for p in (0, 1)]
    for rnd in range(2):
        for split, prio in cases:
            out.zero_()
            for _ in range(2):
                run(split, prio)
            ts = []
            for _ in range(args.reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                a.record(cur)
                run(split, prio)
                b.record(cur)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            same = bool(torch.equal(out, ref))
            ts.sort()
            print(f"round {rnd} split {split:2d} prio {prio}: median {ts[len(ts) // 2]:.3f} ms "
                  f"min {ts[0]:.3f} bit-identical {same}", flush=True)


if __name__ == "__main__":
    main()
