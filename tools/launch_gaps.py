"""Launch overhead of the fused forward at image sizes: one P.fwd step timed
eagerly with and without the library's profiling events, and replayed from a
CUDA graph (the call is stream-ordered and capture-safe with profiling and
check_finite off). L2 flushed before every timed step.
Usage: python tools/launch_gaps.py [flux|sd35|wan13b]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_01077_b200 as P  # noqa: E402

SHAPES = {"flux": (24, 4608, 128), "sd35": (24, 4429, 64), "wan13b": (12, 32760, 128)}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "flux"
    H, L, d = SHAPES[name]
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn((1, H, L, d), generator=g, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    out = torch.empty_like(q)
    ctx = P.Context.get(0)
    kw = dict(sparsity=0.875)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def step():
        P.fwd(q, k, v, out, **kw)

    def timed(fn, n=50):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for a, b in evs:
            flush.zero_()
            a.record()
            fn()
            b.record()
        torch.cuda.synchronize()
        ts = sorted(a.elapsed_time(b) for a, b in evs)
        return sum(ts) / n, ts[n // 2]

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    ref = out.clone()
    ctx.set_profiling(False)
    eager = timed(step)
    ctx.set_profiling(True)
    prof = timed(step)
    kern = ctx.read_profile()
    ctx.set_profiling(False)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        step()
    torch.cuda.current_stream().wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    out.zero_()
    graph.replay()
    torch.cuda.synchronize()
    same = torch.equal(out, ref)
    gr = timed(graph.replay)
    ksum = sum(ms for ms, _ in kern.values()) / 50
    print(f"{name}: eager {eager[0]:.4f} ms (median {eager[1]:.4f}), eager+profiling {prof[0]:.4f}, "
          f"CUDA graph {gr[0]:.4f} (median {gr[1]:.4f}); sum of kernel events {ksum:.4f} ms; "
          f"graph output identical: {same}")


if __name__ == "__main__":
    main()
