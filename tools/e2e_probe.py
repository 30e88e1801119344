"""Where the host path's time goes: the 16-chunk H2D -> compute -> D2H pipeline
of pisa_b200_fwd_host emulated with torch streams at the Wan2.1-14B shape,
with and without the compute step, next to the C-ABI call itself.
Usage: python tools/e2e_probe.py"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_01077_b200 as P  # noqa: E402


def main():
    B, H, L, d = 1, 40, 75600, 128
    g = torch.Generator(device="cuda").manual_seed(0)
    hq, hk, hv = (torch.randn((B, H, L, d), generator=g, device="cuda", dtype=torch.bfloat16).cpu().pin_memory()
                  for _ in range(3))
    ho = torch.empty((B, H, L, d), dtype=torch.bfloat16).pin_memory()
    kw = dict(sparsity=0.875)
    chunk = 3
    starts = list(range(0, H, chunk))
    bufs = [[torch.empty((B, chunk, L, d), device="cuda", dtype=torch.bfloat16) for _ in range(4)] for _ in range(2)]
    s_h2d, s_comp, s_d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()

    def pipeline(compute: bool):
        ev_h2d = [torch.cuda.Event() for _ in starts]
        ev_comp = [torch.cuda.Event() for _ in starts]
        ev_d2h = [torch.cuda.Event() for _ in starts]
        for c, h0 in enumerate(starts):
            hc = min(chunk, H - h0)
            bq, bk, bv, bo = (x[:, :hc] for x in bufs[c & 1])
            with torch.cuda.stream(s_h2d):
                if c >= 2:
                    s_h2d.wait_event(ev_comp[c - 2])
                bq.copy_(hq[:, h0:h0 + hc], non_blocking=True)
                bk.copy_(hk[:, h0:h0 + hc], non_blocking=True)
                bv.copy_(hv[:, h0:h0 + hc], non_blocking=True)
                ev_h2d[c].record(s_h2d)
            with torch.cuda.stream(s_comp):
                s_comp.wait_event(ev_h2d[c])
                if c >= 2:
                    s_comp.wait_event(ev_d2h[c - 2])
                if compute:
                    P.fwd(bq, bk, bv, bo, **kw)
                ev_comp[c].record(s_comp)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(ev_comp[c])
                ho[:, h0:h0 + hc].copy_(bo, non_blocking=True)
                ev_d2h[c].record(s_d2h)
        torch.cuda.synchronize()

    def timed(fn, n=4):
        fn()
        t = time.perf_counter()
        for _ in range(n):
            fn()
        return (time.perf_counter() - t) * 1e3 / n

    print(f"emulated pipeline, copies only      : {timed(lambda: pipeline(False)):.1f} ms")
    print(f"emulated pipeline, with compute     : {timed(lambda: pipeline(True)):.1f} ms")
    print(f"pisa_b200_fwd_host (C ABI)          : {timed(lambda: P.fwd_host(hq, hk, hv, ho, **kw)):.1f} ms")
    dq, dk, dv = (x.cuda() for x in (hq, hk, hv))
    do = torch.empty_like(dq)
    print(f"device-resident fwd                 : {timed(lambda: (P.fwd(dq, dk, dv, do, **kw), torch.cuda.synchronize())):.1f} ms")


if __name__ == "__main__":
    main()
