"""K1c (block norms) probe at the Wan2.1-14B and FLUX shapes.

    PISA_B200_LIB=.../libpisa_b200_cN.so python tools/k1c_probe.py clocks TAG
        (library built with -DPISA_K1C_CLOCKS=N: M_j holds a phase's cycles)
    PISA_B200_LIB=... python tools/k1c_probe.py time TAG
        (ms per call; M_j saved to gpurun_out/k1c_m_TAG_<shape>.pt for A/B)
    python tools/k1c_probe.py compare TAG_A TAG_B"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SHAPES = {"wan14b": (1, 40, 75600, 128), "flux": (1, 24, 4608, 128)}
OUT = "gpurun_out"


def main():
    mode, tag = sys.argv[1], sys.argv[2]
    if mode == "compare":
        for sh in SHAPES:
            a = torch.load(f"{OUT}/k1c_m_{tag}_{sh}.pt")
            b = torch.load(f"{OUT}/k1c_m_{sys.argv[3]}_{sh}.pt")
            rel = ((a - b).abs() / b.abs().clamp_min(1e-30)).max().item()
            print(f"{sh}: max rel diff {tag} vs {sys.argv[3]}: {rel:.3e}")
        return
    import paper_2602_01077_b200 as P
    os.makedirs(OUT, exist_ok=True)
    for sh, (B, H, L, d) in SHAPES.items():
        g = torch.Generator(device="cuda").manual_seed(0)
        q, k, v = (torch.randn((B, H, L, d), generator=g, device="cuda", dtype=torch.bfloat16) for _ in range(3))
        m = P.block_norms(q, k, v)
        torch.cuda.synchronize()
        if mode == "clocks":
            c = m.flatten().double()
            qs = torch.quantile(c[: min(c.numel(), 1 << 24)], torch.tensor([0.1, 0.5, 0.9], dtype=torch.float64, device=c.device))
            print(f"{tag} {sh}: mean {c.mean().item():.0f} cycles, p10/p50/p90 "
                  f"{qs[0].item():.0f}/{qs[1].item():.0f}/{qs[2].item():.0f}")
        else:
            for _ in range(3):
                P.block_norms(q, k, v)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 20
            e0.record()
            for _ in range(n):
                P.block_norms(q, k, v)
            e1.record()
            torch.cuda.synchronize()
            print(f"{tag} {sh}: {e0.elapsed_time(e1) / n:.4f} ms per block_norms call (incl. block stats)")
            torch.save(m.cpu(), f"{OUT}/k1c_m_{tag}_{sh}.pt")


if __name__ == "__main__":
    main()
