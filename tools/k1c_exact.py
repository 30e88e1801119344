"""K1c accuracy at full scale: GPU M_j (P.block_norms) against exact
sigma_max(H_j - H_bar) from fp64 SVD on the GPU, for a few heads of the
Wan2.1-14B shape (gaussian and clustered-like keys).
Usage: python tools/k1c_exact.py [heads]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_01077_b200 as P  # noqa: E402


def exact_norms(k, v):
    """k, v [L][d] bf16 -> sigma_max(H_j - H_bar) per block (fp64), H_bar over all N blocks."""
    L, d = k.shape
    N = -(-L // 64)
    kf, vf = k.double(), v.double()
    H = torch.empty((N, d, d), dtype=torch.float64, device=k.device)
    for j in range(N):
        kb, vb = kf[j * 64:(j + 1) * 64], vf[j * 64:(j + 1) * 64]
        H[j] = (kb - kb.mean(0)).T @ vb
    Hbar = H.mean(0)
    return torch.linalg.matrix_norm(H - Hbar, ord=2)


def main():
    heads = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    L, d = 75600, 128
    for kind in ("gaussian", "clustered"):
        g = torch.Generator(device="cuda").manual_seed(5)
        shape = (1, heads, L, d)
        if kind == "gaussian":
            k = torch.randn(shape, generator=g, device="cuda").bfloat16()
        else:
            ctr = torch.randn((1, heads, 16, d), generator=g, device="cuda")
            zi = torch.clamp(torch.arange(L, device="cuda") // (-(-L // 16)), max=15)
            k = (ctr[:, :, zi] + 0.15 * torch.randn(shape, generator=g, device="cuda")).bfloat16()
        v = torch.randn(shape, generator=g, device="cuda").bfloat16()
        q = torch.randn(shape, generator=g, device="cuda").bfloat16()
        m = P.block_norms(q, k, v)[0].double()
        worst = 0.0
        errs = []
        for h in range(heads):
            ex = exact_norms(k[0, h], v[0, h])
            rel = ((m[h] - ex).abs() / ex.clamp_min(1e-30))
            errs.append(rel)
            worst = max(worst, rel.max().item())
        rel = torch.cat(errs)
        qs = torch.quantile(rel, torch.tensor([0.5, 0.99, 0.999], dtype=torch.float64, device=rel.device))
        print(f"{kind}: {rel.numel()} blocks, rel. error median {qs[0].item():.2e}, p99 {qs[1].item():.2e}, "
              f"p99.9 {qs[2].item():.2e}, max {worst:.2e}, blocks > 1e-5: {(rel > 1e-5).sum().item()}")


if __name__ == "__main__":
    main()
