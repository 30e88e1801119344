"""Diagnostics and theory checks on GPU outputs (the reference's analysis.hpp).

* ``compare_outputs`` (analysis.hpp:27-57): l1_rel, l2_rel, max_abs, per-row L2.
* ``theorem1_check`` (analysis.hpp:80-164): certifies, row by row, the error
  bound of PISA's global first-order correction against the exact block-wise one
      ||o~_t - o_t||_2 <= C_q * M_max * rho_t / B,   rho_t = tau_t / D_t,
  with the block-wise Jensen inequality alpha_t <= tau_t / B alongside. The
  Hybrid output o~ may be the fused kernel's own output (``hybrid=``), which is
  the point: the bound is checked on what the GPU produced.
* ``jensen_check`` (analysis.hpp:170-207): exp(s q.k_bar_j) <= mean_n exp(s q.k_{j,n})
  for every row and unselected block.

They are O(L^2 d) dense passes by construction (tau needs every exact score),
computed in fp64 with torch on the device in row chunks -- diagnostics for
modest shapes, not part of the attention hot path. The BlockFirst reference
output (per-block H_j correction, engine.hpp:184-192) is formed here in fp64.
Semantics follow the reference line by line (same max shift over exact and
centroid scores, same slack constants kBoundAbsSlack = 1e-9 and
kJensenRelSlack = 1e-9); tests/test_analysis.py pins them to the reference.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import torch

K_BOUND_ABS_SLACK = 1e-9   # analysis.hpp:77
K_JENSEN_REL_SLACK = 1e-9  # analysis.hpp:78


@dataclasses.dataclass
class ErrorReport:  # analysis.hpp:20-25
    l1_rel: float
    l2_rel: float
    max_abs: float
    per_row_l2: torch.Tensor


def compare_outputs(approx: torch.Tensor, ref: torch.Tensor) -> ErrorReport:
    if approx.shape != ref.shape:
        from .pisa import InvalidDimension
        raise InvalidDimension(f"InvalidDimension: output shapes differ: {tuple(approx.shape)} vs "
                               f"{tuple(ref.shape)}")
    a, b = approx.double(), ref.double()
    diff = a - b
    n1, d1 = diff.abs().sum().item(), b.abs().sum().item()
    n2, d2 = diff.pow(2).sum().item(), b.pow(2).sum().item()
    return ErrorReport(
        l1_rel=n1 / d1 if d1 > 0 else (0.0 if n1 == 0 else math.inf),
        l2_rel=math.sqrt(n2) / math.sqrt(d2) if d2 > 0 else (0.0 if n2 == 0 else math.inf),
        max_abs=diff.abs().max().item() if diff.numel() else 0.0,
        per_row_l2=diff.pow(2).sum(-1).sqrt())


@dataclasses.dataclass
class BoundReport:  # analysis.hpp:59-75 (rows as column tensors)
    actual_err: torch.Tensor
    bound: torch.Tensor
    rho: torch.Tensor
    alpha_sum: torch.Tensor
    jensen_rhs: torch.Tensor
    c_q: float
    m_max: float
    block_size: int
    violations: int
    jensen_violations: int
    max_slack_ratio: float


def _block_stats64(k: torch.Tensor, v: torch.Tensor, B: int):
    """fp64 k_bar, v_hat, per-block H_j, H_bar, M_j (exact spectral norms)."""
    L, d = k.shape
    N = L // B
    kb = k.view(N, B, d)
    vb = v.view(N, B, d)
    kbar = kb.mean(1)
    vhat = vb.sum(1)
    kc = kb - kbar[:, None, :]
    H = torch.einsum("nra,nrc->nac", kc, vb)               # [N][d][d]
    hbar = H.sum(0) / N                                     # ascending-order sum / N
    m = torch.linalg.matrix_norm(H - hbar, ord=2)           # sigma_max per block
    return kbar, vhat, H, hbar, m


def theorem1_check(q, k, v, selected: torch.Tensor, B: int = 64, scale: float = 0.0,
                   hybrid: Optional[torch.Tensor] = None, row_chunk: int = 512) -> BoundReport:
    """theorem1_check for one head: q/k/v [L][d] (any float dtype, device),
    selected [N][k] ascending (the routing plan). ``hybrid`` [L][d]: the Hybrid
    output to certify (e.g. the fused kernel's); default: the fp64 Hybrid."""
    # outputs are materialised in the element type T of the inputs, as the
    # reference's pisa_reference<T> does (engine.hpp:212: orow[c] = T(num / denom))
    t_out = q.dtype if q.dtype in (torch.float32, torch.float64) else torch.float32
    q, k, v = (x.double() for x in (q, k, v))
    L, d = q.shape
    N = L // B
    if L % B:
        from .pisa import BlockDivisibility
        raise BlockDivisibility(f"BlockDivisibility: seq_len {L} not divisible by block size {B}")
    scale = scale if scale > 0 else 1.0 / math.sqrt(d)
    dev = q.device
    kbar, vhat, H, hbar, m = _block_stats64(k, v, B)
    m_max = float(m.max().item())
    c_q = scale * float(q.norm(dim=1).max().item())
    sel = torch.zeros((N, N), dtype=torch.bool, device=dev)
    sel.scatter_(1, selected.long().to(dev), True)
    out = {n: torch.empty(L, dtype=torch.float64, device=dev)
           for n in ("actual_err", "bound", "rho", "alpha_sum", "jensen_rhs")}
    hyb_out = torch.empty((L, d), dtype=torch.float64, device=dev) if hybrid is None else None
    for r0 in range(0, L, row_chunk):
        r1 = min(L, r0 + row_chunk)
        qr = q[r0:r1]
        qblk = torch.arange(r0, r1, device=dev) // B
        s = scale * (qr @ k.T)                               # exact scores [R][L]
        cent = scale * (qr @ kbar.T)                         # centroid scores [R][N]
        insel = sel[qblk]                                    # [R][N]
        cent_u = torch.where(insel, torch.full_like(cent, -math.inf), cent)
        mrow = torch.maximum(s.max(1).values, cent_u.max(1).values)   # one shift (analysis.hpp:118-126)
        pexp = torch.exp(s - mrow[:, None]).view(-1, N, B)
        blk = pexp.sum(-1)                                   # [R][N]
        tau = torch.where(insel, torch.zeros_like(blk), blk).sum(1)
        exact_sel = torch.where(insel, blk, torch.zeros_like(blk)).sum(1)
        a = torch.where(insel, torch.zeros_like(cent), torch.exp(cent_u - mrow[:, None]))  # [R][N]
        alpha = a.sum(1)
        denom = exact_sel + B * alpha
        rho = torch.where(denom > 0, tau / denom, torch.zeros_like(tau))
        # Hybrid / BlockFirst numerators over the identical piecewise denominator
        # (pisa_reference, engine.hpp:163-209)
        pe = torch.where(insel[:, :, None], pexp, torch.zeros_like(pexp)).view(r1 - r0, L)
        num_exact = pe @ v + a @ vhat
        qh = qr @ hbar
        num_hyb = num_exact + (alpha * scale)[:, None] * qh
        # sum_j a_j * scale * (q . H_j)  ==  ((a (x) q) flattened) @ H.view(N*d, d)
        w = (a[:, :, None] * qr[:, None, :]).reshape(r1 - r0, N * d)
        num_bf = num_exact + scale * (w @ H.reshape(N * d, d))
        o_bf = (num_bf / denom[:, None]).to(t_out).double()
        o_hy = (num_hyb / denom[:, None]).to(t_out).double() if hybrid is None else hybrid[r0:r1].double()
        if hyb_out is not None:
            hyb_out[r0:r1] = o_hy
        lift = torch.exp(mrow)
        out["actual_err"][r0:r1] = (o_hy - o_bf).norm(dim=1)
        out["rho"][r0:r1] = rho
        out["bound"][r0:r1] = c_q * m_max * rho / B
        out["alpha_sum"][r0:r1] = alpha * lift
        out["jensen_rhs"][r0:r1] = tau * lift / B
    viol = int((out["actual_err"] > out["bound"] + K_BOUND_ABS_SLACK).sum().item())
    jv = int((out["alpha_sum"] > out["jensen_rhs"] * (1.0 + K_JENSEN_REL_SLACK)).sum().item())
    pos = out["bound"] > 0
    slack = float((out["actual_err"][pos] / out["bound"][pos]).max().item()) if bool(pos.any()) else 0.0
    return BoundReport(c_q=c_q, m_max=m_max, block_size=B, violations=viol, jensen_violations=jv,
                       max_slack_ratio=slack, **out)


def pisa_fp64(q, k, v, selected: torch.Tensor, variant: str = "hybrid", B: int = 64, scale: float = 0.0,
              row_chunk: int = 512) -> torch.Tensor:
    """fp64 piecewise attention of one head (pisa_reference, engine.hpp:103-223)
    for SparseOnly / Zeroth / Hybrid on the given plan: the exact softmax over
    the selected key blocks, the zeroth-order centroid tail with weight B per
    unselected block, and (Hybrid) the global first-order term
    scale * ell_tail * (q . H_bar). q/k/v [L][d], L % B == 0; [L][d] fp64."""
    q, k, v = q.double(), k.double(), v.double()
    L, d = q.shape
    N = L // B
    scale = scale if scale > 0 else 1.0 / math.sqrt(d)
    kbar, vhat, _, hbar, _ = _block_stats64(k, v, B)
    sel = torch.zeros((N, N), dtype=torch.bool, device=q.device)
    sel.scatter_(1, selected.long().to(q.device), True)
    out = torch.empty((L, d), dtype=torch.float64, device=q.device)
    for r0 in range(0, L, row_chunk):
        r1 = min(L, r0 + row_chunk)
        qr = q[r0:r1]
        insel = sel[torch.arange(r0, r1, device=q.device) // B]
        s = (scale * (qr @ k.T)).view(r1 - r0, N, B)
        s = torch.where(insel[:, :, None], s, torch.full_like(s, -math.inf))
        cent = scale * (qr @ kbar.T)
        cent = torch.where(insel, torch.full_like(cent, -math.inf), cent)
        if variant == "sparse_only":
            cent = torch.full_like(cent, -math.inf)
        mrow = torch.maximum(s.amax((1, 2)), cent.amax(1))
        pe = torch.exp(s - mrow[:, None, None]).view(r1 - r0, L)
        a = torch.exp(cent - mrow[:, None])
        num = pe @ v + a @ vhat
        den = pe.sum(1) + B * a.sum(1)
        if variant == "hybrid":
            num = num + (scale * a.sum(1))[:, None] * (qr @ hbar)
        out[r0:r1] = num / den[:, None]
    return out


def jensen_check(q, k, selected: torch.Tensor, B: int = 64, scale: float = 0.0,
                 row_chunk: int = 512) -> int:
    """jensen_check (analysis.hpp:170-207): violation count (0 when correct)."""
    q, k = q.double(), k.double()
    L, d = q.shape
    if k.shape[0] % B:
        from .pisa import BlockDivisibility
        raise BlockDivisibility("BlockDivisibility: seq_len not divisible by block size")
    N = k.shape[0] // B
    scale = scale if scale > 0 else 1.0 / math.sqrt(d)
    kbar = k.view(N, B, d).mean(1)
    sel = torch.zeros((N, N), dtype=torch.bool, device=q.device)
    sel.scatter_(1, selected.long().to(q.device), True)
    viol = 0
    for r0 in range(0, L, row_chunk):
        r1 = min(L, r0 + row_chunk)
        qr = q[r0:r1]
        s = (scale * (qr @ k.T)).view(r1 - r0, N, B)
        lhs_arg = scale * (qr @ kbar.T)                      # [R][N]
        mm = torch.maximum(s.max(-1).values, lhs_arg)        # per (row, block) shift
        rhs = torch.exp(s - mm[:, :, None]).sum(-1) / B
        lhs = torch.exp(lhs_arg - mm)
        bad = (lhs > rhs * (1.0 + K_JENSEN_REL_SLACK)) & ~sel[torch.arange(r0, r1, device=q.device) // B]
        viol += int(bad.sum().item())
    return viol


def theorem1_multihead(q, k, v, plans: List[torch.Tensor], hybrid=None, **kw) -> List[BoundReport]:
    """theorem1_check per head of [H][L][d] tensors (plans[h] [N][k])."""
    return [theorem1_check(q[h], k[h], v[h], plans[h], hybrid=None if hybrid is None else hybrid[h], **kw)
            for h in range(q.shape[0])]
