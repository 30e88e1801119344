"""DiT integration surface: the caller side of the PISA attention path.

A diffusion transformer calls attention once per (layer, denoising step) with
DiT-layout tensors [B, L, H, d]. The paper's recipe (PAPER.md:599 and the
warmup tables at):

* a warmup policy keeps the first ``dense_layers`` transformer layers and the
  first ``dense_steps`` denoising steps on dense attention, PISA elsewhere
  (video models: 1 layer + 10-15 steps; image models: 4 layers, 0 steps);
* image models use the covariance-aware router ("We only employ
  the Covariance-Aware Block Selection ... for image generation");
* MMDiT models (FLUX.1, SD3.5) attend jointly over the concatenated
  [text tokens; image tokens] sequence; PISA then routes over that sequence
  like any other (the ragged last block is handled exactly).

The sparse path is the fused sm_100a forward (``paper_2602_01077_b200.fwd``,
strided [B, L, H, d] through the C ABI, no copy). The dense warmup path is the
plain dense attention the model would otherwise run (torch SDPA, i.e. the
cuDNN / flash library kernel), exactly as in the paper's setup; it is not part
of the PISA hot path.
"""
from __future__ import annotations

import dataclasses
from typing import Optional, Tuple

import torch
import torch.nn.functional as F

from . import pisa as _p


@dataclasses.dataclass(frozen=True)
class WarmupPolicy:
    """Dense for layer < dense_layers or step < dense_steps."""
    dense_layers: int = 0
    dense_steps: int = 0

    def is_dense(self, layer: Optional[int], step: Optional[int]) -> bool:
        if layer is not None and layer < self.dense_layers:
            return True
        if step is not None and step < self.dense_steps:
            return True
        return False


@dataclasses.dataclass(frozen=True)
class Preset:
    policy: WarmupPolicy
    router: _p.RouterStrategy
    density: float = 0.125  # 87.5 % sparsity, the paper's setting


# Table "Configuration of Video/Image Generation" and the
# router choice of PAPER.md:599.
PRESETS = {
    "wan2.1-1.3b": Preset(WarmupPolicy(1, 15), _p.RouterStrategy.Plain),
    "wan2.1-14b": Preset(WarmupPolicy(1, 10), _p.RouterStrategy.Plain),
    "hunyuanvideo-13b": Preset(WarmupPolicy(1, 10), _p.RouterStrategy.Plain),
    "sd3.5-medium": Preset(WarmupPolicy(4, 0), _p.RouterStrategy.CovarianceAware),
    "sd3.5-turbo": Preset(WarmupPolicy(4, 0), _p.RouterStrategy.CovarianceAware),
    "flux.1-schnell": Preset(WarmupPolicy(4, 0), _p.RouterStrategy.CovarianceAware),
    "flux.1-dev": Preset(WarmupPolicy(4, 0), _p.RouterStrategy.CovarianceAware),
}


def dense_attention(q, k, v, scale: float = 0.0, layout: str = "blhd") -> torch.Tensor:
    """Dense softmax attention (the warmup path), same layout in and out."""
    if layout == "blhd":
        q, k, v = (t.transpose(1, 2) for t in (q, k, v))
    o = F.scaled_dot_product_attention(q, k, v, scale=scale if scale > 0 else None)
    return o.transpose(1, 2) if layout == "blhd" else o


class PisaAttention:
    """Drop-in attention call for a DiT block.

    ``attn(q, k, v, layer=i, step=s)`` with q/k/v bf16 CUDA tensors
    [B, L, H, d] (``layout="blhd"``, the DiT default) or [B, H, L, d]
    (``layout="bhld"``); returns O in the same layout. Warmup layers / steps
    run dense attention, all others the fused PISA forward.
    """

    def __init__(self, density: float = 0.125, policy: WarmupPolicy = WarmupPolicy(),
                 router: _p.RouterOptions = _p.RouterOptions(),
                 variant: _p.PisaVariant = _p.PisaVariant.Hybrid,
                 cfg: _p.AttentionConfig = _p.AttentionConfig(), layout: str = "blhd",
                 ragged: bool = True):
        if not 0.0 < density <= 1.0:
            raise _p.InvalidSparsity(f"InvalidSparsity: density must lie in (0, 1], got {density}")
        if layout not in ("blhd", "bhld"):
            raise _p.InvalidDimension(f"InvalidDimension: unknown layout {layout}")
        self.density = density
        self.policy = policy
        self.router = router
        self.variant = variant
        self.cfg = cfg
        self.layout = layout
        self.ragged = ragged  # L % 64 != 0 (e.g. 4096 image + 333 text tokens) is exact
        self.calls = {"dense": 0, "pisa": 0}

    @classmethod
    def from_preset(cls, name: str, density: Optional[float] = None, **kw) -> "PisaAttention":
        if name not in PRESETS:
            raise KeyError(f"unknown preset {name!r}; known: {sorted(PRESETS)}")
        p = PRESETS[name]
        return cls(density=p.density if density is None else density, policy=p.policy,
                   router=_p.RouterOptions(strategy=p.router), **kw)

    def __call__(self, q, k, v, *, layer: Optional[int] = None, step: Optional[int] = None,
                 out: Optional[torch.Tensor] = None) -> torch.Tensor:
        if self.policy.is_dense(layer, step) or self.density >= 1.0:
            self.calls["dense"] += 1
            o = dense_attention(q, k, v, self.cfg.scale, self.layout)
            if out is not None:
                out.copy_(o)
                return out
            return o
        self.calls["pisa"] += 1
        if self.router.row_level:
            raise _p.Unsupported("Unsupported: row-level routing is not on the GPU path")
        return _p.fwd(q, k, v, out, layout=self.layout, sparsity=1.0 - self.density,
                      variant=self.variant, router=self.router.strategy,
                      epsilon=self.router.epsilon, force_diagonal=self.router.force_diagonal,
                      block_size=self.cfg.block_size, group_size=self.cfg.group_size,
                      scale=self.cfg.scale, literal_phase3=self.cfg.literal_phase3,
                      ragged=self.ragged)

    def joint(self, txt: Tuple[torch.Tensor, torch.Tensor, torch.Tensor],
              img: Tuple[torch.Tensor, torch.Tensor, torch.Tensor], *,
              layer: Optional[int] = None, step: Optional[int] = None
              ) -> Tuple[torch.Tensor, torch.Tensor]:
        """MMDiT joint attention (FLUX.1 / SD3.5): attention over the concatenated
        [text; image] token sequence; returns (out_text, out_image)."""
        dim = 1 if self.layout == "blhd" else 2
        n_txt = txt[0].shape[dim]
        q, k, v = (torch.cat([a, b], dim=dim) for a, b in zip(txt, img))
        o = self(q, k, v, layer=layer, step=step)
        return o.narrow(dim, 0, n_txt), o.narrow(dim, n_txt, o.shape[dim] - n_txt)
