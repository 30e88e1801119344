"""(batch x head) sharding across ranks -- the only multi-GPU decomposition the
path needs: heads are independent in pisa_multihead
(engine.hpp:432-468), so each rank runs the full K1 -> K2 -> K3 sequence on a
contiguous range of (b, h) units with no data-path collective. The optional
final gather of O is one all_gather over NCCL (NVLink/NVSwitch) or gloo.
"""
from __future__ import annotations

from typing import Tuple

import torch


def unit_range(units: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous [lo, hi) range of (b, h) units for `rank` (balanced to +-1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return rank * units // world, (rank + 1) * units // world


def shard_heads(x: torch.Tensor, world: int, rank: int, head_dim: int = 1) -> torch.Tensor:
    """This rank's slice of a [B][H][L][d] (head_dim=1) tensor, flattened over (b, h)."""
    B, H = x.shape[0], x.shape[head_dim]
    lo, hi = unit_range(B * H, world, rank)
    flat = x.reshape(B * H, *x.shape[2:]) if head_dim == 1 else x.transpose(1, 2).reshape(
        B * H, *x.shape[1:2], *x.shape[3:])
    return flat[lo:hi]


def gather_heads(local: torch.Tensor, units: int, world: int, group=None) -> torch.Tensor:
    """All-gathers per-rank [units_r][L][d] slices into [units][L][d] (rank order).
    Uneven ranks are padded to the largest share for the collective."""
    import torch.distributed as dist

    if world == 1:
        return local
    shares = [unit_range(units, world, r) for r in range(world)]
    mx = max(hi - lo for lo, hi in shares)
    pad = torch.zeros((mx, *local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[: hi - lo] for b, (lo, hi) in zip(bufs, shares)], 0)
