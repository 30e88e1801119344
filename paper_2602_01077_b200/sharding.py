"""(batch x head) sharding across ranks -- the only multi-GPU decomposition the
path needs: heads are independent in pisa_multihead
(engine.hpp:432-468), so each rank runs the full K1 -> K2 -> K3 sequence on a
contiguous range of (b, h) units with no data-path collective. The optional
final gather of O is one all_gather over NCCL (NVLink/NVSwitch) or gloo.

When the units do not divide evenly (Wan2.1-1.3B: 12 heads on 8 GPUs), the
work is split in (unit x query-block) space instead: query blocks of a head are
independent too (engine.hpp:272), so a rank may own a range of query blocks of
a head, computed by pisa_b200_fwd_qrange (statistics and routing still see the
head's full K / V, recomputed by every rank that touches the head).
"""
from __future__ import annotations

from typing import List, NamedTuple, Tuple

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


class Piece(NamedTuple):
    """Units [u0, u1) of one batch index b (heads h0 = u0 % H ...), query blocks [qb0, qb1)."""
    b: int
    h0: int
    h1: int
    qb0: int
    qb1: int


def unit_qblock_pieces(B: int, H: int, N: int, world: int, rank: int) -> List[Piece]:
    """This rank's share of the B*H*N query blocks (balanced to +-1 block), as
    at most a few (batch, head range, query-block range) calls: a partial first
    head, whole heads, a partial last head (split again at batch boundaries)."""
    total = B * H * N
    lo, hi = unit_range(total, world, rank)
    pieces: List[Piece] = []
    x = lo
    while x < hi:
        u, qb = divmod(x, N)
        b, h = divmod(u, H)
        if qb != 0 or hi - x < N:  # partial head
            end = min(hi, (u + 1) * N)
            pieces.append(Piece(b, h, h + 1, qb, end - u * N))
            x = end
        else:  # whole heads up to the end of this batch index or of the share
            nh = min((hi - x) // N, H - h)
            pieces.append(Piece(b, h, h + nh, 0, N))
            x += nh * N
    return pieces


def fwd_pieces(q, k, v, out, pieces: List[Piece], fwd=None, **kw):
    """Runs this rank's pieces on [B][H][L][d] device tensors (views per piece,
    no copies); rows of `out` outside the pieces are not written. ``fwd`` is
    the forward with P.fwd's signature (default P.fwd)."""
    if fwd is None:
        from . import pisa as P
        fwd = P.fwd

    for pc in pieces:
        sl = (slice(pc.b, pc.b + 1), slice(pc.h0, pc.h1))
        N = -(-q.shape[2] // 64)
        rng = None if (pc.qb0, pc.qb1) == (0, N) else (pc.qb0, pc.qb1)
        fwd(q[sl], k[sl], v[sl], out[sl], q_blocks=rng, **kw)
    return out


def _piece_rows(pc: Piece, L: int):
    return pc.qb0 * 64, min(L, pc.qb1 * 64)


def gather_pieces(out: torch.Tensor, B: int, H: int, N: int, world: int, rank: int, group=None) -> torch.Tensor:
    """The optional final gather for (unit x query-block) sharding: every rank
    holds a full-size [B][H][L][d] ``out`` in which only its pieces are written;
    the rows of all ranks' pieces are exchanged with one all_gather (packed
    per rank in piece order, padded to the largest share) and the assembled
    output is returned on every rank. The piece lists are recomputed locally
    (unit_qblock_pieces is deterministic), so no metadata travels."""
    import torch.distributed as dist

    if world == 1:
        return out
    L, d = out.shape[2], out.shape[3]

    def pack_len(r):
        return sum((pc.h1 - pc.h0) * (lambda a: a[1] - a[0])(_piece_rows(pc, L))
                   for pc in unit_qblock_pieces(B, H, N, world, r))

    mx = max(pack_len(r) for r in range(world))
    buf = torch.zeros((mx, d), dtype=out.dtype, device=out.device)
    o = 0
    for pc in unit_qblock_pieces(B, H, N, world, rank):
        r0, r1 = _piece_rows(pc, L)
        rows = out[pc.b, pc.h0:pc.h1, r0:r1].reshape(-1, d)
        buf[o:o + rows.shape[0]] = rows
        o += rows.shape[0]
    bufs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf, group=group)
    full = torch.empty_like(out)
    for r in range(world):
        o = 0
        for pc in unit_qblock_pieces(B, H, N, world, r):
            r0, r1 = _piece_rows(pc, L)
            n = (pc.h1 - pc.h0) * (r1 - r0)
            full[pc.b, pc.h0:pc.h1, r0:r1] = bufs[r][o:o + n].reshape(pc.h1 - pc.h0, r1 - r0, d)
            o += n
    return full
