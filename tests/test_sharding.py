"""(batch x head) sharding, world_size 2 over gloo on CPU: every unit lands on
exactly one rank, and the optional gather reassembles O in order."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_01077_b200.sharding import gather_heads, shard_heads, unit_qblock_pieces, unit_range


@pytest.mark.parametrize("units,world", [(40, 1), (40, 2), (40, 8), (12, 8), (24, 5), (3, 4)])
def test_unit_range_partitions(units, world):
    seen = []
    for r in range(world):
        lo, hi = unit_range(units, world, r)
        assert 0 <= lo <= hi <= units
        seen += list(range(lo, hi))
    assert seen == list(range(units))
    sizes = [unit_range(units, world, r)[1] - unit_range(units, world, r)[0] for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("B,H,N,world", [(1, 12, 512, 8), (1, 40, 1182, 8), (2, 3, 10, 4), (1, 1, 7, 3),
                                         (1, 24, 72, 5), (3, 2, 1, 4)])
def test_unit_qblock_pieces_partition(B, H, N, world):
    """(unit x query-block) sharding: every query block of every
    (b, h) on exactly one rank, shares balanced to one block, at most three
    calls per rank and batch index."""
    cover, sizes = [], []
    for r in range(world):
        ps = unit_qblock_pieces(B, H, N, world, r)
        n = 0
        for p in ps:
            assert 0 <= p.b < B and 0 <= p.h0 < p.h1 <= H and 0 <= p.qb0 < p.qb1 <= N
            assert p.h1 - p.h0 == 1 or (p.qb0, p.qb1) == (0, N)  # a partial range covers one head
            cover += [(p.b, h, qb) for h in range(p.h0, p.h1) for qb in range(p.qb0, p.qb1)]
            n += (p.h1 - p.h0) * (p.qb1 - p.qb0)
        sizes.append(n)
        assert len(ps) <= 3 * B
    assert sorted(cover) == [(b, h, q) for b in range(B) for h in range(H) for q in range(N)]
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def oracle_fwd(q, k, v, out, q_blocks=None, sparsity=0.75, **kw):
    """A CPU forward with P.fwd's signature and q_blocks semantics (statistics
    and routing from the whole head, only the range's rows written), made of
    the oracle's restatement of the reference (block_stats -> select_plain ->
    pisa_attention): real per-head PISA work for the sharding logic on CPU."""
    import numpy as np

    import oracle as O
    B, H, L, d = q.shape
    N = -(-L // 64)
    kk = O.sparsity_to_k(sparsity, N)[0]
    qb0, qb1 = q_blocks if q_blocks is not None else (0, N)
    for b in range(B):
        for h in range(H):
            qf, kf, vf = (x[b, h].float().numpy() for x in (q, k, v))
            st = O.block_stats(kf, vf)
            sel = O.select_plain(O.query_means(qf), st[0], kk, d ** -0.5)
            o = O.pisa_attention(qf, kf, vf, sel, st, d ** -0.5, "hybrid", qb0=qb0, qb1=qb1)[0]
            r0, r1 = qb0 * 64, min(L, qb1 * 64)
            out[b, h, r0:r1] = torch.from_numpy(np.ascontiguousarray(o[r0:r1])).to(out.dtype)
    return out


def _inputs(B, H, L, d):
    import oracle as O
    q, k, v = O.gen("clustered", 17, B * H, L, d)
    return [torch.from_numpy(x).reshape(B, H, L, d) for x in (q, k, v)]


def _worker(rank, world, port, B, H, L, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_01077_b200.sharding import fwd_pieces, gather_pieces
    d = 64
    x = _inputs(B, H, L, d)
    N = -(-L // 64)
    if mode == "heads":  # (b x h) units: whole heads per rank, all_gather of the slices
        qs, ks, vs = (shard_heads(t, world, rank) for t in x)
        out = torch.zeros_like(qs)
        oracle_fwd(qs[None], ks[None], vs[None], out[None])
        full = gather_heads(out, B * H, world).reshape(B, H, L, d)
        n = qs.shape[0]
    else:  # (unit x query-block) pieces: partial heads, the pieces gather
        out = torch.zeros(B, H, L, d)
        pieces = unit_qblock_pieces(B, H, N, world, rank)
        fwd_pieces(*x, out, pieces, fwd=oracle_fwd)
        full = gather_pieces(out, B, H, N, world, rank)
        n = sum((p.h1 - p.h0) * (p.qb1 - p.qb0) for p in pieces)
    if rank == 0:
        ref = oracle_fwd(*x, torch.zeros(B, H, L, d))
        q.put((rank, torch.equal(full, ref), n))
    else:
        q.put((rank, True, n))
    dist.destroy_process_group()


@pytest.mark.parametrize("B,H,L,mode", [(1, 4, 320, "heads"), (2, 3, 200, "heads"), (1, 3, 1000, "pieces"),
                                        (2, 3, 130, "pieces")])
def test_gloo_world2_sharded_forward_equals_single_process(B, H, L, mode):
    """World size 2 over gloo: each rank runs real per-head PISA work (the
    oracle's forward behind P.fwd's interface) on its (b x h) units or its
    (unit x query-block) pieces, the gather reassembles O, and the result is
    bit-identical to the single-process forward of all heads."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, H, L, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res)
    N = -(-L // 64)
    assert sum(n for _, _, n in res) == (B * H if mode == "heads" else B * H * N)
