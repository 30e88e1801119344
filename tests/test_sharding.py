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


def _worker(rank, world, port, units, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    B, H, L, d = 2, units // 2, 8, 4
    x = torch.arange(B * H * L * d, dtype=torch.float32).reshape(B, H, L, d)
    local = shard_heads(x, world, rank)
    # a per-unit computation (stands in for the per-head PISA forward)
    out_local = local * 2.0 + 1.0
    full = gather_heads(out_local, B * H, world)
    ok = torch.equal(full, (x * 2.0 + 1.0).reshape(B * H, L, d))
    q.put((rank, ok, local.shape[0]))
    dist.destroy_process_group()


@pytest.mark.parametrize("units", [10, 7 * 2])
def test_gloo_world2_shard_and_gather(units):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, units, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res)
    assert sum(n for _, _, n in res) == units
