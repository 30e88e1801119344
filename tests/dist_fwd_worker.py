"""torchrun worker for tests/test_gpu.py::test_torchrun_world2_same_gpu: two
ranks on ONE GPU (gloo; rank-to-GPU mapping is the only thing an 8-GPU box
changes) run the head-sharded and the (head x query-block) sharded forward and
gather O; rank 0 compares with the single-rank forward and writes a JSON verdict.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port P tests/dist_fwd_worker.py result.json
"""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2602_01077_b200 as P  # noqa: E402
from paper_2602_01077_b200.sharding import (fwd_pieces, gather_heads, gather_pieces, shard_heads,  # noqa: E402
                                            unit_qblock_pieces)


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    res = {}
    # (b x h) sharding: 6 heads over 2 ranks; whole heads per rank
    B, H, L, d = 1, 6, 2000, 128
    q, k, v = (x.reshape(B, H, L, d) for x in P.gen_gaussian(3, B * H, L, d))
    qs, ks, vs = (shard_heads(x, world, rank).unsqueeze(0).cuda() for x in (q, k, v))
    out = P.fwd(qs, ks, vs, sparsity=0.875)
    # gloo collectives on fp32 copies (bf16 -> fp32 is exact)
    full = gather_heads(out[0].cpu().float(), B * H, world).reshape(B, H, L, d)
    if rank == 0:
        ref = P.fwd(q.cuda(), k.cuda(), v.cuda(), sparsity=0.875).cpu().float()
        res["heads_bit_equal"] = bool(torch.equal(full, ref))
    # (head x query-block) pieces: 3 heads x 16 query blocks over 2 ranks
    B, H, L = 1, 3, 1000
    N = -(-L // 64)
    q, k, v = (x.reshape(B, H, L, d).cuda() for x in P.gen_clustered(5, B * H, L, d))
    out = torch.zeros((B, H, L, d), dtype=torch.bfloat16, device="cuda")
    fwd_pieces(q, k, v, out, unit_qblock_pieces(B, H, N, world, rank), sparsity=0.75)
    full = gather_pieces(out.cpu().float(), B, H, N, world, rank)
    if rank == 0:
        ref = P.fwd(q, k, v, sparsity=0.75).cpu()
        res["pieces_max_abs_diff"] = float((full.float() - ref.float()).abs().max())
        res["world"] = world
        with open(sys.argv[1], "w") as f:
            json.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
