"""Command-line harness of the GPU path, mirroring the reference CLI
(tools/pisa_cli.cpp: gen / run / sweep / bench / verify) so its parity,
benchmark and invariant workflows run unchanged against the sm_100a kernels.

    python -m paper_2602_01077_b200.cli gen   --kind clustered --len 4096 --out x.pqkv
    python -m paper_2602_01077_b200.cli run   --in x.pqkv --sparsity 0.875
    python -m paper_2602_01077_b200.cli sweep --lengths 2048,4096 --sparsities 0.5,0.875
    python -m paper_2602_01077_b200.cli bench --len 75600 --heads 40 --dim 128
    python -m paper_2602_01077_b200.cli verify [--only theorem1] [--seeds 5]

Same options and JSON / CSV keys as the reference (pisa_cli.cpp:27-125,
:222-262, :268-290, :703-767) and the same exit codes (:844-851): 0 ok,
2 validation error, 3 I/O error, 1 invariant / other error. Differences, by
design of the GPU path: tensors run in bf16 (inputs are rounded once); the
dense baseline of `run` / `sweep` is an fp32 GPU computation on the same bf16
inputs; `bench` times dense attention with the library SDPA kernel and PISA
with CUDA events, and reports the prepare / select / attention phases from the
per-kernel events (the fused kernel does exact + approximate + normalise in
one launch, so those three are reported together as phase_attention_ms).
`gen` draws from torch's generator, not the reference's xoshiro stream; for
bit-identical inputs pass a file written by the reference's `pisa gen`.
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
import time
from typing import List

import numpy as np
import torch

from . import pisa as P
from . import pqkv


# ------------------------------------------------------------- flop model --
def flop_model(L: int, d: int, b: int, k: int, variant: P.PisaVariant) -> dict:
    """flop_model (analysis.hpp:309-355): 2mnp convention, exp ignored."""
    if b <= 0 or L % b:
        raise P.BlockDivisibility(f"BlockDivisibility: seq_len {L} not divisible by block size {b}")
    n = L / b
    if k <= 0 or k > n:
        raise P.InvalidSparsity("InvalidSparsity: k out of range")
    dense = 4.0 * L * L * d
    prep_centroids, select, normalize = 2.0 * L * d, 2.0 * n * n * d, 1.0 * L * d
    exact = 4.0 * L * (k * b) * d
    has_tail = variant != P.PisaVariant.SparseOnly
    has_h = variant in (P.PisaVariant.BlockFirst, P.PisaVariant.Hybrid, P.PisaVariant.GlobalCentroid)
    zeroth = 4.0 * L * (n - k) * d if has_tail else 0.0
    h_prep = 2.0 * L * d * d if has_h else 0.0
    first = 2.0 * L * (n - k) * d * d if variant == P.PisaVariant.BlockFirst else (2.0 * L * d * d if has_h else 0.0)
    sparse = exact + select + prep_centroids + normalize
    pisa = sparse + zeroth + h_prep + first
    return {"dense_flops": dense, "sparse_flops": sparse, "pisa_flops": pisa,
            "sparse_ratio": sparse / dense, "pisa_ratio": pisa / dense,
            "overhead_ratio": (pisa - sparse) / dense}


VARIANTS = {"sparse_only": P.PisaVariant.SparseOnly, "zeroth": P.PisaVariant.Zeroth,
            "block_first": P.PisaVariant.BlockFirst, "hybrid": P.PisaVariant.Hybrid,
            "global_centroid": P.PisaVariant.GlobalCentroid}
STRATEGIES = {"plain": P.RouterStrategy.Plain, "cov": P.RouterStrategy.CovarianceAware}


# ------------------------------------------------------------ generation --
def generate(kind: str, seed: int, heads: int, L: int, d: int, std: float = 1.0,
             clusters: int = 16, concentration: float = 2.0, noise_std: float = 0.15,
             device: str = "cuda") -> tuple:
    """Synthetic [H][L][d] bundle with the reference generators' structure
    (generate.hpp:104-190): gaussian N(0, std^2), or clustered keys around
    `clusters` centres per head (contiguous runs), queries drawn around a subset
    of the centres scaled by `concentration`, values gaussian."""
    g = torch.Generator(device=device).manual_seed(seed)
    shape = (heads, L, d)
    if kind == "gaussian":
        return tuple(std * torch.randn(shape, generator=g, device=device) for _ in range(3))
    if kind != "clustered":
        raise P.InvalidDimension(f"InvalidDimension: unknown generator {kind}")
    if clusters < 1:
        raise P.DegenerateScale("DegenerateScale: clusters must be >= 1")
    ctr = torch.randn((heads, clusters, d), generator=g, device=device)
    run = -(-L // clusters)
    zi = torch.clamp(torch.arange(L, device=device) // run, max=clusters - 1)
    k = ctr[:, zi] + noise_std * torch.randn(shape, generator=g, device=device)
    sub = torch.randint(0, clusters, (heads, max(1, clusters // 4)), generator=g, device=device)
    pick = torch.gather(sub, 1, torch.randint(0, sub.shape[1], (heads, L), generator=g, device=device))
    q = concentration * torch.gather(ctr, 1, pick.unsqueeze(-1).expand(heads, L, d)) + \
        torch.randn(shape, generator=g, device=device)
    v = torch.randn(shape, generator=g, device=device)
    return q, k, v


def _bundle(args):
    if getattr(args, "input", None):
        q, k, v, _ = pqkv.read_bundle(args.input)
        return tuple(torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda() for x in (q, k, v))
    return generate(args.kind, args.seed, args.heads, args.len, args.dim, args.std, args.clusters,
                    args.concentration, args.noise_std)


def _dense_fp32(q, k, v, scale: float, chunk: int = 2048) -> torch.Tensor:
    """Dense softmax attention in fp32 on the GPU, row chunks ([H][L][d])."""
    out = torch.empty_like(q, dtype=torch.float32)
    for r0 in range(0, q.shape[1], chunk):
        s = torch.einsum("hld,hmd->hlm", q[:, r0:r0 + chunk].float(), k.float()) * scale
        out[:, r0:r0 + chunk] = torch.softmax(s, -1) @ v.float()
    return out


# -------------------------------------------------------------- commands --
def _run_cell(qb, kb, vb, rc, dense) -> dict:
    """run_cell (pisa_cli.cpp:146-192): one (variant, sparsity) over all heads."""
    H, L, d = qb.shape
    variant = VARIANTS[rc.variant]
    router = P.RouterOptions(strategy=STRATEGIES[rc.strategy], epsilon=rc.epsilon)
    cfg = P.AttentionConfig(block_size=rc.block, group_size=rc.group)
    ctx = P.Context.get(0)
    ctx.set_profiling(True)
    ctx.read_profile()
    t0 = time.perf_counter()
    res = P.pisa_multihead(P.TensorBundle(qb, kb, vb), rc.sparsity, router, variant, cfg,
                           rc.streaming, out_dtype=torch.float32, diagnostics=False)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    prof = ctx.read_profile()
    ctx.set_profiling(False)
    out = torch.stack([h.output for h in res.heads]).double()
    ref = dense.double()
    diff = out - ref
    per_head_l1 = (diff.abs().sum((1, 2)) / ref.abs().sum((1, 2)).clamp_min(1e-300)).tolist()
    fl = flop_model(L, d, rc.block, res.k, variant) if L % rc.block == 0 else None
    ms = lambda *names: sum(prof.get(n, (0.0, 0))[0] for n in names)
    return {
        "sparsity_realized": res.sparsity_realized,
        "l1_rel": float(diff.abs().sum() / ref.abs().sum()),
        "l2_rel": float(diff.pow(2).sum().sqrt() / ref.pow(2).sum().sqrt()),
        "max_abs": float(diff.abs().max()),
        "per_head_l1": per_head_l1,
        "flops_ratio": fl["pisa_ratio"] if fl else None,
        "flops_sparse_ratio": fl["sparse_ratio"] if fl else None,
        "flops_overhead_ratio": fl["overhead_ratio"] if fl else None,
        "wall": wall,
        "wall_prepare": ms("block_stats_kernel", "hbar_reduce_kernel", "block_norms_kernel"),
        "wall_select": ms("select_kernels", "pairing_kernels"),
        "wall_attention": ms("fused_attn_kernel"),
    }


def cmd_gen(args) -> int:
    if args.len % args.block:
        raise P.BlockDivisibility(f"BlockDivisibility: seq_len {args.len} must be divisible by block "
                                  f"size {args.block}")
    q, k, v = generate(args.kind, args.seed, args.heads, args.len, args.dim, args.std, args.clusters,
                       args.concentration, args.noise_std)
    nbytes = pqkv.write_bundle(args.out, q, k, v, args.dtype)
    print(json.dumps({"path": args.out, "bytes": nbytes, "dtype": args.dtype, "kind": args.kind,
                      "seed": args.seed, "num_heads": args.heads, "seq_len": args.len,
                      "head_dim": args.dim, "generator": "torch"}))
    return 0


def cmd_run(args) -> int:
    q, k, v = _bundle(args)
    qb, kb, vb = (x.to(torch.bfloat16) for x in (q, k, v))
    H, L, d = qb.shape
    t0 = time.perf_counter()
    dense = _dense_fp32(qb, kb, vb, P.AttentionConfig().resolved_scale(d))
    mx = _run_cell(qb, kb, vb, args, dense)
    wall = (time.perf_counter() - t0) * 1e3
    z = args.deterministic
    print(json.dumps({
        "variant": args.variant, "strategy": args.strategy, "seq_len": L, "head_dim": d,
        "num_heads": H, "block_size": args.block, "group_size": args.group,
        "sparsity_requested": args.sparsity, "sparsity_realized": mx["sparsity_realized"],
        "l1_rel": mx["l1_rel"], "l2_rel": mx["l2_rel"], "max_abs": mx["max_abs"],
        "flops_ratio": mx["flops_ratio"], "flops_sparse_ratio": mx["flops_sparse_ratio"],
        "flops_overhead_ratio": mx["flops_overhead_ratio"],
        "wall_ms": 0.0 if z else wall, "wall_ms_prepare": 0.0 if z else mx["wall_prepare"],
        "wall_ms_select": 0.0 if z else mx["wall_select"],
        "wall_ms_attention": 0.0 if z else mx["wall_attention"]}))
    return 0


def _fmt(x) -> str:  # pisa::fmt_double: shortest round-trip
    return repr(float(x))


def cmd_sweep(args) -> int:
    """cmd_sweep (pisa_cli.cpp:268-360): CSV rows in fixed (seed, length,
    sparsity, variant, head) order; failed cells keep their row with status."""
    rows = ["method,strategy,seed,head,seq_len,block_size,sparsity_requested,sparsity_realized,"
            "l1_rel,l2_rel,max_abs,flops_ratio,wall_ms,status"]
    seeds = [0] if args.input else args.seeds
    lengths = [0] if args.input else args.lengths
    for seed in seeds:
        for L in lengths:
            a = argparse.Namespace(**vars(args))
            a.seed, a.len = seed, L
            q, k, v = _bundle(a)
            qb, kb, vb = (x.to(torch.bfloat16) for x in (q, k, v))
            H, LL, d = qb.shape
            dense = _dense_fp32(qb, kb, vb, P.AttentionConfig().resolved_scale(d))
            for sp in args.sparsities:
                for var in args.variants:
                    c = argparse.Namespace(**vars(args))
                    c.sparsity, c.variant = sp, var
                    try:
                        mx = _run_cell(qb, kb, vb, c, dense)
                        for h in range(H):
                            rows.append(",".join([var, args.strategy, str(seed), str(h), str(LL),
                                                  str(args.block), _fmt(sp),
                                                  _fmt(mx["sparsity_realized"]),
                                                  _fmt(mx["per_head_l1"][h]), _fmt(mx["l2_rel"]),
                                                  _fmt(mx["max_abs"]),
                                                  _fmt(mx["flops_ratio"] or 0.0),
                                                  _fmt(0.0 if args.deterministic else mx["wall"]),
                                                  "ok"]))
                    except P.Error as e:
                        status = type(e).__name__
                        for h in range(H):
                            rows.append(",".join([var, args.strategy, str(seed), str(h), str(LL),
                                                  str(args.block), _fmt(sp), "", "", "", "", "", "",
                                                  status]))
    text = "\n".join(rows) + "\n"
    if args.out in (None, "-"):
        sys.stdout.write(text)
    else:
        with open(args.out, "w") as f:
            f.write(text)
    return 0


def cmd_bench(args) -> int:
    """cmd_bench (pisa_cli.cpp:703-767) on the GPU: dense attention vs PISA
    Hybrid, medians over `reps` after one warmup, CUDA-event timed."""
    if args.len % args.block and not args.ragged:
        raise P.BlockDivisibility("BlockDivisibility: seq_len must be divisible by block size")
    q, k, v = generate(args.kind, args.seed, args.heads, args.len, args.dim, args.std, args.clusters,
                       args.concentration, args.noise_std)
    qb, kb, vb = (x.to(torch.bfloat16).unsqueeze(0) for x in (q, k, v))
    del q, k, v
    router = STRATEGIES[args.strategy]
    kw = dict(sparsity=args.sparsity, variant=P.PisaVariant.Hybrid, router=router,
              epsilon=args.epsilon, block_size=args.block, group_size=args.group,
              ragged=args.ragged)
    ctx = P.Context.get(0)
    dense_ms, hybrid_ms = [], []
    phases = {"prepare": 0.0, "select": 0.0, "attention": 0.0}
    ev = lambda: torch.cuda.Event(enable_timing=True)
    for rep in range(args.reps + 1):
        a, b_ = ev(), ev()
        a.record()
        torch.nn.functional.scaled_dot_product_attention(qb, kb, vb)
        b_.record()
        ctx.set_profiling(rep > 0)
        c, d_ = ev(), ev()
        c.record()
        P.fwd(qb, kb, vb, **kw)
        d_.record()
        torch.cuda.synchronize()
        if rep == 0:
            continue
        prof = ctx.read_profile()
        ctx.set_profiling(False)
        dense_ms.append(a.elapsed_time(b_))
        hybrid_ms.append(c.elapsed_time(d_))
        g = lambda *n: sum(prof.get(x, (0.0, 0))[0] for x in n)
        phases["prepare"] += g("block_stats_kernel", "hbar_reduce_kernel", "block_norms_kernel")
        phases["select"] += g("select_kernels", "pairing_kernels")
        phases["attention"] += g("fused_attn_kernel")
    dm, hm = statistics.median(dense_ms), statistics.median(hybrid_ms)
    print(json.dumps({
        "seq_len": args.len, "head_dim": args.dim, "num_heads": args.heads, "block_size": args.block,
        "group_size": args.group, "sparsity": args.sparsity, "dtype": "bf16", "accum": "f32",
        "reps": args.reps, "dense_ms": dm, "dense_impl": "torch SDPA (cuDNN / flash)",
        "hybrid_ms": hm, "speedup": dm / hm,
        "phase_prepare_ms": phases["prepare"] / args.reps,
        "phase_select_ms": phases["select"] / args.reps,
        "phase_attention_ms": phases["attention"] / args.reps,
        "strategy": args.strategy, "device": torch.cuda.get_device_name(0)}))
    return 0


# ------------------------------------------------------------------ main --
def _csv(tp):
    return lambda s: [tp(x) for x in s.split(",") if x]


def _gen_opts(p, seed=True):
    p.add_argument("--kind", default="gaussian", choices=["gaussian", "clustered"])
    if seed:
        p.add_argument("--seed", type=int, default=0)
    p.add_argument("--heads", type=int, default=2)
    p.add_argument("--len", type=int, default=4096)
    p.add_argument("--dim", type=int, default=64)
    p.add_argument("--std", type=float, default=1.0)
    p.add_argument("--clusters", type=int, default=16)
    p.add_argument("--concentration", type=float, default=2.0)
    p.add_argument("--noise-std", dest="noise_std", type=float, default=0.15)


def _run_opts(p, sparsity=True):
    p.add_argument("--variant", default="hybrid", choices=list(VARIANTS))
    p.add_argument("--strategy", default="plain", choices=list(STRATEGIES))
    if sparsity:
        p.add_argument("--sparsity", type=float, default=0.75)
    p.add_argument("--block", type=int, default=64)
    p.add_argument("--group", type=int, default=8)
    p.add_argument("--epsilon", type=float, default=1e-6)
    p.add_argument("--streaming", action="store_true")
    p.add_argument("--deterministic", action="store_true")
    p.add_argument("--ragged", action="store_true", help="allow L % block != 0 (GPU-path extension)")


# ----------------------------------------------------------------- verify --
# The reference's invariant suite (cmd_verify, pisa_cli.cpp:668-693) on the GPU
# path: the same checks, at the GPU path's shapes (block 64, d 64 / 128; the
# reference runs them at block 16, d 16-32) and with the bf16 tolerance of
# north_star (max-abs <= 2e-2, cosine >= 0.999) where it compares against a
# dense or fp64 computation. "cancellation" (a BlockFirst property) has no
# GPU-path counterpart: BlockFirst is not on the GPU path.
VERIFY_ATOL, VERIFY_COS = 2e-2, 0.999


def _close(got: torch.Tensor, ref: torch.Tensor):
    g, r = got.double().flatten(), ref.double().flatten()
    err = float((g - r).abs().max().item())
    cos = float((g @ r / (g.norm() * r.norm())).item())
    return err, cos


def _dense_fp32(q, k, v, scale):
    s = scale * (q.float() @ k.float().transpose(-1, -2))
    return torch.softmax(s, -1) @ v.float()


def _verify_inputs(kind: str, seed: int, L: int, d: int):
    from .generate import gen_clustered, gen_gaussian
    gen = gen_clustered if kind == "clustered" else gen_gaussian
    return tuple(x.cuda() for x in gen(seed, 1, L, d))


def check_oracle_equivalence(seeds: int):
    from .analysis import pisa_fp64
    worst_err, worst_cos = 0.0, 1.0
    for s in range(seeds):
        for d in (64, 128):
            q, k, v = _verify_inputs("clustered", s, 1024, d)
            for name, var in (("sparse_only", P.PisaVariant.SparseOnly), ("zeroth", P.PisaVariant.Zeroth),
                              ("hybrid", P.PisaVariant.Hybrid)):
                o, ex = P.fwd(q[None], k[None], v[None], sparsity=0.75, variant=var, out_dtype=torch.float32,
                              return_plan=True)
                ref = pisa_fp64(q[0], k[0], v[0], ex["selected"][0, 0], name)
                err, cos = _close(o[0, 0], ref)
                worst_err, worst_cos = max(worst_err, err), min(worst_cos, cos)
    return ("oracle_equivalence", worst_err <= VERIFY_ATOL and worst_cos >= VERIFY_COS,
            f"max_abs={worst_err:.3e} min_cos={worst_cos:.7f} vs fp64 piecewise attention on the GPU plan")


def check_full_coverage(seeds: int):
    worst = 0.0
    for s in range(seeds):
        q, k, v = _verify_inputs("gaussian", s, 512, 64)
        dense = _dense_fp32(q[0], k[0], v[0], 64 ** -0.5)
        for var in (P.PisaVariant.SparseOnly, P.PisaVariant.Zeroth, P.PisaVariant.Hybrid,
                    P.PisaVariant.GlobalCentroid):
            o = P.fwd(q[None], k[None], v[None], sparsity=0.0, variant=var, out_dtype=torch.float32)
            worst = max(worst, _close(o[0, 0], dense)[0])
    return ("full_coverage", worst <= VERIFY_ATOL, f"max_abs={worst:.3e}")


def check_constant_key(seeds: int):
    worst = 0.0
    L, d, B = 1024, 64, 64
    for s in range(seeds):
        q, _, v = _verify_inputs("gaussian", s, L, d)
        g = torch.Generator().manual_seed(s + 7777)
        kb = torch.randn((L // B, d), generator=g).to(torch.bfloat16).cuda()
        k = kb.repeat_interleave(B, 0)[None]
        dense = _dense_fp32(q[0], k[0], v[0], d ** -0.5)
        for var in (P.PisaVariant.Zeroth, P.PisaVariant.Hybrid):
            o = P.fwd(q[None], k[None], v[None], sparsity=0.75, variant=var, out_dtype=torch.float32)
            worst = max(worst, _close(o[0, 0], dense)[0])
    return ("constant_key_exactness", worst <= VERIFY_ATOL, f"max_abs={worst:.3e}")


def _normalized(seed: int, L: int, d: int):
    q, k, v = _verify_inputs("clustered", seed, L, d)
    q = (q.double() / q.double().norm(dim=-1, keepdim=True)).to(torch.bfloat16)
    k = (k.double() / k.double().norm(dim=-1, keepdim=True)).to(torch.bfloat16)
    return q, k, v


def check_theorem1(seeds: int):
    from .analysis import theorem1_check
    viol, slack = 0, 0.0
    for s in range(seeds):
        q, k, v = _normalized(s, 1024, 64)
        _, ex = P.fwd(q[None], k[None], v[None], sparsity=0.875, return_plan=True)
        rep = theorem1_check(q[0], k[0], v[0], ex["selected"][0, 0])
        viol += rep.violations
        slack = max(slack, rep.max_slack_ratio)
    return ("theorem1", viol == 0, f"violations={viol} max_slack_ratio={slack:.4g} seeds={seeds}")


def check_jensen(seeds: int):
    from .analysis import jensen_check
    viol = 0
    for s in range(seeds):
        q, k, v = _normalized(s, 1024, 64)
        _, ex = P.fwd(q[None], k[None], v[None], sparsity=0.875, return_plan=True)
        viol += jensen_check(q[0], k[0], ex["selected"][0, 0])
    return ("jensen", viol == 0, f"violations={viol} seeds={seeds}")


def check_streaming(seeds: int):
    worst = 0.0
    for s in range(seeds):
        q, k, v = _verify_inputs("clustered", s, 1024, 64)
        st = P.compute_prepare(q, k, v)
        plan = P.select_topk_plain(st.q_bar, st.k_bar, 4, 64 ** -0.5)
        ref, _ = P.pisa_reference(q, k, v, plan, st, P.PisaVariant.Hybrid, out_dtype=torch.float32)
        stream, _ = P.pisa_streaming(q, k, v, plan, st, out_dtype=torch.float32)
        worst = max(worst, _close(stream, ref)[0])
    return ("streaming_equivalence", worst <= 1e-6, f"max_abs={worst:.3e}")


def check_router_properties():
    ok, notes = True, []
    q, k, v = _verify_inputs("clustered", 3, 1024, 64)
    st = P.compute_prepare(q, k, v)
    m = P.block_norms(q, k, v)
    scale = 0.25
    base = P.select_topk_covariance(st.q_bar, st.k_bar, m, 1e-6, 4, scale)
    scaled = P.select_topk_covariance(st.q_bar, st.k_bar, m * 37.5, 37.5e-6, 4, scale)
    if not torch.equal(base, scaled):
        ok = False
        notes.append("joint-(M,eps)-scaling changed the plan")
    zq = torch.zeros((1, 8, 64), device="cuda")  # (square: the GPU select scores N x N blocks)
    zk = torch.zeros((1, 8, 64), device="cuda")
    tie = P.select_topk_plain(zq, zk, 3, scale)
    if not bool((tie == torch.tensor([0, 1, 2], device="cuda", dtype=tie.dtype)).all()):
        ok = False
        notes.append("tie-break mismatch")
    plain = P.select_topk_plain(st.q_bar, st.k_bar, 4, scale)
    cov_const = P.select_topk_covariance(st.q_bar, st.k_bar, torch.full_like(m, 2.0), 1e-6, 4, scale)
    if not torch.equal(plain, cov_const):
        ok = False
        notes.append("constant-M covariance plan differs from plain")
    return ("router_properties", ok, "; ".join(notes) if notes else "all router invariants hold")


VERIFY_CHECKS = ("oracle_equivalence", "full_coverage", "constant_key_exactness", "theorem1", "jensen",
                 "streaming_equivalence", "router_properties")


def cmd_verify(args) -> int:
    """cmd_verify (pisa_cli.cpp:668-693): each check prints pass / FAIL and a
    detail; exit 0 when all pass, 1 on a failure, 2 for an unknown check."""
    if args.only and args.only not in VERIFY_CHECKS:
        sys.stderr.write(f"unknown check: {args.only}\n")
        return 2
    run = {"oracle_equivalence": lambda: check_oracle_equivalence(min(args.seeds, 3)),
           "full_coverage": lambda: check_full_coverage(min(args.seeds, 5)),
           "constant_key_exactness": lambda: check_constant_key(min(args.seeds, 5)),
           "theorem1": lambda: check_theorem1(args.seeds),
           "jensen": lambda: check_jensen(min(args.seeds, 20)),
           "streaming_equivalence": lambda: check_streaming(min(args.seeds, 5)),
           "router_properties": check_router_properties}
    results = [run[n]() for n in VERIFY_CHECKS if not args.only or args.only == n]
    ok = True
    for name, passed, detail in results:
        print(f"{'pass  ' if passed else 'FAIL  '}{name}  ({detail})")
        ok = ok and passed
    print("verify: all checks passed" if ok else "verify: FAILURES")
    return 0 if ok else 1


def main(argv: List[str] | None = None) -> int:
    ap = argparse.ArgumentParser(prog="pisa-b200", description=__doc__.split("\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("gen", help="Generate a PQKV tensor file")
    _gen_opts(g)
    g.add_argument("--dtype", default="f32", choices=list(pqkv.TAG_OF))
    g.add_argument("--block", type=int, default=64)
    g.add_argument("--out", required=True)
    r = sub.add_parser("run", help="Run one configuration, print JSON metrics")
    r.add_argument("--in", dest="input")
    _gen_opts(r)
    _run_opts(r)
    s = sub.add_parser("sweep", help="Sweep a grid, emit CSV")
    _gen_opts(s, seed=False)
    _run_opts(s, sparsity=False)
    s.add_argument("--lengths", type=_csv(int), default=[1024, 2048])
    s.add_argument("--sparsities", type=_csv(float), default=[0.5, 0.75, 0.875])
    s.add_argument("--variants", type=_csv(str), default=["hybrid"])
    s.add_argument("--seeds", type=_csv(int), default=[0])
    s.add_argument("--in", dest="input")
    s.add_argument("--out", default="-")
    b = sub.add_parser("bench", help="Phase benchmark (GPU events)")
    _gen_opts(b)
    _run_opts(b)
    b.add_argument("--reps", type=int, default=5)
    vf = sub.add_parser("verify", help="Invariant suite on the GPU path")
    vf.add_argument("--only", default="", help="run one check (" + ", ".join(VERIFY_CHECKS) + ")")
    vf.add_argument("--seeds", type=int, default=5)
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    try:
        if args.cmd in ("run", "sweep", "bench"):
            for v in ([args.variant] if args.cmd != "sweep" else args.variants):
                if v not in VARIANTS:
                    raise P.InvalidDimension(f"InvalidDimension: unknown variant {v}")
        return {"gen": cmd_gen, "run": cmd_run, "sweep": cmd_sweep, "bench": cmd_bench,
                "verify": cmd_verify}[args.cmd](args)
    except P.Error as e:  # exit codes of pisa_cli.cpp:844-851
        sys.stderr.write(f"error: {e}\n")
        return {P.ErrorKind.Validation: 2, P.ErrorKind.Io: 3, P.ErrorKind.Invariant: 1}[e.kind]
    except Exception as e:  # noqa: BLE001
        sys.stderr.write(f"error: {e}\n")
        return 1


if __name__ == "__main__":
    sys.exit(main())
