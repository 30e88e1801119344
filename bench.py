#!/usr/bin/env python3
"""PISA attention forward benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A step is one PISA forward (Hybrid, block 64, density 12.5 %) over the whole
workload: prepare (K1) -> select (K2) -> fused piecewise attention (K3). Default
workload: Wan2.1-14B 720p attention, B=1 H=40 L=75600 d=128 (BASELINE.json
configs[3]; it fits one B200). Heads are sharded across ranks (no data-path
collective); the reported latency is the max over ranks.

value = dense-equivalent TFLOPS of the whole job = H * 4 L^2 d / t.
Inputs (2.3 GB) are larger than L2 (126 MB), so no L2 flush between steps.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PISA attn fwd latency (ms) & dense-equiv TFLOPS at Wan2.1-14B shape, 1/2/4/8 B200"
WORKLOADS = {
    # name: (B, H, L, d, density, BASELINE.json config)
    "wan14b": (1, 40, 75600, 128, 0.125, "Wan2.1-14B 720p 81-frame video attention"),
    "wan13b": (1, 12, 32760, 128, 0.125, "Wan2.1-1.3B 480p 81-frame video attention"),
    "flux": (1, 24, 4608, 128, 0.125, "FLUX.1 1024px image DiT attention"),
    "sd35": (1, 24, 4429, 64, 0.125, "SD3.5-Medium 1024px joint attention (4096 image + 333 text tokens, d=64)"),
    "hunyuan": (1, 24, 118800, 128, 0.125, "HunyuanVideo 720p 129-frame attention"),
    "smoke": (1, 2, 4096, 64, 0.25, "CPU-oracle smoke"),
}


def flops_dense(L, d):
    return 4.0 * L * L * d  # analysis.hpp:322


def flops_fused(L, d, N, k):
    # exact + full Phase-2 scan + first-order + normalize, per head
    return 4.0 * L * k * 64 * d + 4.0 * L * N * d + 2.0 * L * d * d + L * d


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return j["bf16_tflops"], j["bf16_tflops_sustained"], j["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """SM clock + throttle reasons sampled during the timed region: NVML polled
    every 0.5 ms from a thread (so a few-millisecond region of image-size steps
    still gets samples), nvidia-smi at 100 ms when NVML is unavailable. The NVML
    device is found by the CUDA device's PCI bus id (NVML ignores
    CUDA_VISIBLE_DEVICES)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int, pci_bus_id: str | None = None):
        self.gpu = gpu_index
        self.pci = pci_bus_id
        self.proc = None
        self.lines = []
        self.samples = []  # (sm MHz, reasons bitmask) from NVML
        self.nv = None
        self.stop = threading.Event()

    def _nvml_handle(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = None
            if self.pci:
                try:
                    h = nv.nvmlDeviceGetHandleByPciBusId_v2(self.pci.encode())
                except Exception:
                    h = None
            if h is None:
                h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                         "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                         "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                         "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            self.nv = nv
            return h
        except Exception:
            return None

    def _poll(self, h):
        nv = self.nv
        while True:
            try:
                self.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                                     int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))))
            except Exception:
                pass
            if self.stop.wait(0.0005):
                break

    def __enter__(self):
        h = self._nvml_handle()
        if h is not None:
            self.t = threading.Thread(target=self._poll, args=(h,), daemon=True)
            self.t.start()
            time.sleep(0.005)  # a first sample before the timed work starts
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.nv is not None:
            self.stop.set()
            self.t.join(timeout=1)
            return
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        if self.nv is not None:
            for mhz, bits in self.samples:
                sm.append(mhz)
                for n in self.NAMES:
                    if bits & self.bits[n]:
                        reasons.add(n)
            mx = self.max_mhz
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(self.NAMES, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml 0.5 ms" if self.nv is not None else "nvidia-smi 100 ms"}


# ------------------------------------------------------------ CPU legs --
def cpu_reference_sample(wl, steps, warmup, log, data="gaussian", density=None):
    """Times the unmodified reference (oracle/_ref, compiled from /root/reference)
    on the host cores: prepare over a full head + route + pisa_streaming for a
    bounded range of query blocks (pisa_cli.cpp:728-729 semantics, accum F32).
    Inputs: head 0 of the GPU arm's bundle (gen_gaussian / gen_clustered seed 0,
    bf16-rounded), floored to whole blocks."""
    import numpy as np  # noqa: F401

    import oracle as O

    B, H, L, d, dens0, _ = WORKLOADS[wl]
    density = dens0 if density is None else density
    Lf = (L // 64) * 64  # the reference rejects L % 64 != 0 (attention.hpp:43-47)
    N = Lf // 64
    threads = os.cpu_count() or 1
    os.environ.setdefault("PISA_THREADS", str(threads))
    if not O.ref_available():
        O.build()
    R = O.ref()
    if data == "gaussian":  # head 0 of gen_gaussian(0, B*H, L, d) without the other heads
        q, k, v = O.gen_gaussian_head(0, B * H, L, d, 0, rows=Lf)
    else:  # gen_clustered draws head 0 first: a one-head bundle has the same head 0
        q, k, v = (x[0, :Lf].copy() for x in O.gen("clustered", 0, 1, L, d))
    # Bounded sample: prepare over the full head, routing + streaming attention for a
    # range of query blocks sized to ~2 s of CPU work. The full-head time is
    # extrapolated linearly in query blocks (heads are serial, engine.hpp:432, and
    # query blocks are independent, engine.hpp:272): t_head = t_prep + t_qb * N / n_qb.
    out = np.zeros((N * 64, d), np.float32)
    ms = np.zeros(3)

    def run(nqb):
        st = R.ref_bench_sample(q, k, v, Lf, d, 1.0 - density, 0, nqb, threads, out, ms)  # noqa: B023
        if st != 0:
            raise RuntimeError(f"ref_bench_sample status {st}")
        return ms.copy()

    m = run(16)
    per_block = max(1e-3, (m[1] + m[2]) / 16)
    qb1 = int(max(16, min(N, 2000.0 / per_block)))
    heads = []
    for i in range(warmup + steps):
        m = run(qb1)
        if i >= warmup:
            heads.append(m[0] + (m[1] + m[2]) * N / qb1)
    tm = statistics.median(heads)
    value = 4.0 * Lf * Lf * d / (tm * 1e-3) / 1e12  # dense-equivalent TFLOPS of one head
    sample = (f"head 0 of {wl} (the GPU arm's gen_{data} seed-0 bundle, bf16-rounded) floored to "
              f"L={Lf}: prepare over the full head + routing and Hybrid streaming (accum f32) for "
              f"query blocks [0,{qb1}) of {N}, extrapolated to the head (t_prep + t_blocks*N/{qb1}); "
              f"median of {len(heads)} after {warmup} warmup; PISA_THREADS={threads}")
    return {"value": value, "unit": "TFLOPS (dense-equivalent)", "cores": threads,
            "kind": "reference", "sample": sample, "ms_per_sample": tm,
            "lib": os.path.basename(R._path), "ms_per_head": tm}


def gen_inputs(P, kind, heads, L, d):
    """Host bf16 [heads][L][d] q, k, v: the reference's gen_gaussian / gen_clustered
    values (seed 0; generate.hpp:29-116) through pisa_b200_gen_* (bit-identical,
    tests/test_generate.py)."""
    import torch
    if kind == "gaussian":
        return P.gen_gaussian(0, heads, L, d, 1.0, dtype=torch.bfloat16)
    return P.gen_clustered(0, heads, L, d, 16, 2.0, 0.15, dtype=torch.bfloat16)


def plan_parity(P, q, k, v, plan, density, d):
    """The GPU's routing plan of every head against the CPU restatement of the
    reference's prepare + select_topk_plain at the workload's own (ragged) length
    (oracle, pinned to oracle/_ref in tests/test_oracle.py): rows that differ,
    and how many of them are near-ties (fp64 gap to the k-th score <= 1e-6 |s_k|)."""
    import concurrent.futures as cf

    import oracle as O
    from oracle import parity

    H, N, ksel = plan.shape
    scale = d ** -0.5

    def head(h):
        qf, kf, vf = (x[0, h].float().numpy() for x in (q, k, v))
        st = O.block_stats(kf, vf)
        qb = O.query_means(qf)
        return parity.classify_rows(plan[h], O.select_plain(qb, st[0], ksel, scale), qb, st[0], ksel, scale)

    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(min(H, os.cpu_count() or 1)) as ex:
        res = list(ex.map(head, range(H)))
    return {"plan_rows": H * N, "rows_differing": sum(r[0] for r in res),
            "near_tie_rows": sum(r[1] for r in res), "near_tie_swaps": sum(r[2] for r in res),
            "non_tie_rows": sum(len(r[3]) for r in res),
            "against": "oracle restatement of compute_block_stats + select_topk_plain at this L "
                       "(PARITY_r02.json: the unmodified reference at the floored length)",
            "seconds": round(time.perf_counter() - t0, 1)}


# ---------------------------------------------------------- GPU arm ----
def executed_flops(tiles, ctas, d, first_order=True):
    """Executed MMA FLOPs of the fused kernel from its device tile counter: every
    64-key tile (union block or centroid chunk, pair padding included) is an
    S = Q K^T and a P V over 128 query rows, plus one Q.H_bar per CTA."""
    return tiles * (4.0 * 128 * 64 * d) + (ctas * 2.0 * 128 * d * d if first_order else 0.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="wan14b", choices=list(WORKLOADS))
    ap.add_argument("--data", default="gaussian", choices=["gaussian", "clustered"])
    ap.add_argument("--density", type=float, default=None)
    ap.add_argument("--router", default="plain", choices=["plain", "covariance"],
                    help="routing strategy (the headline is plain; covariance adds K1c)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    args = ap.parse_args()
    warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test-only: exercise the multi-rank path on one GPU (every rank on cuda:0,
    # gloo instead of NCCL); timings from such a run mean nothing
    if os.environ.get("PISA_BENCH_SAME_DEVICE") == "1":
        local_rank = 0
    B, H, L, d, density, cfg_name = WORKLOADS[args.workload]
    if args.density is not None:
        density = args.density

    if args.impl == "reference":
        if rank != 0:
            return
        res = cpu_reference_sample(args.workload, args.steps, warmup, None, args.data, density)
        line = {"impl": "reference", "metric": METRIC, "value": res["value"], "unit": res["unit"],
                "n_gpus": args.gpus, "steps": args.steps, "warmup": warmup,
                "ms_per_step": res["ms_per_sample"] * H, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": f"synthetic gen_{args.data}(seed 0) rounded to bf16 (head 0 of the GPU arm's bundle)",
                "config": {"workload": f"{cfg_name} (bounded CPU sample)", "B": B, "H": H,
                           "L": L, "d": d, "density": density, "block": 64,
                           "variant": "hybrid", "router": "plain"},
                "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": res["value"], "unit": res["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist

    import paper_2602_01077_b200 as P

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        backend = os.environ.get("PISA_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    from paper_2602_01077_b200.sharding import Piece, unit_qblock_pieces

    N = -(-L // 64)
    k = P.sparsity_to_k(1.0 - density, N).k
    C2 = -(-N // 64)
    # (batch x head) sharding: contiguous head ranges per rank; when the heads do
    # not divide over the ranks, (head x query-block range) units
    even = (B * H) % world == 0
    if even:
        h0, h1 = rank * H // world, (rank + 1) * H // world
        pieces = [Piece(0, h0, h1, 0, N)]
    else:
        assert B == 1, "query-block sharding in bench.py assumes B == 1"
        pieces = unit_qblock_pieces(B, H, N, world, rank)
        h0, h1 = min(p.h0 for p in pieces), max(p.h1 for p in pieces)
    Hr = h1 - h0  # heads whose Q/K/V this rank holds

    # The reference's own synthetic bundle (gen_gaussian(seed 0, std 1) or
    # gen_clustered(seed 0, 16 clusters, concentration 2, noise 0.15), the CLI
    # defaults, pisa_cli.cpp:27-39), bf16-rounded, from the library's
    # bit-identical generator on the host cores; this rank's heads are uploaded.
    # The reference arm times the same values (head 0, floored to whole blocks).
    shape = (B, Hr, L, d)
    t_gen = time.perf_counter()
    host = gen_inputs(P, args.data, B * H, L, d)
    hq, hk, hv = (x[h0:h1].unsqueeze(0).pin_memory() for x in host)
    del host
    q, kk, v = (x.to(dev) for x in (hq, hk, hv))
    t_gen = time.perf_counter() - t_gen
    out = torch.empty(shape, device=dev, dtype=torch.bfloat16)
    ctx = P.Context.get(local_rank)
    kw = dict(sparsity=1.0 - density, variant=P.PisaVariant.Hybrid)
    if args.router == "covariance":
        kw["router"] = P.RouterStrategy.CovarianceAware

    def step():
        n = 0
        for pc in pieces:
            sl = (slice(None), slice(pc.h0 - h0, pc.h1 - h0))
            rng = None if (pc.qb0, pc.qb1) == (0, N) else (pc.qb0, pc.qb1)
            P.fwd(q[sl], kk[sl], v[sl], out[sl], q_blocks=rng, **kw)
            n += ctx.last_launch_count()
        return n

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()

    # L2 (126 MB on B200): inputs larger than it stream from HBM every step;
    # smaller ones get a flush between timed steps
    in_bytes = 3 * B * Hr * L * d * 2
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if in_bytes < 2 * (126 << 20) else None
    l2_note = (f"inputs {in_bytes / 1e9:.2f} GB per rank > 126 MB L2, no flush" if flush is None else
               f"inputs {in_bytes / 1e6:.0f} MB per rank fit in L2: 512 MB written between timed steps")

    stream = torch.cuda.current_stream()

    def timed_steps(fn, n):
        """Average ms of n steps: back to back, or each alone after an L2 flush."""
        if flush is None:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(n):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / n
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for ea, eb in evs:
            flush.zero_()
            ea.record(stream)
            fn()
            eb.record(stream)
        torch.cuda.synchronize()
        return sum(ea.elapsed_time(eb) for ea, eb in evs) / n

    # Per-kernel events (the library's profiling mode) cost ~2 us each on the
    # device: invisible in a 26 ms step, +15 % on a 0.16 ms FLUX step. Short
    # steps are therefore timed without them, and the per-kernel durations come
    # from a profiling pass of the same steps right after the timed region.
    ctx.set_profiling(False)
    est_ms = timed_steps(step, 1)
    inline_prof = est_ms >= 5.0

    # timed region
    ctx.set_profiling(inline_prof)
    ctx.read_profile()
    launches = 0
    props = torch.cuda.get_device_properties(dev)
    pci = None
    if hasattr(props, "pci_bus_id"):
        pci = f"{getattr(props, 'pci_domain_id', 0):08X}:{props.pci_bus_id:02X}:{getattr(props, 'pci_device_id', 0):02X}.0"
    with ClockSampler(local_rank, pci) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        # inputs that fit in L2: each step timed alone, an L2-sized buffer
        # written between steps (outside the events)
        counted = []
        step_ms = timed_steps(lambda: counted.append(step()), args.steps)
        launches = sum(counted)
        if world > 1:
            dist.barrier()
    if not inline_prof:  # per-kernel durations: the same steps again, with events
        ctx.set_profiling(True)
        ctx.read_profile()
        timed_steps(step, args.steps)
    ctx.set_profiling(False)
    prof = ctx.read_profile()
    tiles = ctx.fused_tiles() / args.steps  # per step (all pieces)
    graph_ms = None
    if not inline_prof:
        # the same step replayed from a CUDA graph (P.fwd is stream-ordered and
        # capture-safe with profiling and check_finite off): launch gaps removed
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            step()
        stream.wait_stream(side)
        cg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(cg):
            step()
        torch.cuda.synchronize()
        graph_ms = timed_steps(cg.replay, args.steps)
        del cg
    ctas = B * sum((p.h1 - p.h0) * (-(-(p.qb1 - p.qb0) // 2)) for p in pieces)
    exec_flops = executed_flops(tiles, ctas, d)
    union_ratio = (tiles / ctas - 2 * (-(-C2 // 2))) / k  # union blocks (incl. pair padding) per tile / k
    t_ms = step_ms
    t = torch.tensor([t_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms = float(t.item())
    clocks = clk.summary()

    total_dense = H * B * flops_dense(L, d)
    value = total_dense / (t_ms * 1e-3) / 1e12
    # roofline of the dominant kernel (fused) on this rank: against the measured
    # BURST dense bf16 peak (MEASURED_PEAKS.json bf16_tflops); the sustained
    # figure (cuBLAS back to back under the power cap) is reported beside it
    peak_burst, peak_sus, hbm, peak_src = load_peaks()
    capped = "sw_power_cap" in (clocks.get("reasons") or [])
    peak = peak_burst
    peak_src = f"{peak_src} burst (bf16_tflops); sustained in peak_sustained / frac_sustained"
    fused_ms, fused_n = prof.get("fused_attn_kernel", (0.0, 0))
    fused_avg = fused_ms / max(1, fused_n)
    fused_step = fused_ms / args.steps  # one launch per piece, pieces per step
    alg = B * flops_fused(L, d, N, k) * sum((p.h1 - p.h0) * (p.qb1 - p.qb0) for p in pieces) / N
    achieved = alg / (fused_step * 1e-3) / 1e12 if fused_step > 0 else None
    executed = exec_flops / (fused_step * 1e-3) / 1e12 if fused_step > 0 else None
    # DRAM bytes per launch from the committed ncu --set full capture of this
    # workload (profiles/traffic.json names the capture); not measured live
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                tj = json.load(f)
            ent = tj.get(args.workload, {})
            traffic = ent.get("fused_attn_kernel_bytes")
            if traffic is not None:
                traffic_src = ent.get("source") or (
                    f"not measured in this run: dram__bytes_read.sum + dram__bytes_write.sum of "
                    f"fused_attn_kernel from the {ent.get('round', '?')} ncu --set full capture "
                    f"(profiles/{ent.get('round', '?')}_ncu_summary.md), default gaussian workload")
        except Exception:
            traffic = None
    # The stream that bounds the fused kernel (profiles/r02_k3_variants.log,
    # tools/k3_variants/README.md): K and V tiles from L2 into shared memory,
    # 2 x 64 rows x d x 2 B per 64-key tile (the tile counter is live)
    kv_step = tiles * 2 * 64 * d * 2
    kv_bytes = kv_step / max(1, len(pieces))
    kv_tbps = kv_step / (fused_step * 1e-3) / 1e12 if fused_step > 0 else None
    kernels = {n: {"ms_per_launch": ms / max(1, c), "launches": c,
                   "share": ms / max(1e-9, sum(x[0] for x in prof.values()))}
               for n, (ms, c) in prof.items()}
    # HBM rooflines of the prepare (K1) and select (K2) kernels, SURVEY §8(d):
    # K1 reads Q, K, V (3 L d 2 B) and writes k_bar / v_hat / q_bar fp32 and the
    # bf16 k_bar / v_hat copies (3 N d 4 + 2 N d 2 B) per head; K2 reads q_bar /
    # k_bar (2 N d 4 B) and writes the plan (N k 4 B) per head
    units = B * sum((p.h1 - p.h0) for p in pieces)
    k1_bytes = units * (3 * L * d * 2 + 3 * N * d * 4 + 2 * N * d * 2)
    k2_bytes = units * (2 * N * d * 4 + N * k * 4)
    hbm_rooflines = {}
    for name, nbytes, extra in (("block_stats_kernel", k1_bytes, {}),
                                ("select_kernels", k2_bytes, {"fp32_flops_per_launch": units * 2.0 * N * N * d})):
        ms, c = prof.get(name, (0.0, 0))
        if c:
            gbs = nbytes / (ms / c * 1e-3) / 1e9
            hbm_rooflines[name] = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                                   "algorithmic_bytes_per_launch": nbytes, "ms_per_launch": ms / c, **extra}

    # dense attention baseline on the same B200 (cuDNN/flash SDPA via torch), this rank's heads
    dense = None
    if not args.no_dense:
        import torch.nn.functional as F
        try:
            F.scaled_dot_product_attention(q, kk, v)
            torch.cuda.synchronize()
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(3):
                F.scaled_dot_product_attention(q, kk, v)
            a1.record(stream)
            torch.cuda.synchronize()
            dms = a0.elapsed_time(a1) / 3
            dense = {"impl": "torch SDPA (cuDNN / flash backend)", "ms": dms,
                     "pisa_speedup": dms / t_ms, "tflops": Hr * B * flops_dense(L, d) / (dms * 1e-3) / 1e12}
        except Exception as e:  # noqa: BLE001
            dense = {"error": str(e)[:200]}

    # end to end through the C-ABI host path: pinned host buffers, H2D + D2H timed
    e2e = None
    if not args.no_e2e:
        ho = torch.empty(shape, dtype=torch.bfloat16).pin_memory()
        for _ in range(2):
            P.fwd_host(hq, hk, hv, ho, device=local_rank, **kw)
        if world > 1:
            dist.barrier()
        ts = time.perf_counter()
        for _ in range(args.steps):
            P.fwd_host(hq, hk, hv, ho, device=local_rank, **kw)
        te = (time.perf_counter() - ts) * 1e3 / args.steps
        tt = torch.tensor([te], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        te = float(tt.item())
        hs = torch.tensor([Hr], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(hs)
        nb = 2 * B * int(hs.item()) * L * d  # bytes of one tensor over all ranks
        e2e = {"value": total_dense / (te * 1e-3) / 1e12, "unit": "TFLOPS (dense-equivalent)",
               "ms_per_step": te, "h2d_bytes_per_step": 3 * nb, "d2h_bytes_per_step": nb,
               "path": "pisa_b200_fwd_host (pinned host Q/K/V/O; H2D, compute, D2H overlapped per head chunk)"
                       + ("" if even else "; whole heads of each rank's span (partial heads computed in full)")}

    # routing plan of the timed inputs vs the CPU restatement of the reference
    # (every head; near-tie swaps counted), rank 0 at N = 1
    parity_res = None
    if rank == 0 and world == 1 and not args.no_cpu and args.router == "plain":
        try:
            _, exq = P.fwd(q, kk, v, return_plan=True, **kw)
            parity_res = plan_parity(P, hq, hk, hv, exq["selected"][0].cpu().numpy(), density, d)
            del exq
        except Exception as e:  # noqa: BLE001
            parity_res = {"error": str(e)[:200]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_reference_sample(args.workload, 3, 1, None, args.data, density)
            cpu.pop("ms_per_sample", None)
            cpu.pop("lib", None)
        except Exception as e:  # noqa: BLE001
            cpu = {"error": str(e)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOPS (dense-equivalent)",
            "n_gpus": world, "steps": args.steps, "warmup": warmup, "ms_per_step": t_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": f"synthetic gen_{args.data}(seed 0) values of the reference's generator, bf16-rounded",
            "input_generation_s": t_gen,
            "config": {"workload": cfg_name, "B": B, "H": H, "L": L, "d": d, "N": N, "k": k,
                       "density": density, "block": 64, "variant": "hybrid", "router": args.router,
                       "parallelism": (f"head-sharded x{world}" if even
                                       else f"head x query-block sharded x{world}"),
                       "heads_per_gpu": Hr, "pieces_rank0": [list(p) for p in pieces],
                       "l2": l2_note},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "kernel": "fused_attn_kernel", "kernel_ms": fused_avg,
                         "algorithmic_flops_per_launch": alg, "executed_flops_per_launch": exec_flops,
                         "executed_tflops": executed,
                         "executed_frac": (executed / peak) if executed else None,
                         "frac_sustained": (achieved / peak_sus) if achieved else None,
                         "executed_frac_sustained": (executed / peak_sus) if executed else None,
                         "power_capped": capped,
                         "union_over_k": union_ratio, "peak_source": peak_src, "peak_burst": peak_burst,
                         "l2_to_smem_kv": {"bytes_per_launch": kv_bytes, "achieved_TBps": kv_tbps,
                                           "note": "K/V tiles streamed L2 -> shared memory by TMA (live tile "
                                                   "count); on gaussian routing this stream, not the tensor "
                                                   "pipe, sets the kernel's time (tools/k3_variants/README.md)"},
                         "peak_sustained": peak_sus,
                         "kernel_timing": ("library events around each launch inside the timed region"
                                           if inline_prof else
                                           f"library events around each launch in a pass of the same "
                                           f"{args.steps} steps after the timed region (step < 5 ms)")},
            "kernels": kernels,
            "hbm_rooflines": hbm_rooflines,
            "plan_parity": parity_res,
            "graph": (None if graph_ms is None else
                      {"ms_per_step": graph_ms, "value": total_dense / (graph_ms * 1e-3) / 1e12,
                       "note": "the same step replayed from a CUDA graph (rank 0); not the headline value"}),
            "dense_baseline": dense,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
