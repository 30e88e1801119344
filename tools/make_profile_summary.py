"""Turns an ncu --set full report + launch-list CSV into profiles/<tag>_*.md/json.
Usage: python tools/make_profile_summary.py TAG gpurun_out/prof_TAG.ncu-rep gpurun_out/launches_TAG.csv"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "TMA bytes L2->SM"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
]


def main(tag, rep, launches):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary, {tag}", "",
             f"Source: `{os.path.basename(rep)}` (gpurun_out/, not committed); command:",
             "`ncu --set full --clock-control none --import-source on -k regex:... -s 4 -c 4 "
             "python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-dense` (Wan2.1-14B, 1 B200).",
             "Per-launch values (ncu replays each kernel; cold-cache, serialised).", ""]
    traffic = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        short = name.split("(")[0].split("::")[-1].split("<")[0]
        lines.append(f"## {short}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        vals = {}
        for key, label in METRICS:
            if key in hdr:
                i = hdr.index(key)
                lines.append(f"| {label} (`{key}`) | {r[i]} | {units[i]} |")
                vals[key] = (r[i], units[i])
        stalls = [(h, r[i]) for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warps_issue_stalled_") and
                  h.endswith("per_issue_active.ratio")]
        stalls = sorted(stalls, key=lambda x: -float(x[1] or 0))[:5]
        lines.append("")
        lines.append("Top stall reasons (warps per issue): " + ", ".join(
            f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} "
            f"{float(v):.2f}" for h, v in stalls))
        lines.append("")

        def tobytes(v):
            x, u = float(v[0]), v[1]
            return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        if "dram__bytes_read.sum" in vals:
            traffic[short] = tobytes(vals["dram__bytes_read.sum"]) + tobytes(vals["dram__bytes_write.sum"])
    # launch list
    if launches and os.path.exists(launches):
        with open(launches) as f:
            txt = f.read()
        body = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
        lr = list(csv.reader(io.StringIO(body)))
        h = lr[0]
        agg = {}
        for r in lr[1:]:
            if len(r) < len(h):
                continue
            k = r[h.index("Kernel Name")].split("(")[0].split("::")[-1]
            v = float(r[h.index("Metric Value")])
            agg.setdefault(k, []).append(v)
        tot = sum(sum(v) for v in agg.values())
        lines.append("## Launch list (gpu__time_duration.sum, `--clock-control none`)")
        lines.append("")
        lines.append("| kernel | launches | mean | share |")
        lines.append("|---|---|---|---|")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| {k} | {len(v)} | {sum(v)/len(v):.1f} | {sum(v)/tot*100:.1f}% |")
        unit = h.index("Metric Unit")
        lines.append("")
        lines.append(f"(unit: {lr[1][unit]})")
        with open(os.path.join(ROOT, "profiles", f"{tag}_launches.csv"), "w") as f:
            f.write(body)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    j = {}
    if os.path.exists(tp):
        j = json.load(open(tp))
    j["wan14b"] = {"round": tag, "fused_attn_kernel_bytes": traffic.get("fused_attn_kernel"),
                   "per_kernel_bytes": traffic,
                   "source": ("not measured in this run: dram__bytes_read.sum + dram__bytes_write.sum of "
                              f"fused_attn_kernel from the {tag} ncu --set full capture "
                              f"(profiles/{tag}_ncu_summary.md), default gaussian Wan2.1-14B workload")}
    json.dump(j, open(tp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
