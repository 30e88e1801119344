"""Summarise an ncu report: key raw metrics (with units) and the top stall
sources from the source page. Usage: python tools/ncu_summary.py rep.ncu-rep [-k name]"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers", "sm__cycles_active.avg", "smsp__cycles_active.avg",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size",
]


def raw(rep, kname=None):
    cmd = ["ncu", "-i", rep, "--page", "raw", "--csv"]
    if kname:
        cmd += ["-k", kname]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print("==", name[:100])
        for kk in KEYS:
            if kk in hdr:
                i = hdr.index(kk)
                print(f"  {kk:90s} {r[i]:>16s} {units[i]}")
        stalls = [(h, r[i], units[i]) for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warp_latency_issue_stalled") or
                  (h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio"))]
        stalls = sorted(stalls, key=lambda x: -float(x[1] or 0))[:12]
        for h, v, u in stalls:
            print(f"  {h:90s} {v:>16s} {u}")


if __name__ == "__main__":
    rep = sys.argv[1]
    k = sys.argv[sys.argv.index("-k") + 1] if "-k" in sys.argv else None
    raw(rep, k)
