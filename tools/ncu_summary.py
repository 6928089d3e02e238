"""Summarise an ncu report (raw page) into the metrics we judge kernels by."""
import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_shared_mem",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__average_warp_latency_issue_stalled_barrier",
]


def main(path, pattern=""):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        if pattern and pattern not in name:
            continue
        print("===", name[:100])
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k:90s} {r[i]:>16s} {units[i]}")
        stall = [(h[i], r[i]) for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled_")
                 and not h[i].endswith("_not_issued")]
        vals = []
        for k, v in stall:
            try:
                vals.append((float(v.replace(",", "")), k))
            except ValueError:
                pass
        vals.sort(reverse=True)
        print("  top stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')}={v:.0f}" for v, k in vals[:8]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
