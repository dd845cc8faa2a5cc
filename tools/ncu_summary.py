"""Summarise ncu reports (run here, no GPU): per report the kernel, duration,
DRAM bytes, throughputs, occupancy and top stall reasons.

    python tools/ncu_summary.py gpurun_out/prof_*.ncu-rep > profiles/rXX_ncu_summary.txt
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return [dict(zip(rows[0], r)) for r in rows[2:]], dict(zip(rows[0], rows[1]))


def main():
    for path in sys.argv[1:]:
        recs, units = raw(path)
        for d in recs:
            print(f"== {path}: {d.get('Kernel Name', '')[:110]}")
            for k in KEYS:
                if k in d:
                    print(f"   {k:70s} {d[k]:>16s} {units.get(k, '')}")
            st = [(float(v), k) for k, v in d.items()
                  if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                  and v.replace('.', '', 1).isdigit()]
            for v, k in sorted(st, reverse=True)[:5]:
                print(f"   stall {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:30s} {v:.2f}")


if __name__ == "__main__":
    main()
