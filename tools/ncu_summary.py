"""Summarise ncu --set full reports (one or more kernels each) into key metrics + top stalls.

    python tools/ncu_summary.py report.ncu-rep [...] > summary.txt
"""
import csv
import io
import subprocess
import sys

KEYS = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "launch__registers_per_thread",
        "smsp__inst_executed.sum"]


def main():
    for rep in sys.argv[1:]:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        if len(rows) < 3:
            continue
        hdr, units = rows[0], rows[1]
        print(f"== {rep}")
        for vals in rows[2:]:
            d = dict(zip(hdr, vals))
            u = dict(zip(hdr, units))
            for k in KEYS:
                if k in d:
                    print(f"  {k} = {d[k]} {u.get(k, '')}".rstrip())
            stalls = {k.split("issue_stalled_")[1]: float(v) for k, v in d.items()
                      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and
                      not k.endswith("_not_issued") and v not in ("", "0")}
            tot = sum(stalls.values()) or 1.0
            top = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
            print("  top stall reasons (pc sampling share): " +
                  ", ".join(f"{k} {v / tot:.3f}" for k, v in top))
            print()


if __name__ == "__main__":
    main()
