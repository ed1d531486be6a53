"""Summarise an ncu report: python profiles/ncu_summary.py <report.ncu-rep>"""
import csv
import io
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_hit_rate.pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum", "launch__grid_size", "launch__block_size",
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"# {name[:100]}")
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                print(f"{w:70s} {vals[i]:>18s} {units[i]}")
    stalls = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv", "--section", "WarpStateStats"],
                            capture_output=True, text=True).stdout
    for r in csv.reader(io.StringIO(stalls)):
        if len(r) > 3 and "Stall" in r[-4]:
            print("  ", r[-4], r[-2], r[-1])


if __name__ == "__main__":
    main(sys.argv[1])
