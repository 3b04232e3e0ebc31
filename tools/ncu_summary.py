"""Key metrics of an ncu report (details page) as `name = value unit` lines.
usage: python tools/ncu_summary.py report.ncu-rep [kernel-regex]"""
import csv
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "Registers Per Thread", "Theoretical Occupancy",
        "Achieved Occupancy", "Executed Ipc Active", "Issue Slots Busy", "Executed Instructions",
        "Avg. Active Threads Per Warp", "Avg. Not Predicated Off Threads Per Warp",
        "L1/TEX Hit Rate", "L2 Hit Rate", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler", "No Eligible", "Branch Efficiency", "Grid Size", "Block Size",
        "Static Shared Memory Per Block"]


def main():
    kf = ["-k", "regex:" + sys.argv[2]] if len(sys.argv) > 2 else []
    out = subprocess.run(["ncu", "-i", sys.argv[1], *kf, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    iname, iunit, ival = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    seen = set()
    for r in rows[1:]:
        if len(r) <= ival:
            continue
        if r[iname] in KEYS and r[iname] not in seen:
            seen.add(r[iname])
            print(f"{r[iname]:45s} = {r[ival]} {r[iunit]}")
    raw = subprocess.run(["ncu", "-i", sys.argv[1], *kf, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    if len(raw) >= 3:
        h = next(csv.reader([raw[0]]))
        v = next(csv.reader([raw[2]]))
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
                  "l1tex__t_bytes.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
                  "sm__warps_active.avg.pct_of_peak_sustained_active"):
            if k in h:
                print(f"{k:45s} = {v[h.index(k)]}")


if __name__ == "__main__":
    main()
