"""Write profiles/render_traffic.json (DRAM bytes per march launch, read by bench.py's
roofline.traffic) from an `ncu --set full` capture of one march launch.

  python tools/traffic_from_ncu.py report.ncu-rep [--out profiles/render_traffic.json]
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _source_hash():
    """the library-source digest the capture was taken with (paper_2302_12249_b200.build)"""
    from paper_2302_12249_b200.build import source_hash
    return source_hash()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--out", default="profiles/render_traffic.json")
    ap.add_argument("--kernel", default="march_kernel", help="kernel-name regex (report may hold several)")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.report, "-k", "regex:" + a.kernel, "--page", "raw", "--csv", "--print-units", "base", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,"
                          "lts__t_sectors.sum,sm__cycles_elapsed.avg"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    r = dict(zip(hdr, data[0]))
    rd, wr = float(r["dram__bytes_read.sum"]), float(r["dram__bytes_write.sum"])
    d = {"source": f"{a.report.split('/')[-1]} (ncu --set full --clock-control none, {r['Kernel Name'].split('(')[0]},"
                   " one launch = 16 views at 1080p, tools/prof_render.py --views 16)",
         "dram_bytes_read_per_launch": rd, "dram_bytes_write_per_launch": wr, "dram_bytes_per_launch": rd + wr,
         "ncu_duration_ns": float(r["gpu__time_duration.sum"]),
         "warp_inst_per_launch": float(r["smsp__inst_executed.sum"]),
         "l2_bytes_per_launch": 32.0 * float(r["lts__t_sectors.sum"]),
         "sm_cycles_per_launch": float(r["sm__cycles_elapsed.avg"]),
         "note": "includes the workspace (segments read, accumulators written); scene texels hit L1/L2",
         "source_sha16": _source_hash()}
    with open(a.out, "w") as f:
        json.dump(d, f, indent=1)
    print(json.dumps(d))


if __name__ == "__main__":
    main()
