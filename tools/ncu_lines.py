"""Aggregate an ncu report's source page by CUDA source line (stall samples, executed
instructions).  usage: python tools/ncu_lines.py report.ncu-rep [top] [kernel-regex]"""
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    kf = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
    out = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                         capture_output=True, text=True).stdout
    rows = []
    path = None
    hdr = None
    for line in out.splitlines():
        if line.startswith('"File Path"'):
            path = next(csv.reader([line]))[1].split("/")[-1]
            continue
        if line.startswith('"Line No"'):
            hdr = next(csv.reader([line]))
            continue
        if hdr is None or not line.startswith('"'):
            continue
        r = next(csv.reader([line]))
        if len(r) < 8 or r[2] != "-":
            continue
        try:
            stall = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            inst = int(r[hdr.index("Instructions Executed")])
            tinst = int(r[hdr.index("Thread Instructions Executed")])
        except (ValueError, IndexError):
            continue
        rows.append((stall, inst, tinst, path, r[0], r[1].strip()[:90]))
    tot_s = sum(x[0] for x in rows) or 1
    tot_i = sum(x[1] for x in rows) or 1
    print(f"total stall samples {tot_s}, warp instructions {tot_i}")
    print(f"{'stall%':>7} {'inst%':>6} {'thr/inst':>8}  location / source")
    for s, i, t, p, ln, src in sorted(rows, reverse=True)[:top]:
        print(f"{100*s/tot_s:7.2f} {100*i/tot_i:6.2f} {t/max(i,1):8.1f}  {p}:{ln}  {src}")


if __name__ == "__main__":
    main()
