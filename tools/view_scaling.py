"""Per-view cost of the pipeline kernels against the number of views per merf_render call
(the same 1080p orbit view repeated n times, and n distinct orbit views): separates the
per-launch fixed cost (persistent march ramp and tail, launch gaps) from the per-view cost.
Each configuration is rendered repeatedly, so calls of <= 4 views run with the frame-sequence
tile order; MERF_TILE_ORDER=raster measures raster order.

  python tools/view_scaling.py [--reps 20] [--out FILE]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import numpy as np
    import torch
    from merf_inputs import make_scene, orbit_cameras
    import paper_2302_12249_b200 as M
    s = M.Scene(make_scene("c2"))
    st = torch.cuda.Stream()
    lines = []
    for mode in ("same", "distinct"):
        for n in (1, 2, 4, 8, 16):
            cams = (np.repeat(orbit_cameras(256, indices=[0]), n, axis=0) if mode == "same"
                    else orbit_cameras(256, indices=list(range(0, 16 * n, 16))[:n]))
            out = torch.empty((n, 1080, 1920, 4), dtype=torch.uint8, device="cuda")
            with torch.cuda.stream(st):
                for _ in range(3):
                    M.merf_render(s.handle, cams, 1920, 1080, out, fmt=M.MERF_RGBA_U8, stream=st)
                torch.cuda.synchronize()
                M.merf_kernel_times_get(s.handle, reset=True)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(a.reps):
                    M.merf_render(s.handle, cams, 1920, 1080, out, fmt=M.MERF_RGBA_U8, stream=st,
                                  flags=M.MERF_TIMED)
                e1.record(st)
            torch.cuda.synchronize()
            kt = M.merf_kernel_times_get(s.handle, reset=True)
            call = e0.elapsed_time(e1) / a.reps
            stc = M.merf_render(s.handle, cams, 1920, 1080, out, fmt=M.MERF_RGBA_U8, stream=st, stats=True)
            ln = {"mode": mode, "views": n, "call_ms": call, "call_ms_per_view": call / n,
                  "setup_ms_per_view": kt["setup_ms"] / a.reps / n, "march_ms_per_view": kt["march_ms"] / a.reps / n,
                  "shade_ms_per_view": kt["shade_ms"] / a.reps / n,
                  "march_busy_ms": stc["march_busy_ns"] / 1e6, "march_tail_ms": stc["march_tail_ns"] / 1e6,
                  "note": "busy/tail from the counter instance: first warp start -> tile queue dry -> last exit"}
            print(json.dumps(ln), flush=True)
            lines.append(ln)
    s.close()
    if a.out:
        with open(a.out, "w") as f:
            for ln in lines:
                f.write(json.dumps(ln) + "\n")


if __name__ == "__main__":
    main()
