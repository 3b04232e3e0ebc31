"""NEXT-4 measurement: progressive rendering on the bench workload (paper-scale scene,
orbit views at 1920x1080, RGBA8).  For stride s: the first preview (pass 0 with nearest
fill) latency per view, and the whole s^2-pass cycle vs one full render.

  python tools/bench_progressive.py [--views 8] [--strides 2,4,8] [--out f.jsonl]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, default=8)
    ap.add_argument("--strides", default="2,4,8")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    from merf_inputs import make_scene, orbit_cameras
    import paper_2302_12249_b200 as M
    s = M.Scene(make_scene("c2"))
    W, H = 1920, 1080
    cams = orbit_cameras(256, indices=range(0, 256, 256 // a.views))
    out = torch.empty((len(cams), H, W, 4), dtype=torch.uint8, device="cuda")

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    full = timed(lambda: M.merf_render(s.handle, cams, W, H, out, fmt=M.MERF_RGBA_U8))
    lines = [dict(mode="full", ms_per_view=full / len(cams), fps=len(cams) / (full / 1e3))]
    for st in [int(x) for x in a.strides.split(",")]:
        pre = timed(lambda: M.merf_render_progressive(s.handle, cams, W, H, st, 0, out, fill=True,
                                                      fmt=M.MERF_RGBA_U8))

        def cycle():
            for p in range(st * st):
                M.merf_render_progressive(s.handle, cams, W, H, st, p, out, fmt=M.MERF_RGBA_U8)
        cyc = timed(cycle, reps=1)
        lines.append(dict(mode=f"progressive_s{st}", first_preview_ms_per_view=pre / len(cams),
                          preview_fps=len(cams) / (pre / 1e3), preview_speedup=full / pre,
                          full_cycle_ms_per_view=cyc / len(cams), cycle_overhead=cyc / full - 1.0))
    for d in lines:
        print(json.dumps(d))
    if a.out:
        with open(a.out, "w") as f:
            for d in lines:
                f.write(json.dumps(d) + "\n")
    s.close()


if __name__ == "__main__":
    main()
