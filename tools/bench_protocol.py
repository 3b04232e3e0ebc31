"""The paper's benchmark protocol (App. C) on the synthetic scenes: one
fixed camera pose per configuration, identical intrinsics, the average frame rate over 150
frames (after 10 warm-up frames), progressive rendering off.  Each frame is ONE merf_render
call for one view (RGBA8, device output), i.e. interactive single-frame latency -- unlike
bench.py, which renders batches of 16 moving orbit views per call.  Times are CUDA events on
the render stream around the 150 calls.  From the second call of a pose on, the library
dispatches tiles longest first by the previous frame's measured tile costs (frame-sequence
tile order; output byte-identical); MERF_TILE_ORDER=raster times raster order.

  python tools/bench_protocol.py [--frames 150] [--out profiles/r01_protocol.jsonl]

Configurations: C2 = 1280x720 from (0.3, 0.1, -0.7) (the paper's M1 setting),
C3a/C3b = 1920x1080 poses crossing all contraction regions, and orbit view 0 at 1080p.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def protocol_poses():
    """(name, camera, W, H) of the protocol's four poses (shared with single_view_timed.py)"""
    from merf_inputs import config_cameras, orbit_cameras
    c2, W2, H2 = config_cameras("c2")
    c3, W3, H3 = config_cameras("c3")
    return [("c2_720p", c2[0], W2, H2), ("c3a_1080p_outward", c3[0], W3, H3),
            ("c3b_1080p_outside_cube", c3[1], W3, H3),
            ("orbit0_1080p", orbit_cameras(256, indices=[0])[0], 1920, 1080)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=150)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    from merf_inputs import make_scene, config_cameras, orbit_cameras
    import paper_2302_12249_b200 as M
    s = M.Scene(make_scene("c2"))
    poses = protocol_poses()
    stream = torch.cuda.Stream()
    lines = []
    for name, cam, W, H in poses:
        out = torch.empty((1, H, W, 4), dtype=torch.uint8, device="cuda")
        cams = cam[None]
        with torch.cuda.stream(stream):
            for _ in range(a.warmup):
                M.merf_render(s.handle, cams, W, H, out, fmt=M.MERF_RGBA_U8, stream=stream)
            st = M.merf_render(s.handle, cams, W, H, out, fmt=M.MERF_RGBA_U8, stream=stream, stats=True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(a.frames):
                M.merf_render(s.handle, cams, W, H, out, fmt=M.MERF_RGBA_U8, stream=stream)
            e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.frames
        rays = W * H
        lines.append({"pose": name, "W": W, "H": H, "frames": a.frames, "ms_per_frame": ms,
                      "fps": 1e3 / ms, "rays_per_sec": rays / (ms / 1e3),
                      "mean_evaluated_samples_per_ray": st["evaluated"] / rays,
                      "density_only_fraction": st["density_only"] / max(st["evaluated"], 1),
                      "protocol": "PAPER P:583: fixed pose, identical intrinsics, average over "
                                  f"{a.frames} frames after {a.warmup} warm-up, progressive off",
                      "tile_order": ("raster (MERF_TILE_ORDER=raster)" if os.environ.get("MERF_TILE_ORDER") == "raster"
                                     else "frame-sequence history: tiles dispatched longest first by the previous "
                                          "frame's measured tile durations (output byte-identical to raster)")})
        print(json.dumps(lines[-1]), flush=True)
    s.close()
    if a.out:
        with open(a.out, "w") as f:
            for ln in lines:
                f.write(json.dumps(ln) + "\n")


if __name__ == "__main__":
    main()
