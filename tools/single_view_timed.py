"""Per-kernel times (MERF_TIMED CUDA events) of single-view calls on the protocol poses of
tools/bench_protocol.py: where a one-view frame's time goes (setup / march / shade).

  python tools/single_view_timed.py [--frames 50]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=50)
    a = ap.parse_args()
    import torch
    import paper_2302_12249_b200 as M
    from merf_inputs import make_scene
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from bench_protocol import protocol_poses
    s = M.Scene(make_scene("c2"))
    for name, cam, W, H in protocol_poses():
        out = torch.empty((1, H, W, 4), dtype=torch.uint8, device="cuda")
        for _ in range(10):
            M.merf_render(s.handle, cam[None], W, H, out, fmt=M.MERF_RGBA_U8)
        torch.cuda.synchronize()
        M.merf_kernel_times_get(s.handle, reset=True)
        for _ in range(a.frames):
            M.merf_render(s.handle, cam[None], W, H, out, fmt=M.MERF_RGBA_U8, flags=M.MERF_TIMED)
        torch.cuda.synchronize()
        kt = M.merf_kernel_times_get(s.handle, reset=True)
        print(json.dumps({"pose": name, **{k: round(v / a.frames, 4) for k, v in kt.items() if k.endswith("_ms")}}))
    s.close()


if __name__ == "__main__":
    main()
