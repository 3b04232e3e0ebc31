"""Config-5 sweep (BASELINE.json configs[4]; the paper's Fig. 6 VRAM/resolution trade-off,
P:345-351): throughput and device memory of the render path over plane resolution R,
grid resolution L, the dense-3D-only (SNeRG++-style) and the planes-only variants.

  python tools/sweep_c5.py [--views 8] [--out profiles/r01_c5_sweep.jsonl]

Each point renders `--views` orbit views at 1920x1080 (config 4's orbit, config 2's world),
Delta = 2 / max(R, L) (reading D5).  Throughput is CUDA-event timed over 3 repeats after a
warm-up; counters (samples/ray) come from an untimed pass.  Scenes for the grid reuse the
3D grid of a given L and the planes of a given R (both are functions of the same world).
"""
import argparse
import copy
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, default=8)
    ap.add_argument("--out", default="")
    ap.add_argument("--R", default="512,1024,2048,4096")
    ap.add_argument("--L", default="256,512,1024")
    args = ap.parse_args()
    import torch
    from merf_inputs import make_scene, orbit_cameras
    import paper_2302_12249_b200 as M

    Rs = [int(x) for x in args.R.split(",")]
    Ls = [int(x) for x in args.L.split(",")]
    t0 = time.time()
    vscenes = {L: make_scene("c2", L=L, R=512) for L in Ls}          # V of each L
    pscenes = {R: make_scene("c2", L=0, R=R, source_mask=14) for R in Rs}
    print(f"# generated in {time.time() - t0:.0f} s", file=sys.stderr)

    cams = orbit_cameras(256, indices=range(0, 256, 256 // args.views))
    W, H = 1920, 1080
    points = [(L, R, 15) for L in Ls for R in Rs] + [(L, 0, 1) for L in Ls] + [(0, R, 14) for R in Rs]
    lines = []
    for (L, R, mask) in points:
        if mask == 15:
            sc = copy.copy(vscenes[L])
            sc.planes = _noise_planes(pscenes[R])
            sc.R = R
        elif mask == 1:
            sc = copy.copy(vscenes[L])
            sc.R = 0
        else:
            sc = copy.copy(pscenes[R])
        sc.source_mask = mask
        sc.step = 2.0 / max(sc.R if mask & 14 else 0, sc.L if mask & 1 else 0)
        s = M.Scene(sc)
        info = s.info()
        out = torch.empty((len(cams), H, W, 4), dtype=torch.uint8, device="cuda")
        st = M.merf_render(s.handle, cams, W, H, out, fmt=M.MERF_RGBA_U8, stats=True)
        M.merf_render(s.handle, cams, W, H, out, fmt=M.MERF_RGBA_U8)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            M.merf_render(s.handle, cams, W, H, out, fmt=M.MERF_RGBA_U8)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        rays = len(cams) * W * H
        d = dict(variant={15: "merf", 1: "3d_grid_only", 14: "planes_only"}[mask], L=sc.L if mask & 1 else 0,
                 R=sc.R if mask & 14 else 0, step=sc.step, n_blocks=info["n_blocks"],
                 device_mb=info["device_bytes"] / 1e6, rays_per_s=rays / (ms / 1e3),
                 fps=len(cams) / (ms / 1e3), samples_per_ray=st["evaluated"] / rays,
                 density_only_fraction=st["density_only"] / max(st["evaluated"], 1))
        lines.append(d)
        print(json.dumps(d), flush=True)
        s.close()
        del out
    if args.out:
        with open(args.out, "w") as f:
            for d in lines:
                f.write(json.dumps(d) + "\n")


def _noise_planes(pscene):
    """planes of resolution R with the c2-style density noise (not the planes-only projection)."""
    import numpy as np
    from merf_inputs.scene import _hash_u8, SEED
    R = pscene.R
    planes = pscene.planes.copy()
    idx = np.arange(R * R, dtype=np.int64)
    for a in range(3):
        h = _hash_u8(SEED, a, idx, 0).astype(np.int16)
        planes[a, :, :, 0] = (128 + ((h * 13) >> 8) - 6).reshape(R, R).astype(np.uint8)
    return planes


if __name__ == "__main__":
    main()
