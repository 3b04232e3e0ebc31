"""Warm render launches of the bench workload for ncu (--set full) captures: two warm-up
renders, then one render with counters (its stats are printed).  Each render is one setup,
one march and one shade launch, so `-k regex:"march_kernel|shade_mma|setup_kernel" -s 3 -c 3`
captures the second render's three kernels (tools/gpu_profile_round.sh).

  python tools/prof_render.py [--views N] [--first K]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, default=4)
    ap.add_argument("--first", type=int, default=0)
    args = ap.parse_args()
    import torch
    from merf_inputs import make_scene, orbit_cameras
    import paper_2302_12249_b200 as M
    sc = make_scene("c2")
    s = M.Scene(sc)
    cams = orbit_cameras(256, indices=range(args.first, args.first + args.views))
    out = torch.empty((args.views, 1080, 1920, 4), dtype=torch.uint8, device="cuda")
    for _ in range(2):
        M.merf_render(s.handle, cams, 1920, 1080, out, fmt=M.MERF_RGBA_U8)
    torch.cuda.synchronize()
    st = M.merf_render(s.handle, cams, 1920, 1080, out, fmt=M.MERF_RGBA_U8, stats=True)
    print(st)
    s.close()


if __name__ == "__main__":
    main()
