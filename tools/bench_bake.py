"""Throughput of the bake-side structure construction (NEXT-1) on B200:
weighted points -> A (merf_bake_occupancy) at the paper's base resolution 4096^3 and at
256^3, A -> occupancy levels 32/128/256 (merf_build_occupancy, max-pool factors 128/32/16,
P:307), canonical block allocation for L = 512 (merf_build_block_index) and atlas packing
from a dense 512^3 x 8 grid (merf_pack_atlas).  CUDA-event timed, 3 repeats after warm-up.
  python tools/bench_bake.py [--points 16777216]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def timed(fn, reps=3):
    import torch
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", type=int, default=1 << 24)
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2302_12249_b200 as M
    from merf_inputs import MerfScene
    n = args.points
    g = torch.Generator(device="cuda").manual_seed(0)
    # contracted-uniform points near the middle of the domain, mapped to the world
    c = (torch.rand((n, 3), generator=g, device="cuda", dtype=torch.float64) * 3.9 - 1.95)
    j = c.abs().argmax(1)
    aj = c.abs().gather(1, j[:, None])[:, 0]
    scale = torch.where(aj > 1, 1.0 / (2.0 - aj), torch.ones_like(aj))
    x = c.clamp(-1, 1) * scale[:, None]
    x.scatter_(1, j[:, None], (torch.sign(c.gather(1, j[:, None])[:, 0]) * torch.maximum(scale, aj))[:, None])
    tau = torch.exp(torch.randn(n, generator=g, device="cuda", dtype=torch.float64) * 3 + 3)
    w = torch.rand(n, generator=g, device="cuda", dtype=torch.float64) * 0.02
    out = []
    for N in (256, 4096):
        bits = torch.empty((N ** 3 + 31) // 32, dtype=torch.int32, device="cuda")
        ms = timed(lambda: M.merf_bake_occupancy(x, tau, w, N, 2.0 ** -10, bits))
        out.append(dict(op="bake_occupancy", N=N, points=n, ms=ms, points_per_s=n / (ms / 1e3)))
    desc = MerfScene(L=512, R=2048, level_res=(32, 128, 256, 4096), step=2.0 ** -10,
                     planes=np.zeros(1, np.uint8), block_index=np.zeros(1, np.int32),
                     atlas=np.zeros((0, 9, 9, 9, 8), np.uint8), occ_finest=np.zeros(1, np.uint32),
                     mlp=np.zeros(883))
    lv = torch.empty(sum((N ** 3 + 31) // 32 for N in (32, 128, 256)), dtype=torch.int32, device="cuda")
    ms = timed(lambda: M.merf_build_occupancy(bits, desc, lv))
    out.append(dict(op="build_occupancy 4096 -> 32/128/256", ms=ms, bytes_read=4096 ** 3 // 8))
    desc.level_res = (32, 128, 256)
    idx = torch.empty(64 ** 3, dtype=torch.int32, device="cuda")
    fin = lv[((32 ** 3 + 31) // 32) + ((128 ** 3 + 31) // 32):]
    nb = [0]

    def blk():
        nb[0] = M.merf_build_block_index(fin, desc, idx)
    ms = timed(blk)
    out.append(dict(op="build_block_index L=512 from 256^3", ms=ms, n_blocks=nb[0]))
    dense = torch.randint(0, 256, (512, 512, 512, 8), dtype=torch.uint8, device="cuda")
    atlas = torch.empty((max(nb[0], 1), 9, 9, 9, 8), dtype=torch.uint8, device="cuda")
    ms = timed(lambda: M.merf_pack_atlas(dense, 512, idx, nb[0], atlas))
    out.append(dict(op="pack_atlas L=512", ms=ms, n_blocks=nb[0], bytes_written=nb[0] * 729 * 8,
                    gbs=2 * nb[0] * 729 * 8 / (ms / 1e3) / 1e9))
    for d in out:
        print(json.dumps(d))


if __name__ == "__main__":
    main()
