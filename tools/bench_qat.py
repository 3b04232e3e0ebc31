"""NEXT-3 measurement: throughput of the quantisation-aware training step (merf_qat_step:
forward + backward, Eq. 7-8) on a dense toy field.

  python tools/bench_qat.py [--L 128] [--R 512] [--N 64] [--views 4] [--size 256] [--out f.json]

Input recipe: theta ~ N(0, 1.2) (density channel N(-1, 1)), occupancy = the cells
of a contracted-space shell 0.45 <= |c| <= 0.8 (a surface-like band, ~16 % of cells), one
orbit of `--views` cameras at distance 1.6 looking at the origin, Delta = 2 / max(L, R)
(reading D5), target uniform in [0, 1].  Reported: rays/s and samples/s of the full step
(CUDA events over 5 steps after 3 warm-ups).
"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=128)
    ap.add_argument("--R", type=int, default=512)
    ap.add_argument("--N", type=int, default=64)
    ap.add_argument("--views", type=int, default=4)
    ap.add_argument("--size", type=int, default=256)
    ap.add_argument("--max-samples", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import numpy as np
    import torch
    from merf_inputs import look_at_camera, pack_bits
    import paper_2302_12249_b200 as M

    g = torch.Generator().manual_seed(0)
    tv = torch.randn((a.L, a.L, a.L, 8), generator=g) * 1.2
    tv[..., 0] = torch.randn((a.L, a.L, a.L), generator=g) - 1.0
    tp = torch.randn((3, a.R, a.R, 8), generator=g)
    tp[..., 0] = torch.randn((3, a.R, a.R), generator=g) - 1.0
    c = (np.arange(a.N) + 0.5) / a.N * 4 - 2
    r = np.sqrt(c[None, None, :] ** 2 + c[None, :, None] ** 2 + c[:, None, None] ** 2)
    occ_np = (r >= 0.45) & (r <= 0.8)
    occ = torch.from_numpy(np.ascontiguousarray(pack_bits(occ_np)).view(np.int32))
    mlp = torch.empty(883).uniform_(-0.3, 0.3, generator=g)
    W = H = a.size
    cams = []
    for v in range(a.views):
        ang = 2 * math.pi * v / a.views
        cams.append(look_at_camera((1.6 * math.sin(ang), 0.3, -1.6 * math.cos(ang)), target=(0, 0, 0), W=W, H=H,
                                   fov_x_deg=50))
    target = torch.rand((a.views, H, W, 3), generator=g)
    dev = "cuda"
    tv, tp, occ, mlp, target = (x.to(dev) for x in (tv, tp, occ, mlp, target))
    rgb = torch.empty_like(target)
    gv, gp = torch.empty_like(tv), torch.empty_like(tp)
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    ovf = torch.empty(1, dtype=torch.int32, device=dev)
    nsamp = torch.empty(1, dtype=torch.int64, device=dev)
    step = 2.0 / max(a.L, a.R)

    def run():
        M.merf_qat_step(tv, tp, occ, a.N, mlp, cams, W, H, target, rgb, gv, gp, loss, step,
                        max_samples=a.max_samples, overflow=ovf, n_samples=nsamp)

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    rays = a.views * W * H
    ns = int(nsamp.item())
    d = dict(metric="qat_step_rays_per_s", value=rays / (ms / 1e3), unit="rays/s", ms_per_step=ms,
             samples_per_s=ns / (ms / 1e3), samples_per_ray=ns / rays,
             L=a.L, R=a.R, N=a.N, views=a.views, W=W, H=H, step=step, occ_fraction=float(occ_np.mean()),
             overflow_rays=int(ovf.item()), loss=float(loss.item()), dtype="f32 (fp64 quantiser)")
    print(json.dumps(d))
    if a.out:
        with open(a.out, "w") as f:
            f.write(json.dumps(d) + "\n")


if __name__ == "__main__":
    main()
