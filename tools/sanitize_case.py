"""Small render workload for compute-sanitizer (memcheck): C1 frame, a random scene with
ragged size and every source variant, trace + segments APIs, explicit rays."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from merf_inputs import make_scene, random_scene, config_cameras, look_at_camera
    import paper_2302_12249_b200 as M
    sc = make_scene("c1")
    cams, W, H = config_cameras("c1")
    s = M.Scene(sc)
    s.render(cams, W, H, stats=True)
    s.render(cams, W, H, fmt=M.MERF_RGBA_U8, flags=M.MERF_DENSE)
    pid = torch.arange(W * H, device="cuda")
    cells = torch.zeros((W * H, 64), dtype=torch.int64, device="cuda")
    T = torch.zeros((W * H, 64), device="cuda")
    cnt = torch.zeros(W * H, dtype=torch.int32, device="cuda")
    M.merf_trace(s.handle, cams[0], W, pid, 64, cells, T, cnt)
    segs = torch.zeros(W * H * 8 * 72, dtype=torch.uint8, device="cuda")
    M.merf_segments(s.handle, cams[0], W, pid, 8, segs, cnt)
    rng = np.random.default_rng(0)
    o = torch.as_tensor(rng.uniform(-3, 3, (999, 3)), device="cuda")
    d = torch.as_tensor(rng.normal(size=(999, 3)), device="cuda")
    d = d / d.norm(dim=1, keepdim=True)
    rgb = torch.zeros((999, 3), device="cuda")
    M.merf_render_rays(s.handle, o, d, rgb, stats=True)
    s.close()
    for mask in (15, 1, 14):
        r = random_scene(seed=3, L=32, R=64, level_res=(4, 16, 32), occ_fraction=0.3, source_mask=mask)
        s = M.Scene(r)
        c = look_at_camera((1.7, -1.9, 0.3), target=(0, 0, 0), W=37, H=23, fov_x_deg=100)
        s.render(c[None], 37, 23, stats=True)
        s.close()
    torch.cuda.synchronize()
    print("sanitize case done")


if __name__ == "__main__":
    main()
