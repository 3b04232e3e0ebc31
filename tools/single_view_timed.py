import sys, os
sys.path.insert(0, os.getcwd())
import torch
from merf_inputs import make_scene, orbit_cameras
import paper_2302_12249_b200 as M
s = M.Scene(make_scene("c2"))
cam = orbit_cameras(256, indices=[0])
out = torch.empty((1, 1080, 1920, 4), dtype=torch.uint8, device="cuda")
for _ in range(10):
    M.merf_render(s.handle, cam, 1920, 1080, out, fmt=M.MERF_RGBA_U8)
torch.cuda.synchronize()
M.merf_kernel_times_get(s.handle, reset=True)
for _ in range(50):
    M.merf_render(s.handle, cam, 1920, 1080, out, fmt=M.MERF_RGBA_U8, flags=M.MERF_TIMED)
torch.cuda.synchronize()
kt = M.merf_kernel_times_get(s.handle, reset=True)
print({k: (v / 50 if k.endswith("_ms") else v) for k, v in kt.items()})
