"""Config 5 (BASELINE.json: resolution ablation sweep, planes 512^2-4096^2, grid 256^3-1024^3,
incl. the dense-3D-only SNeRG++-style and the planes-only variants) as GPU parity cases at
full size: sampled pixels of C2's 1280x720 view vs the fp64 oracle pixel by pixel, plus
bit-exact traces.  Delta = 2 / max(R, L) (reading D5)."""
import functools

import numpy as np
import pytest

from conftest import psnr
from merf_inputs import make_scene, config_cameras
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@functools.lru_cache(maxsize=None)
def _scene(key):
    if key == "R4096_L256":
        return make_scene("c2", L=256, R=4096, step=2.0 ** -11)
    if key == "R512_L1024":
        return make_scene("c2", L=1024, R=512, step=2.0 ** -10)
    if key == "Vonly_L1024":           # SNeRG++-style: the 3D grid alone (same arrays, planes off)
        import copy
        sc = copy.copy(_scene("R512_L1024"))
        sc.source_mask = 1
        return sc
    if key == "planes_only_R2048":
        return make_scene("c2", L=0, R=2048, source_mask=14)
    raise KeyError(key)


@pytest.fixture(scope="module")
def M():
    import torch
    assert torch.cuda.is_available()
    import paper_2302_12249_b200 as M
    return M


@pytest.mark.parametrize("key", ["R4096_L256", "R512_L1024", "Vonly_L1024", "planes_only_R2048"])
def test_c5_variant_parity(M, key):
    import torch
    sc = _scene(key)
    cams, W, H = config_cameras("c2")
    s = M.Scene(sc)
    out, st = s.render(cams, W, H, stats=True)
    torch.cuda.synchronize()
    got = out[0].reshape(-1, 3).cpu().numpy()
    rng = np.random.default_rng(7)
    pix = np.unique(rng.integers(0, W * H, 3000))
    osc = O.OracleScene(sc)
    ref = O.render(osc, cams[0], W, H, pixels=pix)
    assert np.abs(got[pix] - ref["rgb"]).max() <= 2e-3
    assert psnr(got[pix], ref["rgb"]) >= 50
    assert st["missing_blocks"] == 0 and st["evaluated"] > 0
    tp = pix[:200]
    o = O.render(osc, cams[0], W, H, pixels=tp, max_trace=4096, flags=O.NO_EARLY_TERM)
    pid = torch.as_tensor(tp, device="cuda")
    cells = torch.zeros((len(tp), 4096), dtype=torch.int64, device="cuda")
    cnt = torch.zeros(len(tp), dtype=torch.int32, device="cuda")
    M.merf_trace(s.handle, cams[0], W, pid, 4096, cells, None, cnt, flags=M.MERF_NO_EARLY_TERM)
    torch.cuda.synchronize()
    assert np.array_equal(cnt.cpu().numpy(), o["trace_count"])
    assert np.array_equal(cells.cpu().numpy().view(np.uint64), o["trace_cells"])
    s.close()


def test_finest_512_bordered_skip_table_all_regions(M):
    """the largest skip-table resolution (finest level 512^3: one-cell border, 2^21-unit cells)
    with a small step (Delta = 2^-11: long segments, the most lattice drift) from a pose
    outside the cube whose rays cross every contraction region and end at the grid border:
    colours vs the oracle, bit-exact traces, and the skip-table traversal equal to the level
    search (the same evaluated samples)."""
    import os
    import torch
    sc = make_scene("c2", L=256, R=1024, level_res=(32, 128, 512), step=2.0 ** -11)
    cams, W, H = config_cameras("c3")
    cam = cams[1]
    s = M.Scene(sc)
    out, st = s.render(cams, W, H, stats=True)
    torch.cuda.synchronize()
    got = out[1].reshape(-1, 3).cpu().numpy()
    os.environ["MERF_NO_SKIPTAB"] = "1"
    try:
        out2, st2 = s.render(cams, W, H, stats=True)
        torch.cuda.synchronize()
    finally:
        os.environ.pop("MERF_NO_SKIPTAB", None)
    assert np.array_equal(out2.cpu().numpy(), out.cpu().numpy())
    assert st2["evaluated"] == st["evaluated"] and st["skips"] <= st2["skips"]
    assert all(n > 0 for n in st["region_segments"])          # every region crossed (both poses)
    rng = np.random.default_rng(11)
    pix = np.unique(np.concatenate([rng.integers(0, W * H, 2000), np.arange(0, W * H, 4099)]))
    osc = O.OracleScene(sc)
    ref = O.render(osc, cam, W, H, pixels=pix)
    assert np.abs(got[pix] - ref["rgb"]).max() <= 2e-3
    assert psnr(got[pix], ref["rgb"]) >= 50
    tp = pix[:256]
    o = O.render(osc, cam, W, H, pixels=tp, max_trace=8192, flags=O.NO_EARLY_TERM)
    pid = torch.as_tensor(tp, device="cuda")
    cells = torch.zeros((len(tp), 8192), dtype=torch.int64, device="cuda")
    cnt = torch.zeros(len(tp), dtype=torch.int32, device="cuda")
    M.merf_trace(s.handle, cam, W, pid, 8192, cells, None, cnt, flags=M.MERF_NO_EARLY_TERM)
    torch.cuda.synchronize()
    assert np.array_equal(cnt.cpu().numpy(), o["trace_count"])
    assert np.array_equal(cells.cpu().numpy().view(np.uint64), o["trace_cells"])
    s.close()
