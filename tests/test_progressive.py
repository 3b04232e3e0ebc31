"""NEXT-4: progressive rendering.  CPU pins of the pass geometry
(hand-enumerated cases, partition of the frame, nearest-upsampling blocks) and GPU parity:
the stride^2 passes of merf_render_progressive assemble exactly merf_render's frame, each
pass's pixels match the fp64 oracle, and the preview is the nearest upsampling."""
import numpy as np
import pytest

from conftest import psnr
from oracle import progressive as P


def test_pass_pixels_hand_cases():
    # W = 5, H = 3, stride 2: pass 0 -> (0,0),(2,0),(4,0),(0,2),(2,2),(4,2); pass 3 -> (1,1),(3,1)
    assert P.pass_pixels(5, 3, 2, 0).tolist() == [0, 2, 4, 10, 12, 14]
    assert P.pass_pixels(5, 3, 2, 1).tolist() == [1, 3, 11, 13]
    assert P.pass_pixels(5, 3, 2, 2).tolist() == [5, 7, 9]
    assert P.pass_pixels(5, 3, 2, 3).tolist() == [6, 8]
    assert P.pass_pixels(5, 3, 1, 0).tolist() == list(range(15))
    with pytest.raises(ValueError):
        P.pass_pixels(5, 3, 2, 4)


@pytest.mark.parametrize("W,H,s", [(5, 3, 2), (37, 23, 3), (8, 8, 4), (3, 2, 4)])
def test_passes_partition_the_frame(W, H, s):
    ids = np.concatenate([P.pass_pixels(W, H, s, p) for p in range(s * s)])
    assert np.array_equal(np.sort(ids), np.arange(W * H))


def test_fill_source_blocks():
    src = P.fill_source(5, 3, 2, 0).reshape(3, 5)
    assert src.tolist() == [[0, 0, 2, 2, 4], [0, 0, 2, 2, 4], [10, 10, 12, 12, 14]]
    src = P.fill_source(5, 3, 2, 3).reshape(3, 5)
    assert src.tolist() == [[-1] * 5, [-1, 6, 6, 8, 8], [-1, 6, 6, 8, 8]]
    # every pixel is filled by the pass-0 preview, from a rendered pixel of its block
    W, H, s = 37, 23, 3
    src = P.fill_source(W, H, s, 0)
    rendered = set(P.pass_pixels(W, H, s, 0).tolist())
    assert (src >= 0).all() and set(src.tolist()) <= rendered
    x, y = np.arange(W * H) % W, np.arange(W * H) // W
    assert ((x - src % W >= 0) & (x - src % W < s) & (y - src // W >= 0) & (y - src // W < s)).all()


# ---------------------------------------------------------------------------------------
# GPU
# ---------------------------------------------------------------------------------------
@pytest.fixture(scope="module")
def M():
    import torch
    assert torch.cuda.is_available()
    import paper_2302_12249_b200 as M
    return M


def _cams(W, H):
    from merf_inputs import look_at_camera
    return [look_at_camera((0.3, 0.2, -1.5), target=(0, 0, 0), W=W, H=H, fov_x_deg=55),
            look_at_camera((-0.8, 0.1, -1.1), target=(0.1, 0, 0), W=W, H=H, fov_x_deg=55)]


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", [0, 1])
@pytest.mark.parametrize("stride", [2, 3, 5])
def test_gpu_passes_assemble_the_full_frame(M, c1_scene, fmt, stride):
    import torch
    W, H = 37, 23
    cams = _cams(W, H)
    s = M.Scene(c1_scene)
    shape = (2, H, W, 4 if fmt == M.MERF_RGBA_U8 else 3)
    dt = torch.uint8 if fmt == M.MERF_RGBA_U8 else torch.float32
    full = torch.zeros(shape, dtype=dt, device="cuda")
    M.merf_render(s.handle, cams, W, H, full, fmt=fmt)
    prog = torch.full(shape, 7, dtype=dt, device="cuda")
    for p in range(stride * stride):
        M.merf_render_progressive(s.handle, cams, W, H, stride, p, prog, fmt=fmt)
        if p == 0:
            torch.cuda.synchronize()
            got = prog.cpu().numpy().reshape(2, W * H, -1)
            ids = P.pass_pixels(W, H, stride, 0)
            untouched = np.setdiff1d(np.arange(W * H), ids)
            assert (got[:, untouched] == 7).all()              # only the pass's pixels written
    torch.cuda.synchronize()
    assert np.array_equal(prog.cpu().numpy(), full.cpu().numpy())
    s.close()


@pytest.mark.gpu
def test_gpu_pass_pixels_match_oracle_and_preview_is_nearest(M, c1_scene):
    import torch
    from oracle import oracle as O
    W, H, stride = 61, 34, 4
    cams = _cams(W, H)[:1]
    s = M.Scene(c1_scene)
    osc = O.OracleScene(c1_scene)
    for p in (0, 5, 15):
        out = torch.full((1, H, W, 3), -1.0, dtype=torch.float32, device="cuda")
        M.merf_render_progressive(s.handle, cams, W, H, stride, p, out, fill=True)
        torch.cuda.synchronize()
        got = out.cpu().numpy().reshape(W * H, 3)
        ids = P.pass_pixels(W, H, stride, p)
        ref = O.render(osc, cams[0], W, H, pixels=ids)["rgb"]
        assert np.abs(got[ids] - ref).max() <= 2e-3 and psnr(got[ids], ref) >= 50
        src = P.fill_source(W, H, stride, p)
        on = src >= 0
        assert np.array_equal(got[on], got[src[on]])            # nearest upsampling
        assert (got[~on] == -1.0).all()                         # the rest untouched
    s.close()


@pytest.mark.gpu
def test_gpu_progressive_argument_errors(M, c1_scene):
    import torch
    s = M.Scene(c1_scene)
    out = torch.zeros((1, 8, 8, 3), dtype=torch.float32, device="cuda")
    cams = _cams(8, 8)[:1]
    for stride, p in [(0, 0), (65, 0), (2, 4), (2, -1)]:
        with pytest.raises(M.MerfError):
            M.merf_render_progressive(s.handle, cams, 8, 8, stride, p, out)
    M.merf_render_progressive(s.handle, cams, 3, 2, 4, 15, out)   # empty sub-lattice: no-op
    s.close()
