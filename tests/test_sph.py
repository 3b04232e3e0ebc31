"""NEXT-2: the spherical-contraction comparison variant (Eq. 4).
CPU pins of the oracle (SPEC worked example S:63, identity in the unit ball, continuity at
|x| = 1, range, the contracted speed in closed form, the stepping rule's arc length, and the
uniform-density transmittance) and GPU parity (bit-exact traces, colour within tolerance)."""
import math

import numpy as np
import pytest

from merf_inputs import constant_scene, make_scene, config_cameras
from oracle import oracle as O


def test_contract_sph_examples_and_properties():
    y = O.contract_sph([[3, 4, 0], [0.5, 0, 0], [4, 0, 0]])
    assert np.allclose(y, [[1.08, 1.44, 0], [0.5, 0, 0], [1.75, 0, 0]], atol=1e-15)
    rng = np.random.default_rng(0)
    x = rng.normal(size=(2000, 3))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    inside = x * rng.uniform(0, 1, (2000, 1))
    assert np.array_equal(O.contract_sph(inside), inside)
    far = x * rng.uniform(1, 1e6, (2000, 1))
    c = O.contract_sph(far)
    n = np.linalg.norm(c, axis=1)
    assert (n < 2).all() and (n >= 1).all()
    assert np.allclose(c / n[:, None], x, atol=1e-12)                       # radial map
    assert np.allclose(n, 2 - 1 / np.linalg.norm(far, axis=1), atol=1e-12)
    eps = 1e-9
    assert np.abs(O.contract_sph(x * (1 + eps)) - x).max() < 1e-8          # continuity at |x| = 1


def test_sph_speed_closed_form():
    # |d/dt contract(o + t d)|: 1 inside; radial 1/r^2, tangential (2 - 1/r)/r outside
    for r in (1.5, 2.0, 10.0):
        assert abs(O.sph_speed([r, 0, 0], [1, 0, 0]) - 1 / r ** 2) < 1e-15
        assert abs(O.sph_speed([r, 0, 0], [0, 0, 1]) - (2 - 1 / r) / r) < 1e-15
        d = np.array([0.6, 0.8, 0.0])
        expect = math.sqrt((0.6 / r ** 2) ** 2 + ((2 - 1 / r) / r * 0.8) ** 2)
        assert abs(O.sph_speed([r, 0, 0], d) - expect) < 1e-15
    assert O.sph_speed([0.2, 0.1, 0], [1, 0, 0]) == 1.0
    # finite-difference check of the derivative
    rng = np.random.default_rng(1)
    for _ in range(50):
        x = rng.normal(size=3) * 3
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        h = 1e-6
        fd = np.linalg.norm(O.contract_sph(x + h * d)[0] - O.contract_sph(x - h * d)[0]) / (2 * h)
        assert abs(fd - O.sph_speed(x, d)) < 1e-6 * max(1, fd)


def test_sph_uniform_density_and_arc_length():
    # all cells occupied, constant bytes: every step evaluated, T_n = exp(-n tau Delta)
    step = 2.0 ** -6
    sc = constant_scene(L=16, R=32, level_res=(8, 16), step=step, b_d=118, b_a=128)
    osc = O.OracleScene(sc)
    rng = np.random.default_rng(2)
    d = rng.normal(size=(20, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o = rng.uniform(-0.5, 0.5, (20, 3))
    r = O.render_rays(osc, o, d, mode="sph", flags=O.NO_EARLY_TERM, max_trace=4096)
    tau = math.exp(4 * (28 * 118 / 255 - 14))
    for i in range(20):
        n = r["trace_count"][i]
        assert np.allclose(r["trace_T"][i, :n], np.exp(-np.arange(1, n + 1) * tau * step), rtol=1e-12)
        # steps of contracted arc length Delta: contracted length from the origin's image to
        # radius 2 - Delta is covered in about n steps (Euler, slope <= 1)
        c0 = O.contract_sph(o[i])[0]
        k = O.unpack_trace(r["trace_cells"][i, :n])[1]
        assert np.array_equal(k, np.arange(n))                   # every step evaluated
        assert 0.5 * (2 - np.linalg.norm(c0)) / step <= n <= 3.5 * 2 / step


def test_sph_scene_renders():
    sc = make_scene("c1", contraction="sph")
    cams, W, H = config_cameras("c1")
    r = O.render(O.OracleScene(sc), cams[0], W, H, mode="sph")
    assert r["stats"]["evaluated"] > 0 and r["stats"]["missing"] == 0
    assert 0.05 < r["rgb"].mean() < 0.95


@pytest.mark.gpu
@pytest.mark.parametrize("flags", [0, 1])
def test_gpu_sph_parity_c1(flags):
    import torch
    import paper_2302_12249_b200 as M
    sc = make_scene("c1", contraction="sph")
    cams, W, H = config_cameras("c1")
    s = M.Scene(sc)
    out, st = s.render(cams, W, H, flags=M.MERF_SPHERICAL | flags, stats=True)
    torch.cuda.synchronize()
    osc = O.OracleScene(sc)
    ref = O.render(osc, cams[0], W, H, mode="sph", flags=flags, max_trace=2048)
    assert np.abs(out[0].reshape(-1, 3).cpu().numpy() - ref["rgb"]).max() <= 2e-3
    pid = torch.arange(W * H, device="cuda")
    cells = torch.zeros((W * H, 2048), dtype=torch.int64, device="cuda")
    cnt = torch.zeros(W * H, dtype=torch.int32, device="cuda")
    M.merf_trace(s.handle, cams[0], W, pid, 2048, cells, None, cnt, flags=M.MERF_SPHERICAL | flags)
    torch.cuda.synchronize()
    g = cells.cpu().numpy().view(np.uint64)
    gn = cnt.cpu().numpy()
    if flags:
        assert np.array_equal(gn, ref["trace_count"])
        assert st["evaluated"] == ref["stats"]["evaluated"]
    for p in range(W * H):
        n = min(gn[p], ref["trace_count"][p])
        assert np.array_equal(g[p, :n], ref["trace_cells"][p, :n])
    s.close()


@pytest.mark.gpu
def test_gpu_sph_parity_paper_scale_sampled():
    import torch
    import paper_2302_12249_b200 as M
    sc = make_scene("c2", contraction="sph")
    cams, W, H = config_cameras("c2")
    s = M.Scene(sc)
    out = s.render(cams, W, H, flags=M.MERF_SPHERICAL)
    torch.cuda.synchronize()
    pix = np.unique(np.random.default_rng(3).integers(0, W * H, 3000))
    ref = O.render(O.OracleScene(sc), cams[0], W, H, pixels=pix, mode="sph")
    assert np.abs(out[0].reshape(-1, 3).cpu().numpy()[pix] - ref["rgb"]).max() <= 2e-3
    s.close()


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_gpu_sph_persistent_statistical_parity(cfg):
    """MERF_SPH_PERSISTENT: the same curve march (reading S1) in fp32 inside the persistent
    tile-scheduled march with the production gather.  fp32 sample positions drift from the
    canonical fp64 steps by ~1e-6 contracted units, so a sample near a finest-cell face can
    change sides: parity is statistical -- PSNR, the share of pixels inside the 2e-3 bar, and
    the evaluated-sample count."""
    import torch
    import paper_2302_12249_b200 as M
    from conftest import psnr
    sc = make_scene(cfg, contraction="sph")
    cams, W, H = config_cameras(cfg)
    s = M.Scene(sc)
    out, st = s.render(cams, W, H, flags=M.MERF_SPHERICAL | M.MERF_SPH_PERSISTENT, stats=True)
    exact, st_e = s.render(cams, W, H, flags=M.MERF_SPHERICAL, stats=True)
    torch.cuda.synchronize()
    s.close()
    g = out[0].reshape(-1, 3).cpu().numpy()
    ge = exact[0].reshape(-1, 3).cpu().numpy()
    if cfg == "c1":
        ref = O.render(O.OracleScene(sc), cams[0], W, H, mode="sph")["rgb"]
        pix = np.arange(W * H)
    else:
        pix = np.unique(np.random.default_rng(4).integers(0, W * H, 3000))
        ref = O.render(O.OracleScene(sc), cams[0], W, H, pixels=pix, mode="sph")["rgb"]
    err = np.abs(g[pix] - ref).max(axis=1)
    assert psnr(g[pix], ref) >= 45.0
    assert (err <= 2e-3).mean() >= 0.99
    assert abs(st["evaluated"] - st_e["evaluated"]) <= 0.01 * st_e["evaluated"]
    assert np.abs(ge[pix] - ref).max() <= 2e-3            # the fp64 kernel stays exact
