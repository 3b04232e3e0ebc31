"""GPU parity: the CUDA path (through the C ABI) against the fp64 CPU oracle on the same
seeded scenes and cameras.  Bar (BASELINE.json north_star): bit-exact occupancy levels,
block indirection and per-ray visited-cell traces; colour max |err| <= 2e-3 and
PSNR >= 50 dB."""
import math

import numpy as np
import pytest

from conftest import psnr
from merf_inputs import (make_scene, constant_scene, random_scene, config_cameras,
                         look_at_camera, unpack_bits, orbit_cameras)
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL = 2e-3
MIN_PSNR = 50.0


@pytest.fixture(scope="module")
def M():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2302_12249_b200 import build
    build.build()
    import paper_2302_12249_b200 as M
    return M


@pytest.fixture(scope="module")
def c2():
    return make_scene("c2")


def _gpu_frame(M, sc, cams, W, H, flags=0, fmt=0, stats=True):
    import torch
    s = M.Scene(sc)
    out, st = s.render(cams, W, H, fmt=fmt, flags=flags, stats=True)
    torch.cuda.synchronize()
    s.close()
    return out.cpu().numpy(), st


def _gpu_trace(M, sc, cam, W, pixels, max_per_ray=2048, flags=0):
    import torch
    s = M.Scene(sc)
    pid = torch.as_tensor(np.asarray(pixels, np.int64), device="cuda")
    n = len(pixels)
    cells = torch.zeros((n, max_per_ray), dtype=torch.int64, device="cuda")
    T = torch.zeros((n, max_per_ray), dtype=torch.float32, device="cuda")
    cnt = torch.zeros(n, dtype=torch.int32, device="cuda")
    M.merf_trace(s.handle, cam, W, pid, max_per_ray, cells, T, cnt, flags=flags)
    torch.cuda.synchronize()
    s.close()
    return cells.cpu().numpy().view(np.uint64), T.cpu().numpy(), cnt.cpu().numpy()


# GPU density with 16-bit exact-partition weights (GPU numerical choices):
# |dt0| <= 24 * 127.5 / 65535 * 2m/255 = 0.0051 (m = 14), so optical depth agrees to
# OD_REL = 0.52 % relative (+ fp32 slack), and T at the termination cut (OD = ln 5000) to
# T_CUT_REL = exp(0.0052 * ln 5000) - 1 = 4.5 % (reading D19).
OD_REL = 0.0052
T_CUT_REL = 0.045


def _close_transmittance(Tg, To):
    """GPU vs oracle transmittance after each sample, within the optical-depth bound."""
    Tg, To = np.asarray(Tg, np.float64), np.asarray(To, np.float64)
    live = To > 1e-5
    odg, odo = -np.log(np.maximum(Tg[live], 1e-30)), -np.log(To[live])
    ok = np.all(np.abs(odg - odo) <= OD_REL * odo + 2e-5)
    return ok and np.all(Tg[~live] <= 2e-5)


def _compare_traces(g, o, T_oracle=None, t_min=2e-4):
    """bit-exact visited cells; with termination on, a length may differ only when the
    oracle's transmittance at the cut is within T_CUT_REL of t_min (reading D19)."""
    gc, gT, gn = g
    oc, on = o["trace_cells"], o["trace_count"]
    mism = 0
    for r in range(len(gn)):
        n = min(gn[r], on[r], gc.shape[1])
        assert np.array_equal(gc[r, :n], oc[r, :n]), f"ray {r}: first diff at {np.argmax(gc[r,:n] != oc[r,:n])}"
        if gn[r] != on[r]:
            mism += 1
            k = min(gn[r], on[r]) - 1
            Tcut = o["trace_T"][r, k]
            assert abs(Tcut - t_min) <= T_CUT_REL * t_min, (r, gn[r], on[r], Tcut)
    return mism


# ------------------------------------------------------------------------------------
# structures (bit-exact)
# ------------------------------------------------------------------------------------
def test_occupancy_pyramid_bit_exact(M, c2):
    import torch
    s = M.Scene(c2)
    ref = O.build_pyramid(c2.occ_finest, c2.level_res)
    for lev, N in enumerate(c2.level_res):
        out = torch.zeros(O.n_words(N), dtype=torch.int32, device="cuda")
        M.merf_scene_occupancy(s.handle, lev, out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), ref[lev]), lev
    # the standalone helper too
    fin = torch.as_tensor(c2.occ_finest.view(np.int32), device="cuda")
    tot = sum(O.n_words(N) for N in c2.level_res[:-1])
    lv = torch.zeros(tot, dtype=torch.int32, device="cuda")
    M.merf_build_occupancy(fin, c2, lv)
    torch.cuda.synchronize()
    assert np.array_equal(lv.cpu().numpy().view(np.uint32), np.concatenate(ref[:-1]))
    s.close()


@pytest.mark.parametrize("case", ["c1", "c2", "rand"])
def test_block_index_bit_exact(M, c2, case):
    import torch
    sc = {"c1": lambda: make_scene("c1"), "c2": lambda: c2,
          "rand": lambda: random_scene(seed=9, L=64, R=32, level_res=(8, 32))}[case]()
    ref, n = O.canonical_block_index(sc.occ_finest, sc.level_res[-1], sc.L)
    fin = torch.as_tensor(sc.occ_finest.view(np.int32), device="cuda")
    idx = torch.zeros(len(ref), dtype=torch.int32, device="cuda")
    got_n = M.merf_build_block_index(fin, sc, idx)
    torch.cuda.synchronize()
    assert got_n == n
    assert np.array_equal(idx.cpu().numpy(), ref)
    s = M.Scene(sc)
    assert s.info()["canonical_blocks"] == n
    s.close()


def test_upload_rejects_unsound_block_index(M):
    sc = random_scene(seed=4, L=32, R=32, level_res=(8, 16))
    ref, n = O.canonical_block_index(sc.occ_finest, 16, 32)
    bad = sc.block_index.copy()
    victim = np.nonzero(ref >= 0)[0][0]
    bad[victim] = -1
    sc.block_index = bad
    with pytest.raises(M.MerfError) as e:
        M.merf_scene_upload(sc)
    assert e.value.status == M.MERF_EMISMATCH
    bad = sc.block_index.copy()
    bad[np.nonzero(bad >= 0)[0][0]] = sc.atlas.shape[0] + 5
    sc.block_index = bad
    with pytest.raises(M.MerfError):
        M.merf_scene_upload(sc)


def test_canonical_upload_matches_explicit(M):
    # atlas supplied in canonical order with block_index = NULL renders identically
    import torch
    sc = random_scene(seed=6, L=32, R=32, level_res=(8, 16))
    ref, n = O.canonical_block_index(sc.occ_finest, 16, 32)
    # re-pack the atlas in canonical order
    slots = np.nonzero(ref >= 0)[0]
    atlas = sc.atlas[sc.block_index[slots]]
    import copy
    sc2 = copy.copy(sc)
    sc2.atlas = np.ascontiguousarray(atlas)
    sc2.block_index = ref
    cams, W, H = config_cameras("c1")
    a, _ = _gpu_frame(M, sc, cams, W, H)
    s = M.Scene(sc2, canonical=True)
    b = s.render(cams, W, H)
    torch.cuda.synchronize()
    assert np.array_equal(a, b.cpu().numpy())
    s.close()


def test_contract_helper_bit_exact(M):
    import torch
    rng = np.random.default_rng(0)
    x = rng.standard_cauchy((100000, 3)) * rng.uniform(0.1, 10, (100000, 1))
    x[:10] = [[4, 0, 0], [2, 4, 0], [-3, 1, 0.5], [2, 2, 0], [1, -1, 1], [0, 0, 0], [0, 5, 0],
              [0, 0, -10], [1e30, 1, 1], [-1e-30, 0, 0]]
    y_ref, r_ref = O.contract(x)
    xd = torch.as_tensor(x, device="cuda")
    yd = torch.empty_like(xd)
    rd = torch.empty(len(x), dtype=torch.int32, device="cuda")
    M.merf_contract(xd, yd, rd)
    torch.cuda.synchronize()
    assert np.array_equal(yd.cpu().numpy(), y_ref)
    assert np.array_equal(rd.cpu().numpy(), r_ref)


# ------------------------------------------------------------------------------------
# full frames, C1 (tiny): colour + traces + stats
# ------------------------------------------------------------------------------------
def test_c1_frame_colour(M, c1_scene):
    cams, W, H = config_cameras("c1")
    got, st = _gpu_frame(M, c1_scene, cams, W, H)
    ref = O.render(O.OracleScene(c1_scene), cams[0], W, H)
    g = got[0].reshape(-1, 3)
    assert np.abs(g - ref["rgb"]).max() <= TOL
    assert psnr(g, ref["rgb"]) >= MIN_PSNR
    assert st["rays"] == W * H
    assert st["evaluated"] == ref["stats"]["evaluated"]
    # the default traversal skips with all dyadic levels (reading D23): never more skips than
    # the scene's own levels; the level search (MERF_NO_SKIPTAB) reproduces the oracle's count
    assert st["skips"] <= ref["stats"]["skips"]
    import os
    os.environ["MERF_NO_SKIPTAB"] = "1"
    try:
        _, st_lv = _gpu_frame(M, c1_scene, cams, W, H)
    finally:
        os.environ.pop("MERF_NO_SKIPTAB", None)
    assert st_lv["skips"] == ref["stats"]["skips"] and st_lv["evaluated"] == ref["stats"]["evaluated"]
    assert st["segments"] == ref["stats"]["segments"]
    assert st["missing_blocks"] == 0


@pytest.mark.parametrize("flags", [0, 1])
def test_c1_traces_bit_exact(M, c1_scene, flags):
    cams, W, H = config_cameras("c1")
    pix = np.arange(W * H)
    g = _gpu_trace(M, c1_scene, cams[0], W, pix, max_per_ray=1024, flags=flags)
    o = O.render(O.OracleScene(c1_scene), cams[0], W, H, max_trace=1024, flags=flags)
    mism = _compare_traces(g, o)
    if flags == 1:
        assert mism == 0 and np.array_equal(g[2], o["trace_count"])
    # transmittance after each sample agrees within the optical-depth bound
    n = np.minimum(g[2], o["trace_count"])
    for r in range(0, W * H, 7):
        assert _close_transmittance(g[1][r, :n[r]], o["trace_T"][r, :n[r]]), r


def test_dense_equals_hierarchical_on_gpu(M, c1_scene):
    cams, W, H = config_cameras("c1")
    a, sa = _gpu_frame(M, c1_scene, cams, W, H)
    b, sb = _gpu_frame(M, c1_scene, cams, W, H, flags=M.MERF_DENSE)
    assert np.array_equal(a, b)
    assert sa["evaluated"] == sb["evaluated"] and sb["skips"] == 0
    pix = np.arange(W * H)
    ga = _gpu_trace(M, c1_scene, cams[0], W, pix, 1024)
    gb = _gpu_trace(M, c1_scene, cams[0], W, pix, 1024, flags=M.MERF_DENSE)
    assert np.array_equal(ga[0], gb[0]) and np.array_equal(ga[2], gb[2])


def test_determinism_and_u8(M, c1_scene):
    cams, W, H = config_cameras("c1")
    a, _ = _gpu_frame(M, c1_scene, cams, W, H)
    b, _ = _gpu_frame(M, c1_scene, cams, W, H)
    assert np.array_equal(a, b)
    u8, _ = _gpu_frame(M, c1_scene, cams, W, H, fmt=M.MERF_RGBA_U8)
    assert np.array_equal(u8[..., :3], np.rint(a * 255).astype(np.uint8))
    assert (u8[..., 3] == 255).all()


# ------------------------------------------------------------------------------------
# random scenes with ragged frame sizes and every source variant
# ------------------------------------------------------------------------------------
@pytest.mark.parametrize("seed,mask,WH", [(1, 15, (37, 23)), (2, 15, (64, 48)), (3, 1, (33, 17)),
                                          (4, 14, (40, 40)), (5, 15, (1, 1)), (6, 5, (23, 61))])
def test_random_scenes(M, seed, mask, WH):
    W, H = WH
    sc = random_scene(seed=seed, L=32, R=64, level_res=(4, 16, 32), occ_fraction=0.2,
                      source_mask=mask, density_offset=-10)
    rng = np.random.default_rng(seed)
    cams = np.stack([look_at_camera(rng.uniform(-1.5, 1.5, 3), target=rng.uniform(-0.5, 0.5, 3),
                                    W=W, H=H, fov_x_deg=70) for _ in range(3)])
    got, st = _gpu_frame(M, sc, cams, W, H)
    _, st_all = _gpu_frame(M, sc, cams, W, H, flags=M.MERF_NO_EARLY_TERM)
    osc = O.OracleScene(sc)
    ev, ev_all = 0, 0
    for c in range(3):
        ref = O.render(osc, cams[c], W, H)
        g = got[c].reshape(-1, 3)
        assert np.abs(g - ref["rgb"]).max() <= TOL, c
        ev += ref["stats"]["evaluated"]
        o = O.render(osc, cams[c], W, H, max_trace=2048, flags=O.NO_EARLY_TERM)
        gt = _gpu_trace(M, sc, cams[c], W, np.arange(W * H), 2048, flags=M.MERF_NO_EARLY_TERM)
        assert np.array_equal(gt[2], o["trace_count"])
        assert np.array_equal(gt[0], o["trace_cells"])
        ev_all += int(o["trace_count"].sum())
    # the sample set is integer work (exact); the T < t_min cut is a float decision (D19)
    assert st_all["evaluated"] == ev_all
    assert abs(st["evaluated"] - ev) <= 1e-3 * ev


def test_empty_occupancy(M):
    N = 16
    sc = constant_scene(L=16, R=32, level_res=(8, 16), occ=np.zeros((N, N, N), bool))
    sc.mlp = make_scene("c1").mlp
    cams, W, H = config_cameras("c1")
    got, st = _gpu_frame(M, sc, cams, W, H)
    ref = O.render(O.OracleScene(sc), cams[0], W, H)
    assert st["evaluated"] == 0
    assert np.abs(got[0].reshape(-1, 3) - ref["rgb"]).max() <= 1e-5


@pytest.mark.parametrize("i", range(5))
def test_constant_scene_closed_form_on_gpu(M, i):
    import json, os, torch
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_form.json")))
    case = g["cases"][i]
    sc = constant_scene(L=16, R=32, level_res=(8, 16), step=g["delta"], b_d=case["b_d"], b_a=case["b_a"])
    s = M.Scene(sc)
    o = torch.zeros((1, 3), dtype=torch.float64, device="cuda")
    d = torch.tensor([[1.0, 0.0, 0.0]], dtype=torch.float64, device="cuda")
    rgb = torch.zeros((1, 3), dtype=torch.float32, device="cuda")
    st = M.merf_render_rays(s.handle, o, d, rgb, stats=True)
    torch.cuda.synchronize()
    assert st["evaluated"] == case["n"]
    assert np.allclose(rgb.cpu().numpy()[0], case["C_zero_mlp"], atol=1e-5)
    s.close()


def test_render_rays_matches_oracle(M, c1_scene):
    import torch
    rng = np.random.default_rng(3)
    n = 5000
    o = rng.uniform(-1.2, 1.2, (n, 3))
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    tn = rng.uniform(0, 0.3, n)
    ref = O.render_rays(O.OracleScene(c1_scene), o, d, tn)
    s = M.Scene(c1_scene)
    rgb = torch.zeros((n, 3), dtype=torch.float32, device="cuda")
    st = M.merf_render_rays(s.handle, torch.as_tensor(o, device="cuda"), torch.as_tensor(d, device="cuda"),
                            rgb, t_near=torch.as_tensor(tn, device="cuda"), stats=True)
    torch.cuda.synchronize()
    assert np.abs(rgb.cpu().numpy() - ref["rgb"]).max() <= TOL
    assert st["evaluated"] == ref["stats"]["evaluated"]
    s.close()


# ------------------------------------------------------------------------------------
# paper-scale scenes at full size (sampled pixels the oracle computes one by one)
# ------------------------------------------------------------------------------------
def _sampled(M, sc, cam, W, H, n=6000, seed=0, trace=512):
    import torch
    s = M.Scene(sc)
    out = s.render(cam[None], W, H)
    torch.cuda.synchronize()
    got = out[0].reshape(-1, 3).cpu().numpy()
    s.close()
    rng = np.random.default_rng(seed)
    pix = np.unique(np.concatenate([rng.integers(0, W * H, n), np.arange(0, W * H, 997)]))
    osc = O.OracleScene(sc)
    ref = O.render(osc, cam, W, H, pixels=pix)
    err = np.abs(got[pix] - ref["rgb"])
    assert err.max() <= TOL, err.max()
    assert psnr(got[pix], ref["rgb"]) >= MIN_PSNR
    tp = pix[:trace]
    o = O.render(osc, cam, W, H, pixels=tp, max_trace=4096, flags=O.NO_EARLY_TERM)
    g = _gpu_trace(M, sc, cam, W, tp, 4096, flags=M.MERF_NO_EARLY_TERM)
    assert np.array_equal(g[2], o["trace_count"])
    assert np.array_equal(g[0], o["trace_cells"])
    return got


def test_c2_paper_scale_sampled(M, c2):
    cams, W, H = config_cameras("c2")
    _sampled(M, c2, cams[0], W, H)


@pytest.mark.parametrize("pose", [0, 1])
def test_c3_unbounded_sampled(M, c2, pose):
    cams, W, H = config_cameras("c3")
    _sampled(M, c2, cams[pose], W, H, n=4000, seed=pose)


def test_c3_all_regions(M, c2):
    cams, W, H = config_cameras("c3")
    _, st = _gpu_frame(M, c2, cams, W, H)
    assert all(v > 0 for v in st["region_segments"]), st["region_segments"]


def test_c4_orbit_views_sampled(M, c2):
    cams = orbit_cameras(256, indices=[0, 77, 200])
    for k in range(3):
        _sampled(M, c2, cams[k], 1920, 1080, n=2000, seed=10 + k, trace=128)


def test_render_host_equals_render(M, c1_scene):
    import torch
    cams = orbit_cameras(16, W=64, H=48, indices=range(9))
    s = M.Scene(c1_scene)
    dev = s.render(cams, 64, 48, fmt=M.MERF_RGBA_U8)
    torch.cuda.synchronize()
    host = torch.zeros((9, 48, 64, 4), dtype=torch.uint8).pin_memory()
    M.merf_render_host(s.handle, cams, 64, 48, host, fmt=M.MERF_RGBA_U8)
    assert torch.equal(dev.cpu(), host)
    s.close()


def test_render_host_async_stream_equals_render(M, c1_scene):
    """merf_render_host_async over a stream of calls (buffers alternate, copies overlap the
    next render, a buffer is reused only after its copy) lands every frame intact."""
    import torch
    s = M.Scene(c1_scene)
    batches = [orbit_cameras(16, W=64, H=48, indices=range(i, i + 5)) for i in range(0, 15, 5)]
    hosts = [torch.zeros((5, 48, 64, 4), dtype=torch.uint8).pin_memory() for _ in range(3)]
    for b, h in zip(batches, hosts):
        M.merf_render_host_async(s.handle, b, 64, 48, h, fmt=M.MERF_RGBA_U8)
    M.merf_host_wait(s.handle)
    for b, h in zip(batches, hosts):
        dev = s.render(b, 64, 48, fmt=M.MERF_RGBA_U8)
        torch.cuda.synchronize()
        assert torch.equal(dev.cpu(), h)
    s.close()


def _gpu_segments(M, sc, cam, W, pixels, max_seg=8):
    import torch
    s = M.Scene(sc)
    pid = torch.as_tensor(np.asarray(pixels, np.int64), device="cuda")
    n = len(pixels)
    segs = torch.zeros(n * max_seg * M.merf.SEGMENT_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    cnt = torch.zeros(n, dtype=torch.int32, device="cuda")
    M.merf_segments(s.handle, cam, W, pid, max_seg, segs, cnt)
    torch.cuda.synchronize()
    s.close()
    return segs.cpu().numpy().view(M.merf.SEGMENT_DTYPE).reshape(n, max_seg), cnt.cpu().numpy()


@pytest.mark.parametrize("cfg", ["c1", "c3a", "c3b", "outside"])
def test_segments_bit_exact(M, c1_scene, cfg):
    """contracted segments (region, t interval, lattice Qa/U, K) equal the oracle's bit for bit."""
    if cfg == "c1":
        cams, W, H = config_cameras("c1")
        cam, pix = cams[0], np.arange(W * H)
    elif cfg.startswith("c3"):
        cams, W, H = config_cameras("c3")
        cam = cams[0 if cfg == "c3a" else 1]
        pix = np.random.default_rng(5).integers(0, W * H, 3000)
    else:
        W, H = 64, 64
        cam = look_at_camera((0.0354, 1.3514, -1.0675), target=(0.3, -0.2, 0.1), W=W, H=H, fov_x_deg=90)
        pix = np.arange(W * H)
    segs, cnt = _gpu_segments(M, c1_scene, cam, W, pix)
    for r, p in enumerate(pix):
        o, d = O.raygen(cam, p % W, p // W)
        ref = O.segment_ray(o, d, cam[16], c1_scene.step)
        assert cnt[r] == len(ref), (p, cnt[r], len(ref))
        for a, b in zip(ref, segs[r]):
            assert a["region"] == b["region"] and a["K"] == b["K"], p
            assert a["t_a"] == b["t_a"] and (a["t_b"] == b["t_b"]), p
            assert np.array_equal(a["Qa"], b["Qa"]) and np.array_equal(a["U"], b["U"]), p


def test_upload_copies_inputs_before_returning(M):
    """Regression (stale-upload bug): the render after an upload must see exactly the uploaded
    arrays even if the caller overwrites its host buffers right after merf_scene_upload
    returns (ownership contract in include/merf.h)."""
    import copy
    import torch
    sc = random_scene(seed=8, L=64, R=64, level_res=(8, 32), occ_fraction=0.3)
    ref_sc = copy.deepcopy(sc)
    s = M.Scene(sc)
    sc.atlas[...] = 255
    sc.planes[...] = 255
    sc.occ_finest[...] = 0
    cams, W, H = config_cameras("c1")
    out = s.render(cams, W, H)
    torch.cuda.synchronize()
    ref = O.render(O.OracleScene(ref_sc), cams[0], W, H)
    assert np.abs(out[0].reshape(-1, 3).cpu().numpy() - ref["rgb"]).max() <= TOL
    s.close()


def test_bench_launch_configuration(M, c2):
    """The exact launch bench.py times: 16 orbit views at 1920x1080 in one merf_render call
    (one 16-view chunk of the persistent pipeline), RGBA8 output, MERF_TIMED.  Sampled pixels
    of four views vs the oracle: |u8 - round(255 C_oracle)| <= 1."""
    import torch
    import bench
    cams = orbit_cameras(256, indices=bench.views_for(0, 1, 3, 16))
    s = M.Scene(c2)
    out = torch.empty((16, 1080, 1920, 4), dtype=torch.uint8, device="cuda")
    M.merf_render(s.handle, cams, 1920, 1080, out, fmt=M.MERF_RGBA_U8, flags=M.MERF_TIMED)
    torch.cuda.synchronize()
    kt = M.merf_kernel_times_get(s.handle)
    assert kt["march_launches"] == 1 and kt["setup_launches"] == 1 and kt["shade_launches"] == 1
    osc = O.OracleScene(c2)
    rng = np.random.default_rng(11)
    for v in (0, 7, 8, 15):                      # first, middle and last views
        pix = rng.integers(0, 1920 * 1080, 1500)
        ref = O.render(osc, cams[v], 1920, 1080, pixels=pix)["rgb"]
        got = out[v].reshape(-1, 4)[torch.as_tensor(pix, device="cuda")].cpu().numpy()
        assert (got[:, 3] == 255).all()
        assert np.abs(got[:, :3].astype(int) - np.rint(ref * 255).astype(int)).max() <= 1, v
    s.close()


def test_render_argument_errors(M, c1_scene):
    import torch
    s = M.Scene(c1_scene)
    cams, W, H = config_cameras("c1")
    out = torch.empty((1, H, W, 3), device="cuda")
    for bad in (dict(W=0), dict(H=-1), dict(fmt=7)):
        kw = dict(W=W, H=H, fmt=M.MERF_RGB_F32)
        kw.update(bad)
        with pytest.raises(M.MerfError) as e:
            M.merf_render(s.handle, cams, kw["W"], kw["H"], out, fmt=kw["fmt"])
        assert e.value.status == M.MERF_EINVAL
    with pytest.raises(M.MerfError):
        M.merf_render(s.handle, cams, 70000, 70000, out)            # W*H overflow
    bad_cam = cams.copy()
    bad_cam[0, 12] = 0.0                                            # fx = 0
    with pytest.raises(M.MerfError):
        M.merf_render(s.handle, bad_cam, W, H, out)
    s.close()


def test_skip_table_equals_level_search(M, c2):
    """the per-cell skip table (one 4-bit probe over all dyadic levels) and the coarse -> fine
    search over the scene's levels skip only empty space: identical frames, evaluated samples
    and traces; the table's larger cells need no more skips (MERF_NO_SKIPTAB selects the
    search)."""
    import os
    import torch
    cams, W, H = config_cameras("c2")
    s = M.Scene(c2)
    pix = np.random.default_rng(3).integers(0, W * H, 300)
    outs, stats, traces = [], [], []
    for env in ("0", "1"):
        os.environ["MERF_NO_SKIPTAB"] = env
        try:
            out, st = s.render(cams, W, H, stats=True)
            pid = torch.as_tensor(pix, device="cuda")
            cells = torch.zeros((len(pix), 2048), dtype=torch.int64, device="cuda")
            cnt = torch.zeros(len(pix), dtype=torch.int32, device="cuda")
            M.merf_trace(s.handle, cams[0], W, pid, 2048, cells, None, cnt)
            torch.cuda.synchronize()
        finally:
            os.environ.pop("MERF_NO_SKIPTAB", None)
        outs.append(out.cpu().numpy())
        stats.append({k: st[k] for k in ("evaluated", "skips", "density_only")})
        traces.append((cells.cpu().numpy(), cnt.cpu().numpy()))
    s.close()
    assert np.array_equal(outs[0], outs[1])
    assert stats[0]["evaluated"] == stats[1]["evaluated"]
    assert stats[0]["density_only"] == stats[1]["density_only"]
    assert stats[0]["skips"] <= stats[1]["skips"]
    assert np.array_equal(traces[0][0], traces[1][0]) and np.array_equal(traces[0][1], traces[1][1])


# ------------------------------------------------------------------------------------
# deferred MLP on the tensor cores (merf_shade_mma.cu) vs the FFMA kernel and the oracle
# ------------------------------------------------------------------------------------
# split-fp16 products (hi*hi + hi*lo + lo*hi, fp32 accumulation) drop terms of ~2^-22 relative;
# through three 16-wide layers with |W| <= 0.3 the logits agree with fp32 FFMA chains to ~1e-6
MMA_VS_FFMA = 2e-5


def test_mlp_mma_matches_ffma_and_oracle(M, c1_scene, c2):
    import dataclasses
    cams, W, H = config_cameras("c1")
    a, _ = _gpu_frame(M, c1_scene, cams, W, H)
    b, _ = _gpu_frame(M, c1_scene, cams, W, H, flags=M.MERF_MLP_FFMA)
    assert np.abs(a - b).max() <= MMA_VS_FFMA
    ref = O.render(O.OracleScene(c1_scene), cams[0], W, H)
    assert np.abs(a[0].reshape(-1, 3) - ref["rgb"]).max() <= TOL
    # paper-scale scene, two orbit views, ragged tiles (1080 = 270 x 4 rows, 1920 = 240 x 8)
    oc = orbit_cameras(256, indices=[3, 77])
    a, _ = _gpu_frame(M, c2, oc, 1920, 1080)
    b, _ = _gpu_frame(M, c2, oc, 1920, 1080, flags=M.MERF_MLP_FFMA)
    assert np.abs(a - b).max() <= MMA_VS_FFMA
    # a ragged frame (partial 8x4 tiles: lanes without a pixel still join the warp's mma)
    cam = look_at_camera(np.array([0.1, 0.05, -0.2]), target=np.zeros(3), W=37, H=29, fov_x_deg=60)
    a, _ = _gpu_frame(M, c1_scene, cam[None], 37, 29)
    b, _ = _gpu_frame(M, c1_scene, cam[None], 37, 29, flags=M.MERF_MLP_FFMA)
    assert np.abs(a - b).max() <= MMA_VS_FFMA
    # larger weights (exactly scaled by 4; hidden activations of tens to hundreds): still inside
    # the fp16 operand bound, still fp32-class
    big = dataclasses.replace(c1_scene, mlp=c1_scene.mlp * 4.0)
    a, _ = _gpu_frame(M, big, cams, W, H)
    b, _ = _gpu_frame(M, big, cams, W, H, flags=M.MERF_MLP_FFMA)
    assert np.abs(a - b).max() <= 10 * MMA_VS_FFMA
    ref = O.render(O.OracleScene(big), cams[0], W, H)
    assert np.abs(a[0].reshape(-1, 3) - ref["rgb"]).max() <= TOL


def test_mlp_fp16_overflow_bound_falls_back_to_ffma(M, c1_scene):
    """weights whose activation bound exceeds the fp16 range: the upload keeps no fragment
    table and every render runs the FFMA kernel (identical with and without the flag)."""
    import dataclasses
    cams, W, H = config_cameras("c1")
    huge = dataclasses.replace(c1_scene, mlp=c1_scene.mlp * 2048.0)
    a, _ = _gpu_frame(M, huge, cams, W, H)
    b, _ = _gpu_frame(M, huge, cams, W, H, flags=M.MERF_MLP_FFMA)
    assert np.array_equal(a, b)


def test_mlp_mma_rays_and_u8(M, c1_scene):
    import torch
    rng = np.random.default_rng(11)
    n = 1001                                    # ragged: the last warp is partly empty
    o = rng.uniform(-1.2, 1.2, (n, 3))
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    s = M.Scene(c1_scene)
    outs = []
    for fl in (0, M.MERF_MLP_FFMA):
        rgb = torch.zeros((n, 3), dtype=torch.float32, device="cuda")
        M.merf_render_rays(s.handle, torch.as_tensor(o, device="cuda"), torch.as_tensor(d, device="cuda"),
                           rgb, flags=fl)
        torch.cuda.synchronize()
        outs.append(rgb.cpu().numpy())
    s.close()
    assert np.abs(outs[0] - outs[1]).max() <= MMA_VS_FFMA
    cams, W, H = config_cameras("c1")
    f32, _ = _gpu_frame(M, c1_scene, cams, W, H)
    u8, _ = _gpu_frame(M, c1_scene, cams, W, H, fmt=M.MERF_RGBA_U8)
    assert np.array_equal(u8[..., :3], np.rint(f32 * 255).astype(np.uint8))


# ------------------------------------------------------------------------------------
# single-frame sharding (merf_render_shard): 64x64 blocks interleaved by rank
# ------------------------------------------------------------------------------------
@pytest.mark.parametrize("N,WH", [(2, (1920, 1080)), (3, (130, 70)), (5, (257, 129)), (1, (64, 64))])
def test_render_shard_partition(M, c1_scene, c2, N, WH):
    import torch
    W, H = WH
    sc = c2 if W >= 1000 else c1_scene
    cam = orbit_cameras(256, indices=[9], W=W, H=H) if W >= 1000 else \
        look_at_camera(np.array([0.1, 0.05, -0.2]), target=np.zeros(3), W=W, H=H, fov_x_deg=60)[None]
    s = M.Scene(sc)
    full = torch.zeros((1, H, W, 4), dtype=torch.uint8, device="cuda")
    M.merf_render(s.handle, cam, W, H, full, fmt=M.MERF_RGBA_U8)
    acc = torch.zeros((1, H, W, 4), dtype=torch.int32, device="cuda")
    owner = M.shard_owner(W, H, N)
    for r in range(N):
        part = torch.zeros((1, H, W, 4), dtype=torch.uint8, device="cuda")
        M.merf_render_shard(s.handle, cam, W, H, r, N, part, fmt=M.MERF_RGBA_U8)
        torch.cuda.synchronize()
        p = part.cpu().numpy()[0]
        # the shard writes exactly its own blocks (alpha 255 there, untouched zeros elsewhere)
        assert np.array_equal(p[..., 3] == 255, owner == r)
        acc += part.to(torch.int32)
    torch.cuda.synchronize()
    # disjoint shards sum (e.g. an NCCL reduce) to the unsharded frame, byte for byte
    assert np.array_equal(acc.cpu().numpy().astype(np.uint8), full.cpu().numpy())
    with pytest.raises(M.MerfError):
        M.merf_render_shard(s.handle, cam, W, H, N, N, full, fmt=M.MERF_RGBA_U8)
    s.close()


def test_randomised_stress_one_case_per_geometry(M):
    """tools/stress_parity.py, one random case per geometry (paper geometry, small grids,
    V-only, planes-only, V + one plane): every pixel within 2e-3 of the oracle, every pixel's
    trace (termination off) bit-exact."""
    import importlib.util
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("stress_parity", os.path.join(root, "tools", "stress_parity.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    assert mod.run(len(mod.GEOMS), seed=2026, verbose=False) == 0


@pytest.mark.parametrize("cfg", ["c2", "rand"])
def test_mixed_skip_table_equals_dyadic(M, c2, cfg):
    """reading D23, round 2: the table offers per cell the larger of the coarsest empty dyadic
    cell and the empty Chebyshev cube around it (MERF_SKIP_DYADIC=1 builds the dyadic-only
    table).  Both skip only empty space: identical frames, evaluated samples and visited-cell
    traces, and the mixed table needs fewer skips over the frame."""
    import os
    import torch
    if cfg == "c2":
        sc = c2
        cams, W, H = config_cameras("c2")
    else:
        sc = random_scene(seed=12, L=64, R=128, level_res=(4, 16, 64), occ_fraction=0.05, blob_cells=3)
        W, H = 96, 64
        cams = look_at_camera(np.array([0.3, 1.2, -1.4]), target=np.zeros(3), W=W, H=H, fov_x_deg=80)[None]
    pix = np.random.default_rng(4).integers(0, W * H, 300)
    outs, stats, traces = [], [], []
    for env in ("1", "0"):
        os.environ["MERF_SKIP_DYADIC"] = env           # read when the scene is uploaded
        try:
            s = M.Scene(sc)
        finally:
            os.environ.pop("MERF_SKIP_DYADIC", None)
        out, st = s.render(cams, W, H, stats=True)
        pid = torch.as_tensor(pix, device="cuda")
        cells = torch.zeros((len(pix), 4096), dtype=torch.int64, device="cuda")
        cnt = torch.zeros(len(pix), dtype=torch.int32, device="cuda")
        M.merf_trace(s.handle, cams[0], W, pid, 4096, cells, None, cnt, flags=M.MERF_NO_EARLY_TERM)
        torch.cuda.synchronize()
        s.close()
        outs.append(out.cpu().numpy())
        stats.append({k: st[k] for k in ("evaluated", "skips", "density_only")})
        traces.append((cells.cpu().numpy(), cnt.cpu().numpy()))
    assert np.array_equal(outs[0], outs[1])
    assert stats[0]["evaluated"] == stats[1]["evaluated"] and stats[0]["density_only"] == stats[1]["density_only"]
    assert stats[1]["skips"] < stats[0]["skips"]
    assert np.array_equal(traces[0][0], traces[1][0]) and np.array_equal(traces[0][1], traces[1][1])


def test_tile_cost_history_order_is_bit_identical(M, c2):
    """Frame sequences: a small single-chunk call records its per-tile march durations and the
    next call with the same W, H and views dispatches tiles longest first by them (merf_api.cu,
    kHistMaxViews).  Dispatch order changes no ray's arithmetic: every frame of the sequence,
    whether it ran in raster order (first frame, or after a size change) or in history order,
    is byte-identical, and so are its counters."""
    import torch
    s = M.Scene(c2)
    cams = orbit_cameras(256, W=640, H=360, indices=[5, 77])
    frames, stats = [], []
    for W, H, cs in ((640, 360, cams), (640, 360, cams), (320, 180, cams[:1]), (640, 360, cams), (640, 360, cams)):
        out = torch.zeros((len(cs), H, W, 4), dtype=torch.uint8, device="cuda")
        st = M.merf_render(s.handle, cs, W, H, out, fmt=M.MERF_RGBA_U8, stats=True)
        torch.cuda.synchronize()
        if W == 640:
            frames.append(out.cpu().numpy())
            stats.append((st["evaluated"], st["skips"], st["density_only"]))
    s.close()
    for f, t in zip(frames[1:], stats[1:]):
        assert np.array_equal(f, frames[0])
        assert t == stats[0]
