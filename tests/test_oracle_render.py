"""Pins of the oracle's ray march (Eq. 1-3; traversal P:307-309) against closed
forms (constant scenes), the telescoping identity of Eq. 1, and brute-force dense stepping."""
import json
import math
import os

import numpy as np
import pytest

from merf_inputs import constant_scene, random_scene, make_scene, config_cameras, unpack_bits
from oracle import oracle as O

G = os.path.join(os.path.dirname(__file__), "golden")
AXIS_O = np.zeros((1, 3))
AXIS_D = np.array([[1.0, 0.0, 0.0]])


def _closed():
    with open(os.path.join(G, "closed_form.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("i", range(5))
def test_constant_scene_closed_form(i):
    g = _closed()
    case = g["cases"][i]
    sc = constant_scene(L=16, R=32, level_res=(8, 16), step=g["delta"], b_d=case["b_d"], b_a=case["b_a"])
    osc = O.OracleScene(sc)
    r = O.render_rays(osc, AXIS_O, AXIS_D, max_trace=256)
    assert r["trace_count"][0] == case["n"]
    assert r["stats"]["evaluated"] == case["n"]
    aux = r["aux"][0]
    assert abs(aux[7] - case["T"]) < 1e-12 * max(1.0, case["T"]) + 1e-15
    assert np.allclose(aux[:3], case["C_d"], atol=1e-12)
    assert np.allclose(r["rgb"][0], case["C_zero_mlp"], atol=1e-12)


def test_uniform_density_transmittance_is_exponential():
    # north_star: uniform density -> T = exp(-sigma t); here T_n = exp(-n tau Delta) (Eq. 1)
    for b_d in (110, 118, 124, 126):
        sc = constant_scene(L=16, R=32, level_res=(8, 16), step=2.0 ** -6, b_d=b_d, b_a=128)
        osc = O.OracleScene(sc)
        r = O.render_rays(osc, AXIS_O, AXIS_D, max_trace=256, flags=O.NO_EARLY_TERM)
        tau = math.exp(4 * (28 * b_d / 255 - 14))
        n = r["trace_count"][0]
        assert n == 128
        Ts = r["trace_T"][0, :n]
        expect = np.exp(-np.arange(1, n + 1) * tau * 2.0 ** -6)
        assert np.allclose(Ts, expect, rtol=1e-12, atol=0)


def test_termination_index_closed_form():
    # first n with exp(-n tau Delta) < 2e-4: n* = floor(ln(5000) / (tau Delta)) + 1
    for b_d in (128, 132, 136, 139):
        sc = constant_scene(L=16, R=32, level_res=(8, 16), step=2.0 ** -6, b_d=b_d, b_a=128)
        osc = O.OracleScene(sc)
        r = O.render_rays(osc, AXIS_O, AXIS_D, max_trace=256)
        tau_delta = math.exp(4 * (28 * b_d / 255 - 14)) * 2.0 ** -6
        n_star = math.floor(math.log(5000.0) / tau_delta) + 1
        assert r["trace_count"][0] == min(n_star, 128), b_d


def test_weights_telescope_to_one_minus_T():
    # constant appearance, random density: C_d = c (1 - T) and F = f (1 - T) (sum w = 1 - T)
    sc = random_scene(seed=11, L=16, R=32, level_res=(4, 8, 16), occ_fraction=0.3)
    sc.atlas[..., 1:] = 150
    sc.planes[..., 1:] = 120
    osc = O.OracleScene(sc)
    c = 1 / (1 + math.exp(-(14 * 150 / 255 - 7 + 3 * (14 * 120 / 255 - 7))))
    cams, W, H = config_cameras("c1")
    r = O.render(osc, cams[0], W, H, aux=True, flags=O.NO_EARLY_TERM)
    aux = r["aux"]
    one_minus_T = 1 - aux[:, 7]
    assert np.abs(aux[:, :3] - c * one_minus_T[:, None]).max() < 1e-12
    assert np.abs(aux[:, 3:7] - c * one_minus_T[:, None]).max() < 1e-12
    assert (aux[:, 7] >= 0).all() and (aux[:, 7] <= 1).all()
    assert r["stats"]["evaluated"] > 1000


def test_empty_occupancy_gives_mlp_of_zero():
    N = 16
    sc = constant_scene(L=16, R=32, level_res=(8, 16), occ=np.zeros((N, N, N), bool))
    sc.mlp = make_scene("c1").mlp
    osc = O.OracleScene(sc)
    d = np.array([[0.6, -0.48, 0.64]])
    r = O.render_rays(osc, np.zeros((1, 3)), d)
    assert r["stats"]["evaluated"] == 0
    h = O.mlp(sc.mlp, [0, 0, 0], [0, 0, 0, 0], d[0])
    assert np.allclose(r["rgb"][0], np.clip(h, 0, 1), atol=0)


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_hierarchical_equals_dense_random(seed):
    sc = random_scene(seed=seed, L=16, R=32, level_res=(4, 8, 16), occ_fraction=0.15,
                      density_offset=-20)
    osc = O.OracleScene(sc)
    rng = np.random.default_rng(seed)
    n = 500
    o = rng.uniform(-1.5, 1.5, (n, 3))
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    for flags in (0, O.NO_EARLY_TERM):
        h = O.render_rays(osc, o, d, mode="hier", flags=flags, max_trace=4096)
        g = O.render_rays(osc, o, d, mode="dense", flags=flags, max_trace=4096)
        assert np.array_equal(h["trace_count"], g["trace_count"])
        assert np.array_equal(h["trace_cells"], g["trace_cells"])
        assert np.array_equal(h["rgb"], g["rgb"])
        assert h["stats"]["skips"] > 0 and g["stats"]["skips"] == 0


def test_hierarchical_equals_dense_c1(c1_scene):
    osc = O.OracleScene(c1_scene)
    cams, W, H = config_cameras("c1")
    h = O.render(osc, cams[0], W, H, max_trace=1024, flags=O.NO_EARLY_TERM)
    g = O.render(osc, cams[0], W, H, mode="dense", max_trace=1024, flags=O.NO_EARLY_TERM)
    assert np.array_equal(h["trace_cells"], g["trace_cells"])
    assert np.array_equal(h["rgb"], g["rgb"])
    assert h["stats"]["missing"] == 0


def test_skipping_soundness_and_lattice(c1_scene):
    # every evaluated sample lies in a set finest cell; k strictly increases
    osc = O.OracleScene(c1_scene)
    cams, W, H = config_cameras("c1")
    r = O.render(osc, cams[0], W, H, max_trace=1024)
    N = c1_scene.level_res[-1]
    occ = unpack_bits(c1_scene.occ_finest, N).ravel()
    seg, k, cell = O.unpack_trace(r["trace_cells"])
    for p in range(W * H):
        n = r["trace_count"][p]
        assert n <= 1024
        assert occ[cell[p, :n]].all()
        key = seg[p, :n] * (1 << 21) + k[p, :n]
        assert (np.diff(key) > 0).all()


def test_early_termination_bound(c1_scene):
    # termination changes C_d, F by at most the transmittance left at the cut (<= 2e-4)
    osc = O.OracleScene(c1_scene)
    cams, W, H = config_cameras("c1")
    a = O.render(osc, cams[0], W, H, aux=True)
    b = O.render(osc, cams[0], W, H, aux=True, flags=O.NO_EARLY_TERM)
    assert np.abs(a["aux"][:, :7] - b["aux"][:, :7]).max() <= 2e-4
    assert a["stats"]["evaluated"] < b["stats"]["evaluated"]


def test_determinism(c1_scene):
    osc = O.OracleScene(c1_scene)
    cams, W, H = config_cameras("c1")
    a = O.render(osc, cams[0], W, H, threads=1)
    b = O.render(osc, cams[0], W, H)
    assert np.array_equal(a["rgb"], b["rgb"])


def test_psnr_helper():
    from conftest import psnr
    assert abs(psnr(np.zeros(10), np.full(10, 0.5)) - 6.020599913279624) < 1e-12
    assert psnr(np.zeros(4), np.ones(4)) == 0.0


def test_channel_split_closed_form():
    # Eq. 6 split: channel 0 -> tau, 1..3 -> c_d, 4..7 -> f (reading D12); per-channel bytes
    # constant over all four sources, so t_c = 4 (2 m_c b_c / 255 - m_c) exactly.
    b = [126, 40, 90, 200, 10, 70, 160, 250]
    sc = constant_scene(L=16, R=32, level_res=(8, 16), step=2.0 ** -6, bytes_per_channel=b)
    osc = O.OracleScene(sc)
    r = O.render_rays(osc, AXIS_O, AXIS_D, flags=O.NO_EARLY_TERM)
    m = [14.0] + [7.0] * 7
    t = [4 * (2 * m[c] * b[c] / 255 - m[c]) for c in range(8)]
    sig = lambda v: 1 / (1 + math.exp(-v))
    T = math.exp(-128 * math.exp(t[0]) * 2.0 ** -6)
    aux = r["aux"][0]
    assert abs(aux[7] - T) < 1e-12
    for c in range(3):
        assert abs(aux[c] - sig(t[1 + c]) * (1 - T)) < 1e-12
    for k in range(4):
        assert abs(aux[3 + k] - sig(t[4 + k]) * (1 - T)) < 1e-12
