"""Pins of the oracle's contraction and ray segmentation against the paper's
closed forms, hand-worked examples and brute force (never against the oracle itself)."""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O

G = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    with open(os.path.join(G, name)) as f:
        return json.load(f)


def test_contract_examples():
    g = _golden("contract_examples.json")
    for ex in g["contract"]:
        y, reg = O.contract(np.array([ex["x"]]))
        assert np.allclose(y[0], ex["c"], rtol=0, atol=1e-15), ex
        assert reg[0] == ex["region"], ex


def test_discontinuity_witness():
    g = _golden("contract_examples.json")["discontinuity"]
    ya, _ = O.contract(np.array([g["a"]]))
    yb, _ = O.contract(np.array([g["b"]]))
    assert np.allclose(ya[0], g["ca"], atol=1e-12)
    assert np.allclose(yb[0], g["cb"], atol=1e-12)


def test_identity_on_unit_cube():
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, (10000, 3))
    x[:100, 0] = 1.0
    x[100:200, 2] = -1.0
    y, reg = O.contract(x)
    assert np.array_equal(y, x)            # exact identity, ||x||_inf <= 1
    assert (reg == 0).all()


def test_range_and_cross_shape():
    rng = np.random.default_rng(1)
    x = rng.standard_cauchy((20000, 3)) * rng.uniform(0.1, 100, (20000, 1))
    y, reg = O.contract(x)
    assert np.abs(y).max() < 2.0                              # ||c||_inf < 2
    assert ((np.abs(y) > 1).sum(1) <= 1).all()                # image is cross-shaped
    # independent re-derivation of the region: argmax |x_j| with sign
    a = np.abs(x)
    m = a.max(1)
    j = np.argmax(a, 1)
    expect = np.where(m <= 1, 0, 1 + 2 * j + (x[np.arange(len(x)), j] < 0))
    assert np.array_equal(reg, expect)
    # radial monotonicity of the dominant coordinate: |c_j| = 2 - 1/|x_j|
    out = m > 1
    assert np.allclose(np.abs(y[out, j[out]]), 2 - 1 / m[out], atol=1e-15)


def test_continuity_at_unit_cube_boundary():
    rng = np.random.default_rng(2)
    p = rng.uniform(-1, 1, (5000, 3))
    ax = rng.integers(0, 3, 5000)
    sg = rng.choice([-1.0, 1.0], 5000)
    p[np.arange(5000), ax] = sg                 # points on a face of the unit cube
    eps = 1e-9
    outside = p.copy()
    outside[np.arange(5000), ax] = sg * (1 + eps)
    yin, _ = O.contract(p)
    yout, _ = O.contract(outside)
    assert np.abs(yin - yout).max() < 1e-8      # |x_j| = 1 +- eps: jump O(eps)
    # evaluating both adjacent formulas exactly at the boundary agrees to 1e-12
    for i in range(200):
        g = 1 + 2 * ax[i] + (sg[i] < 0)
        a = O.contract_region(0, p[i])
        b = O.contract_region(g, p[i])
        assert np.abs(a - b).max() < 1e-12


def _collinearity(seg, o, d):
    """max distance of contracted interior points from the segment's line."""
    ta, tb = seg["t_a"], seg["t_b"]
    if math.isinf(tb):
        ts = ta + np.geomspace(1e-6, 1e6, 40)
    else:
        ts = ta + (tb - ta) * np.linspace(0.02, 0.98, 40)
    pts = o[None, :] + ts[:, None] * d[None, :]
    c = np.array([O.contract_region(seg["region"], p) for p in pts])
    rel = c - seg["c_a"][None, :]
    along = rel @ seg["u"]
    perp = rel - along[:, None] * seg["u"][None, :]
    return np.abs(perp).max()


def test_segment_examples():
    g = _golden("segment_examples.json")
    for ray in g["rays"]:
        d = np.array(ray["d"], float)
        d /= np.linalg.norm(d)
        segs = O.segment_ray(np.array(ray["o"], float), d, 0.0, g["step"])
        assert len(segs) == len(ray["segments"])
        for s, e in zip(segs, ray["segments"]):
            assert s["region"] == e["region"]
            assert np.allclose(s["c_a"], e["c_a"], atol=1e-12)
            assert np.allclose(s["c_b"], e["c_b"], atol=1e-12)
            if "len" in e:
                assert abs(s["len"] - e["len"]) < 1e-12
            if "K" in e:
                assert s["K"] == e["K"]
            if "t_b" in e:
                assert (math.isinf(s["t_b"]) if e["t_b"] == "inf" else abs(s["t_b"] - e["t_b"]) < 1e-12)


def test_segments_vs_bruteforce_random_rays():
    rng = np.random.default_rng(3)
    step = 2.0 ** -10
    max_seg = 0
    for r in range(400):
        o = rng.uniform(-3, 3, 3) if r % 2 else rng.uniform(-0.99, 0.99, 3)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        segs = O.segment_ray(o, d, 0.0, step)
        max_seg = max(max_seg, len(segs))
        assert 1 <= len(segs) <= 7
        regs = [s["region"] for s in segs]
        assert len(set(regs)) == len(regs)                  # convex regions: no revisit
        # contiguity in t and brute-force region membership
        assert segs[0]["t_a"] == 0.0
        for a, b in zip(segs, segs[1:]):
            assert a["t_b"] == b["t_a"]
        assert math.isinf(segs[-1]["t_b"])
        for s in segs:
            tb = s["t_b"] if not math.isinf(s["t_b"]) else s["t_a"] + 1e4
            ts = np.linspace(s["t_a"], tb, 200)[1:-1]
            x = o[None, :] + ts[:, None] * d[None, :]
            _, reg = O.contract(x)
            assert (reg == s["region"]).all()
            assert _collinearity(s, o, d) < 1e-7 * max(1.0, s["len"])
            # lattice: U is u * Delta * 2^F rounded, K = ceil(len / Delta)
            assert s["K"] == math.ceil(s["len"] / step)
            assert np.abs(s["U"] - s["u"] * step * 2.0 ** O.F_BITS).max() <= 0.5
            assert np.abs(s["Qa"] - s["c_a"] * 2.0 ** O.F_BITS).max() <= 0.5
            assert abs(np.linalg.norm(s["u"]) - 1) < 1e-14
    assert max_seg >= 3


def test_raygen_hand_values():
    # identity rotation, origin (1,2,3): pixel centre (i+0.5-cx)/fx, (j+0.5-cy)/fy, 1 (D18)
    cam = np.zeros(17)
    cam[:12] = [1, 0, 0, 1, 0, 1, 0, 2, 0, 0, 1, 3]
    cam[12:16] = [2.0, 4.0, 1.0, 1.0]
    o, d = O.raygen(cam, 0, 1)
    v = np.array([(0.5 - 1.0) / 2.0, (1.5 - 1.0) / 4.0, 1.0])
    assert np.array_equal(o, [1, 2, 3])
    assert np.allclose(d, v / np.linalg.norm(v), atol=1e-16)
    # 90 degree rotation about y: camera z -> world +x, camera x -> world -z
    cam[:12] = [0, 0, 1, 0, 0, 1, 0, 0, -1, 0, 0, 0]
    o, d = O.raygen(cam, 1, 1)      # principal-ish pixel: x = (1.5-1)/2 = 0.25, y = 0.125
    v = np.array([1.0, 0.125, -0.25])
    assert np.allclose(d, v / np.linalg.norm(v), atol=1e-16)
