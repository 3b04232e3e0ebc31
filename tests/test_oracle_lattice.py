"""Pins of the oracle's lattice and occupancy-cell helpers against real arithmetic.

The paper samples "along the ray in contracted space ... with a small uniform step size"
 and queries the occupancy grid cell containing each sample, skipping to the first
sample outside an empty cell.  These tests check the oracle's integer
realisation of that (reading D8: lattice Q = Qa + k U with F = 28 fraction bits; D10: cell
index by shift and clamp) against exact rational arithmetic (`fractions.Fraction`), which
shares nothing with the oracle's integer code:

* occ_cell(Q, N) == clamp(floor((Q 2^-F + 2) N / 4), 0, N - 1) for random and face-exact Q,
  including positions beyond the [-2, 2] cube (the clamp);
* every lattice sample Q_k 2^-F lies within (k + 1) 2^-29 per axis of the exact uniform
  sample c_a + k Delta u (the drift bound of D8/D21), and the last sample within Delta of c_b;
* c_a equals contract_g(o + t_a d) evaluated exactly;
* end to end: the finest cell the oracle's dense-mode trace records for every sample equals
  the exact cell of the exact uniform sample, wherever that sample is farther than the
  drift bound from a cell face.
"""
from __future__ import annotations

import math
from fractions import Fraction as Fr

import numpy as np
import pytest

from merf_inputs import constant_scene
from oracle import oracle as O

F = O.F_BITS
ONE = 1 << F


def _exact_cell(p: Fr, N: int) -> int:
    c = math.floor((p + 2) * N / 4)
    return min(max(c, 0), N - 1)


@pytest.mark.parametrize("N", [1, 2, 4, 16, 32, 128, 256, 512, 4096])
def test_occ_cell_matches_real_arithmetic(N):
    rng = np.random.default_rng(N)
    # random positions in [-2.5, 2.5] (beyond the cube: the clamp), as exact lattice values
    Qs = [int(q) for q in rng.integers(-5 * ONE // 2, 5 * ONE // 2, 4000)]
    # every cell face of this level exactly, and one lattice unit either side of it
    for c in range(0, N + 1):
        face = (c * 4 * ONE) // N - 2 * ONE
        Qs += [face - 1, face, face + 1]
    Qs += [-2 * ONE, 2 * ONE - 1, 2 * ONE, 2 * ONE + 1, -2 * ONE - 1]
    for Q in Qs:
        assert O.occ_cell(Q, N) == _exact_cell(Fr(Q, ONE), N), (Q, N)


def _contract_exact(g: int, x):
    """contract_g in exact rational arithmetic: c_j = s (2 - 1/|x_j|), c_k = x_k/|x_j|."""
    if g == 0:
        return list(x)
    j, s = (g - 1) // 2, (-1 if (g - 1) % 2 else 1)
    a = abs(x[j])
    return [s * (2 - 1 / a) if k == j else x[k] / a for k in range(3)]


def _rays(n, seed):
    rng = np.random.default_rng(seed)
    for r in range(n):
        o = rng.uniform(-3, 3, 3) if r % 2 else rng.uniform(-0.95, 0.95, 3)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        yield o, d


def test_lattice_positions_track_uniform_contracted_samples():
    step = 2.0 ** -6
    D = Fr(step)
    n_checked = 0
    for o, d in _rays(60, 5):
        for s in O.segment_ray(o, d, 0.0, step):
            # the oracle's contracted endpoint vs exact contraction of the exact point x(t_a)
            xa = [Fr(o[q]) + Fr(s["t_a"]) * Fr(d[q]) for q in range(3)]
            ca = _contract_exact(s["region"], xa)
            for q in range(3):
                assert abs(Fr(s["c_a"][q]) - ca[q]) <= Fr(1, 1 << 50)
            ca = [Fr(v) for v in s["c_a"]]
            u = [Fr(v) for v in s["u"]]
            cb = [Fr(v) for v in s["c_b"]]
            K = s["K"]
            assert (K - 1) * step < s["len"] <= K * step
            for k in range(K):
                for q in range(3):
                    Qk = int(s["Qa"][q]) + k * int(s["U"][q])
                    exact = ca[q] + k * D * u[q]
                    assert abs(Fr(Qk, ONE) - exact) <= Fr(k + 1, 1 << 29), (k, q)
                n_checked += 1
            # the last sample lies within Delta of c_b, before it along u
            last = [ca[q] + (K - 1) * D * u[q] for q in range(3)]
            dist2 = sum((cb[q] - last[q]) ** 2 for q in range(3))
            assert 0 < dist2 <= D * D * (1 + Fr(1, 1 << 40))
    assert n_checked > 8000


@pytest.mark.parametrize("level_res", [(8, 16), (4, 32)])
def test_trace_cells_are_exact_cells_of_uniform_samples(level_res):
    """Dense mode with every finest cell occupied evaluates every lattice sample, so the trace
    lists (segment, k, cell) for all of them: each recorded cell must be the exact cell of the
    exact uniform sample, except within the drift bound of a face."""
    step = 2.0 ** -6
    N = level_res[-1]
    sc = constant_scene(L=16, R=32, level_res=level_res, step=step, b_d=0, b_a=128)
    osc = O.OracleScene(sc)
    rays = list(_rays(24, 11))
    o = np.array([r[0] for r in rays])
    d = np.array([r[1] for r in rays])
    out = O.render_rays(osc, o, d, mode="dense", flags=O.NO_EARLY_TERM, max_trace=4096)
    seg, k, cell = O.unpack_trace(out["trace_cells"])
    D = Fr(step)
    checked = ambiguous = 0
    for r in range(len(rays)):
        segs = O.segment_ray(o[r], d[r], 0.0, step)
        n = out["trace_count"][r]
        assert n == sum(s["K"] for s in segs)          # every lattice sample evaluated
        i = 0
        for j, s in enumerate(segs):
            ca = [Fr(v) for v in s["c_a"]]
            u = [Fr(v) for v in s["u"]]
            for kk in range(s["K"]):
                assert seg[r, i] == j and k[r, i] == kk
                lin = int(cell[r, i])
                got = (lin % N, (lin // N) % N, lin // (N * N))
                margin = Fr(kk + 1, 1 << 29) + Fr(1, 1 << 48)
                for q in range(3):
                    p = ca[q] + kk * D * u[q]
                    t = (p + 2) * N / 4
                    near_face = abs(t - round(t)) * 4 / N <= margin and -2 < p < 2
                    if near_face:
                        ambiguous += 1
                        assert abs(got[q] - _exact_cell(p, N)) <= 1
                    else:
                        assert got[q] == _exact_cell(p, N), (r, j, kk, q)
                        checked += 1
                i += 1
    assert checked > 8000 and ambiguous < checked // 100
