"""Pins of the oracle's field query (Eq. 5-7), occupancy pyramid, canonical block
allocation and deferred MLP (Eq. 3) against closed forms and independent
brute-force re-derivations in real arithmetic."""
import math

import numpy as np

from merf_inputs import constant_scene, random_scene, unpack_bits, make_scene
from oracle import oracle as O

F = O.F_BITS


def _Q(c):
    return np.array([int(round(v * 2 ** F)) for v in c], np.int64)


def test_constant_field_exact():
    sc = constant_scene(b_d=128, b_a=128)
    osc = O.OracleScene(sc)
    rng = np.random.default_rng(0)
    for _ in range(50):
        c = rng.uniform(-2, 2, 3)
        t, miss = O.query_field(osc, _Q(c))
        assert miss == 0
        # all-128: t0 = 4 (28*128/255 - 14) = 0.219608 (Eq. 7, four sources Eq. 5)
        assert abs(t[0] - 4 * (28 * 128 / 255 - 14)) < 1e-12
        assert abs(t[0] - 0.2196078431372549) < 1e-12
        assert np.allclose(t[1:], 4 * (14 * 128 / 255 - 7), atol=1e-12)


def test_cancelling_sources_give_zero():
    # bytes (V, Px, Py, Pz) = (0, 255, 0, 255) -> -m + m - m + m = 0 -> tau = 1, sigma = 0.5
    sc = constant_scene(bytes_per_source=(0, 255, 0, 255))
    osc = O.OracleScene(sc)
    t, _ = O.query_field(osc, _Q([0.3, -1.2, 0.7]))
    assert np.abs(t).max() < 1e-12


def _brute_field(sc, c):
    """independent trilinear/bilinear in real arithmetic: texel i centred at -2 + (i+0.5)*4/M
    (reading D9), clamp to edge; decode each corner 2m b/255 - m before interpolation."""
    m = np.array([14.0] + [7.0] * 7)

    def coord(v, M):
        u = (v + 2.0) * M / 4.0 - 0.5
        i = math.floor(u)
        f = u - i
        if i < 0:
            return 0, 0.0
        if i > M - 2:
            return M - 2, 1.0
        return i, f

    t = np.zeros(8)
    L = sc.L
    if L:
        idx = [coord(v, L) for v in c]
        nb = L // 8
        blk = sc.block_index[((idx[2][0] // 8) * nb + idx[1][0] // 8) * nb + idx[0][0] // 8]
        A = sc.atlas[blk]
        for dz in (0, 1):
            for dy in (0, 1):
                for dx in (0, 1):
                    w = ((idx[0][1] if dx else 1 - idx[0][1]) * (idx[1][1] if dy else 1 - idx[1][1])
                         * (idx[2][1] if dz else 1 - idx[2][1]))
                    b = A[idx[2][0] % 8 + dz, idx[1][0] % 8 + dy, idx[0][0] % 8 + dx].astype(float)
                    t += w * (2 * m * b / 255 - m)
    R = sc.R
    for a, (ua, va) in enumerate([(1, 2), (0, 2), (0, 1)]):
        iu, fu = coord(c[ua], R)
        iv, fv = coord(c[va], R)
        for dv in (0, 1):
            for du in (0, 1):
                w = (fu if du else 1 - fu) * (fv if dv else 1 - fv)
                b = sc.planes[a, iv + dv, iu + du].astype(float)
                t += w * (2 * m * b / 255 - m)
    return t


def test_field_vs_bruteforce_interpolation():
    sc = random_scene(seed=5, L=16, R=32, level_res=(8, 16), occ_fraction=0.6)
    osc = O.OracleScene(sc)
    occ = unpack_bits(sc.occ_finest, 16)
    rng = np.random.default_rng(1)
    n = 0
    while n < 300:
        # points with dyadic coordinates so the real-valued position is exact
        c = np.round(rng.uniform(-2.05, 2.05, 3) * 2 ** 20) / 2 ** 20
        cell = np.clip(((c + 2) * 4).astype(int), 0, 15)
        if not occ[cell[2], cell[1], cell[0]]:
            continue
        t, miss = O.query_field(osc, _Q(c))
        assert miss == 0
        assert np.abs(t - _brute_field(sc, c)).max() < 1e-12
        n += 1


def test_post_activation_ordering():
    # Eq. 6 applies exp AFTER interpolation: midway between density bytes 0 and 255 of V the
    # summed t0 is the average, so tau = exp(avg) (not avg of exp) -- S:208 witness.
    sc = constant_scene(L=16, R=32, level_res=(8, 16), b_d=128, b_a=128)
    sc.planes[..., 0] = 0     # planes contribute -14 each; V carries a step in x
    sc.atlas[..., 0] = 0
    sc.atlas[:, :, :, 4:, 0] = 255
    osc = O.OracleScene(sc)
    # texel centres x = -2 + (i + .5) / 4: i = 3 -> -1.125, i = 4 -> -0.875; midpoint -1.0
    t, _ = O.query_field(osc, _Q([-1.0, 0.1, 0.1]))
    assert abs(t[0] - (0.0 - 3 * 14)) < 1e-12
    assert abs(math.exp(t[0]) - math.exp(-42.0)) < 1e-30


def test_pyramid_vs_numpy_maxpool():
    rng = np.random.default_rng(2)
    N = 32
    occ = rng.random((N, N, N)) < 0.02
    from merf_inputs import pack_bits
    bits = pack_bits(occ)
    for Nc in (16, 8, 4, 1):
        r = N // Nc
        ref = occ.reshape(Nc, r, Nc, r, Nc, r).max(axis=(1, 3, 5))
        got = unpack_bits(O.maxpool_bits(bits, N, Nc), Nc)
        assert np.array_equal(got, ref)


def test_bit_order_x_fastest():
    # bit index (z*N + y)*N + x, LSB first
    from merf_inputs import pack_bits
    occ = np.zeros((4, 4, 4), bool)
    occ[0, 0, 1] = True     # x = 1 -> bit 1 of word 0
    occ[1, 0, 0] = True     # z = 1 -> bit 16
    w = pack_bits(occ)
    assert w[0] == (1 << 1) | (1 << 16)
    got = unpack_bits(O.maxpool_bits(w, 4, 2), 2)
    assert got[0, 0, 0] and not got[0, 0, 1]


def _canonical_bruteforce(occ, L):
    """blocks hit by the real-valued i0 range of each occupied finest cell (reading D11):
    i0(p) = floor((p + 2) L / 4 - 1/2) clamped to [0, L-2]; block = i0 // 8."""
    N = occ.shape[0]
    nb = L // 8
    need = np.zeros((nb, nb, nb), bool)
    for z, y, x in zip(*np.nonzero(occ)):
        rngs = []
        for c in (x, y, z):
            lo = 0 if c == 0 else min(max(math.floor(c * L / N - 0.5), 0), L - 2)
            hi = L - 2 if c == N - 1 else min(max(math.floor((c + 1) * L / N - 0.5 - 1e-9), 0), L - 2)
            rngs.append((lo // 8, hi // 8))
        need[rngs[2][0]:rngs[2][1] + 1, rngs[1][0]:rngs[1][1] + 1, rngs[0][0]:rngs[0][1] + 1] = True
    return need.ravel()


def test_canonical_block_index_bruteforce():
    for seed, (L, N) in enumerate([(32, 32), (32, 16), (64, 32), (16, 16), (64, 8)]):
        rng = np.random.default_rng(seed)
        occ = rng.random((N, N, N)) < 0.03
        occ[0, 0, 0] = True
        occ[-1, -1, -1] = True
        from merf_inputs import pack_bits
        idx, n = O.canonical_block_index(pack_bits(occ), N, L)
        need = _canonical_bruteforce(occ, L)
        assert np.array_equal(idx >= 0, need)
        assert n == need.sum()
        assert np.array_equal(idx[need], np.arange(n))          # raster-order numbering


def test_generator_allocation_is_sound():
    # the generator's conservative allocation must contain the canonical one
    for sc in (make_scene("c1"), random_scene(seed=3, L=32, R=32, level_res=(8, 16, 32))):
        idx, n = O.canonical_block_index(sc.occ_finest, sc.level_res[-1], sc.L)
        assert ((sc.block_index >= 0) | (idx < 0)).all()


def test_encode_dir_and_zero_mlp():
    e = O.encode_dir([1.0, 0.0, 0.0])
    assert len(e) == 27
    assert abs(e[3 + 2] - math.sin(2.0)) < 1e-15             # (j = x, k = 1, sin)
    assert abs(e[3 + 2] - 0.9092974268256817) < 1e-15
    e = O.encode_dir([0.0, 0.0, 1.0])
    assert np.array_equal(e[:3], [0, 0, 1])
    assert np.array_equal(e[3:11:2], [0, 0, 0, 0]) and np.array_equal(e[4:11:2], [1, 1, 1, 1])
    h = O.mlp(np.zeros(883), [0.3, 0.2, 0.1], [0.1] * 4, [0, 0, 1])
    assert np.allclose(h, 0.5, atol=0)                        # sigmoid(0) = 1/2


def test_hand_computed_mlp():
    # one active path: h0 = relu(C_d[0] * 2 - 0.1); h1 = relu(-3 * h0 + 1); out = 1.5 h1 + b2
    w = np.zeros(883)
    W0, b0, W1, b1, W2, b2 = 0, 544, 560, 816, 832, 880
    w[W0 + 0 * 34 + 0] = 2.0
    w[b0 + 0] = -0.1
    w[W1 + 0 * 16 + 0] = -3.0
    w[b1 + 0] = 1.0
    w[W2 + 1 * 16 + 0] = 1.5
    w[b2:b2 + 3] = [0.25, -0.5, 0.0]
    cd = [0.3, 0.9, 0.9]
    h0 = max(0.0, 0.3 * 2 - 0.1)                               # 0.5
    h1 = max(0.0, -3 * h0 + 1)                                 # 0 -> dead
    sig = lambda v: 1 / (1 + math.exp(-v))
    got = O.mlp(w, cd, [0] * 4, [0, 1, 0])
    assert np.allclose(got, [sig(0.25), sig(-0.5 + 1.5 * h1), sig(0.0)], atol=1e-15)
    cd = [0.1, 0, 0]
    h0 = max(0.0, 0.1 * 2 - 0.1)                               # 0.1
    h1 = max(0.0, -3 * h0 + 1)                                 # 0.7
    got = O.mlp(w, cd, [0] * 4, [0, 1, 0])
    assert np.allclose(got, [sig(0.25), sig(-0.5 + 1.5 * h1), 0.5], atol=1e-15)
