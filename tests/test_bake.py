"""NEXT-1: bake-side structure construction.  CPU pins of the oracle
(hand-computed voxel sets, thresholds, culling soundness S:404, atlas packing vs direct
indexing) and GPU parity (bit-exact A and atlas) plus a bake -> pyramid -> canonical blocks
-> pack -> upload -> render chain checked against the oracle."""
import math

import numpy as np
import pytest

from merf_inputs import unpack_bits, pack_bits
from oracle import oracle as O


def _cell_centred_corners(c, N):
    """real-arithmetic corner voxels of a contracted coordinate (reading D9)."""
    u = (c + 2.0) * N / 4.0 - 0.5
    i0 = min(max(math.floor(u), 0), N - 2)
    return i0, i0 + 1


def test_single_point_marks_its_eight_voxels():
    N, step = 16, 2.0 ** -6
    for world in ([0.3, -0.2, 0.55], [4.0, 0.5, -1.0], [-0.97, 0.99, 0.0]):
        bits = O.bake_occupancy(np.array([world]), np.array([1e3]), np.array([0.5]), N, step)
        occ = unpack_bits(bits, N)
        c, _ = O.contract(np.array([world]))
        expect = np.zeros((N, N, N), bool)
        xs, ys, zs = (_cell_centred_corners(v, N) for v in c[0])
        for z in zs:
            for y in ys:
                for x in xs:
                    expect[z, y, x] = True
        assert np.array_equal(occ, expect), world
        assert occ.sum() == 8


def test_thresholds():
    # alpha = 1 - exp(-tau step) > 0.005 and w > 0.005
    N, step = 16, 2.0 ** -6
    tau_thr = -math.log(1 - 0.005) / step
    x = np.array([[0.1, 0.1, 0.1]] * 4)
    tau = np.array([tau_thr * 1.000001, tau_thr * 0.999999, 1e3, 1e3])
    w = np.array([0.5, 0.5, 0.0051, 0.0049])
    for i, expect in enumerate([True, False, True, False]):
        bits = O.bake_occupancy(x[i:i + 1], tau[i:i + 1], w[i:i + 1], N, step)
        assert (unpack_bits(bits, N).sum() == 8) == expect, i
    a = 1 - math.exp(-tau_thr * 1.000001 * step)
    assert a > 0.005


def test_culling_soundness():
    # every voxel containing a point that passes both thresholds is occupied
    rng = np.random.default_rng(0)
    N, step = 32, 2.0 ** -7
    x = rng.standard_cauchy((5000, 3)) * 0.7
    tau = np.exp(rng.normal(2, 3, 5000))
    w = rng.uniform(0, 0.02, 5000)
    occ = unpack_bits(O.bake_occupancy(x, tau, w, N, step), N)
    c, _ = O.contract(x)
    keep = (w > 0.005) & (1 - np.exp(-tau * step) > 0.005)
    assert 500 < keep.sum() < 5000
    cell = np.clip(np.floor((c + 2) * N / 4).astype(int), 0, N - 1)
    assert occ[cell[keep, 2], cell[keep, 1], cell[keep, 0]].all()


def test_pack_atlas_direct_indexing():
    rng = np.random.default_rng(1)
    L = 32
    dense = rng.integers(0, 256, (L, L, L, 8), dtype=np.uint8)
    occ = rng.random((16, 16, 16)) < 0.05
    idx, n = O.canonical_block_index(pack_bits(occ), 16, L)
    atlas = O.pack_atlas(dense, L, idx, n)
    nb = L // 8
    for slot in np.nonzero(idx >= 0)[0][:20]:
        bz, by, bx = slot // (nb * nb), (slot // nb) % nb, slot % nb
        b = idx[slot]
        for lz in (0, 4, 8):
            for ly in (0, 8):
                for lx in (0, 7, 8):
                    g = [min(v * 8 + l, L - 1) for v, l in ((bz, lz), (by, ly), (bx, lx))]
                    assert np.array_equal(atlas[b, lz, ly, lx], dense[g[0], g[1], g[2]])


def _weighted_points(n, seed):
    """synthetic weighted points: world positions from contracted uniform samples."""
    rng = np.random.default_rng(seed)
    c = rng.uniform(-1.98, 1.98, (n, 3))
    # keep reachable contracted points (at most one |c_j| > 1) and map to the world
    a = np.abs(c)
    bad = (a > 1).sum(1) > 1
    c[bad] = np.clip(c[bad], -1, 1)
    j = np.argmax(np.abs(c), 1)
    aj = np.abs(c[np.arange(n), j])
    scale = np.where(aj > 1, 1 / (2 - aj), 1.0)
    x = c * scale[:, None]
    x[np.arange(n), j] = np.where(aj > 1, np.sign(c[np.arange(n), j]) * scale, c[np.arange(n), j])
    tau = np.exp(rng.normal(3, 3, n))
    w = rng.uniform(0, 0.02, n)
    return x, tau, w


@pytest.mark.gpu
def test_gpu_bake_and_pack_bit_exact():
    import torch
    import paper_2302_12249_b200 as M
    x, tau, w = _weighted_points(200000, 3)
    for N, step in ((32, 2.0 ** -6), (256, 2.0 ** -10)):
        ref = O.bake_occupancy(x, tau, w, N, step)
        bits = torch.empty(O.n_words(N), dtype=torch.int32, device="cuda")
        M.merf_bake_occupancy(torch.as_tensor(x, device="cuda"), torch.as_tensor(tau, device="cuda"),
                              torch.as_tensor(w, device="cuda"), N, step, bits)
        torch.cuda.synchronize()
        assert np.array_equal(bits.cpu().numpy().view(np.uint32), ref), N
    L = 64
    rng = np.random.default_rng(2)
    dense = rng.integers(0, 256, (L, L, L, 8), dtype=np.uint8)
    idx, n = O.canonical_block_index(O.bake_occupancy(x, tau, w, 32, 2.0 ** -6), 32, L)
    ref = O.pack_atlas(dense, L, idx, n)
    atlas = torch.empty((n, 9, 9, 9, 8), dtype=torch.uint8, device="cuda")
    M.merf_pack_atlas(torch.as_tensor(dense, device="cuda"), L, torch.as_tensor(idx, device="cuda"), n, atlas)
    torch.cuda.synchronize()
    assert np.array_equal(atlas.cpu().numpy(), ref)


@pytest.mark.gpu
def test_gpu_bake_to_render_chain():
    """weighted points -> A (bake) -> canonical blocks -> atlas from a dense V -> upload with the
    canonical index (NULL) -> render; the oracle renders the same arrays."""
    import torch
    import paper_2302_12249_b200 as M
    from merf_inputs import MerfScene, config_cameras, make_scene
    N, L, R, step = 32, 32, 64, 2.0 ** -6
    x, tau, w = _weighted_points(20000, 5)
    xd, taud, wd = (torch.as_tensor(a, device="cuda") for a in (x, tau, w))
    bits = torch.empty(O.n_words(N), dtype=torch.int32, device="cuda")
    M.merf_bake_occupancy(xd, taud, wd, N, step, bits)
    desc_scene = MerfScene(L=L, R=R, level_res=(8, N), step=step, planes=np.zeros((3, R, R, 8), np.uint8),
                           block_index=np.zeros(1, np.int32), atlas=np.zeros((0, 9, 9, 9, 8), np.uint8),
                           occ_finest=np.zeros(1, np.uint32), mlp=make_scene("c1").mlp)
    idx = torch.empty((L // 8) ** 3, dtype=torch.int32, device="cuda")
    n = M.merf_build_block_index(bits, desc_scene, idx)
    rng = np.random.default_rng(4)
    dense = rng.integers(0, 256, (L, L, L, 8), dtype=np.uint8)
    dense[..., 0] = np.clip(rng.normal(140, 30, (L, L, L)), 0, 255)
    atlas = torch.empty((max(n, 1), 9, 9, 9, 8), dtype=torch.uint8, device="cuda")
    M.merf_pack_atlas(torch.as_tensor(dense, device="cuda"), L, idx, n, atlas)
    torch.cuda.synchronize()
    sc = MerfScene(L=L, R=R, level_res=(8, N), step=step,
                   planes=rng.integers(100, 156, (3, R, R, 8), dtype=np.uint8),
                   block_index=idx.cpu().numpy(), atlas=atlas.cpu().numpy()[:n],
                   occ_finest=bits.cpu().numpy().view(np.uint32), mlp=make_scene("c1").mlp)
    assert np.array_equal(sc.occ_finest, O.bake_occupancy(x, tau, w, N, step))
    ref_idx, ref_n = O.canonical_block_index(sc.occ_finest, N, L)
    assert n == ref_n and np.array_equal(sc.block_index, ref_idx)
    s = M.Scene(sc, canonical=True)
    cams, W, H = config_cameras("c1")
    out, st = s.render(cams, W, H, stats=True)
    # the sample set is integer work: compare its size without early termination (the
    # T < t_min stop is a float decision, fp32 here vs fp64 in the oracle; reading D19)
    _, st_all = s.render(cams, W, H, flags=M.MERF_NO_EARLY_TERM, stats=True)
    torch.cuda.synchronize()
    osc = O.OracleScene(sc)
    ref = O.render(osc, cams[0], W, H)
    ref_all = O.render(osc, cams[0], W, H, flags=O.NO_EARLY_TERM)
    assert st_all["evaluated"] == ref_all["stats"]["evaluated"] and st["missing_blocks"] == 0
    assert abs(st["evaluated"] - ref["stats"]["evaluated"]) <= 1e-3 * ref["stats"]["evaluated"]
    assert np.abs(out[0].reshape(-1, 3).cpu().numpy() - ref["rgb"]).max() <= 2e-3
    s.close()
