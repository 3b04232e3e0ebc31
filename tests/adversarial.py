"""Adversarial inputs for the GPU's 16-bit fixed-point interpolation weights.

The GPU interpolates with integer weights that partition 65535 exactly per source; each
weight carries a rounding error of at most half a unit per split.  Those errors cancel for
smooth fields and average out along a ray whose fractions change from sample to sample.  The
worst case for colour is the opposite:

* axis-aligned rays (d = +x), so the y and z texel fractions -- and therefore the rounding
  errors of every weight split that involves them -- are the same at every sample;
* fractions chosen where f * 65535 lies near a half-integer (the largest rounding error);
* bytes at 0 and 255 that vary only perpendicular to the ray (a density gradient across it),
  so the per-sample errors all push the optical depth the same way;
* a slab of surfaces with optical depth around 1, where the colour is most sensitive to a
  relative optical-depth error (|dT| <= eps * OD * exp(-OD) <= eps / e);
* appearance bytes at 255 (colour ~1) and an MLP whose output is ~0 (no clamp hides the error),
  or appearance bytes on the same 0/255 pattern (coherent appearance-weight errors).

Only input construction lives here (no method arithmetic); the oracle and the GPU render it.
"""
from __future__ import annotations

import numpy as np

from merf_inputs.scene import MerfScene, pack_bits, _gen_block_index


def _pattern(i, j, phase):
    return (((i + j + phase) & 1) * 255).astype(np.uint8)


def slab_scene(L: int, R: int, level_res, step: float, half: float = 0.25, appearance: str = "bright",
               seed: int = 0) -> MerfScene:
    """Occupied slab |c_x|, |c_y|, |c_z| <= half (contracted); density bytes on 0/255
    patterns that vary only in y and z; appearance 255 ("bright") or the same pattern ("pattern")."""
    rng = np.random.default_rng(seed)
    N = level_res[-1]
    g = (np.arange(N) + 0.5) * (4.0 / N) - 2.0
    inside = np.abs(g) <= half + 4.0 / N
    occ = inside[:, None, None] & inside[None, :, None] & inside[None, None, :]
    block_index = _gen_block_index(occ, L)
    nblk = int((block_index >= 0).sum())
    nb = L // 8
    # atlas: voxel (x, y, z) of block b at global coordinates 8 b + local (apron clamped to L-1)
    slots = np.nonzero(block_index >= 0)[0]
    bz, by, bx = slots // (nb * nb), (slots // nb) % nb, slots % nb
    loc = np.arange(9)
    gz = np.minimum(bz[:, None] * 8 + loc[None, :], L - 1)          # [nblk, 9]
    gy = np.minimum(by[:, None] * 8 + loc[None, :], L - 1)
    atlas = np.empty((nblk, 9, 9, 9, 8), np.uint8)
    dens = _pattern(gy[:, None, :], gz[:, :, None], 0)                # [nblk, z, y]
    atlas[..., 0] = dens[:, :, :, None]
    if appearance == "bright":
        atlas[..., 1:] = 255
    else:
        atlas[..., 1:] = dens[:, :, :, None, None]
    # planes: P_x[z][y], P_y[z][x], P_z[y][x] (row v, column u); density varies only in y, z
    r = np.arange(R)
    planes = np.empty((3, R, R, 8), np.uint8)
    planes[0, ..., 0] = _pattern(r[None, :], r[:, None], 1)           # P_x(y, z): both fixed
    planes[1, ..., 0] = _pattern(0 * r[None, :], r[:, None], 0)       # P_y(x, z): z only
    planes[2, ..., 0] = _pattern(0 * r[None, :], r[:, None], 1)       # P_z(x, y): y only
    if appearance == "bright":
        planes[..., 1:] = 255
    else:
        planes[..., 1:] = planes[..., :1]
    mlp = np.zeros(883)
    mlp[880:883] = -20.0                                              # h = sigmoid(-20) ~ 2e-9
    del rng
    return MerfScene(L=L, R=R, level_res=tuple(level_res), step=step, planes=planes,
                     block_index=block_index, atlas=atlas, occ_finest=pack_bits(occ),
                     mlp=mlp, name=f"slab_{appearance}")


def bad_coordinates(n: int, M: int, seed: int, F: int = 28):
    """n contracted coordinates in [-0.2, 0.2] whose texel fraction on a grid of resolution M
    (cell-centred, spacing 4/M) makes f * 65535 lie within 0.05 of a half-integer."""
    rng = np.random.default_rng(seed)
    out = []
    s = F + 2 - int(np.log2(M))
    while len(out) < n:
        i = int(rng.integers(int(1.8 * M / 4), int(2.2 * M / 4)))
        k = int(rng.integers(0, 65535)) + 0.5 + rng.uniform(-0.05, 0.05)
        f = k / 65535.0
        # position of texel i's centre plus f of a texel, on the 2^-F lattice
        c = (i + 0.5 + f) * (4.0 / M) - 2.0
        Q = int(round(c * 2.0 ** F))
        out.append(Q / 2.0 ** F)
    del s
    return np.array(out)


def axis_rays(sc: MerfScene, n: int, seed: int):
    """n rays along +x through the slab, y/z at adversarial plane-texel fractions (half of
    them) or at adversarial V-voxel fractions (the other half)."""
    ys = np.concatenate([bad_coordinates(n // 2, sc.R, seed), bad_coordinates(n - n // 2, sc.L, seed + 1)])
    zs = np.concatenate([bad_coordinates(n // 2, sc.R, seed + 2), bad_coordinates(n - n // 2, sc.L, seed + 3)])
    o = np.stack([np.full(n, -0.6), ys, zs], axis=1)
    d = np.tile(np.array([1.0, 0.0, 0.0]), (n, 1))
    return o, d
