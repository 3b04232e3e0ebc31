"""Synthetic baked MERF scenes, deterministic from (config, seed).

What a scene is (the hot path's inputs):
  * three R x R planes P_x(y,z), P_y(x,z), P_z(x,y) of C = 8 uint8 channels;
  * an L^3 grid V stored block-sparse: int32 indirection over (L/8)^3 block slots plus an
    atlas of 9^3-voxel blocks (8^3 data + 1-voxel apron on the + side);
  * the finest occupancy level as bits (x fastest, LSB first);
  * 883 deferred-MLP weights.

World content: spheres in [-0.8, 0.8]^3, a ground plane y = -0.6 reaching
to infinity, hills on a ring of radius 10-100 and a sky shell of radius 1000, so content
exists in every contraction region.  The generator needs a contracted-space distance to
place bytes: it maps contracted cell centres to the world with the INVERSE contraction
and divides the world SDF by its contracted-space gradient norm.  None of this is the
renderer's arithmetic (which only runs the forward direction); the renderer sees bytes.

Block allocation here is a conservative geometric rule (a block is stored if it lies
within one voxel of an occupied finest cell), deliberately NOT the canonical allocation
the library and the oracle compute; the soundness check (canonical subset of stored)
is what the tests pin.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

SEED = 230212249

# ------------------------------------------------------------------------------------
# container
# ------------------------------------------------------------------------------------


@dataclasses.dataclass
class MerfScene:
    L: int
    R: int
    level_res: tuple
    step: float
    planes: np.ndarray          # uint8 [3, R, R, C]
    block_index: np.ndarray     # int32 [(L/8)^3]
    atlas: np.ndarray           # uint8 [n_blocks, 9, 9, 9, C]
    occ_finest: np.ndarray      # uint32 words
    mlp: np.ndarray             # float64 [883] (values exactly representable in fp32)
    C: int = 8
    m_density: float = 14.0
    m_appearance: float = 7.0
    t_min: float = 2e-4
    alpha_skip: float = 0.0
    source_mask: int = 15
    name: str = ""

    @property
    def n_blocks(self) -> int:
        return int(self.atlas.shape[0]) if self.L > 0 else 0

    def nbytes(self) -> int:
        n = self.planes.nbytes if self.R > 0 else 0
        if self.L > 0:
            n += self.block_index.nbytes + self.atlas.nbytes
        n += self.occ_finest.nbytes + self.mlp.nbytes // 2
        return n

    def stats(self) -> dict:
        N = self.level_res[-1]
        occ = unpack_bits(self.occ_finest, N)
        d = dict(name=self.name, L=self.L, R=self.R, levels=list(self.level_res), step=self.step,
                 occ_fraction=float(occ.mean()), n_blocks=self.n_blocks,
                 scene_mb=self.nbytes() / 1e6)
        if self.L > 0:
            d["block_fraction"] = self.n_blocks / float((self.L // 8) ** 3)
        return d


def pack_bits(occ: np.ndarray) -> np.ndarray:
    """bool [N,N,N] indexed [z,y,x] -> uint32 words, linear index (z*N+y)*N+x, LSB first."""
    flat = np.ascontiguousarray(occ, dtype=bool).ravel()
    pad = (-len(flat)) % 32
    if pad:
        flat = np.concatenate([flat, np.zeros(pad, bool)])
    by = np.packbits(flat, bitorder="little")
    return by.view("<u4").astype(np.uint32)


def unpack_bits(words: np.ndarray, N: int) -> np.ndarray:
    by = np.ascontiguousarray(words, dtype="<u4").view(np.uint8)
    bits = np.unpackbits(by, bitorder="little")[: N * N * N]
    return bits.reshape(N, N, N).astype(bool)


def _hash_u8(seed: int, source: int, idx: np.ndarray, channel: int) -> np.ndarray:
    """Counter-based hash -> uint8 (splitmix64 finaliser)."""
    with np.errstate(over="ignore"):
        x = idx.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)
        x ^= np.uint64((seed * 1000003 + source * 8191 + channel * 131071) & 0xFFFFFFFFFFFFFFFF)
        x ^= x >> np.uint64(30)
        x *= np.uint64(0xBF58476D1CE4E5B9)
        x ^= x >> np.uint64(27)
        x *= np.uint64(0x94D049BB133111EB)
        x ^= x >> np.uint64(31)
    return (x >> np.uint64(56)).astype(np.uint8)


def _encode(raw: np.ndarray, m: float) -> np.ndarray:
    """byte whose decoded value 2m*b/255 - m is nearest to raw (clipped to [-m, m])."""
    v = (np.clip(raw, -m, m) + m) * (255.0 / (2.0 * m))
    return np.clip(np.floor(v + 0.5), 0, 255).astype(np.uint8)


def _mlp_weights(seed: int, scale: float = 0.3) -> np.ndarray:
    rng = np.random.default_rng(seed + 7)
    w = rng.uniform(-scale, scale, 883)
    w[880:883] = rng.uniform(-2.5, -1.5, 3)   # output bias: h ~ 0.1, so C_d is not clamped away
    return w.astype(np.float32).astype(np.float64)


def _gen_block_index(occ: np.ndarray, L: int) -> np.ndarray:
    """Conservative allocation: block b stored iff the voxel range [c*r-1, (c+1)*r] of an
    occupied finest cell c (r = L/N voxels per cell) meets b's data voxels [8b, 8b+7]."""
    N = occ.shape[0]
    assert L % N == 0 or N % L == 0
    nb = L // 8
    need = np.zeros((nb, nb, nb), bool)
    zz, yy, xx = np.nonzero(occ)
    if len(zz) == 0:
        return np.full(nb ** 3, -1, np.int32)
    rng = []
    for c in (xx, yy, zz):
        lo = np.clip((c.astype(np.int64) * L) // N - 1, 0, L - 1) >> 3
        hi = np.clip(((c.astype(np.int64) + 1) * L) // N, 0, L - 1) >> 3
        rng.append((lo, hi))
    span = max(int((h - l).max()) for l, h in rng)
    for dz in range(span + 1):
        for dy in range(span + 1):
            for dx in range(span + 1):
                bx = np.minimum(rng[0][0] + dx, rng[0][1])
                by = np.minimum(rng[1][0] + dy, rng[1][1])
                bz = np.minimum(rng[2][0] + dz, rng[2][1])
                need[bz, by, bx] = True
    idx = np.full(nb ** 3, -1, np.int32)
    flat = need.ravel()
    idx[flat] = np.arange(int(flat.sum()), dtype=np.int32)
    return idx


def _atlas_coords(block_index: np.ndarray, L: int):
    """Global voxel coordinates (clamped to L-1) of every atlas entry: [n_blocks,9,9,9] x3."""
    nb = L // 8
    slots = np.nonzero(block_index >= 0)[0]
    order = block_index[slots]
    slots = slots[np.argsort(order)]
    bz, by, bx = slots // (nb * nb), (slots // nb) % nb, slots % nb
    l = np.arange(9)
    gx = np.minimum(bx[:, None, None, None] * 8 + l[None, None, None, :], L - 1)
    gy = np.minimum(by[:, None, None, None] * 8 + l[None, None, :, None], L - 1)
    gz = np.minimum(bz[:, None, None, None] * 8 + l[None, :, None, None], L - 1)
    shp = (len(slots), 9, 9, 9)
    return (np.broadcast_to(gx, shp), np.broadcast_to(gy, shp), np.broadcast_to(gz, shp))


# ------------------------------------------------------------------------------------
# synthetic world (generator-only geometry)
# ------------------------------------------------------------------------------------
_AVOID = np.array([[0.1, 0.05, -0.2], [0.3, 0.1, -0.7], [0.95, 0.1, 0.0]] +
                  [[0.9 * math.cos(math.radians(15)) * math.cos(a), 0.9 * math.sin(math.radians(15)),
                    0.9 * math.cos(math.radians(15)) * math.sin(a)]
                   for a in np.linspace(0, 2 * math.pi, 64, endpoint=False)])


class World:
    def __init__(self, seed: int):
        rng = np.random.default_rng(seed)
        cs, rs = [], []
        while len(cs) < 24:
            c = rng.uniform(-0.8, 0.8, 3)
            r = rng.uniform(0.05, 0.35)
            if c[1] - r < -0.6 - 0.5 * r:      # mostly above the ground
                c[1] = -0.6 + 0.5 * r
            if np.min(np.linalg.norm(_AVOID - c, axis=1)) < r + 0.08:
                continue
            cs.append(c)
            rs.append(r)
        for _ in range(16):                      # hills on a ring of radius 10-100
            rho = rng.uniform(10.0, 100.0)
            th = rng.uniform(0, 2 * math.pi)
            r = rho * rng.uniform(0.1, 0.3)
            cs.append(np.array([rho * math.cos(th), -0.6, rho * math.sin(th)]))
            rs.append(r)
        self.centers = np.array(cs)
        self.radii = np.array(rs)
        self.colors = rng.uniform(0.1, 0.9, (len(cs) + 2, 3))
        self.features = rng.uniform(-5.0, 5.0, (len(cs) + 2, 4))
        self.ground_y = -0.6
        self.sky_r = 1000.0

    def sdf(self, x):
        """x [n,3] world (torch float64) -> (sdf [n], grad [n,3], object id [n])."""
        import torch
        n_sph = len(self.radii)
        best = x[:, 1] - self.ground_y
        oid = torch.full((x.shape[0],), n_sph, dtype=torch.int64)
        rn = torch.sqrt((x * x).sum(1))
        sky = self.sky_r - rn
        m = sky < best
        best = torch.where(m, sky, best)
        oid[m] = n_sph + 1
        cs = torch.from_numpy(self.centers)
        rs = torch.from_numpy(self.radii)
        sd = torch.cdist(x, cs) - rs[None, :]             # [n, n_sph]
        smin, sarg = sd.min(dim=1)
        m = smin < best
        best = torch.where(m, smin, best)
        oid = torch.where(m, sarg, oid)
        # gradient of the winning primitive only
        is_sph = oid < n_sph
        ctr = torch.cat([cs, torch.zeros(2, 3, dtype=cs.dtype)], 0)[oid]
        dv = torch.where(is_sph[:, None], x - ctr, -x)
        grad = dv / torch.sqrt((dv * dv).sum(1)).clamp_min(1e-30)[:, None]
        ground = oid == n_sph
        grad[ground] = torch.tensor([0.0, 1.0, 0.0], dtype=x.dtype)
        return best, grad, oid


def _inverse_contract(c):
    """world point of a contracted point (torch).  Generator-only; the renderer never
    inverts the contraction."""
    import torch
    a = c.abs()
    aj, j = a.max(dim=1)
    outer = aj > 1.0
    scale = torch.where(outer, 1.0 / (2.0 - aj).clamp_min(1e-9), torch.ones_like(aj))
    x = c * scale[:, None]
    sj = torch.sign(c.gather(1, j[:, None])[:, 0])
    return x, outer, j, sj, scale


def _contracted_distance_sph(world: World, c: np.ndarray, chunk: int = 1 << 19):
    """as contracted_distance, for the spherical contraction of Eq. 4 (NEXT-2 scenes):
    x = r(rho) c/rho with rho = |c|, r = 1/(2 - rho) outside the unit ball, so
    grad_c f = r^2 (g.c^) c^ + (r / rho) (g - (g.c^) c^)."""
    import torch
    out_d = np.empty(len(c))
    out_id = np.empty(len(c), np.int64)
    for s in range(0, len(c), chunk):
        cc = torch.from_numpy(np.ascontiguousarray(c[s:s + chunk], np.float64))
        rho = torch.sqrt((cc * cc).sum(1)).clamp_min(1e-12)
        outer = rho > 1.0
        r = torch.where(outer, 1.0 / (2.0 - rho).clamp_min(1e-9), rho)
        ch = cc / rho[:, None]
        x = torch.where(outer[:, None], ch * r[:, None], cc)
        f, g, oid = world.sdf(x)
        gr = (g * ch).sum(1)
        gc = torch.where(outer[:, None], (r * r * gr)[:, None] * ch + (r / rho)[:, None] * (g - gr[:, None] * ch), g)
        nrm = torch.sqrt((gc * gc).sum(1)).clamp_min(1e-30)
        out_d[s:s + chunk] = (f / nrm).numpy()
        out_id[s:s + chunk] = oid.numpy()
    return out_d, out_id


_CONTRACTION = ["pi"]     # contraction the generator bakes for (make_scene(contraction=...))


def contracted_distance(world: World, c: np.ndarray, chunk: int = 1 << 19):
    """first-order contracted-space signed distance, object id at contracted points."""
    import torch
    if _CONTRACTION[0] == "sph":
        return _contracted_distance_sph(world, c, chunk)
    out_d = np.empty(len(c))
    out_id = np.empty(len(c), np.int64)
    for s in range(0, len(c), chunk):
        cc = torch.from_numpy(np.ascontiguousarray(c[s:s + chunk], np.float64))
        x, outer, j, sj, a = _inverse_contract(cc)
        f, g, oid = world.sdf(x)
        gc = g * a[:, None]                                   # tangential: a * g_k
        gjj = g.gather(1, j[:, None])[:, 0]
        cjj = cc.gather(1, j[:, None])[:, 0]
        gk = (g * cc).sum(1) - gjj * cjj                      # sum_{k != j} g_k c_k
        gcj = torch.where(outer, a * a * (gjj + gk * sj), gjj)
        gc.scatter_(1, j[:, None], gcj[:, None])
        nrm = torch.sqrt((gc * gc).sum(1)).clamp_min(1e-30)
        out_d[s:s + chunk] = (f / nrm).numpy()
        out_id[s:s + chunk] = oid.numpy()
    return out_d, out_id


def _reachable(c: np.ndarray) -> np.ndarray:
    """contracted points in the image of the contraction: at most one |c_j| > 1 for contract_pi
    (cross-shaped image), |c| < 2 for the spherical contraction."""
    if _CONTRACTION[0] == "sph":
        return np.sqrt((c * c).sum(axis=1)) < 2.0
    return (np.abs(c) > 1.0).sum(axis=1) <= 1


def _occupancy(world: World, N: int, band_cells: float) -> np.ndarray:
    """finest occupancy: cell centre within band_cells cells of a surface (coarse-to-fine)."""
    w = 4.0 / N
    Nc = max(N // 4, 1)
    wc = 4.0 / Nc
    g = (np.arange(Nc) + 0.5) * wc - 2.0
    cz, cy, cx = np.meshgrid(g, g, g, indexing="ij")
    cc = np.stack([cx.ravel(), cy.ravel(), cz.ravel()], 1)
    dc, _ = contracted_distance(world, cc)
    cand = (np.abs(dc) < 1.5 * (band_cells * w + 0.9 * wc)) & _reachable(cc)
    occ = np.zeros((N, N, N), bool)
    ci = np.stack(np.nonzero(cand.reshape(Nc, Nc, Nc)), 1)          # [M, 3] (z, y, x)
    r = N // Nc
    o = np.stack(np.meshgrid(np.arange(r), np.arange(r), np.arange(r), indexing="ij"), -1)
    o = o.reshape(-1, 3)                                             # [r^3, 3]
    step = max(1, (1 << 20) // len(o))
    for s in range(0, len(ci), step):
        fine = (ci[s:s + step, None, :] * r + o[None, :, :]).reshape(-1, 3)   # (z, y, x)
        pts = (fine[:, ::-1] + 0.5) * w - 2.0                                  # (x, y, z)
        d, _ = contracted_distance(world, pts)
        ok = (np.abs(d) < band_cells * w) & _reachable(pts)
        f = fine[ok]
        occ[f[:, 0], f[:, 1], f[:, 2]] = True
    return occ


def _field_targets(world: World, c: np.ndarray, w_ramp: float, density_bias: float):
    """raw (pre-quantisation) V targets at contracted points: density ramp, colour, features."""
    d, oid = contracted_distance(world, c)
    t0 = np.clip(-d / w_ramp, -1.0, 1.0) * 14.0 + density_bias
    col = world.colors[oid]
    rgb = np.log(col / (1.0 - col))                      # sigmoid^-1 of the object colour
    feat = world.features[oid]
    return t0, rgb, feat


# ------------------------------------------------------------------------------------
# configs
# ------------------------------------------------------------------------------------
CONFIGS = {
    # name: (L, R, levels, step, band_cells)
    "c1": dict(L=32, R=128, level_res=(16, 32), step=2.0 ** -6),
    "c2": dict(L=512, R=2048, level_res=(32, 128, 256), step=2.0 ** -10),
}


def make_scene(config: str = "c1", seed: int = SEED, L=None, R=None, level_res=None, step=None,
               band_cells: float = 1.25, ramp_cells: float = 0.5, density_bias: float = 0.0,
               source_mask: int = 15, mlp_scale: float = 0.3, contraction: str = "pi") -> MerfScene:
    """The synthetic world baked at (L, R, levels).  c2/c3/c4 share the paper-scale scene.
    contraction="sph" bakes the same world in the spherical contraction's space (NEXT-2)."""
    assert contraction in ("pi", "sph")
    _CONTRACTION[0] = contraction
    try:
        return _make_scene(config, seed, L, R, level_res, step, band_cells, ramp_cells, density_bias,
                           source_mask, mlp_scale, contraction)
    finally:
        _CONTRACTION[0] = "pi"


def _make_scene(config, seed, L, R, level_res, step, band_cells, ramp_cells, density_bias, source_mask,
                mlp_scale, contraction):
    base = dict(CONFIGS["c1" if config == "c1" else "c2"])
    if L is not None:
        base["L"] = L
    if R is not None:
        base["R"] = R
    if level_res is not None:
        base["level_res"] = tuple(level_res)
    if step is not None:
        base["step"] = step
    L, R, level_res, step = base["L"], base["R"], tuple(base["level_res"]), base["step"]
    world = World(seed)
    N = level_res[-1]
    occ = _occupancy(world, N, band_cells)
    w_ramp = ramp_cells * 4.0 / N
    Cn = 8
    # ---- V: block-sparse atlas ----
    if L > 0 and (source_mask & 1):
        block_index = _gen_block_index(occ, L)
        gx, gy, gz = _atlas_coords(block_index, L)
        vs = 4.0 / L
        pts = np.stack([(gx.ravel() + 0.5) * vs - 2.0, (gy.ravel() + 0.5) * vs - 2.0,
                        (gz.ravel() + 0.5) * vs - 2.0], 1)
        t0, rgb, feat = _field_targets(world, pts, w_ramp, density_bias)
        atlas = np.empty((len(pts), Cn), np.uint8)
        atlas[:, 0] = _encode(t0, 14.0)
        atlas[:, 1:4] = _encode(rgb, 7.0)
        atlas[:, 4:8] = _encode(feat, 7.0)
        atlas = atlas.reshape(gx.shape + (Cn,))
    else:
        L = L if (source_mask & 1) else 0
        block_index = np.zeros(0, np.int32)
        atlas = np.zeros((0, 9, 9, 9, Cn), np.uint8)
        L = 0
    # ---- planes: small structured noise around the zero level ----
    if R > 0 and (source_mask & 14):
        planes = np.empty((3, R, R, Cn), np.uint8)
        idx = np.arange(R * R, dtype=np.int64)
        for a in range(3):
            for ch in range(Cn):
                h = _hash_u8(seed, a, idx, ch).astype(np.int16)
                amp = 6 if ch == 0 else 12
                v = 128 + ((h * (2 * amp + 1)) >> 8) - amp
                if L == 0 and ch == 0:
                    pass
                planes[a, :, :, ch] = v.reshape(R, R).astype(np.uint8)
        if L == 0:
            # planes-only variant: the density must come from the planes (3 sources)
            planes = _planes_only_density(occ, planes, R)
    else:
        planes = np.zeros((3, 0, 0, Cn), np.uint8)
        R = 0
    sc = MerfScene(L=L, R=R, level_res=level_res, step=step, planes=planes,
                   block_index=block_index, atlas=atlas, occ_finest=pack_bits(occ),
                   mlp=_mlp_weights(seed, mlp_scale), source_mask=source_mask,
                   name=config + ("_sph" if contraction == "sph" else ""))
    return sc


def _planes_only_density(occ, planes, R):
    """Planes-only variant (config 5, "without 3D grid"): each plane's density is the
    projection of the finest occupancy along its normal (upsampled to R x R): +2 where some
    occupied cell projects, -14 elsewhere, so the 3-plane sum (6) is high only where all three
    projections agree.  A synthetic stand-in for throughput/parity (quality is out of scope)."""
    N = occ.shape[0]
    rep = max(R // N, 1)
    for a in range(3):
        proj = occ.any(axis=2 - a)            # occ is [z, y, x]; axis a -> numpy axis 2 - a
        # P_x is indexed [z][y], P_y [z][x], P_z [y][x]: proj rows are the higher axis
        img = np.repeat(np.repeat(proj, rep, axis=0), rep, axis=1)[:R, :R]
        if img.shape[0] < R:
            idx = (np.arange(R) * N) // R
            img = proj[np.ix_(idx, idx)]
        planes[a, :, :, 0] = _encode(np.where(img, 2.0, -14.0), 14.0)
    return planes


def constant_scene(L: int = 16, R: int = 32, level_res=(8, 16), step: float = 2.0 ** -6,
                   b_d: int = 128, b_a: int = 128, mlp=None, occ=None, source_mask: int = 15,
                   bytes_per_source=None, bytes_per_channel=None) -> MerfScene:
    """Every stored byte of every source equal (b_d density, b_a appearance); all blocks
    stored; occupancy all-set unless `occ` (bool [N,N,N]) is given.  Used by closed-form pins.
    bytes_per_source: optional (V, Px, Py, Pz) density bytes."""
    N = level_res[-1]
    if occ is None:
        occ = np.ones((N, N, N), bool)
    nb = L // 8
    block_index = np.arange(nb ** 3, dtype=np.int32)
    atlas = np.empty((nb ** 3, 9, 9, 9, 8), np.uint8)
    planes = np.empty((3, R, R, 8), np.uint8)
    atlas[..., 0] = b_d
    atlas[..., 1:] = b_a
    planes[..., 0] = b_d
    planes[..., 1:] = b_a
    if bytes_per_channel is not None:
        atlas[...] = np.asarray(bytes_per_channel, np.uint8)
        planes[...] = np.asarray(bytes_per_channel, np.uint8)
    if bytes_per_source is not None:
        atlas[..., :] = bytes_per_source[0]
        for a in range(3):
            planes[a, ..., :] = bytes_per_source[1 + a]
    if mlp is None:
        mlp = np.zeros(883)
    return MerfScene(L=L, R=R, level_res=tuple(level_res), step=step, planes=planes,
                     block_index=block_index, atlas=atlas, occ_finest=pack_bits(occ),
                     mlp=np.asarray(mlp, np.float64), source_mask=source_mask, name="constant")


def random_scene(seed: int = 1, L: int = 16, R: int = 32, level_res=(4, 8, 16),
                 step: float = 2.0 ** -6, occ_fraction: float = 0.2, blob_cells: int = 2,
                 density_offset: int = 0, source_mask: int = 15) -> MerfScene:
    """Random blobby occupancy and random bytes (density biased so rays both pass through
    and terminate).  Small enough for dense-mode oracle runs in seconds."""
    rng = np.random.default_rng(seed)
    N = level_res[-1]
    occ = np.zeros((N, N, N), bool)
    target = occ_fraction * N ** 3
    while occ.sum() < target:
        c = rng.integers(0, N, 3)
        r = rng.integers(1, blob_cells + 1, 3)
        occ[max(c[2] - r[2], 0):c[2] + r[2], max(c[1] - r[1], 0):c[1] + r[1],
            max(c[0] - r[0], 0):c[0] + r[0]] = True
    # remove unreachable cells (two or more |c_j| > 1) like the real generator
    g = (np.arange(N) + 0.5) * (4.0 / N) - 2.0
    Z, Y, X = np.meshgrid(g, g, g, indexing="ij")
    unreach = ((np.abs(X) > 1).astype(int) + (np.abs(Y) > 1) + (np.abs(Z) > 1)) >= 2
    occ &= ~unreach
    if L > 0 and (source_mask & 1):
        block_index = _gen_block_index(occ, L)
        nblk = int((block_index >= 0).sum())
        atlas = rng.integers(0, 256, (nblk, 9, 9, 9, 8), dtype=np.uint8)
        atlas[..., 0] = np.clip(rng.normal(150 + density_offset, 40, (nblk, 9, 9, 9)), 0, 255)
    else:
        L = 0
        block_index = np.zeros(0, np.int32)
        atlas = np.zeros((0, 9, 9, 9, 8), np.uint8)
    if R > 0 and (source_mask & 14):
        planes = rng.integers(0, 256, (3, R, R, 8), dtype=np.uint8)
        planes[..., 0] = np.clip(rng.normal(128 + density_offset / 3, 20, (3, R, R)), 0, 255)
    else:
        R = 0
        planes = np.zeros((3, 0, 0, 8), np.uint8)
    return MerfScene(L=L, R=R, level_res=tuple(level_res), step=step, planes=planes,
                     block_index=block_index, atlas=atlas, occ_finest=pack_bits(occ),
                     mlp=_mlp_weights(seed), source_mask=source_mask, name=f"random{seed}")
