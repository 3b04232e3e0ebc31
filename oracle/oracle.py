"""ctypes wrapper of the fp64 CPU oracle (oracle/merf_oracle.c).

TEST INFRASTRUCTURE ONLY: the product path (paper_2302_12249_b200/) never imports this
module.  Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may call it.  Paper citations (P:<line> = PAPER.md line) live
in merf_oracle.c next to each function.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "merf_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

F_BITS = 28
NO_EARLY_TERM = 1


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, no FMA contraction, no fast-math, OpenMP)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-o", _LIB_PATH + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


class _Scene(C.Structure):
    _fields_ = [
        ("L", C.c_int32), ("R", C.c_int32), ("C", C.c_int32), ("n_levels", C.c_int32),
        ("level_res", C.c_int32 * 4),
        ("m_density", C.c_double), ("m_appearance", C.c_double), ("step", C.c_double),
        ("t_min", C.c_double), ("alpha_skip", C.c_double),
        ("source_mask", C.c_uint32),
        ("planes", C.c_void_p), ("block_index", C.c_void_p), ("atlas", C.c_void_p),
        ("n_blocks", C.c_int64),
        ("occ", C.c_void_p * 4),
        ("mlp", C.c_void_p),
    ]


class _Segment(C.Structure):
    _fields_ = [
        ("region", C.c_int32), ("ordinal", C.c_int32),
        ("t_a", C.c_double), ("t_b", C.c_double),
        ("c_a", C.c_double * 3), ("c_b", C.c_double * 3),
        ("len", C.c_double), ("u", C.c_double * 3),
        ("Qa", C.c_int64 * 3), ("U", C.c_int64 * 3), ("K", C.c_int64),
    ]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB_PATH)
            vp, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_double
            L.orc_region_of.argtypes = [vp]
            L.orc_region_of.restype = C.c_int
            L.orc_contract.argtypes = [vp, i64, vp, vp]
            L.orc_contract_region.argtypes = [C.c_int, vp, vp]
            L.orc_raygen.argtypes = [vp, i32, i32, vp, vp]
            L.orc_segment_ray.argtypes = [vp, vp, dbl, dbl, vp]
            L.orc_segment_ray.restype = C.c_int
            L.orc_occ_cell.argtypes = [i64, i32]
            L.orc_occ_cell.restype = i64
            L.orc_maxpool_bits.argtypes = [vp, i32, vp, i32]
            L.orc_canonical_block_index.argtypes = [vp, i32, i32, vp]
            L.orc_canonical_block_index.restype = i64
            L.orc_query_field.argtypes = [vp, vp, vp]
            L.orc_query_field.restype = C.c_int
            L.orc_encode_dir.argtypes = [vp, vp]
            L.orc_mlp.argtypes = [vp, vp, vp, vp, vp]
            L.orc_render_pixels.argtypes = [vp, vp, i32, vp, i64, C.c_int, C.c_uint32, vp, vp,
                                            i32, vp, vp, vp, vp, vp, i32]
            L.orc_render_rays.argtypes = [vp, vp, vp, vp, i64, C.c_int, C.c_uint32, vp, vp,
                                          i32, vp, vp, vp, vp]
            L.orc_max_threads.restype = i32
            L.orc_contract_sph.argtypes = [vp, vp]
            L.orc_contract_sph.restype = dbl
            L.orc_sph_speed.argtypes = [vp, vp]
            L.orc_sph_speed.restype = dbl
            L.orc_bake_occupancy.argtypes = [vp, vp, vp, i64, dbl, dbl, i32, vp]
            L.orc_pack_atlas.argtypes = [vp, i32, vp, i64, vp]
            _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ------------------------------------------------------------------------------------
# contraction / rays / segmentation
# ------------------------------------------------------------------------------------
def region_of(x) -> int:
    x = _c(x, np.float64)
    return lib().orc_region_of(_p(x))


def contract(x):
    """contract_pi of an [n,3] array -> (y [n,3], region [n])."""
    x = _c(x, np.float64).reshape(-1, 3)
    y = np.empty_like(x)
    reg = np.empty(len(x), np.int32)
    lib().orc_contract(_p(x), len(x), _p(y), _p(reg))
    return y, reg


def contract_region(g: int, x):
    x = _c(x, np.float64)
    y = np.empty(3, np.float64)
    lib().orc_contract_region(int(g), _p(x), _p(y))
    return y


def raygen(cam, i: int, j: int):
    cam = _c(cam, np.float64)
    o = np.empty(3, np.float64)
    d = np.empty(3, np.float64)
    lib().orc_raygen(_p(cam), int(i), int(j), _p(o), _p(d))
    return o, d


def segment_ray(o, d, t_near: float, step: float):
    o = _c(o, np.float64)
    d = _c(d, np.float64)
    segs = (_Segment * 16)()
    n = lib().orc_segment_ray(_p(o), _p(d), float(t_near), float(step), C.cast(segs, C.c_void_p))
    out = []
    for s in segs[:n]:
        out.append(dict(region=s.region, ordinal=s.ordinal, t_a=s.t_a, t_b=s.t_b,
                        c_a=np.array(s.c_a[:]), c_b=np.array(s.c_b[:]), len=s.len,
                        u=np.array(s.u[:]), Qa=np.array(s.Qa[:], np.int64),
                        U=np.array(s.U[:], np.int64), K=int(s.K)))
    return out


# ------------------------------------------------------------------------------------
# occupancy pyramid / block index
# ------------------------------------------------------------------------------------
def occ_cell(Q: int, N: int) -> int:
    """occupancy cell index at resolution N of the (unbiased) lattice coordinate Q (D10)."""
    return int(lib().orc_occ_cell(int(Q), int(N)))


def n_words(N: int) -> int:
    return (N * N * N + 31) // 32


def maxpool_bits(fine, f: int, N: int):
    fine = _c(fine, np.uint32)
    out = np.zeros(n_words(N), np.uint32)
    lib().orc_maxpool_bits(_p(fine), int(f), _p(out), int(N))
    return out


def build_pyramid(finest, level_res):
    """Levels coarse->fine; each coarser level max-pooled from the finest."""
    f = int(level_res[-1])
    finest = _c(finest, np.uint32)
    levels = [maxpool_bits(finest, f, int(N)) for N in level_res[:-1]]
    return levels + [finest]


def canonical_block_index(finest, N: int, L: int):
    finest = _c(finest, np.uint32)
    nb = L // 8
    idx = np.empty(nb ** 3, np.int32)
    n = lib().orc_canonical_block_index(_p(finest), int(N), int(L), _p(idx))
    return idx, int(n)


# ------------------------------------------------------------------------------------
# scene + field + MLP
# ------------------------------------------------------------------------------------
class OracleScene:
    """Keeps numpy arrays alive and exposes the C struct."""

    def __init__(self, sc):
        self.sc = sc
        self.planes = _c(sc.planes, np.uint8) if sc.R > 0 else np.zeros(1, np.uint8)
        self.block_index = _c(sc.block_index, np.int32) if sc.L > 0 else np.zeros(1, np.int32)
        self.atlas = _c(sc.atlas, np.uint8) if sc.L > 0 and sc.atlas.size else np.zeros(1, np.uint8)
        self.levels = build_pyramid(sc.occ_finest, sc.level_res)
        self.mlp = _c(sc.mlp, np.float64)
        s = _Scene()
        s.L, s.R, s.C, s.n_levels = sc.L, sc.R, sc.C, len(sc.level_res)
        for i, r in enumerate(sc.level_res):
            s.level_res[i] = r
        s.m_density, s.m_appearance = sc.m_density, sc.m_appearance
        s.step, s.t_min, s.alpha_skip = sc.step, sc.t_min, sc.alpha_skip
        s.source_mask = sc.source_mask
        s.planes, s.block_index, s.atlas = (self.planes.ctypes.data, self.block_index.ctypes.data,
                                            self.atlas.ctypes.data)
        s.n_blocks = sc.n_blocks
        for i, lv in enumerate(self.levels):
            s.occ[i] = lv.ctypes.data
        s.mlp = self.mlp.ctypes.data
        self.struct = s

    @property
    def ptr(self):
        return C.cast(C.pointer(self.struct), C.c_void_p)


def query_field(osc: OracleScene, Q):
    Q = _c(Q, np.int64)
    t = np.empty(8, np.float64)
    miss = lib().orc_query_field(osc.ptr, _p(Q), _p(t))
    return t, miss


def encode_dir(d):
    d = _c(d, np.float64)
    e = np.empty(27, np.float64)
    lib().orc_encode_dir(_p(d), _p(e))
    return e


def mlp(w, cd, F, d):
    w, cd, F, d = (_c(a, np.float64) for a in (w, cd, F, d))
    h = np.empty(3, np.float64)
    lib().orc_mlp(_p(w), _p(cd), _p(F), _p(d), _p(h))
    return h


# ------------------------------------------------------------------------------------
# renderers
# ------------------------------------------------------------------------------------
_MODES = {"hier": 0, "dense": 1, "sph": 2}
STAT_KEYS = ("rays", "segments", "evaluated", "density_only", "skips", "missing")


def render(osc: OracleScene, cam, W: int, H: int, *, pixels=None, mode: str = "hier",
           flags: int = 0, max_trace: int = 0, threads: int = 0, aux: bool = False,
           region_masks: bool = False):
    """Render pixels (default: the whole W x H frame) of camera `cam` (17 doubles).

    Returns dict(rgb [n,3] float64, stats, optional trace_cells/trace_T/trace_count, aux).
    """
    cam = _c(cam, np.float64)
    if pixels is None:
        pixels = np.arange(W * H, dtype=np.int64)
    pixels = _c(pixels, np.int64)
    n = len(pixels)
    rgb = np.empty((n, 3), np.float64)
    auxa = np.empty((n, 8), np.float64) if aux else None
    tc = np.zeros((n, max_trace), np.uint64) if max_trace else None
    tT = np.zeros((n, max_trace), np.float64) if max_trace else None
    cnt = np.zeros(n, np.int32) if max_trace else None
    rm = np.zeros(n, np.int32) if region_masks else None
    st = np.zeros(6, np.int64)
    nullp = C.c_void_p(0)
    lib().orc_render_pixels(osc.ptr, _p(cam), int(W), _p(pixels), n, _MODES[mode],
                            int(flags), _p(rgb), _p(auxa) if aux else nullp, int(max_trace),
                            _p(tc) if max_trace else nullp, _p(tT) if max_trace else nullp,
                            _p(cnt) if max_trace else nullp, _p(st),
                            _p(rm) if region_masks else nullp, int(threads))
    out = dict(rgb=rgb, stats=dict(zip(STAT_KEYS, st.tolist())))
    if aux:
        out["aux"] = auxa
    if max_trace:
        out.update(trace_cells=tc, trace_T=tT, trace_count=cnt)
    if region_masks:
        out["region_masks"] = rm
    return out


def render_rays(osc: OracleScene, o, d, t_near=None, *, mode: str = "hier", flags: int = 0,
                max_trace: int = 0):
    o = _c(o, np.float64).reshape(-1, 3)
    d = _c(d, np.float64).reshape(-1, 3)
    n = len(o)
    tn = _c(np.zeros(n) if t_near is None else t_near, np.float64)
    rgb = np.empty((n, 3), np.float64)
    auxa = np.empty((n, 8), np.float64)
    tc = np.zeros((n, max_trace), np.uint64) if max_trace else None
    tT = np.zeros((n, max_trace), np.float64) if max_trace else None
    cnt = np.zeros(n, np.int32) if max_trace else None
    st = np.zeros(6, np.int64)
    nullp = C.c_void_p(0)
    lib().orc_render_rays(osc.ptr, _p(o), _p(d), _p(tn), n, _MODES[mode], int(flags),
                          _p(rgb), _p(auxa), int(max_trace), _p(tc) if max_trace else nullp,
                          _p(tT) if max_trace else nullp, _p(cnt) if max_trace else nullp, _p(st))
    out = dict(rgb=rgb, aux=auxa, stats=dict(zip(STAT_KEYS, st.tolist())))
    if max_trace:
        out.update(trace_cells=tc, trace_T=tT, trace_count=cnt)
    return out


def max_threads() -> int:
    return int(lib().orc_max_threads())


def unpack_trace(cells: np.ndarray):
    """(segment ordinal, k, finest cell) from packed trace words."""
    cells = cells.astype(np.uint64)
    return ((cells >> np.uint64(61)).astype(np.int64),
            ((cells >> np.uint64(40)) & np.uint64((1 << 21) - 1)).astype(np.int64),
            (cells & np.uint64((1 << 40) - 1)).astype(np.int64))


# ------------------------------------------------------------------------------------
# baking (NEXT-1)
# ------------------------------------------------------------------------------------
def tau_threshold(step: float, alpha_thr: float = 0.005) -> float:
    """alpha = 1 - exp(-tau step) > alpha_thr  <=>  tau > -ln(1 - alpha_thr) / step."""
    import math
    return -math.log1p(-alpha_thr) / step


def bake_occupancy(x, tau, w, N: int, step: float, w_thr: float = 0.005, alpha_thr: float = 0.005):
    x = _c(x, np.float64).reshape(-1, 3)
    tau = _c(tau, np.float64)
    w = _c(w, np.float64)
    bits = np.zeros(n_words(N), np.uint32)
    lib().orc_bake_occupancy(_p(x), _p(tau), _p(w), len(x), tau_threshold(step, alpha_thr), float(w_thr),
                             int(N), _p(bits))
    return bits


def pack_atlas(dense, L: int, block_index, n_blocks: int):
    dense = _c(dense, np.uint8)
    bi = _c(block_index, np.int32)
    atlas = np.zeros((n_blocks, 9, 9, 9, 8), np.uint8)
    lib().orc_pack_atlas(_p(dense), int(L), _p(bi), int(n_blocks), _p(atlas))
    return atlas


# ------------------------------------------------------------------------------------
# NEXT-2: spherical contraction (Eq. 4)
# ------------------------------------------------------------------------------------
def contract_sph(x):
    x = _c(x, np.float64).reshape(-1, 3)
    y = np.empty_like(x)
    for i in range(len(x)):
        lib().orc_contract_sph(_p(x[i]), _p(y[i]))
    return y


def sph_speed(x, d) -> float:
    return float(lib().orc_sph_speed(_p(_c(x, np.float64)), _p(_c(d, np.float64))))
