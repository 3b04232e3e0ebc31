"""Thin ctypes binding of libmerf.so (include/merf.h).  Argument marshalling only: every
step of the render path runs in the library's CUDA kernels.  There is no CPU fallback --
if the library is missing or no CUDA device is present, calls raise.

Function names mirror the C ABI (merf_scene_upload, merf_render, ...).  Device buffers are
torch CUDA tensors (PyTorch is used for device memory and streams only).
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MERF_LIB: another in-tree build of the same library (A/B timing of kernel variants, e.g.
# `tools/ab_bench.sh`); default: the library next to this file
LIB_PATH = os.environ.get("MERF_LIB") or os.path.join(_HERE, "libmerf.so")

MERF_OK, MERF_EINVAL, MERF_ENOMEM, MERF_ECUDA, MERF_ENCCL, MERF_EMISMATCH, MERF_EIO = range(7)
MERF_RGB_F32, MERF_RGBA_U8 = 0, 1
MERF_NO_EARLY_TERM, MERF_COUNTERS, MERF_DENSE, MERF_TIMED, MERF_SPHERICAL, MERF_MLP_FFMA = 1, 2, 4, 8, 16, 32
MERF_SPH_PERSISTENT = 64
MAX_LEVELS = 4

_STATUS = {1: "MERF_EINVAL", 2: "MERF_ENOMEM", 3: "MERF_ECUDA", 4: "MERF_ENCCL", 5: "MERF_EMISMATCH", 6: "MERF_EIO"}


class MerfError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class merf_scene_desc(C.Structure):
    _fields_ = [("L", C.c_int32), ("R", C.c_int32), ("C", C.c_int32), ("n_levels", C.c_int32),
                ("level_res", C.c_int32 * MAX_LEVELS),
                ("m_density", C.c_float), ("m_appearance", C.c_float),
                ("step", C.c_double), ("t_min", C.c_float), ("alpha_skip", C.c_float),
                ("source_mask", C.c_uint32)]


class merf_qat_desc(C.Structure):
    _fields_ = [("L", C.c_int32), ("R", C.c_int32), ("occ_res", C.c_int32), ("quantize", C.c_int32),
                ("max_samples", C.c_int32), ("pad_", C.c_int32), ("step", C.c_double),
                ("m_density", C.c_double), ("m_appearance", C.c_double)]


class merf_camera(C.Structure):
    _fields_ = [("c2w", C.c_double * 12), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("t_near", C.c_double)]


class merf_stats(C.Structure):
    _fields_ = [("rays", C.c_int64), ("segments", C.c_int64), ("evaluated", C.c_int64),
                ("density_only", C.c_int64), ("skips", C.c_int64), ("missing_blocks", C.c_int64),
                ("region_segments", C.c_int64 * 7), ("march_rounds", C.c_int64), ("march_steps", C.c_int64),
                ("march_lane_rounds", C.c_int64), ("march_busy_ns", C.c_int64), ("march_tail_ns", C.c_int64)]

    def as_dict(self):
        d = {k: int(getattr(self, k)) for k, _ in self._fields_ if k != "region_segments"}
        d["region_segments"] = [int(v) for v in self.region_segments]
        return d


class merf_kernel_times(C.Structure):
    _fields_ = [("setup_ms", C.c_double), ("march_ms", C.c_double), ("shade_ms", C.c_double),
                ("setup_launches", C.c_int64), ("march_launches", C.c_int64), ("shade_launches", C.c_int64)]


class merf_scene_info(C.Structure):
    _fields_ = [("L", C.c_int32), ("R", C.c_int32), ("C", C.c_int32), ("n_levels", C.c_int32),
                ("level_res", C.c_int32 * MAX_LEVELS), ("n_blocks", C.c_int64),
                ("canonical_blocks", C.c_int64), ("device_bytes", C.c_int64), ("device", C.c_int32)]


_lib = None
_lock = threading.Lock()

# (name, restype, argtypes) of every exported symbol of include/merf.h
_vp, _i32, _i64, _u32 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32
SIGNATURES = [
    ("merf_last_error", C.c_char_p, []),
    ("merf_version", _i32, []),
    ("merf_scene_upload", C.c_int, [C.POINTER(merf_scene_desc), _vp, _vp, _vp, _i64, _vp, _vp, _i32,
                                    C.POINTER(_vp)]),
    ("merf_scene_free", C.c_int, [_vp]),
    ("merf_scene_info_get", C.c_int, [_vp, C.POINTER(merf_scene_info)]),
    ("merf_kernel_times_get", C.c_int, [_vp, C.POINTER(merf_kernel_times), _i32]),
    ("merf_scene_occupancy", C.c_int, [_vp, _i32, _vp, _vp]),
    ("merf_scene_block_index", C.c_int, [_vp, _vp, _vp]),
    ("merf_render", C.c_int, [_vp, C.POINTER(merf_camera), _i32, _i32, _i32, _i32, _vp, _u32, _vp,
                              C.POINTER(merf_stats)]),
    ("merf_render_progressive", C.c_int, [_vp, C.POINTER(merf_camera), _i32, _i32, _i32, _i32, _i32, _i32, _i32,
                                          _vp, _u32, _vp]),
    ("merf_render_shard", C.c_int, [_vp, C.POINTER(merf_camera), _i32, _i32, _i32, _i32, _i32, _i32, _vp, _u32,
                                    _vp]),
    ("merf_render_host", C.c_int, [_vp, C.POINTER(merf_camera), _i32, _i32, _i32, _i32, _vp, _u32, _vp]),
    ("merf_render_rays", C.c_int, [_vp, _vp, _vp, _vp, _i64, _vp, _u32, _vp, C.POINTER(merf_stats)]),
    ("merf_trace", C.c_int, [_vp, C.POINTER(merf_camera), _i32, _vp, _i64, _i32, _vp, _vp, _vp, _u32,
                             _vp]),
    ("merf_segments", C.c_int, [_vp, C.POINTER(merf_camera), _i32, _vp, _i64, _i32, _vp, _vp, _vp]),
    ("merf_contract", C.c_int, [_vp, _i64, _vp, _vp, _vp]),
    ("merf_build_occupancy", C.c_int, [_vp, C.POINTER(merf_scene_desc), _vp, _vp]),
    ("merf_bake_occupancy", C.c_int, [_vp, _vp, _vp, _i64, _i32, C.c_double, C.c_double, C.c_double, _vp, _vp]),
    ("merf_pack_atlas", C.c_int, [_vp, _i32, _vp, _i64, _vp, _vp]),
    ("merf_qat_step", C.c_int, [C.POINTER(merf_qat_desc), _vp, _vp, _vp, _vp, C.POINTER(merf_camera), _i32,
                                _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("merf_bundle_write", C.c_int, [C.c_char_p, C.POINTER(merf_scene_desc), _vp, _vp, _vp, _i64, _vp, _vp]),
    ("merf_bundle_read", C.c_int, [C.c_char_p, C.POINTER(merf_scene_desc), C.POINTER(_i64), _vp, _vp, _vp, _vp,
                                   _vp]),
    ("merf_scene_load", C.c_int, [C.c_char_p, _i32, C.POINTER(_vp)]),
    ("merf_cameras_read", C.c_int, [C.c_char_p, C.POINTER(merf_camera), _i32, C.POINTER(_i32), _vp, _vp]),
    ("merf_build_block_index", C.c_int, [_vp, C.POINTER(merf_scene_desc), _vp, C.POINTER(_i64), _vp]),
    ("merf_render_host_async", C.c_int, [_vp, C.POINTER(merf_camera), _i32, _i32, _i32, _i32, _vp, _u32, _vp]),
    ("merf_host_wait", C.c_int, [_vp]),
    ("merf_render_workspace_bytes", C.c_int, [_vp, C.POINTER(merf_camera), _i32, _i32, _i32, C.POINTER(_i64),
                                              C.POINTER(_i64)]),
    ("merf_render_shard_blocks", C.c_int, [_vp, C.POINTER(merf_camera), _i32, _i32, _i32, _i32, _i32, _i32, _vp,
                                           _u32, _vp]),
    ("merf_shard_slots", _i32, [_i32, _i32, _i32]),
    ("merf_shard_assemble", C.c_int, [_vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp]),
    ("merf_comm_unique_id", C.c_int, [_vp]),
    ("merf_comm_init", C.c_int, [_vp, _i32, _i32, _i32, C.POINTER(_vp)]),
    ("merf_comm_free", C.c_int, [_vp]),
    ("merf_comm_info", C.c_int, [_vp, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32)]),
    ("merf_gather_frames", C.c_int, [_vp, _vp, _vp, _i64, _i32, _vp]),
    ("merf_comm_wait", C.c_int, [_vp, _vp, _i32]),
]


def lib():
    """Load libmerf.so (fails loudly if it was not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; "
                                  f"g.build()'` (there is no fallback path)")
            L = C.CDLL(LIB_PATH)
            for name, res, args in SIGNATURES:
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def _check(status):
    if status != MERF_OK:
        raise MerfError(status, lib().merf_last_error().decode())


def merf_last_error() -> str:
    return lib().merf_last_error().decode()


def merf_version() -> int:
    return int(lib().merf_version())


def _ptr(t):
    """data pointer of a torch tensor or numpy array (or None)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream(stream):
    import torch
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def make_desc(scene) -> merf_scene_desc:
    d = merf_scene_desc()
    d.L, d.R, d.C = int(scene.L), int(scene.R), int(getattr(scene, "C", 8))
    lv = list(scene.level_res)
    d.n_levels = len(lv)                 # validated by the library (1..MAX_LEVELS)
    for i, v in enumerate(lv[:MAX_LEVELS]):
        d.level_res[i] = int(v)
    d.m_density = float(getattr(scene, "m_density", 14.0))
    d.m_appearance = float(getattr(scene, "m_appearance", 7.0))
    d.step = float(scene.step)
    d.t_min = float(getattr(scene, "t_min", 2e-4))
    d.alpha_skip = float(getattr(scene, "alpha_skip", 0.0))
    d.source_mask = int(getattr(scene, "source_mask", 15))
    return d


def cameras_to_c(cams) -> "C.Array":
    cams = np.ascontiguousarray(np.asarray(cams, np.float64).reshape(-1, 17))
    arr = (merf_camera * len(cams))()
    C.memmove(arr, cams.ctypes.data, cams.nbytes)
    return arr


def merf_scene_upload(scene, device: int = 0, canonical: bool = False) -> int:
    """Upload host arrays of `scene` (attributes: L, R, level_res, step, planes, block_index,
    atlas, occ_finest, mlp, ...).  canonical=True passes block_index=NULL.  Returns the handle."""
    desc = make_desc(scene)
    planes = np.ascontiguousarray(scene.planes, np.uint8)
    atlas = np.ascontiguousarray(scene.atlas, np.uint8)
    bidx = None if canonical else np.ascontiguousarray(scene.block_index, np.int32)
    occ = np.ascontiguousarray(scene.occ_finest, np.uint32)
    mlp = np.ascontiguousarray(scene.mlp, np.float32)
    n_blocks = int(atlas.shape[0]) if atlas.ndim else 0
    h = C.c_void_p()
    _check(lib().merf_scene_upload(C.byref(desc), _ptr(planes) if planes.size else None,
                                   _ptr(bidx) if bidx is not None and bidx.size else None,
                                   _ptr(atlas) if atlas.size else None, n_blocks, _ptr(occ),
                                   _ptr(mlp), int(device), C.byref(h)))
    return h.value


def merf_scene_free(handle) -> None:
    _check(lib().merf_scene_free(handle))


def merf_scene_info_get(handle) -> dict:
    info = merf_scene_info()
    _check(lib().merf_scene_info_get(handle, C.byref(info)))
    return dict(L=info.L, R=info.R, n_levels=info.n_levels, level_res=list(info.level_res)[:info.n_levels],
                n_blocks=info.n_blocks, canonical_blocks=info.canonical_blocks,
                device_bytes=info.device_bytes, device=info.device)


def merf_kernel_times_get(handle, reset: bool = True) -> dict:
    t = merf_kernel_times()
    _check(lib().merf_kernel_times_get(handle, C.byref(t), int(bool(reset))))
    return {k: getattr(t, k) for k, _ in t._fields_}


def merf_scene_occupancy(handle, level: int, out, stream=None) -> None:
    _check(lib().merf_scene_occupancy(handle, int(level), _ptr(out), _stream(stream)))


def merf_scene_block_index(handle, out, stream=None) -> None:
    _check(lib().merf_scene_block_index(handle, _ptr(out), _stream(stream)))


def merf_render(handle, cams, W: int, H: int, out, fmt: int = MERF_RGB_F32, flags: int = 0,
                stream=None, stats: bool = False):
    """Render frames into the device tensor `out`; returns a stats dict if stats=True."""
    carr = cameras_to_c(cams)
    st = merf_stats() if stats else None
    _check(lib().merf_render(handle, carr, len(carr), int(W), int(H), int(fmt), _ptr(out), int(flags),
                             _stream(stream), C.byref(st) if st is not None else None))
    return st.as_dict() if st is not None else None


def merf_render_progressive(handle, cams, W: int, H: int, stride: int, pass_: int, out, fill: bool = False,
                            fmt: int = MERF_RGB_F32, flags: int = 0, stream=None) -> None:
    """Render pass `pass_` of stride x stride progressive rendering into `out`."""
    carr = cameras_to_c(cams)
    _check(lib().merf_render_progressive(handle, carr, len(carr), int(W), int(H), int(stride), int(pass_),
                                         int(bool(fill)), int(fmt), _ptr(out), int(flags), _stream(stream)))


def shard_owner(W: int, H: int, part_count: int):
    """Owner rank of every pixel under merf_render_shard's partition (host-side indexing, for
    assembling / checking sharded frames): 64x64 blocks, row-major, block b -> rank b % N."""
    by = np.arange(H)[:, None] // 64
    bx = np.arange(W)[None, :] // 64
    return ((by * ((W + 63) // 64) + bx) % part_count).astype(np.int32)


def merf_render_shard(handle, cams, W: int, H: int, part_rank: int, part_count: int, out,
                      fmt: int = MERF_RGB_F32, flags: int = 0, stream=None) -> None:
    """Render the 64x64-pixel blocks b with b % part_count == part_rank of every view into the
    full-size `out` (SURVEY 8(e) single-frame sharding); other pixels are left untouched."""
    carr = cameras_to_c(cams)
    _check(lib().merf_render_shard(handle, carr, len(carr), int(W), int(H), int(part_rank), int(part_count),
                                   int(fmt), _ptr(out), int(flags), _stream(stream)))


def merf_render_workspace_bytes(handle, cams, W: int, H: int) -> dict:
    """device workspace of a merf_render(cams, W, H) call: bytes per chunk and rays per chunk."""
    b, r = C.c_int64(), C.c_int64()
    carr = cameras_to_c(cams)
    _check(lib().merf_render_workspace_bytes(handle, carr, len(carr), int(W), int(H), C.byref(b), C.byref(r)))
    return {"bytes": b.value, "rays_per_chunk": r.value, "bytes_per_ray": b.value / max(r.value, 1)}


def merf_shard_slots(W: int, H: int, part_count: int) -> int:
    """64x64 block slots per part of a W x H frame split into part_count parts."""
    return int(lib().merf_shard_slots(int(W), int(H), int(part_count)))


def merf_render_shard_blocks(handle, cams, W: int, H: int, part_rank: int, part_count: int, out,
                             fmt: int = MERF_RGBA_U8, flags: int = 0, stream=None) -> None:
    """Render this part's 64x64 blocks into the compact slot buffer `out`
    ([n_cams][merf_shard_slots][64][64] pixels), ready for merf_gather_frames."""
    carr = cameras_to_c(cams)
    _check(lib().merf_render_shard_blocks(handle, carr, len(carr), int(W), int(H), int(part_rank),
                                          int(part_count), int(fmt), _ptr(out), int(flags), _stream(stream)))


def merf_shard_assemble(blocks, n_views: int, W: int, H: int, part_count: int, frame_out,
                        fmt: int = MERF_RGBA_U8, stream=None) -> None:
    """Rebuild [n_views][H][W] frames from the gathered [part_count][n_views][slots][64][64] blocks."""
    _check(lib().merf_shard_assemble(_ptr(blocks), int(n_views), int(W), int(H), int(part_count), int(fmt),
                                     _ptr(frame_out), _stream(stream)))


COMM_ID_BYTES = 128


def merf_comm_unique_id() -> bytes:
    """A new NCCL unique id (rank 0 creates it; the caller distributes it)."""
    buf = (C.c_uint8 * COMM_ID_BYTES)()
    _check(lib().merf_comm_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


class Comm:
    """The library's NCCL communicator (merf_comm_init / merf_comm_free); the frame gather of
    SURVEY 8(e) runs through merf_gather_frames on it."""

    def __init__(self, unique_id: bytes, n_ranks: int, rank: int, device: int):
        assert len(unique_id) == COMM_ID_BYTES
        buf = (C.c_uint8 * COMM_ID_BYTES).from_buffer_copy(unique_id)
        h = C.c_void_p()
        _check(lib().merf_comm_init(C.cast(buf, C.c_void_p), int(n_ranks), int(rank), int(device), C.byref(h)))
        self.handle = h.value
        self.n_ranks, self.rank, self.device = n_ranks, rank, device

    def info(self) -> dict:
        n, r, v = C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().merf_comm_info(self.handle, C.byref(n), C.byref(r), C.byref(v)))
        return {"n_ranks": n.value, "rank": r.value, "nccl_version": v.value}

    def gather(self, local, root_buf, nbytes: int = None, root: int = 0, stream=None) -> None:
        """merf_gather_frames: `local` (device tensor) of every rank -> root_buf[rank] on the root."""
        n = int(nbytes if nbytes is not None else local.numel() * local.element_size())
        _check(lib().merf_gather_frames(self.handle, _ptr(local), _ptr(root_buf), n, int(root), _stream(stream)))

    def wait(self, stream=None, timeout_ms: int = 60000) -> None:
        """merf_comm_wait: block until `stream` completes, polling NCCL's async error state."""
        _check(lib().merf_comm_wait(self.handle, _stream(stream), int(timeout_ms)))

    def close(self):
        if getattr(self, "handle", None):
            lib().merf_comm_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def merf_render_host_async(handle, cams, W: int, H: int, out_host, fmt: int = MERF_RGBA_U8,
                           flags: int = 0, stream=None) -> None:
    """Render and enqueue the copy to `out_host` (pinned); returns at once (merf_host_wait)."""
    carr = cameras_to_c(cams)
    _check(lib().merf_render_host_async(handle, carr, len(carr), int(W), int(H), int(fmt), _ptr(out_host),
                                        int(flags), _stream(stream)))


def merf_host_wait(handle) -> None:
    """Wait for every copy merf_render_host_async enqueued on this scene."""
    _check(lib().merf_host_wait(handle))


def merf_render_host(handle, cams, W: int, H: int, out_host, fmt: int = MERF_RGBA_U8,
                     flags: int = 0, stream=None) -> None:
    """End-to-end: render into scene-owned device staging and copy to the host tensor/array."""
    carr = cameras_to_c(cams)
    _check(lib().merf_render_host(handle, carr, len(carr), int(W), int(H), int(fmt), _ptr(out_host),
                                  int(flags), _stream(stream)))


def merf_render_rays(handle, o, d, rgb, t_near=None, flags: int = 0, stream=None, stats: bool = False):
    st = merf_stats() if stats else None
    _check(lib().merf_render_rays(handle, _ptr(o), _ptr(d), _ptr(t_near), int(o.shape[0]), _ptr(rgb),
                                  int(flags), _stream(stream), C.byref(st) if st is not None else None))
    return st.as_dict() if st is not None else None


def merf_trace(handle, cam, W: int, pixel_ids, max_per_ray: int, cells_out, T_out, counts_out,
               flags: int = 0, stream=None) -> None:
    carr = cameras_to_c(cam)
    _check(lib().merf_trace(handle, carr, int(W), _ptr(pixel_ids), int(pixel_ids.shape[0]),
                            int(max_per_ray), _ptr(cells_out), _ptr(T_out), _ptr(counts_out),
                            int(flags), _stream(stream)))


SEGMENT_DTYPE = np.dtype([("t_a", "<f8"), ("t_b", "<f8"), ("Qa", "<i8", 3), ("U", "<i8", 3),
                          ("K", "<i4"), ("region", "<i4")])


def merf_segments(handle, cam, W: int, pixel_ids, max_seg: int, segs_out, counts_out, stream=None) -> None:
    """segs_out: device buffer of n * max_seg * 72 bytes (view as SEGMENT_DTYPE on the host)."""
    carr = cameras_to_c(cam)
    _check(lib().merf_segments(handle, carr, int(W), _ptr(pixel_ids), int(pixel_ids.shape[0]),
                               int(max_seg), _ptr(segs_out), _ptr(counts_out), _stream(stream)))


def merf_contract(x, y, region=None, stream=None) -> None:
    _check(lib().merf_contract(_ptr(x), int(x.shape[0]), _ptr(y), _ptr(region), _stream(stream)))


def merf_build_occupancy(finest_bits, scene, levels_out, stream=None) -> None:
    desc = make_desc(scene)
    _check(lib().merf_build_occupancy(_ptr(finest_bits), C.byref(desc), _ptr(levels_out), _stream(stream)))


def merf_build_block_index(finest_bits, scene, index_out, stream=None) -> int:
    desc = make_desc(scene)
    n = C.c_int64()
    _check(lib().merf_build_block_index(_ptr(finest_bits), C.byref(desc), _ptr(index_out), C.byref(n),
                                        _stream(stream)))
    return int(n.value)


def merf_bake_occupancy(x, tau, w, N: int, step: float, bits_out, w_thr: float = 0.005,
                        alpha_thr: float = 0.005, stream=None) -> None:
    """A from weighted points; x [n,3] / tau / w float64 device tensors."""
    _check(lib().merf_bake_occupancy(_ptr(x), _ptr(tau), _ptr(w), int(x.shape[0]), int(N), float(step),
                                     float(w_thr), float(alpha_thr), _ptr(bits_out), _stream(stream)))


def merf_pack_atlas(dense, L: int, index, n_blocks: int, atlas_out, stream=None) -> None:
    _check(lib().merf_pack_atlas(_ptr(dense), int(L), _ptr(index), int(n_blocks), _ptr(atlas_out),
                                 _stream(stream)))


def merf_qat_step(theta_v, theta_p, occ, N: int, mlp, cams, W: int, H: int, target, rgb_out, grad_v,
                  grad_p, loss, step: float, quantize: bool = True, max_samples: int = 1024,
                  overflow=None, n_samples=None, m_density: float = 14.0, m_appearance: float = 7.0,
                  stream=None) -> None:
    """NEXT-3 quantisation-aware forward + backward (Eq. 7-8) on dense grids; every tensor is a
    device tensor: theta_v [L,L,L,8] / theta_p [3,R,R,8] float32, occ uint32 bits of N^3,
    target / rgb_out [n,H,W,3] float32, grad_* like theta, loss float64 [1], overflow int32 [1],
    n_samples int64 [1]."""
    d = merf_qat_desc()
    d.L, d.R, d.occ_res = int(theta_v.shape[0]), int(theta_p.shape[1]), int(N)
    d.quantize, d.max_samples, d.step = int(bool(quantize)), int(max_samples), float(step)
    d.m_density, d.m_appearance = float(m_density), float(m_appearance)
    carr = cameras_to_c(cams)
    _check(lib().merf_qat_step(C.byref(d), _ptr(theta_v), _ptr(theta_p), _ptr(occ), _ptr(mlp), carr, len(carr),
                               int(W), int(H), _ptr(target), _ptr(rgb_out), _ptr(grad_v), _ptr(grad_p),
                               _ptr(loss), _ptr(overflow), _ptr(n_samples), _stream(stream)))


def merf_bundle_write(directory: str, scene) -> None:
    """Write the host arrays of `scene` (as for merf_scene_upload; block_index required when
    L > 0) as a PNG bundle (Sec. 5.3)."""
    desc = make_desc(scene)
    planes = np.ascontiguousarray(scene.planes, np.uint8)
    atlas = np.ascontiguousarray(scene.atlas, np.uint8)
    bidx = np.ascontiguousarray(scene.block_index, np.int32)
    occ = np.ascontiguousarray(scene.occ_finest, np.uint32)
    mlp = np.ascontiguousarray(scene.mlp, np.float32)
    n_blocks = int(atlas.shape[0]) if atlas.ndim else 0
    _check(lib().merf_bundle_write(os.fsencode(directory), C.byref(desc), _ptr(planes) if planes.size else None,
                                   _ptr(bidx) if bidx.size else None, _ptr(atlas) if atlas.size else None,
                                   n_blocks, _ptr(occ), _ptr(mlp)))


class BundleScene:
    """host arrays read from a bundle; attributes as merf_scene_upload expects."""


def merf_bundle_read(directory: str) -> BundleScene:
    d = merf_scene_desc()
    nb = _i64(0)
    path = os.fsencode(directory)
    _check(lib().merf_bundle_read(path, C.byref(d), C.byref(nb), None, None, None, None, None))
    sc = BundleScene()
    sc.L, sc.R, sc.C = d.L, d.R, d.C
    sc.level_res = tuple(d.level_res[i] for i in range(d.n_levels))
    sc.m_density, sc.m_appearance = d.m_density, d.m_appearance
    sc.step, sc.t_min, sc.alpha_skip, sc.source_mask = d.step, d.t_min, d.alpha_skip, d.source_mask
    n = int(nb.value)
    Nf = sc.level_res[-1]
    sc.planes = np.zeros((3, d.R, d.R, 8) if d.R else (0,), np.uint8)
    sc.block_index = np.zeros(((d.L // 8) ** 3,) if d.L else (0,), np.int32)
    sc.atlas = np.zeros((n, 9, 9, 9, 8), np.uint8)
    sc.occ_finest = np.zeros((Nf ** 3 + 31) // 32, np.uint32)
    sc.mlp = np.zeros(883, np.float32)
    _check(lib().merf_bundle_read(path, C.byref(d), C.byref(nb), _ptr(sc.planes) if sc.planes.size else None,
                                  _ptr(sc.block_index) if sc.block_index.size else None,
                                  _ptr(sc.atlas) if sc.atlas.size else None, _ptr(sc.occ_finest), _ptr(sc.mlp)))
    return sc


def merf_scene_load(directory: str, device: int = 0) -> int:
    """read a bundle and upload it; returns the scene handle."""
    h = C.c_void_p()
    _check(lib().merf_scene_load(os.fsencode(directory), int(device), C.byref(h)))
    return h.value


def merf_cameras_read(path: str):
    """-> (cams float64 [n, 17] as merf_camera, widths int32 [n], heights int32 [n])."""
    n = _i32(0)
    p = os.fsencode(path)
    _check(lib().merf_cameras_read(p, None, 0, C.byref(n), None, None))
    k = int(n.value)
    arr = (merf_camera * max(k, 1))()
    w = np.zeros(max(k, 1), np.int32)
    h = np.zeros(max(k, 1), np.int32)
    _check(lib().merf_cameras_read(p, arr, k, C.byref(n), _ptr(w), _ptr(h)))
    cams = np.frombuffer(bytes(arr), np.float64).reshape(-1, 17)[:k].copy()
    return cams, w[:k], h[:k]


class Scene:
    """RAII wrapper of a device scene handle."""

    def __init__(self, scene, device: int = 0, canonical: bool = False):
        self.handle = merf_scene_upload(scene, device=device, canonical=canonical)
        self.device = device

    @classmethod
    def load(cls, directory: str, device: int = 0) -> "Scene":
        """a scene from a PNG bundle (merf_scene_load)."""
        self = cls.__new__(cls)
        self.handle = merf_scene_load(directory, device)
        self.device = device
        return self

    def info(self) -> dict:
        return merf_scene_info_get(self.handle)

    def render(self, cams, W, H, fmt=MERF_RGB_F32, flags=0, out=None, stream=None, stats=False):
        import torch
        n = len(np.asarray(cams).reshape(-1, 17))
        if out is None:
            shape = (n, H, W, 3) if fmt == MERF_RGB_F32 else (n, H, W, 4)
            out = torch.empty(shape, dtype=torch.float32 if fmt == MERF_RGB_F32 else torch.uint8,
                              device=f"cuda:{self.device}")
        with torch.cuda.device(self.device):      # the scene's device's current stream
            s = merf_render(self.handle, cams, W, H, out, fmt=fmt, flags=flags, stream=stream, stats=stats)
        return (out, s) if stats else out

    def close(self):
        if self.handle:
            merf_scene_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
