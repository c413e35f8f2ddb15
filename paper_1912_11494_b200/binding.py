"""Thin ctypes binding of libsegb200.so (include/seg.h), same names as the C ABI.

Argument marshalling only: every step of the hot path runs in the library's CUDA
kernels.  There is no CPU fallback -- if the library cannot be loaded the import
of this module fails loudly.
"""
from __future__ import annotations

import ctypes
import os

from . import _build

SEG_OK, SEG_EINVAL, SEG_ENOMEM, SEG_ECUDA = 0, -1, -2, -3
SEG_NPTS = 21
SEG_MODE_EXACT, SEG_MODE_PAPER = 0, 1
SEG_KEY_NONE, SEG_KEY_NONFINITE = 0x7FFFFFFFFFFFFFFF, 0x7FFFFFFFFFFFFFFE
SEG_NSTATS = 22
STAT_NAMES = ("fibers", "warp_tiles_listed", "warp_tiles_computed", "lane_tile_pass", "lane_test1",
              "lane_test2", "lane_test34", "lane_full21", "best_updates", "lane_point_dists",
              "lane_bound_tests", "ctas",
              "cyc_consumer", "cyc_full_wait", "cyc_hit_select", "cyc_cand_rounds", "cyc_tile_test", "cyc_ingest",
              "rounds", "round_lanes", "hit_fibers", "reserved21")


class SegError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class seg_atlas_info(ctypes.Structure):
    _fields_ = [("n_centroids", ctypes.c_int64), ("n_bundles", ctypes.c_int32),
                ("n_tiles", ctypes.c_int32), ("tile_size", ctypes.c_int32),
                ("device", ctypes.c_int32), ("device_bytes", ctypes.c_int64), ("mode", ctypes.c_int32)]


def _load() -> ctypes.CDLL:
    override = os.environ.get("SEG_LIB")   # an alternative build of the same sources (the checked build)
    if override:
        if not os.path.exists(override):
            raise ImportError(f"SEG_LIB={override} does not exist")
        path = override
    else:
        path = _build.LIB
    if not override and _build.stale():
        _build.build()          # compiles the CUDA library; raises if nvcc is unavailable
    if not os.path.exists(path):
        raise ImportError(f"libsegb200.so missing at {path}; run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
    lib.seg_create.restype = ctypes.c_int
    lib.seg_create.argtypes = [vp, vp, i64, vp, i32, ctypes.c_int, ctypes.POINTER(vp)]
    lib.seg_create_ex.restype = ctypes.c_int
    lib.seg_create_ex.argtypes = [vp, vp, i64, vp, i32, ctypes.c_int, ctypes.c_uint32, ctypes.POINTER(vp)]
    lib.seg_group_by_bundle.restype = ctypes.c_int
    lib.seg_group_by_bundle.argtypes = [vp, vp, i64, i32, vp, vp, vp, vp, vp, vp]
    lib.seg_resample.restype = ctypes.c_int
    lib.seg_resample.argtypes = [vp, vp, i64, vp, vp]
    lib.seg_classify_keys.restype = ctypes.c_int
    lib.seg_classify_keys.argtypes = [vp, vp, i64, vp, vp]
    lib.seg_classify_multi.restype = ctypes.c_int
    lib.seg_classify_multi.argtypes = [vp, vp, i64, vp, i32, vp]
    lib.seg_keys_to_labels.restype = ctypes.c_int
    lib.seg_keys_to_labels.argtypes = [vp, i64, i32, vp, vp, vp]
    lib.seg_classify.restype = ctypes.c_int
    lib.seg_classify.argtypes = [vp, vp, i64, vp, vp, vp]
    lib.seg_classify_stats.restype = ctypes.c_int
    lib.seg_classify_stats.argtypes = [vp, vp, i64, vp, vp, vp, vp]
    lib.seg_get_atlas_info.restype = ctypes.c_int
    lib.seg_get_atlas_info.argtypes = [vp, ctypes.POINTER(seg_atlas_info)]
    lib.seg_plan_tiles.restype = ctypes.c_int
    lib.seg_plan_tiles.argtypes = [vp, vp, i64, i32, i32, ctypes.POINTER(i32), vp, vp, vp]
    lib.seg_debug_classify_seeded.restype = ctypes.c_int
    lib.seg_debug_classify_seeded.argtypes = [vp, vp, i64, vp, vp, vp, vp, vp]
    lib.seg_profile_enable.restype = ctypes.c_int
    lib.seg_profile_enable.argtypes = [vp, i32]
    lib.seg_profile_read.restype = ctypes.c_int
    lib.seg_profile_read.argtypes = [vp, vp, vp, vp, i32, ctypes.POINTER(i32)]
    lib.seg_destroy.restype = None
    lib.seg_destroy.argtypes = [vp]
    lib.seg_last_error.restype = ctypes.c_char_p
    lib.seg_last_error.argtypes = []
    return lib


LIB = _load()
EXPORTS = ("seg_create", "seg_create_ex", "seg_classify", "seg_classify_stats", "seg_get_atlas_info", "seg_plan_tiles",
           "seg_profile_enable", "seg_profile_read", "seg_group_by_bundle", "seg_resample", "seg_classify_keys", "seg_classify_multi", "seg_keys_to_labels", "seg_debug_classify_seeded", "seg_destroy", "seg_last_error")


def seg_last_error() -> str:
    return LIB.seg_last_error().decode()


def _check(rc: int) -> None:
    if rc != SEG_OK:
        raise SegError(rc, seg_last_error())


def _ptr(x) -> int | None:
    """Raw address of a torch tensor or numpy array (no copies, no dtype conversion)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        return x.ctypes.data
    raise TypeError(f"unsupported buffer type {type(x)}")


def seg_create_ex(centroids, bundle_id, M: int, thresh, B: int, device: int = -1, flags: int = SEG_MODE_EXACT) -> int:
    """seg_create with a scoring mode (SEG_MODE_EXACT / SEG_MODE_PAPER); returns the handle."""
    out = ctypes.c_void_p()
    _check(LIB.seg_create_ex(_ptr(centroids), _ptr(bundle_id), int(M), _ptr(thresh), int(B), int(device),
                             int(flags), ctypes.byref(out)))
    return out.value


def seg_create(centroids, bundle_id, M: int, thresh, B: int, device: int = -1) -> int:
    """Returns an opaque seg_atlas handle (int).  Buffers: host or device, see seg.h."""
    out = ctypes.c_void_p()
    _check(LIB.seg_create(_ptr(centroids), _ptr(bundle_id), int(M), _ptr(thresh), int(B), int(device),
                          ctypes.byref(out)))
    return out.value


def seg_classify(atlas: int, fibers, N: int, label, dist, stream: int | None = None) -> None:
    _check(LIB.seg_classify(atlas, _ptr(fibers), int(N), _ptr(label), _ptr(dist), stream))


def seg_classify_stats(atlas: int, fibers, N: int, label, dist, stats, stream: int | None = None) -> None:
    _check(LIB.seg_classify_stats(atlas, _ptr(fibers), int(N), _ptr(label), _ptr(dist), _ptr(stats), stream))


def seg_get_atlas_info(atlas: int) -> dict:
    info = seg_atlas_info()
    _check(LIB.seg_get_atlas_info(atlas, ctypes.byref(info)))
    return {k: getattr(info, k) for k, _ in seg_atlas_info._fields_}


def seg_plan_tiles(centroids, bundle_id, M: int, B: int, max_tiles: int, tile_bundle=None, tile_members=None,
                   tile_spheres=None) -> int:
    nt = ctypes.c_int32()
    _check(LIB.seg_plan_tiles(_ptr(centroids), _ptr(bundle_id), int(M), int(B), int(max_tiles),
                              ctypes.byref(nt), _ptr(tile_bundle), _ptr(tile_members), _ptr(tile_spheres)))
    return nt.value


def seg_debug_classify_seeded(atlas: int, fibers, N: int, seed_keys, label, dist, stats=None,
                              stream: int | None = None) -> None:
    _check(LIB.seg_debug_classify_seeded(atlas, _ptr(fibers), int(N), _ptr(seed_keys), _ptr(label), _ptr(dist),
                                         _ptr(stats), stream))


def seg_profile_enable(atlas: int, capacity: int) -> None:
    _check(LIB.seg_profile_enable(atlas, int(capacity)))


def seg_profile_read(atlas: int, prepass_ms, cull_ms, classify_ms, capacity: int) -> int:
    cnt = ctypes.c_int32()
    _check(LIB.seg_profile_read(atlas, _ptr(prepass_ms), _ptr(cull_ms), _ptr(classify_ms), int(capacity),
                                ctypes.byref(cnt)))
    return cnt.value


def seg_destroy(atlas: int | None) -> None:
    LIB.seg_destroy(atlas)


def seg_group_by_bundle(label, dist, N: int, B: int, order, offsets, dmin=None, dmax=None, dsum=None,
                        stream: int | None = None) -> None:
    _check(LIB.seg_group_by_bundle(_ptr(label), _ptr(dist), int(N), int(B), _ptr(order), _ptr(offsets),
                                   _ptr(dmin), _ptr(dmax), _ptr(dsum), stream))


def seg_resample(points, offsets, N: int, out, stream: int | None = None) -> None:
    _check(LIB.seg_resample(_ptr(points), _ptr(offsets), int(N), _ptr(out), stream))


def seg_classify_keys(atlas: int, fibers, N: int, keys, stream: int | None = None) -> None:
    _check(LIB.seg_classify_keys(atlas, _ptr(fibers), int(N), _ptr(keys), stream))


def seg_classify_multi(atlas: int, fibers, N: int, masks, words: int, stream: int | None = None) -> None:
    _check(LIB.seg_classify_multi(atlas, _ptr(fibers), int(N), _ptr(masks), int(words), stream))


def seg_keys_to_labels(keys, N: int, mode: int, label, dist, stream: int | None = None) -> None:
    _check(LIB.seg_keys_to_labels(_ptr(keys), int(N), int(mode), _ptr(label), _ptr(dist), stream))

