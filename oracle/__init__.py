"""CPU oracle for the segmentation hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke(), bench.py's cpu_baseline / --impl
reference legs and scripts/oracle_full.py (which caches oracle outputs) may import
this package.  It shares no code with
paper_1912_11494_b200/ (the CUDA product path) and the product never imports it.

oracle.c holds the arithmetic (plain definition of Eq. 1-2 and Alg. 1's
closest-bundle labelling in double precision, and the sound-discard variants that
reach the same labels bitwise; see its header for citations).
This module only compiles it with gcc, marshals numpy arrays through ctypes and
splits a fiber batch into contiguous chunks over host threads (each thread
writes only its own output slots, as PAPER.md:152 describes for the paper's own
threads).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

DELTA_MM = 1e-3   # tie band (BASELINE.json north_star)


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain C, -O2, no FP contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared",
                               _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            f32p = ctypes.POINTER(ctypes.c_float)
            lib.oracle_point_d2.restype = ctypes.c_double
            lib.oracle_point_d2.argtypes = [f32p, f32p]
            lib.oracle_max_pointwise_d2.restype = ctypes.c_double
            lib.oracle_max_pointwise_d2.argtypes = [f32p, f32p, ctypes.c_int]
            lib.oracle_dme_d2.restype = ctypes.c_double
            lib.oracle_dme_d2.argtypes = [f32p, f32p]
            lib.oracle_dme.restype = ctypes.c_double
            lib.oracle_dme.argtypes = [f32p, f32p]
            cls_args = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                        ctypes.c_void_p, ctypes.c_int32, ctypes.c_double,
                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
            lib.oracle_classify.restype = ctypes.c_int
            lib.oracle_classify.argtypes = cls_args + [ctypes.c_void_p]
            lib.oracle_classify_paper.restype = ctypes.c_int
            lib.oracle_classify_paper.argtypes = cls_args + [ctypes.c_void_p] * 3
            for fn in (lib.oracle_classify_sound, lib.oracle_classify_paper_sound):
                fn.restype = ctypes.c_int
                fn.argtypes = cls_args
            lib.oracle_classify_multi.restype = ctypes.c_int
            lib.oracle_classify_multi.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                                  ctypes.c_int64, ctypes.c_void_p, ctypes.c_int32, ctypes.c_double,
                                                  ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]
            lib.oracle_orientation_ambiguous.restype = ctypes.c_int
            lib.oracle_orientation_ambiguous.argtypes = [f32p, f32p]
            lib.oracle_polyline_length.restype = ctypes.c_double
            lib.oracle_polyline_length.argtypes = [f32p]
            lib.oracle_tn.restype = ctypes.c_double
            lib.oracle_tn.argtypes = [ctypes.c_double, ctypes.c_double]
            lib.oracle_endpoint_orientation.restype = ctypes.c_int
            lib.oracle_endpoint_orientation.argtypes = [f32p, f32p]
            lib.oracle_paper_score.restype = ctypes.c_double
            lib.oracle_paper_score.argtypes = [f32p, f32p]
            _lib = lib
    return _lib


def _f32(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float32)


def _fp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def point_d2(p, q) -> float:
    """Eq. 1 squared for two 3-vectors."""
    p, q = _f32(p).reshape(3), _f32(q).reshape(3)
    return _load().oracle_point_d2(_fp(p), _fp(q))


def max_pointwise(a, b, inverse: bool = False) -> float:
    """max_i d_E(a_i, b_i) (direct) or max_i d_E(a_i, b_{20-i}) (inverse), in mm."""
    a, b = _f32(a).reshape(21, 3), _f32(b).reshape(21, 3)
    return float(np.sqrt(_load().oracle_max_pointwise_d2(_fp(a), _fp(b), int(inverse))))


def d_me(a, b) -> float:
    """Eq. 2 in mm (double)."""
    a, b = _f32(a).reshape(21, 3), _f32(b).reshape(21, 3)
    return float(_load().oracle_dme(_fp(a), _fp(b)))


def polyline_length(a) -> float:
    """Chord length of a 21-point fiber in mm (reading R16)."""
    a = _f32(a).reshape(21, 3)
    return float(_load().oracle_polyline_length(_fp(a)))


def tn(ls: float, lc: float) -> float:
    """Eq. 3 length term."""
    return float(_load().oracle_tn(float(ls), float(lc)))


def endpoint_orientation(a, c) -> int:
    """1 = inverse, 0 = direct: argmin of the end-point maxima, ties -> direct, in double (reading R17)."""
    a, c = _f32(a).reshape(21, 3), _f32(c).reshape(21, 3)
    return int(_load().oracle_endpoint_orientation(_fp(a), _fp(c)))


def orientation_ambiguous(a, c) -> bool:
    """True iff the pair's orientation decision lies in the band of reading R20 (both orientations valid)."""
    a, c = _f32(a).reshape(21, 3), _f32(c).reshape(21, 3)
    return bool(_load().oracle_orientation_ambiguous(_fp(a), _fp(c)))


def paper_score(a, c) -> float:
    """The complete metric d_ME (inferred orientation) + TN, in mm."""
    a, c = _f32(a).reshape(21, 3), _f32(c).reshape(21, 3)
    return float(_load().oracle_paper_score(_fp(a), _fp(c)))


def classify(fibers, centroids, bundle_id, thresh, delta: float = DELTA_MM,
             threads: int | None = None, want_d2b: bool = False, mode: str = "exact",
             sound: bool = False, want_bands: bool = False):
    """Classification of fibers [n,21,3] against the atlas.

    mode "exact": Eq. 2 d_ME (the north_star metric); mode "paper": the paper's complete metric
    d_ME in the end-point-inferred orientation + TN (Eq. 3), SURVEY.md Sec. 8(f) row f1.
    sound=False runs the plain definition (every pair, no discarding); sound=True the sound-discard
    variant (Alg. 1's cascade cut at thr + 2 delta), bitwise the same label / dist / decidable.
    Returns dict(label int32[n], dist float64[n], decidable bool[n]) plus, plain only:
      want_d2b   -> d2b float64[n,B]: exact mode the per-bundle minimum of d_ME^2, paper mode the
                    per-bundle minimum score S_b (mm);
      want_bands -> lo, hi float64[n,B]: the per-bundle interval of correct values in mm (exact mode
                    lo = hi = sqrt(d2b); paper mode [L_b, H_b] of reading R20).
    """
    if mode not in ("exact", "paper"):
        raise ValueError(f"unknown oracle mode {mode!r}")
    if sound and (want_d2b or want_bands):
        raise ValueError("the sound-discard variant does not produce per-bundle values")
    lib = _load()
    fib = _f32(fibers).reshape(-1, 21, 3)
    cen = _f32(centroids).reshape(-1, 21, 3)
    bid = np.ascontiguousarray(bundle_id, dtype=np.int32)
    thr = _f32(thresh).reshape(-1)
    n, m, b = fib.shape[0], cen.shape[0], thr.shape[0]
    label = np.empty(n, np.int32)
    dist = np.empty(n, np.float64)
    dec = np.empty(n, np.uint8)
    per_b = want_d2b or want_bands
    d2b = np.empty((n, b), np.float64) if per_b else None
    lo = np.empty((n, b), np.float64) if (want_bands and mode == "paper") else None
    hi = np.empty((n, b), np.float64) if (want_bands and mode == "paper") else None
    if threads is None:
        threads = os.cpu_count() or 1
    threads = max(1, min(threads, n))

    def ptr(a, lo_):
        return a[lo_:].ctypes.data if a is not None else None

    def run(lo_, hi_):
        if hi_ <= lo_:
            return 0
        args = (fib[lo_:].ctypes.data, hi_ - lo_, cen.ctypes.data, bid.ctypes.data, m,
                thr.ctypes.data, b, float(delta),
                label[lo_:].ctypes.data, dist[lo_:].ctypes.data, dec[lo_:].ctypes.data)
        if sound:
            fn = lib.oracle_classify_sound if mode == "exact" else lib.oracle_classify_paper_sound
            return fn(*args)
        if mode == "exact":
            return lib.oracle_classify(*args, ptr(d2b, lo_))
        return lib.oracle_classify_paper(*args, ptr(d2b, lo_), ptr(lo, lo_), ptr(hi, lo_))

    # more chunks than threads: fibers differ in cost (the sound variant), so small chunks balance
    nchunk = threads if (threads == 1 or not sound) else min(n, threads * 16)
    bounds = np.linspace(0, n, nchunk + 1).astype(np.int64)
    if threads == 1:
        rcs = [run(0, n)]
    else:
        with ThreadPoolExecutor(threads) as ex:
            rcs = list(ex.map(lambda i: run(int(bounds[i]), int(bounds[i + 1])), range(nchunk)))
    if any(rcs):
        raise ValueError("oracle_classify: invalid arguments (bundle id out of range)")
    out = dict(label=label, dist=dist, decidable=dec.astype(bool))
    if want_d2b:
        out["d2b"] = d2b
    if want_bands:
        if mode == "exact":
            out["lo"] = np.sqrt(d2b)
            out["hi"] = out["lo"]
        else:
            out["lo"], out["hi"] = lo, hi
    return out


def classify_multi(fibers, centroids, bundle_id, thresh, delta: float = DELTA_MM, words: int | None = None,
                   threads: int | None = None):
    """Multi-label masks (row f4's optional half, PAPER.md:163's original DWM behaviour): bit b of
    mask[n] set iff D_b(n) <= thr_b; amb[n] marks the bits within delta of the threshold (either value is
    a correct answer there).  Returns dict(mask uint32[n, words], amb uint32[n, words])."""
    lib = _load()
    fib = _f32(fibers).reshape(-1, 21, 3)
    cen = _f32(centroids).reshape(-1, 21, 3)
    bid = np.ascontiguousarray(bundle_id, dtype=np.int32)
    thr = _f32(thresh).reshape(-1)
    n, m, b = fib.shape[0], cen.shape[0], thr.shape[0]
    words = words if words is not None else (b + 31) // 32
    mask = np.zeros((n, words), np.uint32)
    amb = np.zeros((n, words), np.uint32)
    threads = max(1, min(threads or os.cpu_count() or 1, max(n, 1)))
    bounds = np.linspace(0, n, threads + 1).astype(np.int64)

    def run(lo, hi):
        if hi <= lo:
            return 0
        return lib.oracle_classify_multi(fib[lo:].ctypes.data, hi - lo, cen.ctypes.data, bid.ctypes.data, m,
                                         thr.ctypes.data, b, float(delta), words, mask[lo:].ctypes.data,
                                         amb[lo:].ctypes.data)

    with ThreadPoolExecutor(threads) as ex:
        rcs = list(ex.map(lambda i: run(int(bounds[i]), int(bounds[i + 1])), range(threads)))
    if any(rcs):
        raise ValueError("oracle_classify_multi: invalid arguments")
    return dict(mask=mask, amb=amb)
