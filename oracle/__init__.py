"""CPU oracle for the segmentation hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  It shares no code with
paper_1912_11494_b200/ (the CUDA product path) and the product never imports it.

oracle.c holds the arithmetic (plain definition of Eq. 1-2 and Alg. 1's
closest-bundle labelling in double precision; see its header for citations).
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
            for fn in (lib.oracle_classify, lib.oracle_classify_paper):
                fn.restype = ctypes.c_int
                fn.argtypes = [
                    ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                    ctypes.c_void_p, ctypes.c_int32, ctypes.c_double,
                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
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
    """1 = inverse, 0 = direct: argmin of the end-point maxima, decided in FP32 (reading R17)."""
    a, c = _f32(a).reshape(21, 3), _f32(c).reshape(21, 3)
    return int(_load().oracle_endpoint_orientation(_fp(a), _fp(c)))


def paper_score(a, c) -> float:
    """The complete metric d_ME (inferred orientation) + TN, in mm."""
    a, c = _f32(a).reshape(21, 3), _f32(c).reshape(21, 3)
    return float(_load().oracle_paper_score(_fp(a), _fp(c)))


def classify(fibers, centroids, bundle_id, thresh, delta: float = DELTA_MM,
             threads: int | None = None, want_d2b: bool = False, mode: str = "exact"):
    """Plain-definition classification of fibers [n,21,3] against the atlas.

    mode "exact": Eq. 2 d_ME (the north_star metric); mode "paper": the paper's complete metric
    d_ME in the end-point-inferred orientation + TN (Eq. 3), SURVEY.md Sec. 8(f) row f1.
    Returns dict(label int32[n], dist float64[n], decidable bool[n][, d2b float64[n,B]]);
    in paper mode d2b holds the per-bundle minimum *score* (mm), not a squared distance.
    """
    if mode not in ("exact", "paper"):
        raise ValueError(f"unknown oracle mode {mode!r}")
    lib = _load()
    fn = lib.oracle_classify if mode == "exact" else lib.oracle_classify_paper
    fib = _f32(fibers).reshape(-1, 21, 3)
    cen = _f32(centroids).reshape(-1, 21, 3)
    bid = np.ascontiguousarray(bundle_id, dtype=np.int32)
    thr = _f32(thresh).reshape(-1)
    n, m, b = fib.shape[0], cen.shape[0], thr.shape[0]
    label = np.empty(n, np.int32)
    dist = np.empty(n, np.float64)
    dec = np.empty(n, np.uint8)
    d2b = np.empty((n, b), np.float64) if want_d2b else None
    if threads is None:
        threads = os.cpu_count() or 1
    threads = max(1, min(threads, n))

    def run(lo, hi):
        if hi <= lo:
            return 0
        return fn(
            fib[lo:].ctypes.data, hi - lo, cen.ctypes.data, bid.ctypes.data, m,
            thr.ctypes.data, b, float(delta),
            label[lo:].ctypes.data, dist[lo:].ctypes.data, dec[lo:].ctypes.data,
            d2b[lo:].ctypes.data if d2b is not None else None)

    bounds = np.linspace(0, n, threads + 1).astype(np.int64)
    if threads == 1:
        rcs = [run(0, n)]
    else:
        with ThreadPoolExecutor(threads) as ex:
            rcs = list(ex.map(lambda i: run(int(bounds[i]), int(bounds[i + 1])), range(threads)))
    if any(rcs):
        raise ValueError("oracle_classify: invalid arguments (bundle id out of range)")
    out = dict(label=label, dist=dist, decidable=dec.astype(bool))
    if d2b is not None:
        out["d2b"] = d2b
    return out
