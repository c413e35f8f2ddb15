"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/seg.h
declares, rejects bad arguments before touching CUDA, and its host-side tile plan
 satisfies the soundness invariant of the cull (row a2)."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import oracle
from paper_1912_11494_b200 import binding
from synth import atlas_for_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "seg.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(seg_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("seg_create", "seg_classify", "seg_destroy", "seg_last_error"):
        assert s in syms
    assert set(syms) == set(binding.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(binding.LIB._name)
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", binding.LIB._name], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_create_rejects_bad_arguments_without_cuda():
    at = atlas_for_config(0)
    c, b, t = at.centroids, at.bundle_id, at.thresh
    out = ctypes.c_void_p(123)
    L = binding.LIB
    assert L.seg_create(None, b.ctypes.data, at.M, t.ctypes.data, at.B, -1, ctypes.byref(out)) == binding.SEG_EINVAL
    assert out.value is None
    assert L.seg_create(c.ctypes.data, b.ctypes.data, 0, t.ctypes.data, at.B, -1, ctypes.byref(out)) == binding.SEG_EINVAL
    assert L.seg_create(c.ctypes.data, b.ctypes.data, at.M, t.ctypes.data, 0, -1, ctypes.byref(out)) == binding.SEG_EINVAL
    assert "B must be" in binding.seg_last_error()
    assert L.seg_create(c.ctypes.data, b.ctypes.data, at.M, t.ctypes.data, at.B, -1, None) == binding.SEG_EINVAL


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU error path")
def test_no_cpu_fallback_without_gpu():
    at = atlas_for_config(0)
    with pytest.raises(binding.SegError) as ei:
        binding.seg_create(at.centroids, at.bundle_id, at.M, at.thresh, at.B)
    assert ei.value.code == binding.SEG_ECUDA
    assert binding.LIB.seg_classify(None, None, 0, None, None, None) == binding.SEG_EINVAL


def test_classify_rejects_null_atlas():
    f = np.zeros((4, 21, 3), np.float32)
    lab = np.zeros(4, np.int32)
    d = np.zeros(4, np.float32)
    with pytest.raises(binding.SegError) as ei:
        binding.seg_classify(None, f, 4, lab, d)
    assert ei.value.code == binding.SEG_EINVAL


def _plan(at):
    T = binding.seg_plan_tiles(at.centroids, at.bundle_id, at.M, at.B, 0)
    tb = np.zeros(T, np.int32)
    tm = np.zeros((T, 32), np.int32)
    ts = np.zeros((T, 12), np.float32)
    assert binding.seg_plan_tiles(at.centroids, at.bundle_id, at.M, at.B, T, tb, tm, ts) == T
    return T, tb, tm, ts


@pytest.mark.parametrize("cfg", [0, 1, 3])
def test_tile_plan_partitions_the_atlas(cfg):
    at = atlas_for_config(cfg)
    T, tb, tm, _ = _plan(at)
    # every tile lies in one bundle; every centroid appears; padding repeats a member
    assert np.all(at.bundle_id[tm] == tb[:, None])
    assert np.array_equal(np.unique(tm), np.arange(at.M))
    counts = np.bincount(at.bundle_id, minlength=at.B)
    assert T == int(np.sum((counts + 31) // 32))
    assert np.all(np.diff(tb) >= 0)           # tiles grouped by ascending bundle


@pytest.mark.parametrize("cfg", [0, 1, 3])
def test_tile_spheres_bound_their_members(cfg):
    """Soundness invariant of row a2: the spheres of points 0/10/20 contain every member
    (in one consistent orientation per member -- the library may store a centroid
    reversed, which Eq. 2 is invariant to)."""
    at = atlas_for_config(cfg)
    T, tb, tm, ts = _plan(at)
    c = at.centroids.astype(np.float64)[tm]                       # [T, 32, 21, 3]
    S = ts.astype(np.float64).reshape(T, 3, 4)
    def inside(pts, s):
        return np.linalg.norm(pts - s[:, None, :3], axis=-1) <= s[:, None, 3]
    in10 = inside(c[:, :, 10], S[:, 1])
    fwd = inside(c[:, :, 0], S[:, 0]) & inside(c[:, :, 20], S[:, 2])
    rev = inside(c[:, :, 20], S[:, 0]) & inside(c[:, :, 0], S[:, 2])
    assert np.all(in10)
    assert np.all(fwd | rev)


def test_tile_bound_is_a_lower_bound_of_dme():
    """The cull's inequality, evaluated in double on random fibers: whenever the sphere
    bound of a tile exceeds a distance s, every member's d_ME (oracle) exceeds s."""
    at = atlas_for_config(0)
    T, tb, tm, ts = _plan(at)
    rng = np.random.default_rng(7)
    from synth import fibers_for_config
    fib = fibers_for_config(0, 0, 60).astype(np.float64)
    S = ts.astype(np.float64).reshape(T, 3, 4)
    checked = 0
    for f in fib:
        for t in rng.choice(T, 6, replace=False):
            d = lambda p, k: np.linalg.norm(f[p] - S[t, k, :3]) - S[t, k, 3]
            lb = max(d(10, 1), min(max(d(0, 0), d(20, 2)), max(d(0, 2), d(20, 0))))
            true = min(oracle.d_me(f.astype(np.float32), at.centroids[m]) for m in tm[t])
            assert true >= lb - 1e-9
            checked += 1
    assert checked == 360


def test_new_entry_points_reject_bad_arguments_without_cuda():
    """Rows f1-f4 argument checks that fire before any CUDA call."""
    at = atlas_for_config(0)
    c, b, t = at.centroids, at.bundle_id, at.thresh
    out = ctypes.c_void_p(123)
    L = binding.LIB
    assert L.seg_create_ex(c.ctypes.data, b.ctypes.data, at.M, t.ctypes.data, at.B, -1, 0x10,
                           ctypes.byref(out)) == binding.SEG_EINVAL
    assert "flags" in binding.seg_last_error() and out.value is None
    assert L.seg_group_by_bundle(None, None, 10, 0, None, None, None, None, None, None) == binding.SEG_EINVAL
    assert L.seg_group_by_bundle(None, None, 10, 4096, None, None, None, None, None, None) == binding.SEG_EINVAL
    assert L.seg_group_by_bundle(None, None, -1, 5, None, None, None, None, None, None) == binding.SEG_EINVAL
    assert L.seg_resample(None, None, -1, None, None) == binding.SEG_EINVAL
    assert L.seg_resample(None, None, 5, None, None) == binding.SEG_EINVAL
    assert L.seg_resample(None, None, 0, None, None) == binding.SEG_OK        # N = 0: no-op
    assert L.seg_keys_to_labels(None, 5, 7, None, None, None) == binding.SEG_EINVAL   # unknown mode
    assert L.seg_classify_keys(None, None, 5, None, None) == binding.SEG_EINVAL       # null atlas


def test_seg_lib_override_fails_loudly():
    """SEG_LIB (the checked build, scripts/checked_build.sh) must name an existing library: a missing
    one is an ImportError, never a silent fallback to another build or to the CPU."""
    import subprocess, sys
    env = dict(os.environ, SEG_LIB="/nonexistent/libsegb200.so")
    r = subprocess.run([sys.executable, "-c", "import paper_1912_11494_b200.binding"], env=env,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       capture_output=True, text=True)
    assert r.returncode != 0 and "SEG_LIB" in r.stderr
