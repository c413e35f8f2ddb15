"""A/B of the host-buffer pipeline (seg_classify with pinned host buffers) across library builds with extra
nvcc defines, interleaved on one box: python scripts/ab_e2e.py CFG "" "-DX" ...  Prints ms per call."""
import ctypes, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1912_11494_b200 import _build
from synth import atlas_for_config, fibers_for_config

cfg = int(sys.argv[1])
defs = sys.argv[2:] or [""]
os.makedirs("build/ab", exist_ok=True)
at = atlas_for_config(cfg)
fib = torch.from_numpy(fibers_for_config(cfg)).pin_memory()
N = fib.shape[0]
lab = torch.empty(N, dtype=torch.int32).pin_memory()
dd = torch.empty(N, dtype=torch.float32).pin_memory()
c, b, t = (torch.from_numpy(x).cuda() for x in (at.centroids, at.bundle_id, at.thresh))
libs = []
for k, d in enumerate(defs):
    out = os.path.abspath(f"build/ab/libe{k}.so")
    subprocess.check_call([_build.nvcc(), *_build.NVCC_FLAGS, *d.split(), "-o", out, *_build.SOURCES],
                          stderr=subprocess.DEVNULL)
    L = ctypes.CDLL(out)
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
    L.seg_create.argtypes = [vp, vp, i64, vp, i32, ctypes.c_int, ctypes.POINTER(vp)]
    L.seg_classify.argtypes = [vp, vp, i64, vp, vp, vp]
    h = vp()
    assert L.seg_create(c.data_ptr(), b.data_ptr(), at.M, t.data_ptr(), at.B, -1, ctypes.byref(h)) == 0
    libs.append((d, L, h))
st = torch.cuda.current_stream().cuda_stream
res = {d: [] for d in defs}
ref = None
for rep in range(6):
    for d, L, h in libs:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        assert L.seg_classify(h, fib.data_ptr(), N, lab.data_ptr(), dd.data_ptr(), st) == 0
        t1 = time.perf_counter()
        if rep:
            res[d].append((t1 - t0) * 1e3)
        if ref is None:
            ref = (lab.clone(), dd.clone())
        else:
            assert torch.equal(ref[0], lab) and torch.equal(ref[1].view(torch.int32), dd.view(torch.int32))
dev = torch.empty_like(fib, device="cuda")
hv = []
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev.copy_(fib, non_blocking=True)
    torch.cuda.synchronize()
    hv.append((time.perf_counter() - t0) * 1e3)
print(f"cfg{cfg} pure H2D of the fibers ({fib.numel() * 4 / 1e9:.3f} GB): median {np.median(hv[1:]):.3f} ms", flush=True)
for d in defs:
    v = np.array(res[d])
    print(f"cfg{cfg} e2e [{d or 'production'}] median {np.median(v):.3f} ms  min {v.min():.3f}  (n={len(v)})", flush=True)
