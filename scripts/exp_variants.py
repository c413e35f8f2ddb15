"""Timing experiments on instrumented builds of the library (results of variants are NOT valid
classifications; only the timing is of interest).  Builds build/exp/libseg_exp{1,2}.so with
-DSEG_EXP=k and times seg_classify on a config against the production build."""
import ctypes, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1912_11494_b200 import _build, Atlas
from synth import atlas_for_config, fibers_for_config

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
variants = {0: _build.LIB}
os.makedirs("build/exp", exist_ok=True)
for k in (1, 2, 3):
    out = f"build/exp/libseg_exp{k}.so"
    subprocess.check_call([_build.nvcc(), *_build.NVCC_FLAGS, f"-DSEG_EXP={k}", "-o", out, *_build.SOURCES],
                          stderr=subprocess.DEVNULL)
    variants[k] = out
at = atlas_for_config(cfg)
fib = torch.from_numpy(fibers_for_config(cfg)).cuda()
N = fib.shape[0]
lab = torch.empty(N, dtype=torch.int32, device="cuda"); d = torch.empty(N, dtype=torch.float32, device="cuda")
c, b, t = (torch.from_numpy(x).cuda() for x in (at.centroids, at.bundle_id, at.thresh))
for k, path in variants.items():
    L = ctypes.CDLL(os.path.abspath(path))
    vp = ctypes.c_void_p
    L.seg_create.argtypes = [vp, vp, ctypes.c_int64, vp, ctypes.c_int32, ctypes.c_int, ctypes.POINTER(vp)]
    L.seg_classify.argtypes = [vp, vp, ctypes.c_int64, vp, vp, vp]
    h = vp()
    assert L.seg_create(c.data_ptr(), b.data_ptr(), at.M, t.data_ptr(), at.B, -1, ctypes.byref(h)) == 0
    st = torch.cuda.current_stream().cuda_stream
    f = lambda: L.seg_classify(h, fib.data_ptr(), N, lab.data_ptr(), d.data_ptr(), st)
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    print(f"cfg{cfg} variant {k}: {e0.elapsed_time(e1)/10:.3f} ms  ({['production','tile-loop only','no candidate rounds','dense only (no hit processing)'][k]})")
