"""A/B timing of library builds with extra nvcc defines: python scripts/ab_build.py CFG "-DX" "-DY" ...
(the empty string = production; "lib:PATH" = a prebuilt library).  AB_MODE=paper: paper-semantics atlases.  Prints the per-kernel event times from seg_profile_read."""
import ctypes, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1912_11494_b200 import _build
from synth import atlas_for_config, fibers_for_config

cfg = int(sys.argv[1])
defs = sys.argv[2:] or [""]
os.makedirs("build/ab", exist_ok=True)
at = atlas_for_config(cfg)
fib = torch.from_numpy(fibers_for_config(cfg)).cuda()
N = fib.shape[0]
c, b, t = (torch.from_numpy(x).cuda() for x in (at.centroids, at.bundle_id, at.thresh))
ref = None
for k, d in enumerate(defs):
    if d.startswith("lib:"):   # a prebuilt library (e.g. the previous commit's, built here before the call)
        out = os.path.abspath(d[4:])
    else:
        out = os.path.abspath(f"build/ab/lib{k}.so")
        subprocess.check_call([_build.nvcc(), *_build.NVCC_FLAGS, *d.split(), "-o", out, *_build.SOURCES],
                              stderr=subprocess.DEVNULL)
    L = ctypes.CDLL(out)
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
    L.seg_create.argtypes = [vp, vp, i64, vp, i32, ctypes.c_int, ctypes.POINTER(vp)]
    L.seg_create_ex.argtypes = [vp, vp, i64, vp, i32, ctypes.c_int, ctypes.c_uint32, ctypes.POINTER(vp)]
    L.seg_classify.argtypes = [vp, vp, i64, vp, vp, vp]
    L.seg_profile_enable.argtypes = [vp, i32]
    L.seg_profile_read.argtypes = [vp, vp, vp, vp, i32, ctypes.POINTER(i32)]
    h = vp()
    flags = 1 if os.environ.get("AB_MODE") == "paper" else 0   # SEG_MODE_PAPER
    assert L.seg_create_ex(c.data_ptr(), b.data_ptr(), at.M, t.data_ptr(), at.B, -1, flags, ctypes.byref(h)) == 0
    lab = torch.empty(N, dtype=torch.int32, device="cuda"); dd = torch.empty(N, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        L.seg_classify(h, fib.data_ptr(), N, lab.data_ptr(), dd.data_ptr(), st)
    R = 10
    L.seg_profile_enable(h, R)
    for _ in range(R):
        L.seg_classify(h, fib.data_ptr(), N, lab.data_ptr(), dd.data_ptr(), st)
    pre, cul, cls = (np.zeros(R, np.float32) for _ in range(3))
    cnt = ctypes.c_int32()
    L.seg_profile_read(h, pre.ctypes.data, cul.ctypes.data, cls.ctypes.data, R, ctypes.byref(cnt))
    same = None
    if ref is None:
        ref = (lab.clone(), dd.clone())
    else:
        same = bool(torch.equal(ref[0], lab)) and bool(torch.equal(ref[1].view(torch.int32), dd.view(torch.int32)))
    print(f"cfg{cfg} [{d or 'production'}] prepass {pre.mean():.3f} cull {cul.mean():.3f} classify {cls.mean():.3f} "
          f"total {pre.mean() + cul.mean() + cls.mean():.3f} ms  same_as_first={same}", flush=True)
