"""A/B timing of library builds on one config: python scripts/ab.py CFG lib1.so lib2.so ..."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import atlas_for_config, fibers_for_config
cfg = int(sys.argv[1])
at = atlas_for_config(cfg)
fib = torch.from_numpy(fibers_for_config(cfg)).cuda()
N = fib.shape[0]
lab = torch.empty(N, dtype=torch.int32, device="cuda"); d = torch.empty(N, dtype=torch.float32, device="cuda")
c, b, t = (torch.from_numpy(x).cuda() for x in (at.centroids, at.bundle_id, at.thresh))
res, ref = {}, None
for rep in range(2):
    for path in sys.argv[2:]:
        L = ctypes.CDLL(os.path.abspath(path)); vp = ctypes.c_void_p
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
        res.setdefault(path, []).append(e0.elapsed_time(e1) / 10)
        out = (lab.clone(), d.clone())
        if ref is None: ref = out
        same = torch.equal(ref[0], out[0]) and torch.equal(ref[1].view(torch.int32), out[1].view(torch.int32))
        if not same: print(f"WARNING {path}: results differ from {sys.argv[2]}")
for path, v in res.items():
    print(f"cfg{cfg} {path}: " + " ".join(f"{x:.3f}" for x in v) + " ms")
