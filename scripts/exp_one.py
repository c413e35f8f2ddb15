"""Run seg_classify from a given library build a few times (for ncu on experiment builds)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import atlas_for_config, fibers_for_config
path, cfg, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
at = atlas_for_config(cfg)
fib = torch.from_numpy(fibers_for_config(cfg)).cuda()
N = fib.shape[0]
lab = torch.empty(N, dtype=torch.int32, device="cuda"); d = torch.empty(N, dtype=torch.float32, device="cuda")
c, b, t = (torch.from_numpy(x).cuda() for x in (at.centroids, at.bundle_id, at.thresh))
L = ctypes.CDLL(os.path.abspath(path)); vp = ctypes.c_void_p
L.seg_create.argtypes = [vp, vp, ctypes.c_int64, vp, ctypes.c_int32, ctypes.c_int, ctypes.POINTER(vp)]
L.seg_classify.argtypes = [vp, vp, ctypes.c_int64, vp, vp, vp]
h = vp()
assert L.seg_create(c.data_ptr(), b.data_ptr(), at.M, t.data_ptr(), at.B, -1, ctypes.byref(h)) == 0
for _ in range(reps):
    assert L.seg_classify(h, fib.data_ptr(), N, lab.data_ptr(), d.data_ptr(), torch.cuda.current_stream().cuda_stream) == 0
torch.cuda.synchronize()
print("ok")
