"""B200-native hot path of atlas-based white-matter fiber segmentation (arXiv 1912.11494).

    from paper_1912_11494_b200 import Atlas
    atlas = Atlas(centroids, bundle_id, thresh)      # float32 [M,21,3], int32 [M], float32 [B]
    label, dist = atlas.classify(fibers)             # float32 [N,21,3] torch CUDA tensor

`binding` is the 1:1 ctypes binding of include/seg.h; `Atlas` only checks dtypes and
shapes and passes raw pointers.  `dist` holds the multi-GPU driver.
"""
from __future__ import annotations

import numpy as np

from . import binding
from .binding import SegError, STAT_NAMES  # noqa: F401

__all__ = ["Atlas", "SegError", "binding", "group_by_bundle", "keys_to_labels", "resample"]


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _check_array(x, dtype_np, shape_tail, name):
    if _is_torch(x):
        import torch
        want = {np.float32: torch.float32, np.int32: torch.int32}[dtype_np]
        if x.dtype != want:
            raise TypeError(f"{name}: dtype {x.dtype}, expected {want}")
        if not x.is_contiguous():
            raise ValueError(f"{name}: must be contiguous")
    else:
        if not isinstance(x, np.ndarray):
            raise TypeError(f"{name}: expected a torch tensor or numpy array")
        if x.dtype != dtype_np:
            raise TypeError(f"{name}: dtype {x.dtype}, expected {np.dtype(dtype_np)}")
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError(f"{name}: must be C-contiguous")
    if tuple(x.shape[1:]) != tuple(shape_tail):
        raise ValueError(f"{name}: shape {tuple(x.shape)}, expected [*, {', '.join(map(str, shape_tail))}]")


class Atlas:
    """An immutable atlas on one CUDA device (seg_create / seg_destroy)."""

    MODES = {"exact": binding.SEG_MODE_EXACT, "paper": binding.SEG_MODE_PAPER}

    def __init__(self, centroids, bundle_id, thresh, device: int = -1, mode: str = "exact"):
        """mode "exact": Eq. 2 d_ME (the north_star metric); "paper": the paper's final classifier,
        d_ME in the end-point-inferred orientation + TN (Eq. 3), see include/seg.h SEG_MODE_PAPER."""
        if mode not in self.MODES:
            raise ValueError(f"mode must be one of {sorted(self.MODES)}")
        self.mode = mode
        _check_array(centroids, np.float32, (21, 3), "centroids")
        _check_array(bundle_id, np.int32, (), "bundle_id")
        _check_array(thresh, np.float32, (), "thresh")
        if bundle_id.shape[0] != centroids.shape[0]:
            raise ValueError("bundle_id and centroids disagree on M")
        self.M = int(centroids.shape[0])
        self.B = int(thresh.shape[0])
        self._h = binding.seg_create_ex(centroids, bundle_id, self.M, thresh, self.B, device, self.MODES[mode])
        self.info = binding.seg_get_atlas_info(self._h)
        self.device = self.info["device"]

    @property
    def handle(self) -> int:
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None):
            binding.seg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _outputs(self, fibers, label, dist):
        n = int(fibers.shape[0])
        if _is_torch(fibers):
            import torch
            if label is None:
                label = torch.empty(n, dtype=torch.int32, device=fibers.device)
            if dist is None:
                dist = torch.empty(n, dtype=torch.float32, device=fibers.device)
        else:
            if label is None:
                label = np.empty(n, np.int32)
            if dist is None:
                dist = np.empty(n, np.float32)
        _check_array(label, np.int32, (), "label")
        _check_array(dist, np.float32, (), "dist")
        if label.shape[0] != n or dist.shape[0] != n:
            raise ValueError("label/dist length must equal the number of fibers")
        return n, label, dist

    @staticmethod
    def _stream(fibers, stream):
        if stream is not None:
            return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)
        if _is_torch(fibers) and fibers.is_cuda:
            import torch
            return int(torch.cuda.current_stream(fibers.device).cuda_stream)
        return None

    def classify(self, fibers, label=None, dist=None, stream=None):
        """Label fibers [N,21,3] float32 -> (label int32[N], dist float32[N]).

        CUDA tensors: asynchronous on `stream` (default: torch's current stream).
        Host arrays/tensors: streamed through the device; returns when results are on the host.
        """
        _check_array(fibers, np.float32, (21, 3), "fibers")
        n, label, dist = self._outputs(fibers, label, dist)
        binding.seg_classify(self._h, fibers, n, label, dist, self._stream(fibers, stream))
        return label, dist

    def classify_stats(self, fibers, label=None, dist=None, stream=None):
        """classify() through the counting kernel; returns (label, dist, {counter: value})."""
        _check_array(fibers, np.float32, (21, 3), "fibers")
        n, label, dist = self._outputs(fibers, label, dist)
        stats = np.zeros(binding.SEG_NSTATS, np.uint64)
        binding.seg_classify_stats(self._h, fibers, n, label, dist, stats, self._stream(fibers, stream))
        return label, dist, dict(zip(binding.STAT_NAMES, (int(v) for v in stats)))

    def classify_keys(self, fibers, keys=None, stream=None):
        """Row f4: each fiber's best key over this atlas (seg_classify_keys), int64 CUDA tensor [N].

        The element-wise minimum of the keys of several atlas shards is the key of their union
        (see include/seg.h); keys_to_labels() decodes it.
        """
        import torch
        _check_array(fibers, np.float32, (21, 3), "fibers")
        if not (_is_torch(fibers) and fibers.is_cuda):
            raise TypeError("fibers: classify_keys takes CUDA tensors")
        n = int(fibers.shape[0])
        if keys is None:
            keys = torch.empty(n, dtype=torch.int64, device=fibers.device)
        binding.seg_classify_keys(self._h, fibers, n, keys, self._stream(fibers, stream))
        return keys


    def classify_multi(self, fibers, masks=None, stream=None):
        """Row f4's optional half (seg_classify_multi): every bundle within threshold, the original DWM
        assignment.  Returns int32 CUDA tensor [N, ceil(B/32)] of bit masks (bit b of word
        b // 32 = bundle b); exact-mode atlases with B <= 128."""
        import torch
        _check_array(fibers, np.float32, (21, 3), "fibers")
        if not (_is_torch(fibers) and fibers.is_cuda):
            raise TypeError("fibers: classify_multi takes CUDA tensors")
        n, words = int(fibers.shape[0]), (self.B + 31) // 32
        if masks is None:
            masks = torch.empty((n, words), dtype=torch.int32, device=fibers.device)
        binding.seg_classify_multi(self._h, fibers, n, masks, int(masks.shape[1]), self._stream(fibers, stream))
        return masks


def group_by_bundle(label, dist, B: int, stream=None):
    """Row f3: the segmented bundles of a classified subject (seg_group_by_bundle).

    label int32 [N] / dist float32 [N] (torch CUDA tensors, e.g. Atlas.classify's outputs; dist may
    be None).  Returns (order int32 [N], offsets int64 [B+2], dmin float32 [B], dmax float32 [B],
    dsum float64 [B]) on the same device: bundle b's fibers are order[offsets[b]:offsets[b+1]] in
    increasing index, the unassigned ones order[offsets[B]:]; the summaries are None without dist.
    """
    import torch
    if not _is_torch(label) or label.dtype != torch.int32 or not label.is_cuda or label.dim() != 1:
        raise TypeError("label: expected a 1-D int32 CUDA tensor")
    if dist is not None and (dist.dtype != torch.float32 or dist.shape != label.shape or dist.device != label.device):
        raise TypeError("dist: expected a float32 CUDA tensor shaped like label")
    label = label.contiguous()
    dist = dist.contiguous() if dist is not None else None
    n, dev = int(label.shape[0]), label.device
    order = torch.empty(n, dtype=torch.int32, device=dev)
    offsets = torch.empty(B + 2, dtype=torch.int64, device=dev)
    dmin = dmax = dsum = None
    if dist is not None:
        dmin = torch.empty(B, dtype=torch.float32, device=dev)
        dmax = torch.empty(B, dtype=torch.float32, device=dev)
        dsum = torch.empty(B, dtype=torch.float64, device=dev)
    if stream is None:
        stream = torch.cuda.current_stream(dev).cuda_stream
    binding.seg_group_by_bundle(label, dist if n else None, n, B, order, offsets, dmin, dmax, dsum, stream)
    return order, offsets, dmin, dmax, dsum


def resample(points, offsets, stream=None):
    """Row f2: raw streamlines -> [N, 21, 3] float32 fibers (seg_resample).

    points float32 [P, 3] and offsets int64 [N + 1] (CSR: fiber f = points[offsets[f]:offsets[f+1]]),
    torch CUDA tensors on one device.  Invalid fibers (< 2 points, zero length) come out as NaN.
    """
    import torch
    if not (_is_torch(points) and points.is_cuda and points.dtype == torch.float32 and points.dim() == 2
            and points.shape[1] == 3):
        raise TypeError("points: expected a float32 CUDA tensor [P, 3]")
    if not (_is_torch(offsets) and offsets.is_cuda and offsets.dtype == torch.int64 and offsets.dim() == 1):
        raise TypeError("offsets: expected an int64 CUDA tensor [N + 1]")
    points, offsets = points.contiguous(), offsets.contiguous()
    n = int(offsets.shape[0]) - 1
    out = torch.empty((max(n, 0), 21, 3), dtype=torch.float32, device=points.device)
    if stream is None:
        stream = torch.cuda.current_stream(points.device).cuda_stream
    binding.seg_resample(points, offsets, max(n, 0), out, stream)
    return out


def keys_to_labels(keys, mode: str = "exact", stream=None):
    """Row f4: decode best keys (Atlas.classify_keys, possibly min-reduced over atlas shards) into
    (label int32 [N], dist float32 [N]) exactly as seg_classify writes them (seg_keys_to_labels)."""
    import torch
    if not (_is_torch(keys) and keys.is_cuda and keys.dtype == torch.int64 and keys.dim() == 1):
        raise TypeError("keys: expected a 1-D int64 CUDA tensor")
    keys = keys.contiguous()
    n = int(keys.shape[0])
    label = torch.empty(n, dtype=torch.int32, device=keys.device)
    dist = torch.empty(n, dtype=torch.float32, device=keys.device)
    if stream is None:
        stream = torch.cuda.current_stream(keys.device).cuda_stream
    binding.seg_keys_to_labels(keys, n, Atlas.MODES[mode], label, dist, stream)
    return label, dist

