#!/usr/bin/env python
"""Benchmark of the segmentation hot path on B200 (BASELINE.json metric and config).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--mode exact|paper]
                    [--scaling strong|weak] [--impl reference]

One step = one pass of the whole hot path (all rows a1-a9 of SURVEY.md Sec. 8(a)) over one subject:
config 3 by default, 4,145,000 synthetic fibers x the 62-bundle / 44,345-centroid atlas
(BASELINE.json configs[3]; seeded synthetic stand-ins).  Inputs are resident in HBM
when the timed region starts; they are 1.04 GB (> 126 MB L2), so no L2 flush is needed between steps.

Multi-GPU (under torchrun; the north_star partition): ONE subject sharded
contiguously over the ranks (dist.shard_range, boundaries multiples of 4 fibers), the atlas broadcast
from rank 0 over NCCL at setup, and every step = each rank's seg_classify of its shard + the
all_gather of the packed (label, dist) results (dist.classify_sharded, C2) -- "scaling": "strong".
--scaling weak gives every rank its own full-size subject instead (no gather).  Timing: barrier +
synchronize on both sides, CUDA events on the launching stream, max over ranks.

e2e: the same metric through the public API with host buffers: at N=1 the library's pipelined
host-buffer path (pinned H2D -> classify -> D2H, seg_classify with host pointers); at N>1 each rank's
own pinned H2D of its shard, the classification and the all_gather, then rank 0's D2H of the whole
subject's results.

--impl reference times the CPU oracle (oracle/, C, double; the sound-discard variant, which is Alg. 1's
own cascade and returns bitwise the plain definition's labels) on the box's host cores on a bounded
seeded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fiber–centroid comparisons/sec"
UNIT = "comparisons/s"
FP32_LANES_PER_SM = 128          # B200 SM: 4 SMSPs x 32 FP32 lanes (B200_PROFILING.md / guide)
FP32_INSTR_PER_PDIST = 6         # Eq. 1 squared: 3 FADD + 1 FMUL + 2 FFMA
# per-fiber algorithmic FP32 work under the tightest exact pruning the survey assumed
# (≈ 2.5 k / 14.8 k / 18.4 k lane-instructions per fiber, configs 1/3/4).  Fixed per config, so unlike the
# measured-W fraction it does not fall when a better bound prunes more work.
SURVEY_INSTR_PER_FIBER = {1: 2.5e3, 3: 14.8e3, 4: 18.4e3}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--mode", choices=["exact", "paper"], default="exact",
                    help="exact: Eq. 2 d_ME (north_star, default); paper: d_ME (inferred orientation) + TN, row f1")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="strong: one subject sharded over the ranks (north_star); weak: one subject per rank")
    ap.add_argument("--gather", choices=["nccl", "p2p"], default="nccl",
                    help="strong scaling, N>1: NCCL all_gather of the results, or the fused gather (each rank's "
                         "kernel epilogue stores into rank 0's buffer over NVLink, dist.PeerResults)")
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU time of the oracle sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-stats", action="store_true")
    return ap.parse_args()


def workload_name(cfg, mode="exact"):
    from synth import CONFIGS
    c = CONFIGS[cfg]
    return (f"cfg{cfg}: {c['n_fibers']:,} fibers x {c['n_centroids']:,} centroids "
            f"({c['n_bundles']} bundles), 21 pts, synthetic"
            + ("" if mode == "exact" else ", paper-semantics score (d_ME inferred orientation + TN)"))


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ------------------------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline leg and --impl reference)
# ------------------------------------------------------------------------------------------
def time_oracle(cfg, fib, at, target_s, mode="exact", seed=78):
    """The sound-discard oracle (Alg. 1's cascade, bitwise the plain definition's labels) on all host
    cores over a seeded sample sized for ~target_s, scaled to comparisons/s (fibers are i.i.d.)."""
    import oracle
    from synth import sample_indices
    threads = os.cpu_count() or 1
    cal = fib[sample_indices(fib.shape[0], max(threads * 8, 64), seed=77)]
    t0 = time.perf_counter()
    oracle.classify(cal, at.centroids, at.bundle_id, at.thresh, threads=threads, mode=mode, sound=True)
    dt = max(time.perf_counter() - t0, 1e-3)
    per_fiber = dt / cal.shape[0]
    k = int(max(threads * 8, min(fib.shape[0], target_s / per_fiber)))
    idx = sample_indices(fib.shape[0], k, seed=seed)
    sub = fib[idx]
    t0 = time.perf_counter()
    oracle.classify(sub, at.centroids, at.bundle_id, at.thresh, threads=threads, mode=mode, sound=True)
    dt = time.perf_counter() - t0
    n = sub.shape[0]
    pct = 100.0 * n / fib.shape[0]
    label = ("full size" if n == fib.shape[0] else
             f"extrapolated x{fib.shape[0] / n:.1f} from a {pct:.2f}% seeded subsample (synth.sample_indices seed {seed})")
    return dict(value=n * at.M / dt, unit=UNIT, cores=threads, kind="oracle",
                fibers_per_s=n / dt, seconds=dt, cpu_model=cpu_model(),
                sample=f"{n:,} of the {fib.shape[0]:,} fibers of {workload_name(cfg, mode)} against the full atlas, "
                       f"{label}; sound-discard oracle (oracle_classify_sound: Alg. 1 cascade in fp64, cut at "
                       f"thr + 2e-3 mm; bitwise the plain definition's labels), {threads} host threads")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from synth import atlas_for_config, fibers_for_config
    at = atlas_for_config(args.config)
    fib = fibers_for_config(args.config)
    vals = []
    budget = max(2.0, args.cpu_seconds / max(1, args.steps + args.warmup))
    for i in range(args.warmup + args.steps):
        r = time_oracle(args.config, fib, at, budget, args.mode, seed=78 + i)
        if i >= args.warmup:
            vals.append(r)
    v = statistics.median([r["value"] for r in vals])
    line = dict(impl="reference", metric=METRIC, value=v, unit=UNIT, n_gpus=args.gpus, steps=args.steps,
                warmup=args.warmup, ms_per_step=1e3 * statistics.median([r["seconds"] for r in vals]),
                higher_is_better=True, scaling=args.scaling, vs_baseline=None, dtype="f64", data="synthetic",
                config=dict(workload=workload_name(args.config, args.mode), sample=vals[-1]["sample"]),
                fibers_per_s=statistics.median([r["fibers_per_s"] for r in vals]),
                cpu_baseline=dict(value=v, unit=UNIT, cores=vals[-1]["cores"], kind="oracle",
                                  sample=vals[-1]["sample"], cpu_model=vals[-1]["cpu_model"]),
                e2e=dict(value=v, unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0),
                gpu_launches=0)
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------
# clocks during the timed region (NVML, 10 ms period)
# ------------------------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x0000000000000001: "gpu_idle", 0x0000000000000002: "applications_clocks_setting",
        0x0000000000000004: "sw_power_cap", 0x0000000000000008: "hw_slowdown",
        0x0000000000000010: "sync_boost", 0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown", 0x0000000000000080: "hw_power_brake_slowdown",
        0x0000000000000100: "display_clock_setting",
    }

    def __init__(self, dev_index):
        self.samples, self.reasons, self.stop_ev = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv = None
            self.err = str(e)

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return dict(sm_mhz=None, sm_max_mhz=self.max_mhz, reasons=sorted(self.reasons), samples=0)
        return dict(sm_mhz=float(statistics.median(self.samples)), sm_max_mhz=self.max_mhz,
                    reasons=sorted(self.reasons), samples=len(self.samples))


def probe_peak():
    """The committed FP32 peak probe (scripts/probes/fp32_peak.cu, profiles/r02/fp32_peak.txt), if any."""
    p = os.path.join(ROOT, "profiles", "fp32_peak.json")
    try:
        return json.load(open(p))
    except Exception:
        return None


def traffic_record(cfg, mode):
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(tf)).get(f"cfg{cfg}_{mode}")
    except Exception:
        return None


# ------------------------------------------------------------------------------------------
# B200 arm
# ------------------------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SEG_BENCH_ONE_DEVICE=1 + SEG_BENCH_BACKEND=gloo: a functional check of the multi-rank code path with every
    # rank on cuda:0 (no rank waits on another's kernel; the collectives run on the host).  Not a timing
    # configuration: the driver's runs use one GPU per rank and NCCL.
    local_dev = 0 if os.environ.get("SEG_BENCH_ONE_DEVICE") == "1" else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        backend = os.environ.get("SEG_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    from paper_1912_11494_b200 import Atlas, binding
    from paper_1912_11494_b200.dist import (PeerResults, broadcast_atlas, classify_sharded, classify_sharded_p2p,
                                            shard_range)
    from synth import CONFIGS, atlas_for_config, fibers_for_config

    cfg = args.config
    spec = CONFIGS[cfg]
    strong = args.scaling == "strong"
    # atlas: rank 0 generates, NCCL broadcast to the others (setup, untimed)
    at = atlas_for_config(cfg) if rank == 0 else None
    cents, bid, thr = broadcast_atlas(at, spec["n_centroids"], spec["n_bundles"], dev, world)
    atlas = Atlas(cents, bid, thr, mode=args.mode)
    # this rank's fibers: strong -> its contiguous shard of subject 0; weak -> its own full subject r
    workers = max(1, (os.cpu_count() or 1) // world)
    t0 = time.perf_counter()
    n_total = spec["n_fibers"]
    if strong:
        lo, hi = shard_range(n_total, world, rank)
        fib_np = fibers_for_config(cfg, lo, hi, workers=workers)
    else:
        lo, hi = 0, n_total
        fib_np = fibers_for_config(cfg, subject=rank, workers=workers)
    gen_s = time.perf_counter() - t0
    N = fib_np.shape[0]                       # this rank's fibers
    n_job = n_total if strong else n_total * world
    fib = torch.from_numpy(fib_np).to(dev)
    lab = torch.empty(N, dtype=torch.int32, device=dev)
    dst = torch.empty(N, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def classify_into(f, lb=None, ds=None):
        return atlas.classify(f, lb if lb is not None else lab, ds if ds is not None else dst)

    peer = PeerResults(n_total, world, rank, dev) if (strong and world > 1 and args.gather == "p2p") else None

    def step():
        if peer is not None:                                   # fused gather: epilogue stores into rank 0
            return classify_sharded_p2p(atlas.classify, fib, peer)
        if strong and world > 1:
            return classify_sharded(lambda f: classify_into(f), fib, n_total, world, rank)   # + all_gather (C2)
        return classify_into(fib)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    # ---------------- timed region: K steps ----------------
    # inputs smaller than 2x L2 (configs 0-2): every step is timed alone with an L2 flush (a 256 MB write)
    # between steps, outside its events; larger inputs (configs 3-4) stream from HBM anyway
    flush = n_job * 252 < 2 * 126e6
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None
    binding.seg_profile_enable(atlas.handle, args.steps)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)] \
        if flush else []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local_dev) as clk:
        ev0.record(stream)
        for i in range(args.steps):
            if flush:
                scratch.zero_()
                evs[i][0].record(stream)
            out = step()
            if flush:
                evs[i][1].record(stream)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms_total = sum(a.elapsed_time(b) for a, b in evs) if flush else ev0.elapsed_time(ev1)
    pre = np.zeros(args.steps, np.float32)
    cul = np.zeros(args.steps, np.float32)
    cls = np.zeros(args.steps, np.float32)
    binding.seg_profile_read(atlas.handle, pre, cul, cls, args.steps)
    binding.seg_profile_enable(atlas.handle, 0)
    t = torch.tensor([ms_total, float(cls.mean()), float(pre.mean()), float(cul.mean())], dtype=torch.float64,
                     device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total, cls_ms, pre_ms, cull_ms = t.tolist()
    ms_step = ms_total / args.steps
    pairs = float(n_job) * spec["n_centroids"]
    value = pairs / (ms_step * 1e-3)
    fibers_per_s = n_job / (ms_step * 1e-3)
    clocks = clk.summary()
    # hist, scan_blocks, scan_totals, scatter (N >= 4096), cull, cta_order (grids of <= 64 waves), classify
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    launches_per_step = (4 if N >= 4096 else 0) + 2 + (1 if -(-N // 256) <= 64 * 2 * sms else 0)
    res_lab = out[0].cpu().numpy() if isinstance(out, tuple) else lab.cpu().numpy()

    # ---------------- stage counters + roofline of the dominant kernel ----------------
    roofline, st = None, None
    sm_mhz = clocks["sm_mhz"] or clocks["sm_max_mhz"] or 1965.0
    peak = sms * FP32_LANES_PER_SM * sm_mhz * 1e6 / 1e12
    if not args.no_stats:
        _, _, st = atlas.classify_stats(fib)
        torch.cuda.synchronize(dev)
        w_instr = FP32_INSTR_PER_PDIST * st["lane_point_dists"]          # algorithmic FP32 lane-instr
        achieved = w_instr / (cls_ms * 1e-3) / 1e12                      # T lane-instr / s
        tr = traffic_record(cfg, args.mode)
        probe = probe_peak()
        roofline = dict(bound="alu", achieved=achieved, peak=peak, unit="Tinstr/s (FP32 lane-instr)",
                        frac=achieved / peak,
                        traffic=tr["bytes"] if tr else None, traffic_unit="DRAM bytes per k_classify launch",
                        traffic_source=tr["source"] if tr else None,
                        kernel="k_classify (timed by the library's profile events on its stream)",
                        kernel_ms=cls_ms, cull_ms=cull_ms, prepass_ms=pre_ms,
                        peak_basis=f"nominal: {sms} SMs x {FP32_LANES_PER_SM} FP32 lanes x {sm_mhz:.0f} MHz "
                                   f"(median SM clock during the timed region; B200_PROFILING.md unit counts)",
                        work_basis=f"{FP32_INSTR_PER_PDIST} FP32 instr x {st['lane_point_dists']:,} lane point-distance "
                                   f"evaluations the kernel's rules needed (stats kernel, rank {rank} fibers)")
        if probe:
            pk = probe["ffma_lane_tops"] * (sm_mhz / probe["sm_mhz"])
            roofline.update(peak_probe=pk, frac_probe=achieved / pk,
                            peak_probe_basis=f"measured FFMA lanes/s ({probe['source']}), scaled to {sm_mhz:.0f} MHz")
        if cfg in SURVEY_INSTR_PER_FIBER:
            w_fix = SURVEY_INSTR_PER_FIBER[cfg] * N
            roofline["frac_survey_work"] = w_fix / (cls_ms * 1e-3) / 1e12 / peak
            roofline["survey_work_basis"] = (f"SURVEY.md §8(d) fixed {SURVEY_INSTR_PER_FIBER[cfg]:,.0f} FP32 lane-instr "
                                             f"per fiber x {N:,} fibers (secondary; frac above is primary)")

    # ---------------- end to end: host buffers through the public API ----------------
    e2e = None
    if not args.no_e2e:
        hf = torch.from_numpy(fib_np).pin_memory()
        if world == 1:
            hl = torch.empty(N, dtype=torch.int32).pin_memory()
            hd = torch.empty(N, dtype=torch.float32).pin_memory()
            e2e_step = lambda: atlas.classify(hf, hl, hd)        # H2D + classify + D2H, returns on completion
            d2h = N * 8
        else:
            full_n = n_job
            hl = torch.empty(full_n, dtype=torch.int32).pin_memory()
            hd = torch.empty(full_n, dtype=torch.float32).pin_memory()
            fdev = torch.empty_like(fib)

            def e2e_step():
                fdev.copy_(hf, non_blocking=True)                # this rank's own H2D over its own link
                if peer is not None:
                    lb, ds = classify_sharded_p2p(atlas.classify, fdev, peer)
                elif strong:
                    lb, ds = classify_sharded(lambda f: classify_into(f), fdev, n_total, world, rank)
                else:
                    lb, ds = classify_into(fdev)
                if rank == 0 and strong:
                    hl.copy_(lb, non_blocking=True)              # the whole subject's results on rank 0
                    hd.copy_(ds, non_blocking=True)
                elif not strong:
                    hl[:N].copy_(lb, non_blocking=True)
                    hd[:N].copy_(ds, non_blocking=True)
            d2h = n_job * 8 if strong else N * 8 * world
        e2e_step()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        t = torch.tensor([e0.elapsed_time(e1) / args.e2e_steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = t.item()
        if world == 1:
            assert np.array_equal(hl.numpy(), res_lab), "host-buffer path disagrees with device path"
        elif strong and rank == 0:
            assert np.array_equal(hl.numpy(), res_lab), "sharded e2e path disagrees with the device path"
        e2e = dict(value=pairs / (e2e_ms * 1e-3), unit=UNIT, ms_per_step=e2e_ms,
                   fibers_per_s=n_job / (e2e_ms * 1e-3),
                   h2d_bytes_per_step=int(fib_np.nbytes) * world, d2h_bytes_per_step=int(d2h),
                   steps=args.e2e_steps,
                   path=("library host-buffer pipeline (seg_classify, host pointers)" if world == 1 else
                         ("per rank: pinned H2D of its shard, seg_classify storing into rank 0 (fused gather); rank 0 "
                          "D2H of all results" if peer is not None else
                          "per rank: pinned H2D of its shard, seg_classify, NCCL all_gather; rank 0 D2H of all results")
                         if strong else "per rank: pinned H2D of its subject, seg_classify, D2H of its results"))

    # ---------------- CPU baseline (oracle) on rank 0 at N=1 ----------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        at0 = at if at is not None else atlas_for_config(cfg)
        cpu = time_oracle(cfg, fib_np, at0, args.cpu_seconds, args.mode)
        cpu.pop("seconds", None)

    if rank == 0:
        line = dict(
            metric=METRIC, value=value, unit=UNIT, n_gpus=world, steps=args.steps, warmup=args.warmup,
            ms_per_step=ms_step, higher_is_better=True, scaling=args.scaling,
            vs_baseline=None, dtype="f32", data="synthetic",
            config=dict(workload=workload_name(cfg, args.mode), fibers=n_job, fibers_per_gpu=N,
                        centroids=spec["n_centroids"], bundles=spec["n_bundles"],
                        parallelism=("one GPU, the whole subject" if world == 1 else
                                     f"one subject sharded contiguously over {world} ranks (atlas NCCL-broadcast, "
                                     + ("results stored into rank 0 by each rank's kernel epilogue over NVLink "
                                        "(fused gather)" if peer is not None else "results all_gathered (NCCL)")
                                     + " in every step)" if strong else
                                     f"one full subject per rank x{world}"),
                        l2=(f"inputs {n_job * 252 / 1e9:.2f} GB > 2 x 126 MB L2; no flush needed" if not flush else
                            f"inputs {n_job * 252 / 1e6:.1f} MB: each step timed alone after a 256 MB L2 flush"),
                        generator_s=round(gen_s, 1)),
            fibers_per_s=fibers_per_s,
            clocks=clocks, e2e=e2e, gpu_launches=launches_per_step * args.steps,
            roofline=roofline, cpu_baseline=cpu,
            cascade=st, labelled_frac=float((res_lab >= 0).mean()),
        )
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
