#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for kronbatch-b200.

Headline workload (BASELINE.json configs[1]): batched 2-D Kronecker action,
fp32, n = 16, batch 4,194,304 entries PER GPU (weak scaling: every rank owns an
independent contiguous shard, no data-path collective). One "step" = one pass
of kron2 over the rank's batch.

  value  : GFlop/s (paper flop count 4 n^3 per entry) over the whole job, inputs
           resident in HBM, device-timed with CUDA events on the launching
           stream, max over ranks.
  e2e    : same metric through the public API with PINNED HOST buffers
           (host->device copy of X and device->host copy of Y inside every
           step; the library pipelines the staging in chunks).
  roofline, cpu_baseline, clocks, gpu_launches: see DESIGN.md "Measurement".
  extra  : the other BASELINE configs (3-D fp32 n=16 / n=10, 3-D fp64 n=16,
           2-D fp32 n=10) measured the same way, for the record.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libkronref.so = the unmodified kronbatch::kron2<float> compiled
from /root/reference, OpenMP over all host cores) on a bounded sample.

Run:  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
      torchrun --nproc-per-node N bench.py --gpus N ...
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "batched Kron GFlop/s + HBM GB/s (n=16 fp32 2-D & 3-D) at 1/2/4/8 B200"
HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback if MEASURED_PEAKS.json is absent
FP32_PEAK_TFLOPS = 72.5    # measured FFMA peak (tools/microbench/fma_tput.cu, profiles/)
FP64_PEAK_TFLOPS = 33.6    # measured DFMA peak
FFMA2_PEAK_TFLOPS = 67.1   # measured fma.rn.f32x2 (FFMA2) peak -- the instruction the fp32 kernels issue
                           # (profiles/r01_fma_tput.txt); reported beside, never as, the roofline

WORKLOADS = {
    # name: (dims3, n, dtype, batch per GPU)
    "kron2-f32-n16": (False, 16, "f32", 4194304),
    "kron3-f32-n16": (True, 16, "f32", 262144),
    "kron3-f32-n10": (True, 10, "f32", 262144),
    "kron3-f64-n16": (True, 16, "f64", 131072),
    "kron2-f32-n10": (False, 10, "f32", 65536),
}
HEADLINE = "kron2-f32-n16"


def flops_per_entry(dims3, n):
    return 6 * n ** 4 if dims3 else 4 * n ** 3  # bench_support.cpp:31-35


def bytes_per_entry(dims3, n, dtype):
    es = 4 if dtype == "f32" else 8
    return 2 * n ** (3 if dims3 else 2) * es  # X read + Y written (beta = 0)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


def load_traffic():
    """Per-launch DRAM bytes of each workload's kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


# ----------------------------------------------------------------- clocks --

class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region (the
    B200_PROFILING.md clocks line), via NVML in a background thread (2 ms
    period) so that even short timed regions get several samples."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, index, period_s=0.002):
        self.index, self.period = index, period_s
        self.sm, self.reasons, self.smax = [], set(), None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception:
            self.nv = None
        return self

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv is not None:
            self.thread.join(timeout=1)

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.smax,
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


# --------------------------------------------------------------- our arm --

def make_problem(kb, torch, dims3, n, dtype, batch, device, host=False, seed=1):
    tdt = torch.float32 if dtype == "f32" else torch.float64
    e = n ** (3 if dims3 else 2)
    g = torch.Generator(device=device).manual_seed(seed)
    mk = lambda cnt: (torch.rand(cnt, dtype=tdt, device=device, generator=g) * 2 - 1)
    # The constant matrices are small host arrays, as in the reference API: the
    # library folds them into kernel parameters (no per-call device->host sync).
    A, B, Cm = (mk(n * n).cpu() for _ in range(3))
    X = mk(e * batch)
    Y = torch.empty(e * batch, dtype=tdt, device=device)
    if host:
        X = X.cpu().pin_memory()
        Y = torch.empty(e * batch, dtype=tdt).pin_memory()
    MV, BV = kb.MatrixView, kb.BatchView
    if dims3:
        pr = kb.KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n)
        args = (pr, MV(A, n, n, n), MV(B, n, n, n), MV(Cm, n, n, n),
                BV(kb.Array3View(X, n, n, n, n, n * n), batch, e), BV(kb.Array3View(Y, n, n, n, n, n * n), batch, e),
                kb.Workspace(None, n * n * n * batch))
        return kb.kron3, args, (X, Y)
    pr = kb.KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n)
    args = (pr, MV(A, n, n, n), MV(B, n, n, n), BV(MV(X, n, n, n), batch, e), BV(MV(Y, n, n, n), batch, e))
    return kb.kron2, args, (X, Y)


def dist_max(torch, v, world):
    if world <= 1:
        return v
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def time_device(kb, torch, name, steps, warmup, world, rank):
    """Device-resident timing: K launches on our stream between events; returns
    (ms per step (max over ranks), per-launch mean ms, launches)."""
    dims3, n, dtype, batch = WORKLOADS[name]
    fn, args, keep = make_problem(kb, torch, dims3, n, dtype, batch, "cuda")
    stream = torch.cuda.Stream()
    ex = kb.Exec(stream=stream, asynchronous=True)
    for _ in range(max(warmup, 3)):
        fn(*args, exec_=ex)
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    barrier(world)
    torch.cuda.synchronize()
    l0 = kb.launch_count()
    t_all0 = torch.cuda.Event(enable_timing=True)
    t_all1 = torch.cuda.Event(enable_timing=True)
    t_all0.record(stream)
    for i in range(steps):
        starts[i].record(stream)
        fn(*args, exec_=ex)
        ends[i].record(stream)
    t_all1.record(stream)
    torch.cuda.synchronize()
    launches = kb.launch_count() - l0
    barrier(world)
    total_ms = t_all0.elapsed_time(t_all1)
    per_launch = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = dist_max(torch, total_ms, world)
    del keep
    return total_ms / steps, statistics.mean(per_launch), launches, kb.last_path()


def time_graph(kb, torch, name, steps, world):
    """Launch-overhead-free device time: `steps` calls captured into one CUDA
    graph (the library's kernel launches are capturable on the exec stream),
    replayed between events; returns ms per launch (max over ranks)."""
    dims3, n, dtype, batch = WORKLOADS[name]
    fn, args, keep = make_problem(kb, torch, dims3, n, dtype, batch, "cuda")
    stream = torch.cuda.Stream()
    ex = kb.Exec(stream=stream, asynchronous=True)
    for _ in range(3):
        fn(*args, exec_=ex)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(steps):
            fn(*args, exec_=ex)
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    with torch.cuda.stream(stream):
        e0.record(stream)
        g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    ms = dist_max(torch, e0.elapsed_time(e1) / steps, world)
    del keep, g
    return ms


def time_e2e(kb, torch, name, steps, warmup, world):
    """End to end through the public API with pinned host X / Y: H2D of X and
    D2H of Y inside every step (wall time around the synchronous call, which
    returns only after Y is back in host memory), max over ranks."""
    dims3, n, dtype, batch = WORKLOADS[name]
    fn, args, (X, Y) = make_problem(kb, torch, dims3, n, dtype, batch, "cuda", host=True)
    for _ in range(max(1, min(warmup, 2))):
        fn(*args)
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(steps):
        fn(*args)
    dt = time.perf_counter() - t0
    dt = dist_max(torch, dt, world)
    return dt * 1e3 / steps, X.numel() * X.element_size(), Y.numel() * Y.element_size()


def cpu_reference_sample(name, seconds_budget=8.0, threads=None):
    """The reference CPU path (oracle/_ref: unmodified kronbatch::kron2/kron3
    with OpenMP) on a bounded sample of the workload; median of reps after a
    verified-by-the-tests warm-up. Returns (GFlop/s, cores, sample text)."""
    import numpy as np

    from oracle.oracle import Reference

    dims3, n, dtype, _ = WORKLOADS[name]
    ref = Reference()
    if threads:
        ref.set_threads(threads)
    cores = ref.max_threads
    dt = np.float32 if dtype == "f32" else np.float64
    e = n ** (3 if dims3 else 2)
    sample = max(1, int((256 << 20) // (e * dt().itemsize)))  # ~256 MiB of X per rep
    a, b, c, x, y = ref.generate_batch(dt, 1, n, dims3, sample)
    work = np.empty(n * n * n * sample if dims3 else 0, dt)

    def run():
        if dims3:
            ref.kron3("N", "N", "N", n, n, n, n, n, n, sample, dt(1), a, (n, n), n, b, (n, n), n, c, (n, n), n, x,
                      (n, n, n), n, n * n, e, dt(0), y, (n, n, n), n, n * n, e, work)
        else:
            ref.kron2("N", "N", "N", n, n, n, n, sample, dt(1), a, (n, n), n, b, (n, n), n, x, (n, n), n, e, dt(0), y,
                      (n, n), n, e)

    run()  # warm-up (first touch, thread pool)
    times = []
    t_end = time.perf_counter() + seconds_budget
    while len(times) < 3 or (time.perf_counter() < t_end and len(times) < 50):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    med = statistics.median(times)
    gf = flops_per_entry(dims3, n) * sample / med / 1e9
    return gf, cores, f"{sample} entries of {name} (generate_batch seed 1), median of {len(times)} reps", med


# ------------------------------------------------------------------ main --

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extra", action="store_true", help="skip the non-headline configs")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--e2e-steps", type=int, default=3)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dims3, n, dtype, batch = WORKLOADS[HEADLINE]
    fl_e, by_e = flops_per_entry(dims3, n), bytes_per_entry(dims3, n, dtype)

    if args.impl == "reference":
        if rank != 0:
            return 0
        gf, cores, sample, med = cpu_reference_sample(HEADLINE, seconds_budget=max(2.0, 0.5 * args.steps))
        line = {"metric": METRIC, "value": round(gf, 3), "unit": "GFlop/s", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(med * 1e3, 4), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference generate_batch, seed 1)",
                "impl": "reference",
                "config": {"workload": f"{HEADLINE}: 2-D Kronecker action fp32 n=16 (reference CPU, bounded sample)",
                           "batch_per_gpu": batch, "sample": sample},
                "cpu_baseline": {"value": round(gf, 3), "unit": "GFlop/s", "cores": cores, "kind": "reference",
                                 "sample": sample},
                "e2e": {"value": round(gf, 3), "unit": "GFlop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1304_7054_b200 as kb

    hbm_peak, peak_kind = load_peaks()
    traffic = load_traffic()
    with ClockSampler(local) as clk:
        ms, launch_ms, launches, path = time_device(kb, torch, HEADLINE, args.steps, args.warmup, world, rank)
    clocks = clk.summary()
    value = fl_e * batch * world / (ms * 1e-3) / 1e9  # GFlop/s, whole job
    gbs = by_e * batch * world / (ms * 1e-3) / 1e9
    achieved = by_e * batch / (launch_ms * 1e-3) / 1e9  # per launch, this rank
    e2e_ms, h2d, d2h = time_e2e(kb, torch, HEADLINE, args.e2e_steps, args.warmup, world)
    e2e_value = fl_e * batch * world / (e2e_ms * 1e-3) / 1e9

    extra = []
    if not args.no_extra:
        for name in WORKLOADS:
            if name == HEADLINE:
                continue
            d3, nn, dt, bt = WORKLOADS[name]
            xms, xlaunch, _, xpath = time_device(kb, torch, name, max(5, args.steps // 2), args.warmup, world, rank)
            fe, be = flops_per_entry(d3, nn), bytes_per_entry(d3, nn, dt)
            tf = fe * bt / (xlaunch * 1e-3) / 1e12
            gb = be * bt / (xlaunch * 1e-3) / 1e9
            fpeak = FP32_PEAK_TFLOPS if dt == "f32" else FP64_PEAK_TFLOPS
            roof_tf = min(fpeak, hbm_peak * fe / be / 1e3)
            rec = {"workload": name, "value": round(fe * bt * world / (xms * 1e-3) / 1e9, 1), "unit": "GFlop/s",
                   "ms_per_step": round(xms, 4), "hbm_gbs": round(gb, 1), "kernel": xpath,
                   "roofline": {"bound": "hbm" if roof_tf < fpeak else "fp-pipe", "roof_tflops": round(roof_tf, 2),
                                "frac": round(tf / roof_tf, 4), "hbm_frac": round(gb / hbm_peak, 4)}}
            if dt == "f32" and roof_tf >= fpeak:
                rec["roofline"]["ffma2_peak_frac"] = round(tf / FFMA2_PEAK_TFLOPS, 4)
            if bt * be < (256 << 20):  # small batch: host launch cost dominates -> also report a CUDA-graph replay
                gms = time_graph(kb, torch, name, max(20, args.steps), world)
                rec["cuda_graph"] = {"ms_per_launch": round(gms, 4),
                                     "value": round(fe * bt * world / (gms * 1e-3) / 1e9, 1),
                                     "hbm_gbs": round(be * bt / (gms * 1e-3) / 1e9, 1)}
            extra.append(rec)

    cpu = None
    if rank == 0 and not args.no_cpu:
        try:
            gf, cores, sample, _ = cpu_reference_sample(HEADLINE)
            cpu = {"value": round(gf, 3), "unit": "GFlop/s", "cores": cores, "kind": "reference", "sample": sample}
        except Exception as e:  # reference .so missing on this box
            cpu = {"value": None, "unit": "GFlop/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        tr = traffic.get(HEADLINE)
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "GFlop/s", "n_gpus": world if world > 1 else args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (torch uniform[-1,1), seed 1; inputs 4.3 GB/GPU >> 126 MB L2, no flush needed)",
            "config": {"workload": f"{HEADLINE}: 2-D Kronecker action Y=A X B^T, fp32, n=16, batch {batch} per GPU "
                                   "(BASELINE configs[1]), alpha 1 beta 0, tight layout",
                       "batch_per_gpu": batch, "n": n, "l2": "inputs larger than L2"},
            "hbm_gbs": round(gbs, 1),
            "kernel": path,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                         "frac": round(achieved / hbm_peak, 4), "peak_kind": peak_kind,
                         "traffic": tr if tr is None else tr.get("dram_bytes_per_launch"),
                         "algorithmic_bytes_per_launch": by_e * batch},
            "e2e": {"value": round(e2e_value, 1), "unit": "GFlop/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 3)},
            "gpu_launches": launches,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "extra": extra,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
