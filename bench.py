#!/usr/bin/env python
"""Benchmark of the B200 RBD greedy loop (BASELINE.json metric: effective HBM
GB/s = X bytes x greedy steps / time; end-to-end seconds alongside).

One bench "step" = one full rbd::decompose of the workload. Workloads
(BASELINE.json configs, seeded synthetic inputs, paper_1503_05947_b200/configs.py):

* N = 1 (default): C2-tall, 1,048,576 x 4,096 fp64 (32 GiB), d = 512 — the
  largest configuration that is a single-GPU workload (BASELINE.json names no
  config for the metric). `value` is device-resident (X in HBM before the
  timed region); `e2e` goes through the reference-facing host entry
  (rbd_decompose_host_many: pinned host X -> H2D -> loop -> D2H of Y and T,
  the upload of matrix i+1 overlapping the loop of matrix i).
* N > 1 (torchrun): C3-sharded, 262,144 x 65,536 (128 GiB), d = 1024, X split
  by contiguous column blocks over the ranks, Y replicated (strong scaling;
  `--workload C3-sharded` runs the same line at N = 1).

Secondary figures (C1 image-like, the fp32 storage mode, C4 out-of-sample)
ride along in `secondary` and never enter `value`.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                       [--workload NAME]
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rbd_effective_hbm_gbs"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--workload", default=None,
                   help="default: C2-tall at N=1, C3-sharded under torchrun (N>1)")
    p.add_argument("--cpu-seconds", type=float, default=20.0,
                   help="cpu_baseline: bounded single-thread oracle sample (seconds)")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=6,
                   help="matrices per timed rbd_decompose_host_many call (capped at --steps)")
    p.add_argument("--aux-steps", type=int, default=3,
                   help="timed decompositions of each secondary figure")
    p.add_argument("--no-secondary", action="store_true")
    p.add_argument("--d-max", type=int, default=None, help="override d_max (quick runs)")
    p.add_argument("--ref-seconds", type=float, default=3.0,
                   help="reference arm: CPU seconds of greedy steps per bench step")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def default_workload(args, world):
    if args.workload:
        return args.workload
    return "C2-tall" if world == 1 else "C3-sharded"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def wait_first(self, timeout: float = 3.0):
        """Block until nvidia-smi has produced its first sample (its start-up
        takes longer than a short timed region), so the samples cover it."""
        t0 = time.perf_counter()
        while self.proc is not None and not self.lines and time.perf_counter() - t0 < timeout:
            time.sleep(0.02)
        self.begin = len(self.lines)   # samples from here on fall in the timed region

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines[getattr(self, "begin", 0):] or self.lines
        for ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload):
    """dram bytes per launch of the loop kernel from one `ncu --set full`
    capture of the same workload (profiles/traffic.json, keyed by workload)."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
    except Exception:
        return None
    return t.get(workload)


def host_mem_available():
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemAvailable:"):
                    return int(ln.split()[1]) * 1024
    except OSError:
        pass
    return None


def read_peak_gbs(dev, gib: int = 4, reps: int = 10):
    import torch
    try:
        buf = torch.ones(gib * (1 << 27), dtype=torch.float64, device=dev)
    except RuntimeError:
        return None
    best = float("inf")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(reps + 2):
        torch.cuda.synchronize(dev)
        e0.record()
        buf.sum()
        e1.record()
        torch.cuda.synchronize(dev)
        if i >= 2:
            best = min(best, e0.elapsed_time(e1))
    nbytes = buf.numel() * 8
    del buf
    torch.cuda.empty_cache()
    return nbytes / (best / 1e3) / 1e9


# ---------------------------------------------------------------- workloads

NOISE = {"C2": 1e-8, "C3": 1e-10, "C4": 1e-6}
RANK = {"C2": 1024, "C3": 2048, "C4": 512}


def make_workload(name, device, offset=0, n_local=None):
    """(workload, X column-major view on `device`, absolute eps_R). C3 is built
    by column blocks (any shard of it regenerates alone)."""
    import torch
    from paper_1503_05947_b200 import configs
    w = configs.WORKLOADS[name]
    key = name.split("-")[0]
    if key == "C1":
        Xd = configs.c1_matrix(n=w.n, seed=w.seed, device=device)
    elif key == "C0":
        Xd = torch.as_tensor(configs.c0_matrix().T.copy(), device=device).t()
    elif key == "C3":
        Xd = configs.low_rank_shard_torch(w.m, w.n, RANK[key], configs.spectrum(key, RANK[key]),
                                          NOISE[key], w.seed, offset,
                                          w.n if n_local is None else n_local, device=device)
    else:
        Xd = configs.low_rank_matrix_torch(w.m, w.n, RANK[key], configs.spectrum(key, RANK[key]),
                                           NOISE[key], w.seed, device=device)
    if torch.device(device).type == "cuda":
        torch.cuda.synchronize(device)
    eps = w.eps_abs
    if w.eps_rel != 0.0:
        eps = configs.eps_for(w, float(Xd.norm(dim=0).max()))
    return w, Xd, eps


def workload_config(w, eps, world, d_max):
    """The `config` object of BOTH arms (identical dicts)."""
    sharded = w.name.startswith("C3")
    xbytes = w.m * w.n * 8
    return {"workload": w.name, "m": w.m, "n": w.n, "d_max": d_max, "eps_R": eps,
            "dtype_X": "f64", "parallelism": (f"colshard{world}" if sharded else f"replicas{world}"),
            "l2": f"inputs larger than L2 (X {xbytes / 1e9:.1f} GB vs 126 MB L2)",
            "describe": w.describe}


# ---------------------------------------------------------------- reference arm

def run_reference(args):
    """The reference's CPU path on the box's host cores: the oracle port
    (restating decompose.cpp / workspace.cpp with the reference's two X passes
    per step), all host threads, on our arm's workload and config. Each bench
    step is a bounded sample: the first S greedy steps of the full workload."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    import torch
    wname = default_workload(args, world)
    dev = torch.device("cuda", local) if torch.cuda.is_available() else torch.device("cpu")
    from paper_1503_05947_b200 import configs
    wfull = configs.WORKLOADS[wname]
    block = None
    if wfull.m * wfull.n * 8 > 64e9:   # C3 (137 GB): a column block of the same X
        block = 2048
        w, Xd, eps = make_workload(wname, dev, 0, block)
    else:
        w, Xd, eps = make_workload(wname, dev)
    d_max = args.d_max or w.d_max
    X = np.asfortranarray(Xd.cpu().numpy())
    del Xd
    if dev.type == "cuda":
        torch.cuda.empty_cache()
    cores = os.cpu_count() or 1
    import oracle
    per_est = 2.0 * w.m * (block or w.n) * 8 / (8e9 * cores)   # two X passes per greedy step
    S = int(max(1, min(d_max, block or d_max, args.ref_seconds / max(per_est, 1e-6))))
    for _ in range(args.warmup):
        oracle.decompose(X, d_max, eps, nthreads=cores, max_steps=S)
    loops, inits, done = 0.0, 0.0, 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r = oracle.decompose(X, d_max, eps, nthreads=cores, max_steps=S)
        loops += r.t_loop_s
        inits += r.t_init_s
        done += r.d
    wall = time.perf_counter() - t0
    ncols = block or w.n
    bytes_per = w.m * ncols * 8
    val = bytes_per * done / loops / 1e9
    sample = (f"first {S} of {d_max} greedy steps of {w.name} ({w.m}x{ncols} fp64"
              f"{f', the first {block} of its {w.n} columns' if block else ''}) per bench step, "
              f"oracle port (decompose.cpp:53-111, two X passes per step), {cores} threads; "
              f"value = X bytes x steps / greedy-loop time (the per-call validation + "
              f"workspace_init pass, {inits / max(args.steps, 1):.2f} s, is excluded: a full "
              f"decompose runs it once per {d_max} steps)")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wall / max(args.steps, 1) * 1e3, "higher_is_better": True,
        "scaling": "strong" if w.name.startswith("C3") else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(wfull, eps, world, d_max),
        "cpu_baseline": {"value": val, "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "greedy_steps_timed": done,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm (one GPU per workload)

def cpu_baseline_leg(X_host, w, eps, d_max, seconds):
    """Oracle port (two X passes per step), ONE thread, on the first S greedy
    steps of the same workload (S sized for ~`seconds` of CPU work)."""
    import oracle
    per_est = 2.0 * w.m * w.n * 8 / 8e9
    S = int(max(1, min(d_max, seconds / max(per_est, 1e-6))))
    r = oracle.decompose(X_host, d_max, eps, nthreads=1, max_steps=S)
    xb = w.m * w.n * 8
    loop_rate = xb * r.d / r.t_loop_s / 1e9
    full_s = r.t_init_s + d_max * r.t_loop_s / r.d
    return {"value": loop_rate, "unit": "GB/s", "cores": 1, "kind": "port",
            "sample": (f"first {r.d} of {d_max} greedy steps of {w.name} ({w.m}x{w.n} fp64), "
                       f"single-thread oracle restating decompose.cpp (two X passes per step): "
                       f"{r.t_loop_s:.1f} s of greedy loop (value = X bytes x steps / loop time) "
                       f"after a {r.t_init_s:.1f} s validation + workspace_init pass"),
            "steps_sampled": r.d, "loop_s": r.t_loop_s, "init_s": r.t_init_s,
            "extrapolated_full_decompose_s": full_s,
            "cpu_model": cpu_model(), "nproc": os.cpu_count()}


def time_decomposes(rbd, X, d_max, eps, ctx, steps, stream, dev):
    import torch
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    ds, loops = [], []
    for _ in range(steps):
        g = rbd.decompose(X, d_max=d_max, eps_r=eps, ctx=ctx)
        ds.append(g.d)
        loops.append(g.result.loop_ms)
        del g
    e1.record(stream)
    torch.cuda.synchronize(dev)
    return e0.elapsed_time(e1), ds, loops


def secondary_c1(rbd, ctx, dev, stream, args, peak):
    w, Xd, eps = make_workload("C1-image-like", dev)
    for _ in range(3):
        rbd.decompose(Xd, d_max=w.d_max, eps_r=eps, ctx=ctx)
    K = max(args.aux_steps, 5)
    ms, ds, loops = time_decomposes(rbd, Xd, w.d_max, eps, ctx, K, stream, dev)
    xb = w.m * w.n * 8
    lm = float(np.mean(loops))
    out = {"workload": w.name, "m": w.m, "n": w.n, "d_max": w.d_max,
           "value": xb * sum(ds) / (ms / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": ms / K,
           "loop_ms_mean": lm, "roofline_frac": xb * float(np.mean(ds)) / (lm / 1e3) / 1e9 / peak,
           "d_reached": int(np.mean(ds))}
    del Xd
    gc.collect()
    return out


def secondary_c4(rbd, ctx, dev, stream, args):
    """BASELINE config 4: RBD on the 65,536 x 8,192 stage, then the out-of-sample
    stream of 16 batches x 16,384 columns (T_new = Y'X_new + Eq. 3 error
    indicator). Device-resident K5 / K6 rates, and e2e through
    rbd_project_host_many[_f32] from pinned host batches (two distinct pinned
    buffers alternate: 16 distinct 8 GiB batches would need 128 GiB of host RAM;
    every batch is uploaded, contracted and downloaded)."""
    import torch
    from paper_1503_05947_b200 import configs
    w = configs.C4
    X = configs.c4_stage_matrix(dev)
    for _ in range(2):
        g = rbd.decompose(X, d_max=w.d_max, ctx=ctx)
    K = max(args.aux_steps, 3)
    ms, ds, loops = time_decomposes(rbd, X, w.d_max, 0.0, ctx, K, stream, dev)
    xb = w.m * w.n * 8
    out = {"stage": {"workload": "C4 RBD stage 65536x8192", "d": int(ds[0]),
                     "value": xb * sum(ds) / (ms / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": ms / K}}
    g = rbd.decompose(X, d_max=w.d_max, ctx=ctx)
    del X
    rm = rbd.ResidentModel.from_model(g, ctx=ctx)
    Yd = g.Y.t().contiguous().t()
    U, sv = configs.c4_basis(dev)
    B = configs.C4_BATCH
    nb = configs.C4_NEW_COLUMNS // B
    flops = 2.0 * w.m * g.d * B
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # device-resident K5 (fp64 DMMA) and K6 (fp32 tcgen05 3xTF32) on one batch
    Xn = configs.c4_new_batch(U, sv, 0, device=dev)
    rbd.project_batch(Yd, Xn, ctx=ctx)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for _ in range(3):
        rbd.project_batch(Yd, Xn, ctx=ctx)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    k5 = e0.elapsed_time(e1) / 3
    Y32 = Yd.float().t().contiguous().t()
    X32 = Xn.float().t().contiguous().t()
    rbd.project_batch_f32(Y32, X32, ctx=ctx)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for _ in range(3):
        rbd.project_batch_f32(Y32, X32, ctx=ctx)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    k6 = e0.elapsed_time(e1) / 3
    out["device_fp64"] = {"kernel": "K5 k_project_dmma (FP64 DMMA) + Eq. 3", "ms_per_batch": k5,
                          "tflops": flops / (k5 / 1e3) / 1e12}
    out["device_fp32"] = {"kernel": "K6 k_project_tf32x3_pair (tcgen05 cta_group::2 kind::tf32, 3xTF32, 256x256 tile per CTA pair) + Eq. 3",
                          "ms_per_batch": k6, "tflops_fp32_equivalent": flops / (k6 / 1e3) / 1e12}
    # e2e: the pinned host stream through the resident model
    for f32, dt, tdt in ((False, torch.float64, np.float64), (True, torch.float32, np.float32)):
        bufs = []
        for b in range(2):
            xb_dev = configs.c4_new_batch(U, sv, b, device=dev)
            h = torch.empty((B, w.m), dtype=dt, pin_memory=True)
            h.copy_(xb_dev.t())
            bufs.append(h.numpy().T)
            del xb_dev
        outs = [(torch.empty((B, g.d), dtype=dt, pin_memory=True).numpy().T,
                 torch.empty(B, dtype=torch.float64, pin_memory=True).numpy()) for _ in range(nb)]
        batches = [bufs[i % 2] for i in range(nb)]
        rm.project_many(batches[:2], f32=f32, out=outs[:2])   # warm
        t0 = time.perf_counter()
        rm.project_many(batches, f32=f32, out=outs)
        te = time.perf_counter() - t0
        hb = B * w.m * (4 if f32 else 8)
        out["e2e_fp32" if f32 else "e2e_fp64"] = {
            "entry": f"rbd_project_host_many{'_f32' if f32 else ''} ({nb} batches of {B}, pinned)",
            "seconds_all_batches": te, "ms_per_batch": te * 1e3 / nb,
            "tflops": flops * nb / te / 1e12, "h2d_gbs": hb * nb / te / 1e9,
            "h2d_bytes_per_batch": hb, "d2h_bytes_per_batch": B * g.d * (4 if f32 else 8) + 8 * B}
        del bufs, outs, batches
        gc.collect()
    # CPU: the reference's per-vector project (decompose.cpp:113-117), one thread
    import oracle
    ns = 64
    Yh = np.asfortranarray(Yd.cpu().numpy())
    Xs = np.asfortranarray(Xn[:, :ns].cpu().numpy())
    t0 = time.perf_counter()
    for j in range(ns):
        oracle.project(Yh, Xs[:, j])
    tc = time.perf_counter() - t0
    out["cpu_baseline"] = {"value": 2.0 * w.m * g.d * ns / tc / 1e12, "unit": "TFLOP/s",
                           "cores": 1, "kind": "port", "seconds": tc,
                           "sample": f"oracle per-vector project (decompose.cpp:113-117, Y re-read "
                                     f"per vector, one thread) on {ns} of the batch's columns"}
    del Xn, X32, Y32, Yd, U, rm, g
    gc.collect()
    torch.cuda.empty_cache()
    return out


def f32_leg(rbd, Xd, w, d_max, eps, ctx, dev, stream, args, peak):
    """fp32 storage mode on the same workload rounded to fp32 (half the X
    bytes per sweep, fp64 arithmetic): device-resident and e2e."""
    import torch
    m, n = Xd.shape
    Xf = Xd.float()
    gf = rbd.decompose(Xf, d_max=d_max, eps_r=eps, ctx=ctx)
    K = max(1, args.aux_steps)
    ms, fd, fl = time_decomposes(rbd, Xf, d_max, eps, ctx, K, stream, dev)
    fbytes = m * n * 4
    floop = float(np.mean(fl))
    out = {"storage": "f32 X, f64 arithmetic (rbd_decompose_device_f32)",
           "value": fbytes * sum(fd) / (ms / 1e3) / 1e9, "unit": "GB/s",
           "ms_per_step": ms / K, "loop_ms_mean": floop,
           "roofline_frac": fbytes * float(np.mean(fd)) / (floop / 1e3) / 1e9 / peak,
           "d_reached": int(np.mean(fd))}
    if not args.no_e2e:
        Xh_t = torch.empty((n, m), dtype=torch.float32, pin_memory=True)
        Xh_t.copy_(Xf.t())
        Xh32 = Xh_t.numpy().T
        del Xf
        torch.cuda.empty_cache()
        Ke = max(1, min(args.e2e_steps, args.steps))
        from paper_1503_05947_b200.api import output_buffers
        obufs = output_buffers(m, n, d_max, Ke)
        warm = rbd.decompose_many([Xh32] * 2, d_max=d_max, eps_r=eps, ctx=ctx, out=obufs[:2])
        del warm
        gc.collect()
        t0 = time.perf_counter()
        outs = rbd.decompose_many([Xh32] * Ke, d_max=d_max, eps_r=eps, ctx=ctx, out=obufs)
        te = time.perf_counter() - t0
        del obufs
        fe = [o.d for o in outs]
        del outs
        gc.collect()
        out["e2e"] = {"value": fbytes * sum(fe) / te / 1e9, "unit": "GB/s",
                      "ms_per_step": te * 1e3 / Ke, "h2d_bytes_per_step": m * n * 4,
                      "entry": "rbd_decompose_host_many_f32 (numpy float32, pinned)"}
        del Xh_t, Xh32
    else:
        del Xf
    del gf
    gc.collect()
    torch.cuda.empty_cache()
    return out


def run_b200(args):
    import torch
    rank, world, local = dist_env()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    import paper_1503_05947_b200 as rbd
    from paper_1503_05947_b200._lib import check, load_library
    import ctypes as C

    wname = default_workload(args, world)
    w, Xd, eps = make_workload(wname, dev)
    d_max = args.d_max or w.d_max
    ctx = rbd.Context(local)
    lib = load_library()
    m, n = Xd.shape
    bytes_per_gstep = m * n * 8
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)

    for _ in range(max(args.warmup, 0)):
        rbd.decompose(Xd, d_max=d_max, eps_r=eps, ctx=ctx)
    clocks = ClockSampler(local)
    torch.cuda.synchronize(dev)
    clocks.start()
    clocks.wait_first()
    launches0 = ctx.launches
    ms, ds, loop_ms = time_decomposes(rbd, Xd, d_max, eps, ctx, args.steps, stream, dev)
    clk = clocks.stop()
    launches = ctx.launches - launches0
    value = bytes_per_gstep * sum(ds) / (ms / 1e3) / 1e9

    # ---- roofline of the dominant kernel ----
    # Inside the timed region the only kernels are K1 (init, 2 launches) and
    # k_rbd_persistent (the whole greedy loop, 1 launch per decompose). Its
    # algorithmic bytes per launch = m*n*8 per greedy step (X read once) x d;
    # its duration is the CUDA-event time around the launch on the context
    # stream (result.loop_ms).
    peak, peak_src = peak_hbm()
    d_mean = float(np.mean(ds))
    loop_mean = float(np.mean(loop_ms))
    alg_bytes = bytes_per_gstep * d_mean
    ach = alg_bytes / (loop_mean / 1e3) / 1e9
    traffic = ncu_traffic(w.name) or {}
    roofline = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": traffic.get("bytes_per_launch"),
                "kernel": "k_rbd_persistent<2> (whole greedy loop, 1 launch/decompose)",
                "algorithmic_bytes_per_launch": alg_bytes,
                "algorithmic_bytes_note": "m*n*8 per greedy step x d (X read once per step); "
                                          "Y passes and bookkeeping not credited",
                "ms_per_launch": loop_mean, "loop_share_of_step": loop_mean / (ms / args.steps),
                "peak_source": peak_src, "traffic_source": traffic.get("source")}
    # DRAM rate of the loop = the ncu capture's bytes per launch / this run's
    # launch time (context only: `frac` above is the algorithmic one)
    if traffic.get("bytes_per_launch") and abs(d_mean - w.d_max) < 0.5:
        dr = traffic["bytes_per_launch"] / (loop_mean / 1e3) / 1e9
        roofline["dram"] = {"gbs": dr, "frac_of_peak": dr / peak,
                            "note": "ncu dram bytes per launch (traffic) / this run's ms_per_launch: "
                                    "what the HBM moves, X plus the uncredited Y passes"}
    # the fused sweep phase alone, as a standalone kernel (K2), CUDA events
    y = torch.randn(m, dtype=torch.float64, device=dev)
    y /= y.norm()
    torch.cuda.synchronize(dev)
    ms_sweep = C.c_double()
    check(lib.rbd_time_sweep(ctx.handle, C.c_void_p(Xd.data_ptr()), m, n, Xd.stride(1),
                             C.c_void_p(y.data_ptr()), 20, C.byref(ms_sweep)))
    sw = bytes_per_gstep / (ms_sweep.value / 1e3) / 1e9
    roofline["sweep_kernel"] = {"kernel": "k_sweep<2,MODE_DOT,stream> (K2 standalone)",
                                "achieved": sw, "frac": sw / peak, "ms_per_launch": ms_sweep.value,
                                "bytes_per_launch": bytes_per_gstep}
    del y
    rp = read_peak_gbs(dev)
    if rp:
        roofline["read_peak"] = {"gbs": rp, "frac": ach / rp,
                                 "how": "torch.sum over a 4 GiB fp64 buffer (read-only), best of 10, "
                                        "CUDA events"}
    roofline["frac_of_nominal"] = {"gbs": 7700.0, "frac": ach / 7700.0,
                                   "note": "nominal HBM3e 7.7 TB/s (HGX), B200_PROFILING.md"}

    # ---- e2e through the reference-facing host entry (pinned host X) ----
    e2e = None
    Xh = None
    Xh_t = None
    if not args.no_e2e or not args.no_cpu:
        Xh_t = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
        Xh_t.copy_(Xd.t())
        Xh = Xh_t.numpy().T  # (m, n) Fortran view, pinned
        assert Xh.flags["F_CONTIGUOUS"]
    if not args.no_e2e:
        Ke = max(1, min(args.e2e_steps, args.steps))
        # the caller's page-locked output buffers, allocated once and reused
        from paper_1503_05947_b200.api import output_buffers
        obufs = output_buffers(m, n, d_max, Ke)
        warm = rbd.decompose_many([Xh] * 2, d_max=d_max, eps_r=eps, ctx=ctx, out=obufs[:2])
        del warm
        gc.collect()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        outs = rbd.decompose_many([Xh] * Ke, d_max=d_max, eps_r=eps, ctx=ctx, out=obufs)
        wall = time.perf_counter() - t0
        d3 = [o.d for o in outs]
        del outs
        gc.collect()
        dmean = float(np.mean(d3))
        e2e = {"value": bytes_per_gstep * sum(d3) / wall / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": m * n * 8,
               "d2h_bytes_per_step": int(8 * (m * dmean + dmean * n + 2 * dmean)),
               "ms_per_step": wall * 1e3 / Ke, "steps": Ke,
               "seconds_per_decompose": wall / Ke,
               "entry": "rbd_decompose_host_many (numpy, pinned; upload of matrix i+1 overlaps "
                        "the loop of matrix i; Y and T stream back during the loop into the "
                        "caller's page-locked output buffers, allocated before the timed region)"}
        del obufs

    # ---- CPU baseline: oracle port, one thread, bounded sample ----
    cpu = None
    if not args.no_cpu:
        cpu = cpu_baseline_leg(Xh, w, eps, d_max, args.cpu_seconds)
    del Xh, Xh_t
    gc.collect()

    # ---- secondary figures (never part of `value`) ----
    secondary = {}
    if not args.no_secondary:
        try:
            secondary["f32_mode"] = f32_leg(rbd, Xd, w, d_max, eps, ctx, dev, stream, args, peak)
        except Exception as ex:   # reported, not fatal: the headline is already measured
            secondary["f32_mode"] = {"error": repr(ex)[:300]}
        del Xd
        gc.collect()
        torch.cuda.empty_cache()
        if not w.name.startswith("C1"):
            try:
                secondary["C1-image-like"] = secondary_c1(rbd, ctx, dev, stream, args, peak)
            except Exception as ex:
                secondary["C1-image-like"] = {"error": repr(ex)[:300]}
        if not w.name.startswith("C4"):
            try:
                secondary["C4-out-of-sample"] = secondary_c4(rbd, ctx, dev, stream, args)
            except Exception as ex:
                secondary["C4-out-of-sample"] = {"error": repr(ex)[:300]}

    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(w, eps, world, d_max),
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "clocks": clk, "loop_ms_mean": loop_mean, "d_per_step": ds,
        "seconds_per_decompose": ms / 1e3 / args.steps,
        "secondary": secondary,
    }
    print(json.dumps(line), flush=True)
    ctx.close()


# ---------------------------------------------------------------- sharded (C3, N GPUs)

def run_sharded(args):
    """C3: X sharded by contiguous column blocks over the ranks (the exchange
    runs inside the library over NCCL); strong scaling on the whole job."""
    import torch
    rank, world, local = dist_env()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    import paper_1503_05947_b200 as rbd
    from paper_1503_05947_b200 import configs, distributed as rd
    wname = default_workload(args, world)
    r = None
    w0 = configs.WORKLOADS[wname]
    plan = rd.plan_shards(w0.n, world)
    o, nl = plan.offsets[rank], plan.n_locals[rank]
    w, X, eps = make_workload(wname, dev, o, nl)
    d_max = args.d_max or w.d_max
    ctx = rbd.Context(local)
    if world > 1:
        uid = rd.exchange_unique_id(rank)
    else:
        import ctypes as C
        buf = C.create_string_buffer(128)
        from paper_1503_05947_b200._lib import check, load_library
        check(load_library().rbd_comm_unique_id(buf))
        uid = bytes(buf.raw)
    rd.init_comm(ctx, rank, world, uid)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    for _ in range(max(args.warmup, 0)):
        r = rd.decompose_sharded(X, plan, rank, d_max, eps, ctx=ctx)
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    clocks.wait_first()
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launches
    e0.record(stream)
    ds = []
    for _ in range(args.steps):
        r = rd.decompose_sharded(X, plan, rank, d_max, eps, ctx=ctx)
        ds.append(r.d)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    t_max = ms
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = float(t.item())
    total = w.m * w.n * 8 * sum(ds)
    value = total / (t_max / 1e3) / 1e9

    # ---- e2e: this rank's shard from pinned host memory -> HBM, the sharded
    #      decompose, Y and T_local back; only where the host can pin the shards ----
    e2e = None
    shard_bytes = w.m * nl * 8
    avail = host_mem_available()
    local_ranks = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    if not args.no_e2e and avail and avail > 2.0 * shard_bytes * local_ranks:
        Xh_t = torch.empty((nl, w.m), dtype=torch.float64, pin_memory=True)
        Xh_t.copy_(X.t())
        Xd_t = X.t()                         # the device shard buffer, refilled every step
        Ke = max(1, min(args.e2e_steps, args.steps))
        barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        de = []
        for _ in range(Ke):
            Xd_t.copy_(Xh_t, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
            r = rd.decompose_sharded(X, plan, rank, d_max, eps, ctx=ctx)
            Yh = r.Y.cpu()
            Th = r.T_local.cpu()
            de.append(r.d)
        te = time.perf_counter() - t0
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([te], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        e2e = {"value": w.m * w.n * 8 * sum(de) / te / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": shard_bytes,
               "d2h_bytes_per_step": int(Yh.numel() * 8 + Th.numel() * 8),
               "ms_per_step": te * 1e3 / Ke, "steps": Ke,
               "entry": "pinned host shard -> HBM (copy engine), rd.decompose_sharded, Y and "
                        "T_local -> host; per rank, max over ranks"}
        del Xh_t
    elif not args.no_e2e:
        e2e = {"skipped": f"host RAM: {(avail or 0) / 1e9:.0f} GB available, the pinned shards "
                          f"need {2.0 * shard_bytes * local_ranks / 1e9:.0f} GB (2x {local_ranks} x "
                          f"{shard_bytes / 1e9:.1f} GB)"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # single-thread oracle on a column block of the same X (the whole 137 GB
        # does not fit the host): the first 2048 columns
        nb = min(nl, 2048)
        Xs = np.asfortranarray(X[:, :nb].cpu().numpy())
        ws = configs.Workload(w.name + f"[:, :{nb}]", w.m, nb, w.d_max, 0.0, 0.0, w.seed, w.describe)
        cpu = cpu_baseline_leg(Xs, ws, eps, min(d_max, nb), args.cpu_seconds)
        del Xs
    if rank == 0:
        peak, src = peak_hbm()
        per_gpu = value / world
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": workload_config(w, eps, world, d_max),
            "roofline": {"bound": "hbm", "achieved": per_gpu, "peak": peak, "unit": "GB/s",
                         "frac": per_gpu / peak, "traffic": None,
                         "kernel": "k_rbd_persistent<2,true> per step + NCCL record allgather + "
                                   "payload allreduce, 8-step CUDA graph",
                         "note": "per-GPU X bytes x steps / time", "peak_source": src},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": ctx.launches - launches0,
            "clocks": clk, "shard_cols": list(plan.n_locals), "d_per_step": ds,
            "step_graph": bool(r.result.reserved),
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    args = parse()
    rank, world, _ = dist_env()
    if args.impl == "reference":
        run_reference(args)
    elif default_workload(args, world).startswith("C3"):
        run_sharded(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
