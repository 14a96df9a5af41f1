#!/usr/bin/env python
"""Benchmark of the B200 RBD greedy loop (BASELINE.json metric: effective HBM
GB/s = X bytes x greedy steps / time).

One bench "step" = one full rbd::decompose of the workload (default C1, the
BASELINE config the metric is quoted on). `value` is device-resident (X in
HBM before the timed region); `e2e` goes through the reference-facing host
entry (numpy X in pinned memory -> H2D -> loop -> D2H of Y and T).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
For N > 1 launch under torchrun; C1 does not shard (replicas only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--workload", default="C1-image-like")
    p.add_argument("--cpu-seconds", type=float, default=15.0)
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-f32", action="store_true", help="skip the fp32 storage-mode line")
    p.add_argument("--d-max", type=int, default=None, help="override d_max (quick runs)")
    p.add_argument("--ref-seconds", type=float, default=6.0,
                   help="reference arm: CPU seconds of greedy steps per bench step")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


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


def ncu_traffic():
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
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


def make_workload(name, device):
    import torch
    from paper_1503_05947_b200 import configs
    w = configs.WORKLOADS[name]
    if name.startswith("C1"):
        Xd = configs.c1_matrix(n=w.n, seed=w.seed, device=device)
    elif name.startswith("C0"):
        Xh = configs.c0_matrix()
        Xd = torch.as_tensor(Xh.T.copy(), device=device).t()
    else:
        rank = {"C2-tall": 1024, "C3-sharded": 2048, "C4-out-of-sample": 512}[name]
        key = name.split("-")[0]
        Xd = configs.low_rank_matrix_torch(w.m, w.n, rank, configs.spectrum(key, rank),
                                           {"C2": 1e-8, "C3": 1e-10, "C4": 1e-6}[key], w.seed,
                                           device=device)
    if torch.device(device).type == "cuda":
        torch.cuda.synchronize(device)
    colmax = float(Xd.norm(dim=0).max())
    return w, Xd, configs.eps_for(w, colmax)


def cpu_baseline_sample(X_host, w, eps, seconds, nthreads):
    """Oracle (restated reference path, two X passes per step) on the first
    greedy steps of the same workload, bounded to ~`seconds` of CPU work."""
    import oracle
    t0 = time.perf_counter()
    oracle.decompose(X_host, w.d_max, eps, nthreads=nthreads, max_steps=2)
    per = max((time.perf_counter() - t0) / 2.0, 1e-4)
    steps = int(max(2, min(w.d_max, seconds / per)))
    t0 = time.perf_counter()
    r = oracle.decompose(X_host, w.d_max, eps, nthreads=nthreads, max_steps=steps)
    dt = time.perf_counter() - t0
    return r.d, dt


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    import torch
    from paper_1503_05947_b200 import configs
    w = configs.WORKLOADS[args.workload]
    dev = torch.device("cuda", local) if torch.cuda.is_available() else torch.device("cpu")
    _, Xd, eps = make_workload(args.workload, dev)
    X = np.asfortranarray(Xd.cpu().numpy())
    del Xd
    cores = os.cpu_count() or 1
    import oracle
    # bounded sample per step: the first S greedy steps of the full workload
    t0 = time.perf_counter()
    oracle.decompose(X, w.d_max, eps, nthreads=cores, max_steps=2)
    per = max((time.perf_counter() - t0) / 2.0, 1e-4)
    S = int(max(2, min(w.d_max, args.ref_seconds / per)))
    for _ in range(args.warmup):
        oracle.decompose(X, w.d_max, eps, nthreads=cores, max_steps=S)
    t0 = time.perf_counter()
    done = 0
    for _ in range(args.steps):
        r = oracle.decompose(X, w.d_max, eps, nthreads=cores, max_steps=S)
        done += r.d
    dt = time.perf_counter() - t0
    bytes_per = w.m * w.n * 8
    val = bytes_per * done / dt / 1e9
    sample = f"first {S} greedy steps of {w.name} per bench step ({w.m}x{w.n} fp64)"
    line = {
        "impl": "reference", "metric": "rbd_effective_hbm_gbs", "value": val, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "m": w.m, "n": w.n, "d_max": w.d_max, "eps_R": eps},
        "cpu_baseline": {"value": val, "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(args):
    import torch
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    import paper_1503_05947_b200 as rbd
    from paper_1503_05947_b200._lib import load_library
    import ctypes as C

    w, Xd, eps = make_workload(args.workload, dev)
    ctx = rbd.Context(local)
    lib = load_library()
    m, n = Xd.shape
    bytes_per_gstep = m * n * 8

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    for _ in range(max(args.warmup, 0)):
        g = rbd.decompose(Xd, d_max=w.d_max, eps_r=eps, ctx=ctx)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    clocks.wait_first()
    launches0 = ctx.launches
    e0.record(stream)
    ds = []
    loop_ms = []
    for _ in range(args.steps):
        g = rbd.decompose(Xd, d_max=w.d_max, eps_r=eps, ctx=ctx)
        ds.append(g.d)
        loop_ms.append(g.result.loop_ms)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    clk = clocks.stop()
    launches = ctx.launches - launches0
    ms = e0.elapsed_time(e1)
    t_max = ms
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = float(t.item())
    total_bytes = bytes_per_gstep * sum(ds) * world
    value = total_bytes / (t_max / 1e3) / 1e9

    # ---- roofline of the dominant kernel ----
    # Inside the timed region the only kernels are K1 (init, 2 launches) and
    # k_rbd_persistent (the whole greedy loop, 1 launch per decompose). Its
    # algorithmic bytes per launch = m*n*8 per greedy step (X read once) x d;
    # its duration is the CUDA-event time around the launch (loop_ms).
    peak, peak_src = peak_hbm()
    d_mean = float(np.mean(ds))
    loop_mean = float(np.mean(loop_ms))
    alg_bytes = bytes_per_gstep * d_mean
    ach = alg_bytes / (loop_mean / 1e3) / 1e9
    traffic = ncu_traffic()
    roofline = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": (traffic or {}).get("bytes_per_launch"),
                "kernel": "k_rbd_persistent<2> (whole greedy loop, 1 launch/decompose)",
                "algorithmic_bytes_per_launch": alg_bytes,
                "algorithmic_bytes_note": "m*n*8 per greedy step x d (X read once per step); "
                                          "Y passes and bookkeeping not credited",
                "ms_per_launch": loop_mean, "peak_source": peak_src,
                "traffic_source": (traffic or {}).get("source")}
    # the fused sweep phase alone, as a standalone kernel (K2), CUDA events
    y = torch.randn(m, dtype=torch.float64, device=dev)
    y /= y.norm()
    torch.cuda.synchronize(dev)
    ms_sweep = C.c_double()
    from paper_1503_05947_b200._lib import check
    check(lib.rbd_time_sweep(ctx.handle, C.c_void_p(Xd.data_ptr()), m, n, Xd.stride(1),
                             C.c_void_p(y.data_ptr()), 20, C.byref(ms_sweep)))
    sw = bytes_per_gstep / (ms_sweep.value / 1e3) / 1e9
    roofline["sweep_kernel"] = {"kernel": "k_sweep<2,MODE_DOT,stream> (K2 standalone)",
                                "achieved": sw, "frac": sw / peak, "ms_per_launch": ms_sweep.value,
                                "bytes_per_launch": bytes_per_gstep}
    # read-only HBM peak (the copy-based peak under-states a pure
    # read stream): a stock reduction over 4 GiB of fp64, best of 10
    rp = read_peak_gbs(dev)
    if rp:
        roofline["read_peak"] = {"gbs": rp, "frac": ach / rp,
                                 "how": "torch.sum over a 4 GiB fp64 buffer (read-only), best of 10, "
                                        "CUDA events"}
    roofline["frac_of_nominal"] = {"gbs": 7700.0, "frac": ach / 7700.0,
                                   "note": "nominal HBM3e 7.7 TB/s (HGX), B200_PROFILING.md"}

    # ---- fp32 storage mode (rbd_decompose_device_f32), same workload rounded
    #      to fp32: half the X bytes per sweep, fp64 arithmetic; reported beside
    #      the fp64 headline (metric bytes at 4 B/element) ----
    f32_mode = None
    if not args.no_f32:
        Xf = Xd.float()
        for _ in range(2):
            gf = rbd.decompose(Xf, d_max=w.d_max, eps_r=eps, ctx=ctx)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        fl, fd = [], []
        for _ in range(max(1, args.steps)):
            gf = rbd.decompose(Xf, d_max=w.d_max, eps_r=eps, ctx=ctx)
            fd.append(gf.d)
            fl.append(gf.result.loop_ms)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        msf = e0.elapsed_time(e1)
        fbytes = m * n * 4
        floop = float(np.mean(fl))
        f32_mode = {"storage": "f32 X, f64 arithmetic (rbd_decompose_device_f32)",
                    "value": fbytes * sum(fd) / (msf / 1e3) / 1e9, "unit": "GB/s",
                    "ms_per_step": msf / len(fd), "loop_ms_mean": floop,
                    "roofline_frac": fbytes * float(np.mean(fd)) / (floop / 1e3) / 1e9 / peak,
                    "d_reached": int(np.mean(fd)),
                    "same_selection_as_f64_run_on_f32_values": None}
        g64 = rbd.decompose(Xf.double(), d_max=w.d_max, eps_r=eps, ctx=ctx)
        f32_mode["same_selection_as_f64_run_on_f32_values"] = g64.selected == gf.selected
        if not args.no_e2e:   # host entry with a pinned float32 X (half the PCIe bytes)
            Xh32_t = torch.empty((n, m), dtype=torch.float32, pin_memory=True)
            Xh32_t.copy_(Xf.t())
            Xh32 = Xh32_t.numpy().T
            K = max(1, args.steps)
            import gc
            warm = rbd.decompose_many([Xh32] * K, d_max=w.d_max, eps_r=eps, ctx=ctx)
            del warm
            gc.collect()
            t0 = time.perf_counter()
            outs = rbd.decompose_many([Xh32] * K, d_max=w.d_max, eps_r=eps, ctx=ctx)
            te = (time.perf_counter() - t0) * 1e3
            fe = [o.d for o in outs]
            del outs
            gc.collect()
            f32_mode["e2e"] = {"value": fbytes * sum(fe) / (te / 1e3) / 1e9, "unit": "GB/s",
                               "ms_per_step": te / len(fe), "h2d_bytes_per_step": m * n * 4,
                               "entry": "rbd_decompose_host_many_f32 (numpy float32, pinned)"}
            del Xh32_t, Xh32
        del Xf, g64
        torch.cuda.empty_cache()

    # ---- e2e through the reference-facing host entry (pinned host X) ----
    e2e = None
    if not args.no_e2e:
        Xh_t = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
        Xh_t.copy_(Xd.t())
        Xh = Xh_t.numpy().T  # (m, n) Fortran view, pinned
        assert Xh.flags["F_CONTIGUOUS"]
        # warm-up: device buffers and the pinned host outputs (the caching host
        # allocator serves the alternating output sets from its cache afterwards)
        for _ in range(max(3, args.warmup)):
            g2 = rbd.decompose(Xh, d_max=w.d_max, eps_r=eps, ctx=ctx)
        barrier()
        torch.cuda.synchronize(dev)
        e0.record(stream)
        t0 = time.perf_counter()
        d2 = []
        for _ in range(max(1, args.steps)):
            g2 = rbd.decompose(Xh, d_max=w.d_max, eps_r=eps, ctx=ctx)
            d2.append(g2.d)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        wall = time.perf_counter() - t0
        ms2 = e0.elapsed_time(e1)
        t2 = max(ms2, wall * 1e3)
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([t2], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t2 = float(t.item())
        dmean = float(np.mean(d2))
        single = {"value": bytes_per_gstep * sum(d2) * world / (t2 / 1e3) / 1e9, "unit": "GB/s",
                  "ms_per_step": t2 / len(d2),
                  "entry": "rbd_decompose_host, one call per step (upload, loop, download in series)"}
        # the stream of inputs through the pipelined host entry: K matrices (the
        # pinned X, uploaded again for every step) in one rbd_decompose_host_many
        # call; the upload of matrix i+1 overlaps the loop of matrix i
        K = max(1, args.steps)
        import gc
        warm = rbd.decompose_many([Xh] * K, d_max=w.d_max, eps_r=eps, ctx=ctx)
        del warm
        gc.collect()
        barrier()
        torch.cuda.synchronize(dev)
        e0.record(stream)
        t0 = time.perf_counter()
        outs = rbd.decompose_many([Xh] * K, d_max=w.d_max, eps_r=eps, ctx=ctx)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        wall = time.perf_counter() - t0
        t3 = max(e0.elapsed_time(e1), wall * 1e3)
        d3 = [o.d for o in outs]
        del outs
        gc.collect()
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([t3], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t3 = float(t.item())
        e2e = {"value": bytes_per_gstep * sum(d3) * world / (t3 / 1e3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": m * n * 8,
               "d2h_bytes_per_step": int(8 * (m * dmean + dmean * n + 2 * dmean)),
               "ms_per_step": t3 / len(d3),
               "entry": "rbd_decompose_host_many (numpy, pinned; upload of step i+1 overlaps "
                        "the loop of step i)",
               "single_call": single}

    # ---- CPU baseline: oracle port, one thread, bounded sample (rank 0, N=1) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        X_host = np.asfortranarray(Xd.cpu().numpy())
        steps, dt = cpu_baseline_sample(X_host, w, eps, args.cpu_seconds, 1)
        cpu = {"value": bytes_per_gstep * steps / dt / 1e9, "unit": "GB/s", "cores": 1,
               "kind": "port",
               "sample": f"first {steps} greedy steps of {w.name} ({m}x{n} fp64), single-thread "
                         f"oracle restating decompose.cpp (two X passes per step), {dt:.1f}s"}

    if rank == 0:
        line = {
            "metric": "rbd_effective_hbm_gbs", "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": w.name, "m": m, "n": n, "d_max": w.d_max, "eps_R": eps,
                       "d_reached": int(np.mean(ds)), "parallelism": f"replicas{world}",
                       "l2": "inputs larger than L2 (X 627 MB vs 126 MB L2)",
                       "describe": w.describe},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk, "loop_ms_mean": float(np.mean(loop_ms)),
            "d_per_step": ds, "f32_mode": f32_mode,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_sharded(args):
    """C3: X sharded by contiguous column blocks over the ranks (NCCL payload
    allgather inside the library); weak per-GPU data, strong on the job."""
    import torch
    rank, world, local = dist_env()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    import paper_1503_05947_b200 as rbd
    from paper_1503_05947_b200 import configs, distributed as rd
    w = configs.WORKLOADS[args.workload]
    key = w.name.split("-")[0]
    rank_r = {"C2": 1024, "C3": 2048, "C4": 512}.get(key, 64)
    plan = rd.plan_shards(w.n, world)
    o, nl = plan.offsets[rank], plan.n_locals[rank]
    X = configs.low_rank_shard_torch(w.m, w.n, rank_r, configs.spectrum(key, rank_r),
                                     {"C2": 1e-8, "C3": 1e-10, "C4": 1e-6}.get(key, 1e-6), w.seed,
                                     o, nl, device=dev)
    torch.cuda.synchronize(dev)
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
        r = rd.decompose_sharded(X, plan, rank, d_max, 0.0, ctx=ctx)
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
        r = rd.decompose_sharded(X, plan, rank, d_max, 0.0, ctx=ctx)
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
    if rank == 0:
        peak, src = peak_hbm()
        per_gpu = value / world
        line = {
            "metric": "rbd_effective_hbm_gbs", "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": w.name, "m": w.m, "n": w.n, "d_max": d_max,
                       "d_reached": int(np.mean(ds)), "parallelism": f"colshard{world}",
                       "shard_cols": list(plan.n_locals), "describe": w.describe},
            "roofline": {"bound": "hbm", "achieved": per_gpu, "peak": peak, "unit": "GB/s",
                         "frac": per_gpu / peak, "traffic": None,
                         "kernel": "k_rbd_persistent<2,true> per step + payload allgather",
                         "note": "per-GPU X bytes x steps / time", "peak_source": src},
            "cpu_baseline": None, "e2e": None, "gpu_launches": ctx.launches - launches0,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.workload.startswith(("C2", "C3")):
        run_sharded(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
