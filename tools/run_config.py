"""Generate a BASELINE workload on the GPU, decompose it once (plus warm-up),
print timing and full-size, size-independent properties:
orthonormality of Y, T == Y'X on sampled columns, monotone history,
distinct selected columns. Usage: tools/run_config.py C2-tall [d_max] [reps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_05947_b200 as rbd  # noqa: E402
from paper_1503_05947_b200 import configs  # noqa: E402


def make(name, dev, f32=False):
    w = configs.WORKLOADS[name]
    key = name.split("-")[0]
    t0 = time.time()
    if f32 and key == "C3":   # 64 GiB in fp32: generated shard by shard (fp64 never whole)
        rank = 2048
        X = torch.empty((w.n, w.m), dtype=torch.float32, device=dev).t()
        for o in range(0, w.n, 8192):
            blk = configs.low_rank_shard_torch(w.m, w.n, rank, configs.spectrum(key, rank), 1e-10,
                                               w.seed, o, min(8192, w.n - o), device=dev)
            X[:, o:o + blk.shape[1]] = blk
            del blk
        torch.cuda.synchronize()
        print(f"[gen] {name} fp32 {tuple(X.shape)} in {time.time() - t0:.1f}s", flush=True)
        return w, X
    if key == "C1":
        X = configs.c1_matrix(n=w.n, seed=w.seed, device=dev)
    elif key == "C0":
        X = torch.as_tensor(configs.c0_matrix().T.copy(), device=dev).t()
    else:
        rank = {"C2": 1024, "C3": 2048, "C4": 512}[key]
        X = configs.low_rank_matrix_torch(w.m, w.n, rank, configs.spectrum(key, rank),
                                          {"C2": 1e-8, "C3": 1e-10, "C4": 1e-6}[key], w.seed,
                                          device=dev)
    torch.cuda.synchronize()
    print(f"[gen] {name} {tuple(X.shape)} {X.numel() * 8 / 1e9:.1f} GB in {time.time() - t0:.1f}s",
          flush=True)
    return w, X


def main():
    name = sys.argv[1]
    dev = torch.device("cuda:0")
    f32 = "--f32" in sys.argv   # fp32 storage mode: X rounded to fp32, fp64 arithmetic
    if f32:
        sys.argv.remove("--f32")
    w, X = make(name, dev, f32)
    if f32 and X.dtype != torch.float32:
        X32 = X.float()
        del X
        torch.cuda.empty_cache()
        X = X32
    es = 4 if f32 else 8
    d_max = int(sys.argv[2]) if len(sys.argv) > 2 else w.d_max
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    colnorm = torch.cat([X[:, i:i + 1024].double().norm(dim=0) for i in range(0, X.shape[1], 1024)])
    eps = configs.eps_for(w, float(colnorm.max()))
    ctx = rbd.Context(0)
    out = {}
    for r in range(reps):
        g = rbd.decompose(X, d_max=d_max, eps_r=eps, ctx=ctx)
        m, n = X.shape
        gbs = m * n * es * g.d / (g.result.loop_ms / 1e3) / 1e9
        print(f"[run {r}] d={g.d} breakdown={g.result.breakdown} loop {g.result.loop_ms:.1f} ms "
              f"({g.result.loop_ms * 1e3 / max(g.d, 1):.1f} us/step) init {g.result.init_ms:.2f} ms "
              f"-> {gbs:.0f} GB/s", flush=True)
        out = {"workload": name, "storage": "f32" if f32 else "f64", "m": m, "n": n, "d": g.d,
               "loop_ms": g.result.loop_ms,
               "gbs": gbs, "breakdown": g.result.breakdown}
    Y, T = g.Y, g.T
    G = Y.t() @ Y
    out["orth_defect"] = float((G - torch.eye(g.d, device=dev, dtype=G.dtype)).abs().max())
    rng = np.random.default_rng(0)
    cols = torch.as_tensor(np.sort(rng.choice(X.shape[1], size=min(256, X.shape[1]), replace=False)),
                           device=dev)
    Td = Y.t() @ X[:, cols].double()
    out["T_rel_err"] = float(((Td - T[:, cols]).abs() / colnorm[cols]).max())
    h = np.asarray(g.residual_history)
    out["history_monotone"] = bool(np.all(h[1:] <= h[:-1] * (1 + 1e-12) + 1e-12 * float(colnorm.max())))
    out["selected_distinct"] = len(set(g.selected)) == g.d
    out["e_first_last"] = [float(h[0]), float(h[-1])]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
