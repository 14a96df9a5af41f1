"""The bench.py contract: one JSON line per run with the keys the driver reads.
CPU: the reference arm (oracle port, all host cores) on the small C0 workload.
GPU: our arm on the C1 workload (the default C2-tall takes minutes), shortened."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config"}


def run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run(["--impl", "reference", "--workload", "C0-cpu-ref", "--steps", "1", "--warmup", "0",
             "--ref-seconds", "0.5"], 300)
    assert BASE <= set(d)
    assert d["impl"] == "reference" and d["metric"] == "rbd_effective_hbm_gbs"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["dtype"] == "f64"
    assert d["config"]["workload"] == "C0-cpu-ref"
    assert set(d["config"]) >= {"workload", "m", "n", "d_max", "eps_R", "parallelism"}
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(cb) and cb["kind"] == "port"
    assert cb["value"] == d["value"] and cb["cores"] >= 1
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0 == e["d2h_bytes_per_step"]


@pytest.mark.gpu
def test_b200_arm_line(cuda):
    d = run(["--workload", "C1-image-like", "--steps", "2", "--warmup", "3", "--cpu-seconds", "1",
             "--aux-steps", "1", "--no-secondary"], 900)
    assert BASE <= set(d) and "impl" not in d
    assert d["config"]["workload"] == "C1-image-like" and d["n_gpus"] == 1
    assert d["scaling"] == "weak" and d["data"] == "synthetic" and d["dtype"] == "f64"
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9 and 0.3 < r["frac"] < 1.2
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["value"] > 0 and cb["cores"] == 1
    assert cb["steps_sampled"] >= 1 and cb["cpu_model"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 32256 * 2432 * 8
    assert e["d2h_bytes_per_step"] > 0 and e["value"] < d["value"]
    assert d["gpu_launches"] >= 2 * d["steps"]
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)
