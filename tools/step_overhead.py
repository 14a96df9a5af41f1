"""Fixed per-step cost of the greedy loop on small inputs (latency floor)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1503_05947_b200 as rbd  # noqa: E402

ctx = rbd.Context(0)
for (m, n, d) in [(4096, 512, 500), (32256, 512, 500), (32256, 2432, 400)]:
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    X = torch.randn(n, m, dtype=torch.float64, device="cuda", generator=g).t()
    for it in range(2):
        r = rbd.decompose(X, d_max=d, ctx=ctx)
    print(f"m={m} n={n} d={r.d}: loop {r.result.loop_ms:.2f} ms = {1e3 * r.result.loop_ms / r.d:.1f} us/step",
          flush=True)
