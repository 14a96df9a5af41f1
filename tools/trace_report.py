"""Summarise a persistent-kernel trace (RBD_TRACE_STEP / RBD_TRACE_FILE; the
library must be built with RBD_NVCC_DEFS=-DRBD_INSTRUMENT=1), per step."""
import sys

import numpy as np

raw = open(sys.argv[1], "rb").read()
G = int(np.frombuffer(raw[:4], dtype=np.int32)[0])
W = 256
h = np.frombuffer(raw[4:], dtype=np.uint64).reshape(G, W)
steps = [[], []]
for c in range(G):
    cnt = int(h[c, 0])
    si = 0
    for w in h[c, 1:1 + cnt]:
        tag = int(w) >> 40
        t = int(w) & 0xFFFFFFFFFF
        if si < 2:
            steps[si].append((c, tag & 0xFF, tag >> 8, t))
        if tag & 0xFF == 10:
            si += 1
names = {1: "P1 start", 2: "P1 end", 3: "bar1 out", 6: "P2 end", 7: "bar2 out", 8: "P3 end",
         11: "decided", 12: "YAY row",
         9: "bar3 out", 10: "step end"}
for si, ev in enumerate(steps):
    if not ev:
        continue
    t0 = min(e[3] for e in ev if e[1] == 1)
    print(f"--- step {si}")
    for tag in [1, 2, 3, 11, 12, 6, 7, 8, 9, 10]:
        ts = np.array([e[3] - t0 for e in ev if e[1] == tag]) / 1e3
        if len(ts):
            print(f"{names[tag]:10s} min={ts.min():8.2f} med={np.median(ts):8.2f} max={ts.max():8.2f} us")
    dur = []
    for c in range(G):
        cur = None
        for e in [e for e in ev if e[0] == c]:
            if e[1] == 4:
                cur = e
            elif e[1] == 5 and cur is not None:
                dur.append(((e[3] - cur[3]) / 1e3, cur[2], c, (cur[3] - t0) / 1e3))
                cur = None
    ntile = max(x[1] for x in dur) + 1
    d = np.array([x[0] for x in dur])
    print(f"tiles: n={len(d)} (max id {ntile - 1}) mean={d.mean():.2f} p50={np.median(d):.2f} "
          f"p90={np.percentile(d, 90):.2f} max={d.max():.2f} us")
    ylong = sorted(dur, key=lambda x: x[1])[:3]
    print("first tiles (dur, id, cta, start):", [(round(a, 1), b, c, round(s, 1)) for a, b, c, s in ylong])
    late = sorted(dur, key=lambda x: -(x[3] + x[0]))[:5]
    print("last-finishing tiles (dur, id, cta, start):", [(round(a, 1), b, c, round(s, 1)) for a, b, c, s in late])
    per_cta = {}
    for x in dur:
        per_cta[x[2]] = per_cta.get(x[2], 0) + 1
    cnts = np.array(list(per_cta.values()))
    print(f"tiles per CTA: min={cnts.min()} max={cnts.max()} mean={cnts.mean():.1f}")
