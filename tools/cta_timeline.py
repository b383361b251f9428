"""Per-CTA timeline of the streaming kernel from a CP_CTA_TIMELINE build (printf lines
'CTL op mode cta smid enter first loop_end exit', globaltimer ns).  Summarizes each launch:
duration, start spread, first-data latency, loop-end spread (tail), epilogue.
    python tools/cta_timeline.py log"""
import sys

import numpy as np

launches, cur, last_key = [], [], None
for line in open(sys.argv[1]):
    if not line.startswith("CTL "):
        continue
    f = line.split()
    op, mode, cta = int(f[1]), int(f[2]), int(f[3])
    t = [int(x) for x in f[5:9]]
    if cur and (cta in {c[2] for c in cur} or (op, mode) != last_key):
        launches.append(cur)
        cur = []
    cur.append((op, mode, cta, *t))
    last_key = (op, mode)
if cur:
    launches.append(cur)
for L in launches[-6:]:
    a = np.array([x[3:] for x in L], dtype=float)
    t0 = a[:, 0].min()
    a = (a - t0) / 1000.0
    print(f"op {L[0][0]} mode {L[0][1]} ctas {len(L)}: exit max {a[:, 3].max():.2f} us | enter max {a[:, 0].max():.2f}"
          f" | first data med {np.median(a[:, 1]):.2f} max {a[:, 1].max():.2f} | loop end min {a[:, 2].min():.2f}"
          f" med {np.median(a[:, 2]):.2f} p90 {np.percentile(a[:, 2], 90):.2f} max {a[:, 2].max():.2f}"
          f" | epilogue med {np.median(a[:, 3] - a[:, 2]):.2f}")
