"""Critical path of one sweep from a CP_CTA_TIMELINE build (CTK lines: tag block enter wait_released
exit, globaltimer ns): per launch, the earliest griddep release, the last block's exit and the gap
to the previous launch's end.  python tools/sweep_timeline.py log [launches to show]"""
import sys

import numpy as np

recs = {}
for line in open(sys.argv[1]):
    if line.startswith("CTK "):
        f = line.split()
        recs.setdefault(f[1], []).append([int(x) for x in f[2:6]])
launches = []
for tag, rs in recs.items():
    a = np.array(rs, dtype=np.int64)
    a = a[np.argsort(a[:, 2])]
    cut = [0] + [i for i in range(1, len(a)) if a[i, 2] - a[i - 1, 2] > 15000] + [len(a)]
    for lo, hi in zip(cut[:-1], cut[1:]):
        g = a[lo:hi]
        launches.append((int(g[:, 2].min()), int(np.median(g[:, 2])), int(g[:, 3].max()), tag, hi - lo))
launches.sort()
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
sel = launches[-n:]
t0 = sel[0][0]
prev_end = None
tot = 0.0
for w0, wmed, x1, tag, nb in sel:
    gap = (w0 - prev_end) / 1000 if prev_end is not None else 0.0
    print(f"{tag:10s} blocks {nb:4d}  released {(w0 - t0) / 1000:8.2f}  (median {(wmed - t0) / 1000:8.2f})"
          f"  end {(x1 - t0) / 1000:8.2f}  dur {(x1 - w0) / 1000:7.2f}  gap {gap:6.2f} us")
    prev_end = x1
