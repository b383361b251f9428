"""Parse YS printf lines of the timing build (last sweep): per-mode median phase end times (us)
relative to the earliest block start.  Columns: start, gamma-issue, contraction, gamma-store,
chol, sB, apply, cluster."""
import sys

import numpy as np

rows = {}
for line in open(sys.argv[1]):
    if line.startswith("YS "):
        f = [int(x) for x in line.split()[1:]]
        rows.setdefault(f[0], []).append(f[2:])
for m, rs in sorted(rows.items()):
    a = np.array(rs[-128:], dtype=float)
    a[a == 0] = np.nan
    t0 = np.nanmin(a[:, 0])
    a = (a - t0) / 1000.0
    print(f"mode {m}: n={len(a)} medians " + " ".join(f"{np.nanmedian(a[:, c]):.2f}" for c in range(a.shape[1]))
          + "  max " + " ".join(f"{np.nanmax(a[:, c]):.2f}" for c in range(a.shape[1])))
