"""Top SASS instructions by warp-stall samples from an ncu --page source csv.
    python tools/ncu_stalls.py src.csv [topN]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
ia, isrc = hdr.index("Address"), hdr.index("Source")
cols = {k: hdr.index(k) for k in ("Warp Stall Sampling (All Samples)", "stall_long_sb", "stall_wait",
                                  "stall_short_sb", "stall_math", "Instructions Executed")}
seen, data = set(), []
for r in rows[2:]:
    if len(r) < len(hdr) or r[ia] in seen or r[ia] == "Address":
        continue
    seen.add(r[ia])
    try:
        data.append((int(r[ia], 16), {k: float(r[i] or 0) for k, i in cols.items()}, r[isrc][:64]))
    except ValueError:
        continue
base = min(d[0] for d in data)
tot = sum(d[1]["Warp Stall Sampling (All Samples)"] for d in data) or 1
for a, m, src in sorted(data, key=lambda d: -d[1]["Warp Stall Sampling (All Samples)"])[:top]:
    print(f"{a - base:6x} {m['Warp Stall Sampling (All Samples)'] / tot * 100:5.1f}% long={m['stall_long_sb']:5.0f} "
          f"wait={m['stall_wait']:5.0f} short={m['stall_short_sb']:5.0f} math={m['stall_math']:4.0f} "
          f"ex={m['Instructions Executed']:9.0f} {src}")
