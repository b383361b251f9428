"""Summarize an ncu --page source csv: stall samples per instruction and per region.
    ncu -i rep --page source --csv --print-source sass > s.csv; python tools/ncu_source_summary.py s.csv [topN]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
ia, isrc, iss, iex = (hdr.index("Address"), hdr.index("Source"),
                      hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"))
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h]
seen, data = set(), []
for r in rows[2:]:
    if len(r) <= iex or r[ia] in seen:
        continue
    seen.add(r[ia])
    try:
        s = float(r[iss] or 0)
    except ValueError:
        continue
    data.append((int(r[ia], 16), s, r[isrc][:70], r[iex]))
data.sort()
tot = sum(d[1] for d in data) or 1
base = data[0][0]
print("total samples", tot)
for a, s, src, ex in sorted(data, key=lambda d: -d[1])[:top]:
    print(f"{a - base:6x} {s / tot * 100:5.1f}% ex={ex:>9s} {src}")
