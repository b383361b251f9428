"""Distribution of the consumer-loop times of every CTA of the c4a streaming passes (timing build:
python tools/build_variant.py timing "-DCP_STREAM_TIMING=2" stream_mma_inst.cu;
CP_LIB_PATH=alt/timing/libcp.so python tools/one_c4a_sweep.py | python tools/cta_loop_times.py)."""
import collections
import re
import sys

rows = collections.defaultdict(list)
sweep = -1
for line in sys.stdin:
    if line.startswith("--- sweep"):
        sweep += 1
    m = re.match(r"\[cta (\d+) warp 0 op (\d+) sm (\d+)\] consumer: loop (\d+) cycles in (\d+) ns \((\d+) MHz\) wait_full (\d+) stages (\d+) start (\d+)", line)
    if m and sweep >= 1:
        c, op, sm, cyc, ns, mhz, wf, st, t0 = map(int, m.groups())
        rows[op].append((c, sm, ns / 1e3, mhz, wf / cyc, t0))
for op, r in rows.items():
    us = sorted(x[2] for x in r)
    n = len(us)
    t0 = min(x[5] for x in r)
    end = max(x[5] + x[2] * 1e3 for x in r)
    print(f"op {op}: {n} CTAs; loop us min {us[0]:.1f} p10 {us[n // 10]:.1f} median {us[n // 2]:.1f} p90 {us[9 * n // 10]:.1f} max {us[-1]:.1f}; "
          f"mean {sum(us) / n:.1f}; first start -> last end {(end - t0) / 1e3:.1f} us; start spread {(max(x[5] for x in r) - t0) / 1e3:.1f} us")
    # by SM parity / halves of the SM id range, and by row block (cta & 1)
    for name, key in (("sm < 74", lambda x: x[1] < 74), ("even cta (rb 0)", lambda x: x[0] % 2 == 0)):
        a = [x[2] for x in r if key(x)]
        b = [x[2] for x in r if not key(x)]
        if a and b:
            print(f"    {name}: mean {sum(a) / len(a):.1f} us ({len(a)}) vs {sum(b) / len(b):.1f} us ({len(b)})")
    slow = sorted(r, key=lambda x: -x[2])[:8]
    print("    slowest:", ", ".join(f"cta {x[0]} sm {x[1]} {x[2]:.1f}us wait {x[4]:.2f}" for x in slow))
    fast = sorted(r, key=lambda x: x[2])[:8]
    print("    fastest:", ", ".join(f"cta {x[0]} sm {x[1]} {x[2]:.1f}us wait {x[4]:.2f}" for x in fast))
