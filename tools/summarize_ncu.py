"""Summarize ncu reports into profiles/: per-kernel key metrics (markdown) and the DRAM traffic
per launch of the streaming kernel (profiles/ncu_traffic.json, read by bench.py).

    python tools/summarize_ncu.py OUT.md REP.ncu-rep[:label] ... [--traffic KEY]
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    traffic_key = None
    if "--traffic" in sys.argv:
        traffic_key = sys.argv[sys.argv.index("--traffic") + 1]
        args.remove(traffic_key)
    out_md = args[0]
    lines = ["| report | kernel | " + " | ".join(k[1] for k in KEYS) + " |",
             "|" + "---|" * (len(KEYS) + 2)]
    traffic = {}
    for spec in args[1:]:
        rep, _, label = spec.partition(":")
        hdr, units, rows = raw(rep)
        for r in rows:
            name = r[hdr.index("Kernel Name")][:40]
            vals = []
            for k, _ in KEYS:
                if k in hdr:
                    i = hdr.index(k)
                    vals.append(f"{r[i]} {units[i]}".strip())
                else:
                    vals.append("-")
            lines.append(f"| {label or os.path.basename(rep)} | {name} | " + " | ".join(vals) + " |")
            if "stream_" in name and label:
                def val(key):
                    i = hdr.index(key)
                    v = float(r[i].replace(",", ""))
                    u = units[i]
                    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                traffic.setdefault(label, []).append(val("dram__bytes_read.sum") + val("dram__bytes_write.sum"))
    with open(out_md, "a") as f:
        f.write("\n".join(lines) + "\n")
    if traffic_key is not None and traffic:
        path = os.path.join(os.path.dirname(out_md), "ncu_traffic.json")
        cur = json.load(open(path)) if os.path.exists(path) else {}
        # bench reads cur[workload]["dram_bytes_per_launch"]: average over the labelled modes
        vals = [v for t in traffic.values() for v in t]
        cur[traffic_key] = {"dram_bytes_per_launch": sum(vals) / len(vals), "per_launch": vals,
                            "source": [os.path.basename(a.partition(":")[0]) for a in args[1:]]}
        json.dump(cur, open(path, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
