"""Markdown summary of `ncu --page raw --csv` exports (the .ncu-rep files of the closing captures
exceed gpurun's return limit, so the raw pages are exported on the GPU box):
    python tools/summarize_raw_csv.py OUT.md file_raw.csv:label ..."""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration us", 1e-3),
    ("dram__bytes_read.sum", "DRAM read MB", None),
    ("dram__bytes_write.sum", "DRAM write MB", None),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of ncu peak", 1),
    ("sm__inst_executed_pipe_fp64_op_dmma.avg.pct_of_peak_sustained_active", "DMMA pipe %", 1),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1),
    ("lts__t_sector_hit_rate.pct", "L2 hit %", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("launch__grid_size", "grid", 1),
    ("launch__block_size", "block", 1),
]
UNIT = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3,
        "ms": 1e3, "msecond": 1e3}


def main():
    out = sys.argv[1]
    lines = ["| capture | kernel | " + " | ".join(k[1] for k in KEYS) + " |", "|" + "---|" * (len(KEYS) + 2)]
    for spec in sys.argv[2:]:
        path, _, label = spec.partition(":")
        rows = list(csv.reader(open(path)))
        hdr, units, body = rows[0], rows[1], rows[2:]
        # DMMA pipe metric names vary: take any column with "dmma" in it
        dm = [h for h in hdr if "dmma" in h and "pct" in h]
        for r in body:
            vals = []
            for key, _, scale in KEYS:
                k = key
                if key.startswith("sm__inst_executed_pipe_fp64_op_dmma") and key not in hdr and dm:
                    k = dm[0]
                if k not in hdr:
                    vals.append("-")
                    continue
                i = hdr.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    vals.append(r[i])
                    continue
                u = units[i]
                if scale is None or "duration" in key:
                    v *= UNIT.get(u, 1.0)
                vals.append(f"{v:.1f}" if abs(v) < 1e5 else f"{v:.3g}")
            lines.append(f"| {label} | {r[hdr.index('Kernel Name')][:44]} | " + " | ".join(vals) + " |")
    open(out, "a").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
