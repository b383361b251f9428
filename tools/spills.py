"""Register / spill report of the stream kernels (ptxas -v):  python tools/spills.py [inst ...]"""
import os
import re
import subprocess
import sys

CSRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1111_6091_b200", "csrc")
insts = sys.argv[1:] or ["0", "1", "2", "3"]
for i in insts:
    r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                        "--expt-relaxed-constexpr", "-Xptxas", "-v", "-c", os.path.join(CSRC, f"stream_inst_{i}.cu"),
                        "-o", "/dev/null"], capture_output=True, text=True)
    cur = None
    for line in r.stderr.splitlines():
        m = re.search(r"Function properties for (\S+)", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur and "stream_kernel" in cur:
            t = re.search(r"stream_kernelILi(\d+)ELi(\d+)ELi(\d+)", cur)
            st, ld = int(m.group(1)), int(m.group(2))
            if st or ld:
                print(f"R={t.group(1):>2} V={t.group(2)} OP={t.group(3)}  spill st={st} ld={ld}")
