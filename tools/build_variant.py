"""A/B build: libcp.so with extra -D flags on selected sources, into alt/<name>/libcp.so (git-ignored;
travels to the GPU box).  The other objects are reused from paper_1111_6091_b200/lib/obj.
    python tools/build_variant.py NAME "-DCP_AB_NOFCM" stream_mma_inst.cu [more.cu ...]
Run with CP_LIB_PATH=alt/NAME/libcp.so."""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1111_6091_b200 import build as b  # noqa: E402

name, flags, srcs = sys.argv[1], sys.argv[2].split(), sys.argv[3:]
out = os.path.join(ROOT, "alt", name)
os.makedirs(out, exist_ok=True)
objs = []
for src in sorted(glob.glob(os.path.join(b.CSRC, "*.cu"))):
    base = os.path.basename(src)
    if base in srcs:
        obj = os.path.join(out, base[:-3] + ".o")
        subprocess.check_call([b.NVCC] + b.ARCH + b.FLAGS + flags + ["-c", src, "-o", obj])
    else:
        obj = os.path.join(b.OBJDIR, base[:-3] + ".o")
    objs.append(obj)
lib = os.path.join(out, "libcp.so")
subprocess.check_call([b.NVCC] + b.ARCH + ["-shared", "-o", lib] + objs + ["-lcudart_static"])
print(lib)
