"""CPU-side checks of the C-ABI boundary: libcp.so loads, exports every symbol include/cp.h
declares, and rejects bad arguments synchronously (before touching the GPU).  No compute."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "cp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cp_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    import paper_1111_6091_b200 as cp
    return cp.lib()


def test_library_exports_every_header_symbol(L):
    syms = header_symbols()
    assert "cp_mttkrp" in syms and "cp_als_sweep" in syms and "cp_fit" in syms
    assert "cp_mode_product" in syms and "cp_norm2" in syms
    for name in syms:
        assert hasattr(L, name), f"libcp.so does not export {name}"
    from paper_1111_6091_b200._lib import EXPORTS
    assert sorted(EXPORTS) == syms


def test_version_and_status_strings(L):
    assert L.cp_version() == 1
    for code in (0, -1, -2, -3, -4, -5):
        assert len(L.cp_status_string(code)) > 0
    assert b"positive definite" in L.cp_status_string(-3)


def test_library_is_sm100a_native():
    """The shipped library holds sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess
    import paper_1111_6091_b200 as cp
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", cp.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _shape(N, R, dims):
    import paper_1111_6091_b200 as cp
    return cp._shape(dims, R) if N == len(dims) else None


@pytest.mark.parametrize("dims,R,code", [
    ((4, 5, 6), 0, -1),        # R < 1
    ((4, 5, 6), 33, -1),       # R > CP_MAX_R
    ((4,), 3, -1),             # N < 2 for MTTKRP
    ((4, 0, 6), 3, -2),        # a zero dimension
    ((4, -3, 6), 3, -2),
    ((1 << 26, 1 << 26), 3, -2),  # element count overflow guard
])
def test_mttkrp_rejects_bad_shapes(L, dims, R, code):
    import paper_1111_6091_b200 as cp
    s = cp._shape(dims, R)
    dummy = ctypes.c_void_p(256)
    arr = (ctypes.c_void_p * 8)(*([256] * 8))
    rc = L.cp_mttkrp(ctypes.byref(s), dummy, arr, 0, dummy, dummy, 1 << 20, None)
    assert rc == code


def test_rejects_null_pointers_and_bad_mode(L):
    import paper_1111_6091_b200 as cp
    s = cp._shape((4, 5, 6), 3)
    dummy = ctypes.c_void_p(256)
    arr = (ctypes.c_void_p * 8)(*([256] * 8))
    assert L.cp_mttkrp(ctypes.byref(s), None, arr, 0, dummy, dummy, 1 << 20, None) == -1
    assert L.cp_mttkrp(ctypes.byref(s), dummy, None, 0, dummy, dummy, 1 << 20, None) == -1
    assert L.cp_mttkrp(ctypes.byref(s), dummy, arr, 3, dummy, dummy, 1 << 20, None) == -1
    assert L.cp_mttkrp(ctypes.byref(s), dummy, arr, -1, dummy, dummy, 1 << 20, None) == -1
    assert L.cp_als_sweep(ctypes.byref(s), dummy, None, arr, None, dummy, dummy, 1 << 20, None) == -1
    assert L.cp_fit(ctypes.byref(s), dummy, dummy, arr, None, None, None, dummy, 1 << 20, None) == -1
    assert L.cp_mttkrp(None, dummy, arr, 0, dummy, dummy, 1 << 20, None) == -1
    dims = (ctypes.c_int64 * 3)(4, 5, 6)
    assert L.cp_mode_product(3, dims, dummy, 3, dummy, 2, dummy, None, 0, None) == -1
    assert L.cp_mode_product(3, dims, dummy, 0, dummy, 0, dummy, None, 0, None) == -1
    assert L.cp_mode_product(3, dims, None, 0, dummy, 2, dummy, None, 0, None) == -1
    bad = (ctypes.c_int64 * 3)(4, 0, 6)
    assert L.cp_mode_product(3, bad, dummy, 0, dummy, 2, dummy, None, 0, None) == -2


def test_binding_fails_loudly_without_library(monkeypatch, tmp_path):
    """No CPU fallback: a missing libcp.so is an ImportError, never a silent fallback."""
    import paper_1111_6091_b200._lib as l
    monkeypatch.setattr(l, "_LIB", str(tmp_path / "missing.so"))
    monkeypatch.setattr(l, "_lib", None)
    with pytest.raises(ImportError):
        l.lib()


def test_product_path_never_imports_oracle():
    """The product package shares no code with oracle/ (grep of its sources)."""
    pkg = os.path.join(ROOT, "paper_1111_6091_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "cp_oracle" not in txt and "liboracle" not in txt, f


def test_peaks_library_exports_header_symbols():
    """libcppeaks.so (bench.py's fp64 peak microbenchmarks, include/cp_peaks.h) loads and exports
    what its header declares; a bad argument is rejected before any CUDA call."""
    import paper_1111_6091_b200 as cp
    src = open(os.path.join(ROOT, "include", "cp_peaks.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    syms = sorted(set(re.findall(r"\b(cpp_[a-z0-9_]+)\s*\(", src)))
    assert syms == ["cpp_fp64_peaks", "cpp_launch_floor_us"]
    P = ctypes.CDLL(os.path.join(os.path.dirname(cp.lib_path()), "libcppeaks.so"))
    for name in syms:
        assert hasattr(P, name)
    a, b = ctypes.c_double(), ctypes.c_double()
    assert P.cpp_fp64_peaks(ctypes.byref(a), ctypes.byref(b), 0) == -1
    assert P.cpp_fp64_peaks(None, ctypes.byref(b), 1) == -1
    assert P.cpp_launch_floor_us(0, ctypes.byref(a)) == -1


def test_every_path_selector_is_documented_in_cp_h():
    """The environment switches the shipped library reads (path_flag's whitelist in csrc/capi.cu)
    are exactly the ones include/cp.h documents: no undocumented global changes a result path."""
    import re
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = open(os.path.join(root, "paper_1111_6091_b200", "csrc", "capi.cu")).read()
    m = re.search(r"kPaths\[\]\s*=\s*\{(.*?)\};", src, re.S)
    assert m, "path_flag whitelist not found"
    names = re.findall(r'"(CP_[A-Z0-9_]+)"', m.group(1))
    assert len(names) >= 10
    hdr = open(os.path.join(root, "include", "cp.h")).read()
    missing = [n for n in names if n not in hdr]
    assert not missing, f"selectors missing from include/cp.h: {missing}"
    # and every path_flag() call site uses a whitelisted name (others would silently return the default)
    used = set()
    for fn in os.listdir(os.path.join(root, "paper_1111_6091_b200", "csrc")):
        used |= set(re.findall(r'path_flag\("(CP_[A-Z0-9_]+)"', open(os.path.join(root, "paper_1111_6091_b200", "csrc", fn)).read()))
    assert used <= set(names), f"path_flag names not in the whitelist: {sorted(used - set(names))}"
