"""Loader of lib/libcp.so.  No fallback: a missing library or a failed load raises."""
import ctypes
import os

CP_MAX_N = 8
CP_MAX_R = 32
CP_OK, CP_EINVAL, CP_EDIM, CP_ENOTSPD, CP_ECUDA, CP_EWORKSPACE = 0, -1, -2, -3, -4, -5

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.environ.get("CP_LIB_PATH") or os.path.join(_HERE, "lib", "libcp.so")
_lib = None

# every symbol include/cp.h declares (checked by tests/test_capi_symbols.py)
EXPORTS = ["cp_workspace_bytes", "cp_norm2", "cp_mttkrp", "cp_als_sweep", "cp_als_sweeps",
           "cp_als_sweeps_then_gradient",
           "cp_mode_product_workspace_bytes", "cp_mode_product", "cp_fit", "cp_gradient",
           "cp_restrict_workspace_bytes", "cp_restrict_structured",
           "cp_last_launch_count", "cp_profile_enable", "cp_profile_read", "cp_normalize_sort",
           "cp_mg_default_params", "cp_mg_workspace_bytes", "cp_mg_solve",
           "cp_als_solve_workspace_bytes", "cp_als_solve", "cp_status_string", "cp_version"]


class CPError(RuntimeError):
    def __init__(self, code, what=""):
        self.code = code
        msg = _status(code)
        super().__init__(f"{what}: {msg} ({code})" if what else f"{msg} ({code})")


def _status(code):
    try:
        return lib().cp_status_string(int(code)).decode()
    except Exception:
        return "status"


def lib_path():
    return _LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"libcp.so not built ({_LIB}); run `python -m paper_1111_6091_b200.build` "
                              "or __graft_entry__.build() -- there is no CPU fallback")
        L = ctypes.CDLL(_LIB)
        vp, sz, i32, i64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32, ctypes.c_int64
        L.cp_workspace_bytes.argtypes = [vp]
        L.cp_workspace_bytes.restype = sz
        L.cp_norm2.argtypes = [vp, vp, vp, vp, sz, vp]
        L.cp_mttkrp.argtypes = [vp, vp, vp, i32, vp, vp, sz, vp]
        L.cp_als_sweep.argtypes = [vp, vp, vp, vp, vp, vp, vp, sz, vp]
        L.cp_als_sweeps.argtypes = [vp, vp, vp, vp, vp, i32, i32, vp, vp, sz, vp]
        L.cp_als_sweeps_then_gradient.argtypes = [vp, vp, vp, vp, vp, i32, i32, vp, vp, vp, vp, vp, sz, vp]
        L.cp_als_sweeps_then_gradient.restype = ctypes.c_int
        L.cp_mode_product_workspace_bytes.argtypes = [i32, vp, i32, i64]
        L.cp_mode_product_workspace_bytes.restype = sz
        L.cp_mode_product.argtypes = [i32, vp, vp, i32, vp, i64, vp, vp, sz, vp]
        L.cp_fit.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
        L.cp_gradient.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
        L.cp_restrict_workspace_bytes.argtypes = [i32, vp, i32]
        L.cp_restrict_workspace_bytes.restype = sz
        L.cp_restrict_structured.argtypes = [i32, vp, vp, i32, vp, vp, vp, vp, sz, vp]
        L.cp_restrict_structured.restype = ctypes.c_int
        for f in ["cp_norm2", "cp_mttkrp", "cp_als_sweep", "cp_als_sweeps", "cp_mode_product", "cp_fit", "cp_gradient",
                  "cp_last_launch_count", "cp_version"]:
            getattr(L, f).restype = ctypes.c_int
        L.cp_profile_enable.argtypes = [ctypes.c_int]
        L.cp_profile_enable.restype = ctypes.c_int
        L.cp_profile_read.argtypes = [vp, vp, vp]
        L.cp_profile_read.restype = ctypes.c_int
        L.cp_normalize_sort.argtypes = [vp, vp, i32, vp, vp, sz, vp]
        L.cp_normalize_sort.restype = ctypes.c_int
        L.cp_mg_default_params.argtypes = [vp]
        L.cp_mg_default_params.restype = None
        L.cp_mg_workspace_bytes.argtypes = [vp, vp]
        L.cp_mg_workspace_bytes.restype = sz
        L.cp_mg_solve.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
        L.cp_mg_solve.restype = ctypes.c_int
        L.cp_als_solve_workspace_bytes.argtypes = [vp]
        L.cp_als_solve_workspace_bytes.restype = sz
        L.cp_als_solve.argtypes = [vp, vp, vp, ctypes.c_double, i32, i32, vp, vp, sz, vp]
        L.cp_als_solve.restype = ctypes.c_int
        L.cp_status_string.argtypes = [ctypes.c_int]
        L.cp_status_string.restype = ctypes.c_char_p
        _lib = L
    return _lib
