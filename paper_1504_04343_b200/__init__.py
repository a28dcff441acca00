"""B200-native Caffe con Troll convolution hot path (lowering + tcgen05 3xTF32 GEMM).

The product is the native library ``_lib/libcct.so`` (CUDA kernels for sm_100a
+ the C ABI declared in ``include/cct.h``).  This module is a thin ctypes
binding of that ABI for callers that hold torch device tensors (tests, bench,
the multi-GPU driver): torch provides device memory, streams and
torch.distributed; every FLOP runs in libcct.so.  There is no fallback: if the
library is missing or the device is not sm_100, calls raise.

Layouts follow the reference containers (tensor.hpp): x/dx NHWC (b,n,n,d),
w/dw (o,k,k,d), y/dy NCHW (b,o,m,m).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

__all__ = [
    "lib", "ConvDesc", "CctError", "ConfigError", "ResourceError",
    "LOWER_AUTO", "LOWER_T1", "LOWER_T2", "LOWER_T3", "PASS_FWD", "PASS_BWD_DATA", "PASS_BWD_WEIGHT", "PASS_BWD",
    "ROWS_SPEC", "ROWS_INTERNAL", "NCHW", "NHWC", "TUNE", "set_tuning", "get_tuning", "reset_tuning", "tuning",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# $CCT_LIB_DIR selects another in-tree build of libcct.so (A/B profiling of kernel variants)
LIB_PATH = os.path.join(os.environ.get("CCT_LIB_DIR", os.path.join(_HERE, "_lib")), "libcct.so")

LOWER_AUTO, LOWER_T1, LOWER_T2, LOWER_T3 = 0, 1, 2, 3
PASS_FWD, PASS_BWD_DATA, PASS_BWD_WEIGHT, PASS_BWD = 0, 1, 2, 3
ROWS_SPEC, ROWS_INTERNAL = 0, 1
NCHW, NHWC = 0, 1  # cct_layout of y / dy
OK, ERR_CONFIG, ERR_RESOURCE, ERR_CUDA, ERR_UNSUPPORTED = 0, 1, 2, 3, 4
# cct_tuning keys (include/cct.h): explicit process-wide switches between measured variants
TUNE = {"split_producer": 0, "a_tmem": 1, "a_tmem_wide": 2, "cta_pairs": 3, "bn384": 4, "streamk": 5,
        "chain2": 6, "s2d": 7, "implicit_bwd": 8, "wgrad_swap": 9, "dgrad_swap": 10, "fwd_swap": 11,
        "trace_phases": 12, "gather": 13, "fused_t23": 14, "overlap": 15}


class CctError(RuntimeError):
    pass


class ConfigError(CctError):
    """Maps CCT_ERR_CONFIG / CCT_ERR_UNSUPPORTED (convlow::config_error, common.hpp:17-19)."""


class ResourceError(CctError):
    """Maps CCT_ERR_RESOURCE / CCT_ERR_CUDA (convlow::resource_error, common.hpp:22-24)."""


class ConvExt(C.Structure):
    """cct_conv_ext: channel groups and the bias / ReLU epilogue (include/cct.h)."""
    _fields_ = [("groups", C.c_int64), ("bias", C.c_void_p), ("relu", C.c_int)]


class _Desc(C.Structure):
    _fields_ = [(f, C.c_int64) for f in ("n", "k", "d", "o", "b", "stride", "pad", "m", "R", "layout")]


class CostEstimate(C.Structure):
    _fields_ = [
        ("lower_elements_written", C.c_uint64), ("gemm_flops", C.c_uint64), ("lift_adds", C.c_uint64),
        ("lowered_bytes", C.c_uint64), ("hbm_bytes", C.c_uint64), ("total_score", C.c_double),
        ("model_seconds", C.c_double),
    ]


class Calibration(C.Structure):
    _fields_ = [(f, C.c_double) for f in ("alpha", "beta", "hbm_bytes_per_s", "gemm_flops_per_s", "launch_s")]


_lib = None


def lib() -> C.CDLL:
    """Load libcct.so (raises if it was not built: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build() "
                          "(make -C paper_1504_04343_b200/csrc)")
    L = C.CDLL(LIB_PATH)
    P, I64, VP, SZ = C.POINTER, C.c_int64, C.c_void_p, C.c_size_t
    D = P(_Desc)
    sigs = {
        "cct_conv_desc_init": [D] + [I64] * 7,
        "cct_conv_desc_set_layout": [D, C.c_int],
        "cct_workspace_size": [D, C.c_int, C.c_int, P(SZ)],
        "cct_conv_fwd": [D, C.c_int, VP, VP, VP, VP, SZ, VP],
        "cct_conv_bwd_data": [D, C.c_int, VP, VP, VP, VP, SZ, VP],
        "cct_conv_bwd_weight": [D, C.c_int, VP, VP, VP, VP, SZ, VP],
        "cct_lowered_shape": [D, C.c_int, C.c_int, P(I64), P(I64), P(I64)],
        "cct_lower": [D, C.c_int, C.c_int, VP, VP, I64, VP],
        "cct_lower_khat": [D, C.c_int, VP, VP, VP],
        "cct_lift": [D, C.c_int, C.c_int, VP, I64, VP, VP],
        "cct_gemm": [I64, I64, I64, VP, I64, VP, I64, VP, I64, C.c_int, VP, SZ, VP],
        "cct_gemm_workspace_size": [I64, I64, I64, C.c_int, P(SZ)],
        "cct_gemm_passes": [I64, I64, I64, VP, I64, VP, I64, VP, I64, C.c_int, VP],
        "cct_select_lowering": [D, P(Calibration), C.c_int, P(C.c_int), P(CostEstimate)],
        "cct_lowered_cache_size": [D, C.c_int, P(SZ)],
        "cct_conv_fwd_cached": [D, C.c_int, VP, VP, VP, VP, SZ, VP, SZ, VP],
        "cct_conv_bwd": [D, C.c_int, VP, VP, VP, VP, VP, VP, VP, SZ, VP],
        "cct_estimate": [D, C.c_int, P(Calibration), C.c_int, P(CostEstimate)],
        "cct_workspace_size_ex": [D, C.c_int, P(ConvExt), C.c_int, P(SZ)],
        "cct_conv_fwd_ex": [D, C.c_int, P(ConvExt), VP, VP, VP, VP, SZ, VP],
        "cct_conv_bwd_ex": [D, C.c_int, P(ConvExt), VP, VP, VP, VP, VP, VP, VP, VP, SZ, VP],
    }
    for name, args in sigs.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = C.c_int
    L.cct_calibration_default.argtypes = [P(Calibration)]
    L.cct_calibration_default.restype = None
    L.cct_last_error.restype = C.c_char_p
    L.cct_abi_version.restype = C.c_int
    L.cct_set_workspace_limit.argtypes = [C.c_size_t]
    L.cct_set_workspace_limit.restype = None
    L.cct_get_workspace_limit.restype = C.c_size_t
    L.cct_set_implicit_lowering.argtypes = [C.c_int]
    L.cct_set_implicit_lowering.restype = None
    L.cct_get_implicit_lowering.restype = C.c_int
    L.cct_set_tuning.argtypes = [C.c_int, C.c_int]
    L.cct_set_tuning.restype = C.c_int
    L.cct_get_tuning.argtypes = [C.c_int]
    L.cct_get_tuning.restype = C.c_int
    L.cct_reset_tuning.restype = None
    L.cct_launch_count.restype = C.c_uint64
    L.cct_reset_launch_count.restype = None
    _lib = L
    return L


def check(status: int) -> None:
    if status == OK:
        return
    msg = lib().cct_last_error().decode()
    if status in (ERR_CONFIG, ERR_UNSUPPORTED):
        raise ConfigError(msg)
    raise ResourceError(msg)


@dataclass(frozen=True)
class ConvDesc:
    """LayerConfig (tensor.hpp:15-26) + stride/pad (defaults keep reference semantics)."""
    n: int
    k: int
    d: int
    o: int
    b: int
    stride: int = 1
    pad: int = 0
    layout: int = 0  # NCHW (OutputBatch) or NHWC y / dy

    def c(self) -> _Desc:
        d = _Desc()
        check(lib().cct_conv_desc_init(C.byref(d), self.n, self.k, self.d, self.o, self.b, self.stride, self.pad))
        if self.layout:
            check(lib().cct_conv_desc_set_layout(C.byref(d), self.layout))
        return d

    def y_shape(self) -> tuple[int, int, int, int]:
        """Shape of y / dy: (b, o, m, m) for NCHW, (b, m, m, o) for NHWC."""
        m = self.m
        return (self.b, m, m, self.o) if self.layout == NHWC else (self.b, self.o, m, m)

    @property
    def m(self) -> int:
        return (self.n + 2 * self.pad - self.k) // self.stride + 1

    def flops_per_pass(self) -> int:
        """Algorithmic flops of one pass: 2 m^2 k^2 d o per image (Eq. 1)."""
        return 2 * self.b * self.m ** 2 * self.k ** 2 * self.d * self.o


def workspace_size(desc: ConvDesc, lowering: int, pass_: int) -> int:
    out = C.c_size_t()
    check(lib().cct_workspace_size(C.byref(desc.c()), lowering, pass_, C.byref(out)))
    return out.value


def lowered_cache_size(desc: ConvDesc, lowering: int) -> int:
    out = C.c_size_t()
    check(lib().cct_lowered_cache_size(C.byref(desc.c()), lowering, C.byref(out)))
    return out.value


def set_tuning(key: str, value: int) -> None:
    """cct_set_tuning: select a measured kernel variant (see include/cct.h)."""
    check(lib().cct_set_tuning(TUNE[key], int(value)))


def get_tuning(key: str) -> int:
    return int(lib().cct_get_tuning(TUNE[key]))


def reset_tuning() -> None:
    lib().cct_reset_tuning()


class tuning:
    """Context manager: ``with tuning(split_producer=0): ...`` restores the old values on exit."""

    def __init__(self, **kv):
        self.kv = kv
        self.old = {}

    def __enter__(self):
        for k, v in self.kv.items():
            self.old[k] = get_tuning(k)
            set_tuning(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.old.items():
            set_tuning(k, v)
        return False


def launch_count() -> int:
    return int(lib().cct_launch_count())


def reset_launch_count() -> None:
    lib().cct_reset_launch_count()


def default_calibration() -> Calibration:
    cal = Calibration()
    lib().cct_calibration_default(C.byref(cal))
    return cal


def select_lowering(desc: ConvDesc, pass_: int = 3, cal: Calibration | None = None):
    """select_strategy: returns (type, [CostEstimate x 3])."""
    cal = cal or default_calibration()
    out = C.c_int()
    est = (CostEstimate * 3)()
    check(lib().cct_select_lowering(C.byref(desc.c()), C.byref(cal), pass_, C.byref(out), est))
    return out.value, list(est)


def estimate(desc: ConvDesc, lowering: int, pass_: int = 0, cal: Calibration | None = None) -> CostEstimate:
    cal = cal or default_calibration()
    est = CostEstimate()
    check(lib().cct_estimate(C.byref(desc.c()), lowering, C.byref(cal), pass_, C.byref(est)))
    return est
