"""ctypes bindings of the CPU checker (oracle/) for the test-suite.

TEST INFRASTRUCTURE ONLY: the oracle is the parity checker, never the thing
measured or shipped.  ``liboracle.so`` is the C restatement (oracle/cct_oracle.c);
``_ref/libcctref.so`` is the reference's own tensor.cpp/gemm.cpp plus a shim
(oracle/ref_shim.cpp), present only where it was built.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))  # repo root
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libcctref.so")

_fp = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_L = C.c_long


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class Oracle:
    """The C restatement (oracle/cct_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        lib = C.CDLL(path)
        self.lib = lib
        lib.orc_uniform_fill.argtypes = [C.c_uint64, C.c_uint64, _fp, C.c_size_t]
        for name in ("orc_conv_fwd",):
            getattr(lib, name).argtypes = [_fp, _fp, _fp] + [_L] * 7
        lib.orc_conv_bwd_data.argtypes = [_fp, _fp, _fp] + [_L] * 7
        lib.orc_conv_bwd_weight.argtypes = [_fp, _fp, _fp] + [_L] * 7
        lib.orc_direct_convolve_batch.argtypes = [_fp, _L, _L, _L, _fp, _L, _L, _fp]
        lib.orc_multiply.argtypes = [_fp, _fp, _fp, _L, _L, _L]
        lib.orc_lowered_shape.argtypes = [C.c_int] + [_L] * 5 + [C.POINTER(_L)] * 3
        lib.orc_lower.argtypes = [C.c_int, _fp, _fp] + [_L] * 5 + [_fp, _fp]
        lib.orc_lift.argtypes = [C.c_int, _fp] + [_L] * 5 + [_fp]
        lib.orc_convolve_lowered.argtypes = [C.c_int, _fp, _fp] + [_L] * 5 + [_fp]
        lib.orc_estimate.argtypes = [C.c_int] + [_L] * 5 + [C.POINTER(C.c_uint64)] * 3
        lib.orc_lower_internal.argtypes = [C.c_int, _fp] + [_L] * 6 + [_fp, _L]
        for name in ("orc_lowered_fwd", "orc_lowered_bwd_data", "orc_lowered_bwd_weight"):
            getattr(lib, name).argtypes = [C.c_int, _fp, _fp, _fp] + [_L] * 7 + [C.c_void_p, C.c_void_p]

    # -- data -------------------------------------------------------------
    def uniform(self, seed: int, count: int, skip: int = 0) -> np.ndarray:
        out = np.empty(count, np.float32)
        self.lib.orc_uniform_fill(seed, skip, out, count)
        return out

    def random_problem(self, seed, b, n, d, k, o):
        """Same stream as DataBatch::random then KernelBank::random (tensor.cpp:39-64)."""
        v = self.uniform(seed, b * n * n * d + k * k * d * o)
        x = v[: b * n * n * d].copy()
        w = v[b * n * n * d:].copy()
        return x, w

    # -- convolution -------------------------------------------------------
    @staticmethod
    def m_of(n, k, s, p):
        return (n + 2 * p - k) // s + 1

    def direct_convolve_batch(self, x, b, n, d, w, k, o):
        m = n - k + 1
        y = np.empty(b * o * m * m, np.float32)
        rc = self.lib.orc_direct_convolve_batch(_f32(x), b, n, d, _f32(w), k, o, y)
        assert rc == 0
        return y

    def conv_fwd(self, x, w, b, n, d, k, o, s=1, p=0):
        m = self.m_of(n, k, s, p)
        y = np.empty(b * o * m * m, np.float32)
        assert self.lib.orc_conv_fwd(_f32(x), _f32(w), y, b, n, d, k, o, s, p) == 0
        return y

    def conv_bwd_data(self, dy, w, b, n, d, k, o, s=1, p=0):
        dx = np.empty(b * n * n * d, np.float32)
        assert self.lib.orc_conv_bwd_data(_f32(dy), _f32(w), dx, b, n, d, k, o, s, p) == 0
        return dx

    def conv_bwd_weight(self, x, dy, b, n, d, k, o, s=1, p=0):
        dw = np.empty(o * k * k * d, np.float32)
        assert self.lib.orc_conv_bwd_weight(_f32(x), _f32(dy), dw, b, n, d, k, o, s, p) == 0
        return dw

    def lowered(self, pass_, type_, a, bb, b, n, d, k, o, s=1, p=0):
        if pass_ == "fwd":
            m = self.m_of(n, k, s, p)
            out = np.empty(b * o * m * m, np.float32)
            fn = self.lib.orc_lowered_fwd
        elif pass_ == "bwd_data":
            out = np.empty(b * n * n * d, np.float32)
            fn = self.lib.orc_lowered_bwd_data
        else:
            out = np.empty(o * k * k * d, np.float32)
            fn = self.lib.orc_lowered_bwd_weight
        assert fn(type_, _f32(a), _f32(bb), out, b, n, d, k, o, s, p, None, None) == 0
        return out

    # -- gemm / lowering ---------------------------------------------------
    def multiply(self, A, B):
        A = _f32(A)
        B = _f32(B)
        M, K = A.shape
        K2, N = B.shape
        assert K == K2
        Cm = np.empty((M, N), np.float32)
        self.lib.orc_multiply(A, B, Cm, M, K, N)
        return Cm

    def lowered_shape(self, type_, b, n, d, k, o):
        r, c, kc = _L(), _L(), _L()
        rc = self.lib.orc_lowered_shape(type_, b, n, d, k, o, C.byref(r), C.byref(c), C.byref(kc))
        if rc:
            raise ValueError("invalid layer config")
        return r.value, c.value, kc.value

    def lower(self, type_, x, w, b, n, d, k, o):
        rows, cols, kcols = self.lowered_shape(type_, b, n, d, k, o)
        dh = np.empty((rows, cols), np.float32)
        kh = np.empty((cols, kcols), np.float32)
        assert self.lib.orc_lower(type_, _f32(x), _f32(w), b, n, d, k, o, dh, kh) == 0
        return dh, kh

    def lift(self, type_, rhat, b, n, d, k, o):
        m = n - k + 1
        y = np.empty(b * o * m * m, np.float32)
        assert self.lib.orc_lift(type_, _f32(rhat), b, n, d, k, o, y) == 0
        return y

    def convolve_lowered(self, type_, x, w, b, n, d, k, o):
        m = n - k + 1
        y = np.empty(b * o * m * m, np.float32)
        assert self.lib.orc_convolve_lowered(type_, _f32(x), _f32(w), b, n, d, k, o, y) == 0
        return y

    def estimate(self, type_, b, n, d, k, o):
        a, g, l_ = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.lib.orc_estimate(type_, b, n, d, k, o, C.byref(a), C.byref(g), C.byref(l_))
        return a.value, g.value, l_.value

    def lower_internal(self, type_, x, b, n, d, k, s, p):
        N = n + 2 * p
        m = (N - k) // s + 1
        R = s * (m - 1) + k
        rows, cols = {1: (b * m * m, k * k * d), 2: (b * R * m, k * d), 3: (b * R * R, d)}[type_]
        out = np.empty((rows, cols), np.float32)
        assert self.lib.orc_lower_internal(type_, _f32(x), b, n, d, k, s, p, out, cols) == 0
        return out


class Reference:
    """The reference's own tensor.cpp / gemm.cpp (oracle/_ref/libcctref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        lib = C.CDLL(path)
        self.lib = lib
        lib.ref_random_problem.argtypes = [C.c_ulonglong] + [_L] * 5 + [_fp, _fp]
        lib.ref_random_mat.argtypes = [C.c_ulonglong, _L, _L, _fp]
        lib.ref_direct_convolve_batch.argtypes = [_fp, _L, _L, _L, _fp, _L, _L, _fp]
        for name in ("ref_conv_fwd_adapter", "ref_conv_bwd_data_adapter", "ref_conv_bwd_weight_adapter"):
            getattr(lib, name).argtypes = [_fp, _fp, _fp] + [_L] * 7
        lib.ref_multiply.argtypes = [_fp, _fp, _fp, _L, _L, _L, _L]
        lib.ref_multiply_reference.argtypes = [_fp, _fp, _fp, _L, _L, _L]
        lib.ref_lowered.argtypes = [C.c_int, C.c_int, _L, _fp, _fp, _fp] + [_L] * 7
        lib.ref_gemm_throughput_probe.argtypes = [_L, _L, _L, _L, C.c_int]
        lib.ref_gemm_throughput_probe.restype = C.c_double
        lib.ref_memcpy_bandwidth_probe.argtypes = [_L, C.c_int]
        lib.ref_memcpy_bandwidth_probe.restype = C.c_double

    def random_problem(self, seed, b, n, d, k, o):
        x = np.empty(b * n * n * d, np.float32)
        w = np.empty(o * k * k * d, np.float32)
        assert self.lib.ref_random_problem(seed, b, n, d, k, o, x, w) == 0
        return x, w

    def random_mat(self, seed, rows, cols):
        out = np.empty((rows, cols), np.float32)
        self.lib.ref_random_mat(seed, rows, cols, out)
        return out

    def direct_convolve_batch(self, x, b, n, d, w, k, o):
        m = n - k + 1
        y = np.empty(b * o * m * m, np.float32)
        assert self.lib.ref_direct_convolve_batch(_f32(x), b, n, d, _f32(w), k, o, y) == 0
        return y

    def conv_fwd(self, x, w, b, n, d, k, o, s=1, p=0):
        m = (n + 2 * p - k) // s + 1
        y = np.empty(b * o * m * m, np.float32)
        assert self.lib.ref_conv_fwd_adapter(_f32(x), _f32(w), y, b, n, d, k, o, s, p) == 0
        return y

    def conv_bwd_data(self, dy, w, b, n, d, k, o, s=1, p=0):
        dx = np.empty(b * n * n * d, np.float32)
        assert self.lib.ref_conv_bwd_data_adapter(_f32(dy), _f32(w), dx, b, n, d, k, o, s, p) == 0
        return dx

    def conv_bwd_weight(self, x, dy, b, n, d, k, o, s=1, p=0):
        dw = np.empty(o * k * k * d, np.float32)
        assert self.lib.ref_conv_bwd_weight_adapter(_f32(x), _f32(dy), dw, b, n, d, k, o, s, p) == 0
        return dw

    def multiply(self, A, B, threads=1):
        A = _f32(A)
        B = _f32(B)
        M, K = A.shape
        _, N = B.shape
        Cm = np.empty((M, N), np.float32)
        rc = self.lib.ref_multiply(A, B, Cm, M, K, N, threads)
        if rc == 1:
            raise ValueError("config_error")
        assert rc == 0
        return Cm

    def lowered(self, pass_, type_, a, bb, b, n, d, k, o, s=1, p=0, threads=1):
        idx = {"fwd": 0, "bwd_data": 1, "bwd_weight": 2}[pass_]
        m = (n + 2 * p - k) // s + 1
        size = {0: b * o * m * m, 1: b * n * n * d, 2: o * k * k * d}[idx]
        out = np.empty(size, np.float32)
        assert self.lib.ref_lowered(idx, type_, threads, _f32(a), _f32(bb), out, b, n, d, k, o, s, p) == 0
        return out


def grouped_fwd(orc, x, w, b, n, d, k, o, s, p, groups, bias=None, relu=False):
    """Grouped convolution + bias + ReLU (the layer extension) on
    the oracle: group j convolves input channels [j d/G, (j+1) d/G) with kernels
    [j o/G, (j+1) o/G) -- Caffe's `group` semantics (bvlc_reference_caffenet,
    PAPER.md:343, 401) -- then y = act(conv + bias).  Returns (b, o, m, m) float32."""
    dg, og = d // groups, o // groups
    m = (n + 2 * p - k) // s + 1
    xs = np.asarray(x, np.float32).reshape(b, n, n, d)
    ws = np.asarray(w, np.float32).reshape(o, k, k, dg)
    parts = [orc.conv_fwd(_f32(xs[..., j * dg:(j + 1) * dg]).ravel(), _f32(ws[j * og:(j + 1) * og]).ravel(),
                          b, n, dg, k, og, s, p).reshape(b, og, m, m) for j in range(groups)]
    y = np.concatenate(parts, axis=1)
    if bias is not None:
        y = y + np.asarray(bias, np.float32)[None, :, None, None]
    return np.maximum(y, 0).astype(np.float32) if relu else y.astype(np.float32)


def grouped_bwd(orc, dz, x, w, b, n, d, k, o, s, p, groups):
    """(dx, dw, db) of the grouped convolution for dz = the gradient at the conv output
    (the ReLU mask already applied).  dx (b, n, n, d), dw (o, k, k, d/G), db (o), fp64 db."""
    dg, og = d // groups, o // groups
    m = (n + 2 * p - k) // s + 1
    dzs = np.asarray(dz, np.float32).reshape(b, o, m, m)
    xs = np.asarray(x, np.float32).reshape(b, n, n, d)
    ws = np.asarray(w, np.float32).reshape(o, k, k, dg)
    dx = np.empty((b, n, n, d), np.float32)
    dw = np.empty((o, k, k, dg), np.float32)
    for j in range(groups):
        dzj = _f32(dzs[:, j * og:(j + 1) * og]).ravel()
        dx[..., j * dg:(j + 1) * dg] = orc.conv_bwd_data(dzj, _f32(ws[j * og:(j + 1) * og]).ravel(),
                                                         b, n, dg, k, og, s, p).reshape(b, n, n, dg)
        dw[j * og:(j + 1) * og] = orc.conv_bwd_weight(_f32(xs[..., j * dg:(j + 1) * dg]).ravel(), dzj,
                                                      b, n, dg, k, og, s, p).reshape(og, k, k, dg)
    db = dzs.astype(np.float64).sum(axis=(0, 2, 3))
    return dx, dw, db


def rel_l2(a, b) -> float:
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))
