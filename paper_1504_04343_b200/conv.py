"""Host-side mirror of the reference operator API over torch device tensors.

Names and argument meaning follow the reference's ``convlow`` API
(gemm.hpp:56-62): ``lower``, ``lift``, ``convolve_lowered``,
``multiply`` -- plus the backward passes the north star adds.  Each call goes
straight to libcct.so through the C ABI (include/cct.h) on torch's current
CUDA stream; torch only owns the memory.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import (LOWER_AUTO, PASS_BWD, PASS_BWD_DATA, PASS_BWD_WEIGHT, PASS_FWD, ROWS_INTERNAL, ROWS_SPEC,
               ConfigError, ConvDesc, ConvExt, check, lib, lowered_cache_size, workspace_size)

__all__ = ["Workspace", "conv_fwd", "conv_bwd_data", "conv_bwd_weight", "convolve_lowered", "lower",
           "conv_fwd_cached", "conv_bwd", "alloc_cache", "conv_fwd_ex", "conv_bwd_ex",
           "lower_khat", "lift", "lowered_shape", "multiply", "multiply_passes"]


def _ptr(t: torch.Tensor | None):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _need_cuda_f32(*ts):
    for t in ts:
        if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
            raise ConfigError("expected contiguous float32 CUDA tensors")


class Workspace:
    """Grow-only device scratch buffer sized by cct_workspace_size()."""

    def __init__(self, device=None):
        self.device = device
        self.buf: torch.Tensor | None = None

    def get(self, nbytes: int) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes:
            dev = self.device if self.device is not None else torch.cuda.current_device()
            self.buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
        return self.buf


_default_ws: dict[int, Workspace] = {}


def _ws(ws: Workspace | None, dev: torch.device) -> Workspace:
    if ws is not None:
        return ws
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    return _default_ws.setdefault(idx, Workspace(idx))


def _run(fn, desc: ConvDesc, lowering: int, pass_: int, a, b, out, ws, stream):
    _need_cuda_f32(a, b, out)
    nbytes = workspace_size(desc, lowering, pass_)
    buf = _ws(ws, a.device).get(nbytes)
    check(fn(C.byref(desc.c()), lowering, _ptr(a), _ptr(b), _ptr(out), _ptr(buf), buf.numel(), _stream(stream)))
    return out


def conv_fwd(x, w, desc: ConvDesc, lowering: int = LOWER_AUTO, out=None, ws=None, stream=None):
    """convolve_lowered: x (b,n,n,d) NHWC, w (o,k,k,d) -> y (b,o,m,m) NCHW."""
    m = desc.m
    y = out if out is not None else torch.empty(desc.y_shape(), dtype=torch.float32, device=x.device)
    return _run(lib().cct_conv_fwd, desc, lowering, PASS_FWD, x, w, y, ws, stream)


convolve_lowered = conv_fwd


def conv_bwd_data(dy, w, desc: ConvDesc, lowering: int = LOWER_AUTO, out=None, ws=None, stream=None):
    dx = out if out is not None else torch.empty((desc.b, desc.n, desc.n, desc.d), dtype=torch.float32,
                                                 device=dy.device)
    return _run(lib().cct_conv_bwd_data, desc, lowering, PASS_BWD_DATA, dy, w, dx, ws, stream)


def conv_bwd_weight(x, dy, desc: ConvDesc, lowering: int = LOWER_AUTO, out=None, ws=None, stream=None):
    dw = out if out is not None else torch.empty((desc.o, desc.k, desc.k, desc.d), dtype=torch.float32,
                                                 device=x.device)
    return _run(lib().cct_conv_bwd_weight, desc, lowering, PASS_BWD_WEIGHT, x, dy, dw, ws, stream)


def alloc_cache(desc: ConvDesc, lowering: int, device) -> torch.Tensor | None:
    """Buffer for the forward pass's Dhat (None when Dhat is the input itself)."""
    n = lowered_cache_size(desc, lowering)
    return torch.empty(n // 4, dtype=torch.float32, device=device) if n else None


def conv_fwd_cached(x, w, desc: ConvDesc, lowering: int = LOWER_AUTO, cache=None, out=None, ws=None, stream=None):
    """Forward that leaves Dhat in `cache` for conv_bwd (training step)."""
    _need_cuda_f32(x, w)
    m = desc.m
    y = out if out is not None else torch.empty(desc.y_shape(), dtype=torch.float32, device=x.device)
    nbytes = workspace_size(desc, lowering, PASS_FWD) if lowering else max(
        workspace_size(desc, t, PASS_FWD) for t in (1, 2, 3))
    buf = _ws(ws, x.device).get(nbytes)
    cb = cache.numel() * 4 if cache is not None else 0
    check(lib().cct_conv_fwd_cached(C.byref(desc.c()), lowering, _ptr(x), _ptr(w), _ptr(y), _ptr(cache), cb,
                                    _ptr(buf), buf.numel(), _stream(stream)))
    return y


def conv_bwd(dy, w, desc: ConvDesc, lowering: int = LOWER_AUTO, x=None, cache=None, dx=None, dw=None,
             want_dx=True, want_dw=True, ws=None, stream=None):
    """bwd-data + bwd-weight in one call: dy expanded once, Dhat from `cache` if given."""
    dev = dy.device
    if want_dx and dx is None:
        dx = torch.empty((desc.b, desc.n, desc.n, desc.d), dtype=torch.float32, device=dev)
    if want_dw and dw is None:
        dw = torch.empty((desc.o, desc.k, desc.k, desc.d), dtype=torch.float32, device=dev)
    nbytes = workspace_size(desc, lowering, PASS_BWD) if lowering else max(
        workspace_size(desc, t, PASS_BWD) for t in (1, 2, 3))
    buf = _ws(ws, dev).get(nbytes)
    check(lib().cct_conv_bwd(C.byref(desc.c()), lowering, _ptr(x), _ptr(cache), _ptr(dy), _ptr(w),
                             _ptr(dx if want_dx else None), _ptr(dw if want_dw else None), _ptr(buf), buf.numel(),
                             _stream(stream)))
    return dx, dw


def lowered_shape(desc: ConvDesc, lowering: int, order: int = ROWS_SPEC):
    r, c, kc = C.c_int64(), C.c_int64(), C.c_int64()
    check(lib().cct_lowered_shape(C.byref(desc.c()), lowering, order, C.byref(r), C.byref(c), C.byref(kc)))
    return r.value, c.value, kc.value


def lower(x, desc: ConvDesc, lowering: int, order: int = ROWS_SPEC, stream=None):
    """lower: the data-side matrix Dhat (rows x cols)."""
    _need_cuda_f32(x)
    rows, cols, _ = lowered_shape(desc, lowering, order)
    dh = torch.empty((rows, cols), dtype=torch.float32, device=x.device)
    check(lib().cct_lower(C.byref(desc.c()), lowering, order, _ptr(x), _ptr(dh), cols, _stream(stream)))
    return dh


def lower_khat(w, desc: ConvDesc, lowering: int, stream=None):
    """Khat of SPEC.md:112-114 (the transpose of the KernelBank storage)."""
    _need_cuda_f32(w)
    _, cols, kcols = lowered_shape(desc, lowering, ROWS_INTERNAL)
    kh = torch.empty((cols, kcols), dtype=torch.float32, device=w.device)
    check(lib().cct_lower_khat(C.byref(desc.c()), lowering, _ptr(w), _ptr(kh), _stream(stream)))
    return kh


def lift(rhat, desc: ConvDesc, lowering: int, order: int = ROWS_SPEC, stream=None):
    """lift: Rhat (rows x khat_cols) -> OutputBatch (b,o,m,m)."""
    _need_cuda_f32(rhat)
    m = desc.m
    y = torch.empty(desc.y_shape(), dtype=torch.float32, device=rhat.device)
    check(lib().cct_lift(C.byref(desc.c()), lowering, order, _ptr(rhat), rhat.shape[1], _ptr(y), _stream(stream)))
    return y


def _pad4(t: torch.Tensor) -> torch.Tensor:
    """Row stride multiple of 4 floats (TMA 16-byte strides)."""
    rows, cols = t.shape
    if cols % 4 == 0 and t.is_contiguous() and t.data_ptr() % 16 == 0:
        return t
    p = torch.zeros((rows, (cols + 3) // 4 * 4), dtype=t.dtype, device=t.device)
    p[:, :cols] = t
    return p


def multiply(a, b, split_k: int = 0, ws: Workspace | None = None, stream=None):
    """multiply (gemm.cpp:93): C = A B on the tensor cores, fp32-accurate (3xTF32)."""
    _need_cuda_f32(a.contiguous(), b.contiguous())
    M, K = a.shape
    K2, N = b.shape
    if K != K2:
        raise ConfigError(f"gemm dimension mismatch: A is {M}x{K}, B is {K2}x{N}")
    ap, bp = _pad4(a.contiguous()), _pad4(b.contiguous())
    c = torch.empty((M, N), dtype=torch.float32, device=a.device)
    need = C.c_size_t()
    check(lib().cct_gemm_workspace_size(M, N, K, split_k, C.byref(need)))
    buf = _ws(ws, a.device).get(need.value) if need.value else None
    check(lib().cct_gemm(M, N, K, _ptr(ap), ap.shape[1], _ptr(bp), bp.shape[1], _ptr(c), N, split_k,
                         _ptr(buf), buf.numel() if buf is not None else 0, _stream(stream)))
    return c


def multiply_passes(a, b, passes: int, stream=None):
    """Diagnostic: passes=1 is a single TF32 product (shows how the tensor core reads fp32)."""
    M, K = a.shape
    _, N = b.shape
    ap, bp = _pad4(a.contiguous()), _pad4(b.contiguous())
    c = torch.empty((M, N), dtype=torch.float32, device=a.device)
    check(lib().cct_gemm_passes(M, N, K, _ptr(ap), ap.shape[1], _ptr(bp), bp.shape[1], _ptr(c), N, passes,
                                _stream(stream)))
    return c


# ---------------------------------------------------------------- layer extension
def _ext(groups: int, bias, relu: bool) -> ConvExt:
    return ConvExt(int(groups), bias.data_ptr() if bias is not None else None, 1 if relu else 0)


def _ws_ex(desc: ConvDesc, lowering: int, ext: ConvExt, pass_: int) -> int:
    out = C.c_size_t()
    check(lib().cct_workspace_size_ex(C.byref(desc.c()), lowering, C.byref(ext), pass_, C.byref(out)))
    return out.value


def conv_fwd_ex(x, w, desc: ConvDesc, lowering: int = LOWER_AUTO, groups: int = 1, bias=None, relu: bool = False,
                out=None, ws=None, stream=None):
    """Grouped convolution + bias + ReLU (cct_conv_fwd_ex): x (b,n,n,d), w (o,k,k,d/groups),
    bias (o) or None -> y (b,o,m,m) = act(conv + bias)."""
    _need_cuda_f32(x, w, *([bias] if bias is not None else []))
    m = desc.m
    y = out if out is not None else torch.empty(desc.y_shape(), dtype=torch.float32, device=x.device)
    ext = _ext(groups, bias, relu)
    buf = _ws(ws, x.device).get(_ws_ex(desc, lowering, ext, PASS_FWD))
    check(lib().cct_conv_fwd_ex(C.byref(desc.c()), lowering, C.byref(ext), _ptr(x), _ptr(w), _ptr(y), _ptr(buf),
                                buf.numel(), _stream(stream)))
    return y


def conv_bwd_ex(dy, w, desc: ConvDesc, lowering: int = LOWER_AUTO, groups: int = 1, relu: bool = False, x=None,
                y=None, need_dx: bool = True, need_dw: bool = True, need_db: bool = False, ws=None, stream=None):
    """Backward of conv_fwd_ex: dy is the gradient of the layer output y (post-ReLU; y is needed
    when relu).  Returns (dx, dw, db), None for the gradients not requested."""
    dev = dy.device
    dx = torch.empty((desc.b, desc.n, desc.n, desc.d), dtype=torch.float32, device=dev) if need_dx else None
    dw = torch.empty((desc.o, desc.k, desc.k, desc.d // groups), dtype=torch.float32, device=dev) if need_dw else None
    db = torch.empty((desc.o,), dtype=torch.float32, device=dev) if need_db else None
    ext = _ext(groups, None, relu)
    pass_ = PASS_BWD if (need_dx and need_dw) else PASS_BWD_DATA if need_dx else PASS_BWD_WEIGHT
    buf = _ws(ws, dev).get(_ws_ex(desc, lowering, ext, pass_))
    check(lib().cct_conv_bwd_ex(C.byref(desc.c()), lowering, C.byref(ext), _ptr(x), _ptr(y), _ptr(dy), _ptr(w),
                                _ptr(dx), _ptr(dw), _ptr(db), _ptr(buf), buf.numel(), _stream(stream)))
    return dx, dw, db
