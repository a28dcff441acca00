"""CPU: the C-ABI library (libcct.so) -- loads, exports every symbol declared in
include/*.h, validates like the reference (LayerConfig::validate, tensor.cpp:23-30;
check_multiply_dims, gemm.cpp:19-34), sizes workspaces, and implements the cost
model.  No compute call runs here: without a GPU every compute
entry point must fail loudly (there is no CPU fallback)."""
import ctypes as C
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        for m in re.finditer(r"CCT_API\s+[\w\s\*]+?\b(cct_\w+)\s*\(", open(h).read()):
            syms.add(m.group(1))
    return sorted(syms)


def test_every_declared_symbol_is_exported(cct):
    syms = header_symbols()
    assert len(syms) >= 20
    lib = cct.lib()
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, f"symbols declared in include/*.h but not exported: {missing}"


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_1504_04343_b200", "_lib", "libcct.so")
    data = open(so, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_abi_version(cct):
    assert cct.lib().cct_abi_version() == 1


@pytest.mark.parametrize("args", [
    (5, 6, 1, 1, 1, 1, 0),   # k > n + 2 pad
    (5, 0, 1, 1, 1, 1, 0),   # k < 1
    (5, 3, 0, 1, 1, 1, 0),   # d < 1
    (5, 3, 1, 0, 1, 1, 0),   # o < 1
    (5, 3, 1, 1, 0, 1, 0),   # b < 1
    (5, 3, 1, 1, 1, 0, 0),   # stride < 1
    (5, 3, 1, 1, 1, 1, -1),  # pad < 0
])
def test_invalid_layer_config_is_config_error(cct, args):
    with pytest.raises(cct.ConfigError) as e:
        cct.ConvDesc(*args).c()
    assert "invalid layer config" in str(e.value) and "n=5" in str(e.value)


def test_desc_derived_fields(cct):
    d = cct.ConvDesc(227, 11, 3, 96, 256, 4, 0).c()
    assert (d.m, d.R) == (55, 227)
    d = cct.ConvDesc(27, 5, 96, 256, 256, 1, 2).c()
    assert (d.m, d.R) == (27, 31)


def test_lowered_shapes_match_spec(cct):
    from paper_1504_04343_b200.conv import lowered_shape
    # SPEC.md:119-120
    assert lowered_shape(cct.ConvDesc(5, 3, 2, 1, 1), 1) == (9, 18, 1)
    assert lowered_shape(cct.ConvDesc(5, 3, 2, 4, 2), 3) == (50, 2, 36)
    assert lowered_shape(cct.ConvDesc(5, 3, 2, 4, 2), 2) == (50, 6, 12)
    with pytest.raises(cct.ConfigError):   # SPEC order is stride-1 / pad-0 only
        lowered_shape(cct.ConvDesc(5, 3, 2, 4, 2, 2, 0), 1)


def test_workspace_sizes(cct):
    L = cct.lib()
    old = L.cct_get_implicit_lowering()
    try:
        for implicit in (0, 1):
            L.cct_set_implicit_lowering(implicit)
            for t in (1, 2, 3):
                for p in (0, 1, 2):
                    small = cct.workspace_size(cct.ConvDesc(27, 5, 96, 256, 2, 1, 2), t, p)
                    big = cct.workspace_size(cct.ConvDesc(27, 5, 96, 256, 8, 1, 2), t, p)
                    if implicit and t == 1 and p == 0:
                        assert small == big  # implicit lowering: no Dhat, no scratch
                    else:
                        assert 0 < small < big  # footprint grows with the batch
            # implicit Type 1 keeps no lowered cache
            assert (cct.lowered_cache_size(cct.ConvDesc(27, 5, 96, 256, 8, 1, 2), 1) == 0) == bool(implicit)
    finally:
        L.cct_set_implicit_lowering(old)


def test_compute_without_gpu_fails_loudly(cct):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = cct.lib()
    d = cct.ConvDesc(9, 3, 4, 8, 2).c()
    fake = C.c_void_p(1 << 20)
    st = lib.cct_conv_fwd(C.byref(d), 1, fake, fake, fake, fake, 1 << 30, None)
    assert st == 3, "expected CCT_ERR_CUDA without a device (no CPU fallback)"


def test_gemm_argument_checks(cct):
    lib = cct.lib()
    fake = C.c_void_p(1 << 20)
    assert lib.cct_gemm(4, 4, 4, fake, 3, fake, 4, fake, 4, 1, None, 0, None) == 1  # lda < K
    assert lib.cct_gemm(4, 4, 6, fake, 6, fake, 4, fake, 4, 1, None, 0, None) == 1  # lda % 4
    assert b"16-byte" in lib.cct_last_error() or b"leading" in lib.cct_last_error()
    assert lib.cct_gemm(0, 4, 4, fake, 4, fake, 4, fake, 4, 1, None, 0, None) == 0  # empty: no-op


# ------------------------------------------------------------------ cost model
def test_estimate_counts_match_spec(cct):
    e = cct.estimate(cct.ConvDesc(5, 3, 2, 1, 1), 1)
    assert (e.lower_elements_written, e.gemm_flops, e.lift_adds) == (162, 324, 0)


def test_select_strategy_extremes(cct):
    # d >> o -> Type 3 ; d << o -> Type 1 (forward pass, the paper's setting)
    t_hi, _ = cct.select_lowering(cct.ConvDesc(13, 3, 384, 3, 256, 1, 1), 0)
    t_lo, _ = cct.select_lowering(cct.ConvDesc(13, 3, 3, 384, 256, 1, 1), 0)
    assert t_hi == 3 and t_lo == 1


def test_select_strategy_k1_tie_breaks_to_type1(cct):
    # k = 1: identical costs -> lowest type
    t, est = cct.select_lowering(cct.ConvDesc(13, 1, 64, 64, 32), 0)
    assert t == 1
    assert est[0].gemm_flops == est[1].gemm_flops == est[2].gemm_flops


def test_select_strategy_monotone_in_ratio(cct):
    # with d*o fixed, increasing d/o never switches from T3 back to T1
    seq = []
    for e in range(-6, 7):
        d = int(2 ** (8 + e / 2))
        o = max(1, int(2 ** 16 // d))
        seq.append(cct.select_lowering(cct.ConvDesc(13, 3, d, o, 64, 1, 0), 0)[0])
    first3 = next((i for i, t in enumerate(seq) if t == 3), len(seq))
    assert all(t != 1 for t in seq[first3:])


def test_select_scale_invariance(cct):
    # argmin invariant under uniform scaling of the calibration
    desc = cct.ConvDesc(27, 5, 96, 256, 64, 1, 2)
    cal = cct.default_calibration()
    t0, _ = cct.select_lowering(desc, 3, cal)
    cal.hbm_bytes_per_s *= 10
    cal.gemm_flops_per_s *= 10
    cal.launch_s /= 10
    t1, _ = cct.select_lowering(desc, 3, cal)
    assert t0 == t1


def test_split_k_request_is_normalised_to_running_splits():
    """CPU: a split-K request that would leave empty trailing splits (kb 6050 over 96 ->
    64 k-blocks each -> 95 run) is sized for the splits that actually run."""
    import ctypes as C
    import paper_1504_04343_b200 as cct
    out = C.c_size_t()
    M, N, K = 20, 30, 6050 * 16
    assert cct.lib().cct_gemm_workspace_size(M, N, K, 96, C.byref(out)) == 0
    assert out.value == 95 * M * N * 4
    assert cct.lib().cct_gemm_workspace_size(M, N, K, 50, C.byref(out)) == 0
    assert out.value == 50 * M * N * 4  # 121 k-blocks each: all 50 run


def test_tuning_switches_are_explicit():
    """CPU: the kernel-variant switches are set through the ABI (cct_set_tuning), range
    checked, and restored by cct_reset_tuning -- the library reads no environment."""
    import paper_1504_04343_b200 as cct
    L = cct.lib()
    cct.reset_tuning()
    defaults = {k: cct.get_tuning(k) for k in cct.TUNE}
    assert defaults["split_producer"] == 0 and defaults["fwd_swap"] == 0 and defaults["s2d"] == 1
    assert defaults["fused_t23"] == 0 and defaults["gather"] == 1
    assert L.cct_set_tuning(cct.TUNE["fused_t23"], 2) == 1
    with cct.tuning(s2d=2, split_producer=1):
        assert cct.get_tuning("s2d") == 2 and cct.get_tuning("split_producer") == 1
    assert {k: cct.get_tuning(k) for k in cct.TUNE} == defaults
    assert L.cct_set_tuning(7, 3) == 1          # out of range -> CCT_ERR_CONFIG
    assert b"out of range" in L.cct_last_error()
    assert L.cct_set_tuning(99, 0) == 1         # unknown key
    assert L.cct_get_tuning(99) == -1
    assert cct.get_tuning("s2d") == 1


def test_library_reads_no_environment():
    """CPU: no getenv in the library's own sources (results cannot depend on the caller's
    environment; the statically linked CUDA runtime's own CUDA_* handling is not ours)."""
    srcs = glob.glob(os.path.join(ROOT, "paper_1504_04343_b200", "csrc", "**", "*.c*"), recursive=True)
    assert srcs
    offenders = [p for p in srcs if "getenv" in open(p).read()]
    assert not offenders, offenders


def test_fused_t23_resolves_to_implicit_type1():
    """CPU: with CCT_TUNE_FUSED_T23 a Type 2 / 3 request on a layer with the implicit form
    (conv2, d = 96) sizes exactly like implicit Type 1 (no Rhat workspace, no lowered cache);
    conv1 (d = 3) keeps its materialised Type 2 / 3 sizes."""
    import paper_1504_04343_b200 as cct
    conv2 = cct.ConvDesc(27, 5, 96, 256, 32, 1, 2)
    conv1 = cct.ConvDesc(227, 11, 3, 96, 8, 4, 0)
    ws = lambda d, t: [cct.workspace_size(d, t, p) for p in range(3)]
    base2, base1 = {t: ws(conv2, t) for t in (1, 2, 3)}, {t: ws(conv1, t) for t in (1, 2, 3)}
    assert base2[3][0] > base2[1][0] and cct.lowered_cache_size(conv2, 3) > 0
    with cct.tuning(fused_t23=1):
        for t in (2, 3):
            assert ws(conv2, t) == base2[1] and cct.lowered_cache_size(conv2, t) == 0
            assert ws(conv1, t) == base1[t]
    assert ws(conv2, 3) == base2[3]
