// gemm.cu -- warp-specialised, persistent tcgen05 GEMM with 3xTF32 split emulation.
//
// Replaces the reference GEMM (convlow::multiply, gemm.cpp:93-122; hot loop
// gemm_panel gemm.cpp:54-63, fp32 x fp32 -> double accumulate).  fp32 accuracy
// comes from the split a = a_big + a_small (a_big = a with the low 13 mantissa
// bits cleared, which is what the tensor core consumes when reading fp32 data
// as tf32) and three tensor-core products per K slice:
//     C += A_big*B_big + A_big*B_small + A_small*B_big      (fp32 accumulate in TMEM)
//
// CTA = 384 threads, one CTA per SM, persistent over output tiles (m fastest):
//   warp 0      TMA producer   (one lane): raw A/B tiles -> smem ring
//   warp 1      MMA issuer     (one lane): 3 x tcgen05.mma.kind::tf32 per 8-wide K step
//   warp 2      TMEM allocator
//   warps 4-7   epilogue: tcgen05.ld (TMEM lane quarter = warp%4) -> st.global
//   warps 8-11  transform: small = x - big for the A and B tiles of each stage
// Pipelines: smem ring full/tdone/empty (TMA -> transform -> MMA -> TMA) and a
// double-buffered TMEM accumulator tfull/tempty (MMA <-> epilogue), so the
// epilogue of tile i overlaps the MMAs of tile i+1.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "cct.h"
#include "common.cuh"
#include "gemm.cuh"
#include "ptx.cuh"

#include "gemm_kernel.cuh"

namespace cct {

using namespace gk;

namespace {

// ----------------------------------------------------------------------------
// host side
// ----------------------------------------------------------------------------

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// mn_extent x k_extent logical operand; box_mn rows per (K-major) tile
bool make_tmap(CUtensorMap* map, const Operand& op, int64_t mn_extent, int64_t k_extent, int box_mn) {
    auto enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2];
    cuuint64_t strides[1] = {cuuint64_t(op.ld) * 4};
    cuuint32_t box[2];
    cuuint32_t estr[2] = {1, 1};
    CUtensorMapSwizzle sw;
    if (op.major == Major::K) {
        dims[0] = cuuint64_t(k_extent);
        dims[1] = cuuint64_t(mn_extent);
        box[0] = kBK;
        box[1] = cuuint32_t(box_mn);
        sw = CU_TENSOR_MAP_SWIZZLE_64B;
    } else {
        dims[0] = cuuint64_t(mn_extent);
        dims[1] = cuuint64_t(k_extent);
        box[0] = 32;
        box[1] = kBK;
        sw = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
    }
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(op.ptr), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

PFN_cuTensorMapEncodeIm2col_v12000 encode_im2col_fn() {
    static PFN_cuTensorMapEncodeIm2col_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(p);
    }
    return fn;
}

// NHWC input as a 4D (c, w, h, n) im2col map: bounding box lower corner -p,
// upper corner p - (k - 1), traversal stride s (output pixels along W, H, N).
bool make_tmap_im2col(CUtensorMap* map, const Im2col& ic, bool mn_major, int box_pixels = kBM) {
    auto enc = encode_im2col_fn();
    if (!enc) return false;
    const int64_t cs = ic.cs ? ic.cs : ic.d;  // channel group of a wider tensor: extent d, stride cs
    cuuint64_t dims[4] = {cuuint64_t(ic.d), cuuint64_t(ic.n), cuuint64_t(ic.n), cuuint64_t(ic.b)};
    cuuint64_t strides[3] = {cuuint64_t(cs) * 4, cuuint64_t(ic.n * cs) * 4, cuuint64_t(ic.n * ic.n * cs) * 4};
    int lower[2] = {int(-ic.p), int(-ic.p)};
    int upper[2] = {int(ic.p - (ic.k - 1)), int(ic.p - (ic.k - 1))};
    cuuint32_t estr[4] = {1, cuuint32_t(ic.s), cuuint32_t(ic.s), 1};
    const cuuint32_t chans = mn_major ? 32 : kBK;
    const cuuint32_t pixels = mn_major ? kBK : cuuint32_t(box_pixels);
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(ic.x), dims, strides, lower, upper,
                     chans, pixels, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_64B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    // Older drivers mis-handle im2col maps of tensors < 128 KiB unless bit 21 of
    // the second descriptor word is cleared (same workaround as CUTLASS).
    int drv = 0;
    cudaDriverGetVersion(&drv);
    if (drv <= 13010 && ic.b * ic.n * ic.n * cs * 4 < 131072) reinterpret_cast<uint64_t*>(map)[1] &= ~(1ull << 21);
    return true;
}

// CTA-pair mode needs >= 2 row tiles and, for an MN-major B, B halves that are
// whole 32-column TMA boxes.
int choose_cg(const GemmProblem& g, int bn) {
    const int forced = tuning(CCT_TUNE_CTA_PAIRS);
    const bool ok2 = (g.B.major == Major::K) ? (bn / 2) % 8 == 0 : (bn / 2) % 32 == 0;
    if (forced == 1 || !ok2) return 1;
    if (forced == 2) return 2;
    if (g.M <= kBM) return 1;
    // pairs tile M by 256: only when that adds (almost) no padding over 128-row tiles
    const int64_t pad1 = (g.M + kBM - 1) / kBM * kBM - g.M;
    const int64_t pad2 = (g.M + 2 * kBM - 1) / (2 * kBM) * (2 * kBM) - g.M;
    return (pad2 - pad1) * 10 <= g.M ? 2 : 1;  // pairs are ~10-15% faster per useful flop
}

}  // namespace

bool im2col_ok(int64_t d, bool) { return d % kBK == 0; }
int64_t im2col_dk(int64_t d, bool mn_major) { return mn_major ? (d + 31) / 32 * 32 : d; }

int choose_bn(int64_t N) {
    static const int cands[] = {256, 192, 128, 96, 64};
    int best = 256;
    int64_t best_pad = INT64_MAX;
    for (int bn : cands) {
        const int64_t pad = ((N + bn - 1) / bn) * bn;
        if (pad < best_pad) { best_pad = pad; best = bn; }
    }
    return best;
}

// The tensor core accumulates fp32 with truncation, so the error of one
// TMEM accumulation chain grows ~linearly with its length (measured on B200:
// rel-L2 9e-7 at K=96, 1.6e-5 at K=2400).  Chains are therefore capped at
// kMaxChainK; longer reductions are split and the partials summed in fp32
// round-to-nearest by the deterministic reduce kernel.  Short-K problems with
// too few tiles to fill the machine are also split.
// The kernel gives every split ceil(kb / s) k-blocks and drops empty splits, so a request of
// s splits may run as fewer (e.g. kb 6050, s 96 -> 64 k-blocks each -> 95 splits).  Callers
// size and reduce the partial slices with the count that actually runs.
int effective_splits(int64_t kb, int s) {
    if (s <= 1 || kb <= 1) return 1;
    const int64_t per = (kb + s - 1) / s;
    return int((kb + per - 1) / per);
}

int choose_splits(int64_t M, int64_t N, int64_t K, int sms, int bn, int cg, int chains) {
    const int64_t tiles = ((M + kBM * cg - 1) / (kBM * cg)) * ((N + bn - 1) / bn);
    const int64_t slots = sms / cg;  // one CTA (pair) per SM (pair)
    const int64_t kb = (K + kBK - 1) / kBK;
    // accuracy floor: every TMEM chain <= kMaxChainKB k-blocks (chains per unit: 1, or 2 with CH2)
    const int64_t s_min = std::max<int64_t>(1, (kb + int64_t(kMaxChainKB) * chains - 1) / (int64_t(kMaxChainKB) * chains));
    if (kb < 64) return int(s_min);
    // Pick the split count in [s_min, 4 s_min] (>= 16 k-blocks per split) whose
    // (pair-)units fill the last wave of the machine best; ties keep the smaller
    // split count (less partial-sum traffic).
    int64_t best = s_min;
    double best_eff = 0.0;
    for (int64_t s = s_min; s <= 4 * s_min && kb / s >= 16; ++s) {
        const int64_t units = tiles * s;
        const int64_t waves = (units + slots - 1) / slots;
        const double eff = double(units) / double(waves * slots);
        if (eff > best_eff + 0.02) {
            best_eff = eff;
            best = s;
        }
    }
    return int(best);
}

// tile width of a problem: the caller's, else the least-padding candidate (>= 192 for
// the transposing epilogue)
int tile_n(const GemmProblem& g) {
    if (g.bn) return g.bn;
    if (g.C.transposed) return ((g.N + 191) / 192) * 192 < ((g.N + 255) / 256) * 256 ? 192 : 256;
    // N a multiple of 384 (conv3/4 o, conv4/5 d): one 256 + 128 composite tile instead of two
    // 192-wide ones (a 192-wide MMA costs about as much as a 256-wide one); K-major operands,
    // no epilogue transposition, no chain split.  CCT_TUNE_BN384 = 0 disables it (A/B).
    const int bn384 = tuning(CCT_TUNE_BN384);
    // (also 256 < N <= 384: one composite tile pads no more than two 192-wide ones)
    if (bn384 && (g.N % 384 == 0 || (g.N > 256 && g.N <= 384)) && !g.chain2 && g.passes == 3 &&
        !(g.im2col.x && g.im2col.operand != 0))
        return 384;
    return choose_bn(g.N);
}

int plan_splits(const GemmProblem& g) {
    const int bn = tile_n(g);
    return effective_splits((g.K + kBK - 1) / kBK,
                            choose_splits(g.M, g.N, g.K, num_sms(), bn, choose_cg(g, bn), g.chain2 ? 2 : 1));
}

// Stream-K plan: used for an unsplit GEMM of at least one wave whose whole-tile
// waves would leave >= 8% of the machine idle (e.g. 169 tiles on 74 CTA pairs).
struct SkPlan {
    int len = 0;             // k-block iterations per CTA group (0: data-parallel)
    int64_t part_floats = 0;  // two partial tiles per group boundary
    int64_t cnt_ints = 0;
};

SkPlan sk_plan(const GemmProblem& g) {
    SkPlan sp;
    const int enabled = tuning(CCT_TUNE_STREAMK);
    if (!enabled || g.splits > 1 || g.chain2 || g.M <= 0 || g.N <= 0 || g.K <= 0) return sp;
    const int bn = tile_n(g);
    const int cg = choose_cg(g, bn);
    const int64_t tiles = ((g.M + kBM * cg - 1) / (kBM * cg)) * ((g.N + bn - 1) / bn);
    const int64_t slots = num_sms() / cg;
    const int64_t kb = (g.K + kBK - 1) / kBK;
    if (tiles < slots || kb < 4) return sp;
    const int64_t waves = (tiles + slots - 1) / slots;
    if (double(tiles) / double(waves * slots) >= 0.92) return sp;
    const int64_t len = (tiles * kb + slots - 1) / slots;
    if (len < kb || tiles * kb >= (int64_t(1) << 31)) return sp;  // each tile spans <= 2 groups
    sp.len = int(len);
    sp.part_floats = slots * 2 * cg * int64_t(bn) * kBM;
    sp.cnt_ints = slots * cg;
    return sp;
}

size_t gemm_workspace_bytes(const GemmProblem& g) {
    const SkPlan sp = sk_plan(g);
    return sp.len ? size_t(sp.part_floats) * 4 + size_t(sp.cnt_ints) * 4 + 256 : 0;
}

cudaError_t run_gemm(const GemmProblem& g, cudaStream_t stream) {
    if (g.M <= 0 || g.N <= 0 || g.K <= 0) return cudaErrorInvalidValue;
    const int bn = tile_n(g);
    KParams kp{};
    kp.M = int(g.M);
    kp.N = int(g.N);
    kp.K = int(g.K);
    kp.num_m_tiles = int((g.M + kBM - 1) / kBM);
    kp.num_n_tiles = int((g.N + bn - 1) / bn);
    kp.kb_total = int((g.K + kBK - 1) / kBK);
    const int splits = std::max(1, std::min(g.splits, kp.kb_total));
    kp.kb_per_split = (kp.kb_total + splits - 1) / splits;
    kp.splits = (kp.kb_total + kp.kb_per_split - 1) / kp.kb_per_split;  // no empty split
    kp.units = kp.num_m_tiles * kp.num_n_tiles * kp.splits;
    kp.passes = g.passes;
    kp.C = g.C.ptr;
    kp.mdiv = g.C.mdiv;
    kp.s_mq = g.C.s_mq;
    kp.s_mr = g.C.s_mr;
    kp.s_n = g.C.s_n;
    kp.s_split = g.C.s_split;
    kp.ndiv = g.C.ndiv < (int64_t(1) << 31) ? int(g.C.ndiv) : 0;
    kp.s_nq = g.C.s_nq;
    kp.mlim = g.C.mlim;
    kp.nmlim = g.C.nmlim < (int64_t(1) << 31) ? int(g.C.nmlim) : INT32_MAX;
    kp.split_producer = tuning(CCT_TUNE_SPLIT_PRODUCER);
    kp.bias = g.C.bias;
    kp.relu = g.C.relu;

    const int cg = choose_cg(g, bn);
    kp.num_m_tiles = int((g.M + kBM * cg - 1) / (kBM * cg));
    kp.units = kp.num_m_tiles * kp.num_n_tiles * kp.splits;
    if (g.ws) {
        const SkPlan sp = sk_plan(g);
        if (sp.len && kp.splits == 1 && g.ws_bytes >= gemm_workspace_bytes(g)) {
            char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(g.ws) + 255) & ~uintptr_t(255));
            kp.sk_part = reinterpret_cast<float*>(base);
            kp.sk_cnt = reinterpret_cast<int*>(base + sp.part_floats * 4);
            cudaError_t e = cudaMemsetAsync(kp.sk_cnt, 0, size_t(sp.cnt_ints) * 4, stream);
            if (e != cudaSuccess) return e;
            kp.sk_len = sp.len;
        }
    }
    CUtensorMap ta, tb;
    const bool b_im = g.im2col.x && g.im2col.operand >= 1;
    if (g.im2col.x) {
        const Im2col& ic = g.im2col;
        const bool amn = g.A.major == Major::MN;
        const bool imn = (ic.operand == 2) || (ic.operand == 0 && amn);  // the im2col operand is MN-major
        const int64_t dk = ic.dk ? ic.dk : ic.d;
        if (!im2col_ok(ic.d, imn) || dk < ic.d || dk % (imn ? 32 : kBK)) return cudaErrorInvalidValue;
        kp.ic_d = int(dk);
        kp.ic_k = int(ic.k);
        kp.ic_s = int(ic.s);
        kp.ic_p = int(ic.p);
        kp.ic_m = int(ic.m);
        kp.ic_mm = int(ic.m * ic.m);
        kp.ic_cpt = int(dk / kBK);
        if (b_im && ic.operand == 2) {
            if (g.B.major != Major::MN || (bn / cg) % 32 || !make_tmap_im2col(&tb, ic, true) ||
                !make_tmap(&ta, g.A, g.M, g.K, kBM))
                return cudaErrorInvalidValue;
        } else if (b_im) {
            if (amn || g.B.major == Major::MN || !make_tmap_im2col(&tb, ic, false, bn / cg) ||
                !make_tmap(&ta, g.A, g.M, g.K, kBM))
                return cudaErrorInvalidValue;
        } else if (!make_tmap_im2col(&ta, ic, amn)) {
            return cudaErrorInvalidValue;
        }
    } else if (!make_tmap(&ta, g.A, g.M, g.K, kBM)) {
        return cudaErrorInvalidValue;
    }
    if (!b_im && !make_tmap(&tb, g.B, g.N, g.K, bn == 384 ? 64 : bn / cg)) return cudaErrorInvalidValue;
    if (cg == 2) {
        switch (bn) {
        case 384: return dispatch_layout<384, 2>(g, ta, tb, kp, stream);
        case 256: return dispatch_layout<256, 2>(g, ta, tb, kp, stream);
        case 192: return dispatch_layout<192, 2>(g, ta, tb, kp, stream);
        case 128: return dispatch_layout<128, 2>(g, ta, tb, kp, stream);
        case 96: return dispatch_layout<96, 2>(g, ta, tb, kp, stream);
        case 64: return dispatch_layout<64, 2>(g, ta, tb, kp, stream);
        default: return cudaErrorInvalidValue;
        }
    }
    switch (bn) {
    case 384: return dispatch_layout<384, 1>(g, ta, tb, kp, stream);
    case 256: return dispatch_layout<256, 1>(g, ta, tb, kp, stream);
    case 192: return dispatch_layout<192, 1>(g, ta, tb, kp, stream);
    case 128: return dispatch_layout<128, 1>(g, ta, tb, kp, stream);
    case 96: return dispatch_layout<96, 1>(g, ta, tb, kp, stream);
    case 64: return dispatch_layout<64, 1>(g, ta, tb, kp, stream);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace cct
