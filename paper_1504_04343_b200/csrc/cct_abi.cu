// cct_abi.cu -- the extern "C" boundary (include/cct.h): argument validation,
// workspace planning and the per-pass kernel sequences of the lowered
// convolution (lower -> tcgen05 3xTF32 GEMM -> lift, and the adjoints).
//
// Pass / lowering -> GEMM mapping:
//   FWD  T1: M=b m^2  N=o     K=k^2 d  A=Dhat1 (K-major)  B=W (K-major)   C -> y NCHW (lift fused)
//   FWD  T2: M=b R m  N=k o   K=k d    A=Dhat2            B=W as (ok x kd) C -> Rhat^T, lift_t2
//   FWD  T3: M=b R^2  N=k^2 o K=d      A=Dhat3 (=Xp)      B=W as (ok^2 x d) C -> Rhat^T, lift_t3
//   BWD_DATA: M=cols(Dhat) N=rows K=ncols  A=W (MN-major) B=dRhat^T (MN-major) C -> dDhat, col2im
//   BWD_WEIGHT: M=cols N=ncols K=rows   A=Dhat (MN-major) B=dRhat^T (K-major) C -> dW (split-K)
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <string>

#include "cct.h"
#include "common.cuh"
#include "gemm.cuh"
#include "lowering.cuh"
#include "reduce.cuh"
#include "s2d.cuh"
#include "epilogue.cuh"
#include "gather.cuh"
#include "dgrad.cuh"

namespace cct {
uint64_t launch_count();
void reset_launch_count();
}  // namespace cct

using namespace cct;

namespace {

cct_status fail(cct_status s, const std::string& msg) {
    set_error(msg);
    return s;
}

cct_status cuda_status(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return CCT_OK;
    return fail(CCT_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CCT_TRY(expr, where)                                     \
    do {                                                         \
        cct_status _s = cuda_status((expr), (where));            \
        if (_s != CCT_OK) return _s;                             \
    } while (0)

std::string desc_str(const cct_conv_desc* d) {
    std::ostringstream os;
    os << "(n=" << d->n << ", k=" << d->k << ", d=" << d->d << ", o=" << d->o << ", b=" << d->b
       << ", stride=" << d->stride << ", pad=" << d->pad << ")";
    return os.str();
}

cct_status check_desc(const cct_conv_desc* d) {
    if (!d) return fail(CCT_ERR_CONFIG, "null conv descriptor");
    if (d->k < 1 || d->d < 1 || d->o < 1 || d->b < 1 || d->stride < 1 || d->pad < 0 ||
        d->k > d->n + 2 * d->pad || (d->layout != CCT_LAYOUT_NCHW && d->layout != CCT_LAYOUT_NHWC))
        return fail(CCT_ERR_CONFIG, "invalid layer config " + desc_str(d) +
                                        ": need 1 <= k <= n + 2 pad, d >= 1, o >= 1, b >= 1, stride >= 1, pad >= 0");
    return CCT_OK;
}

Geo geo_of(const cct_conv_desc* d) {
    Geo g;
    g.b = d->b; g.n = d->n; g.d = d->d; g.k = d->k; g.o = d->o; g.s = d->stride; g.p = d->pad;
    g.N = g.n + 2 * g.p;
    g.m = (g.N - g.k) / g.s + 1;
    g.R = g.s * (g.m - 1) + g.k;
    g.yl = d->layout == CCT_LAYOUT_NHWC ? 1 : 0;
    return g;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// bump allocator over the caller's workspace; base == nullptr -> size query.
// Real workspaces are first aligned up to 256 bytes (hence +256 in the size).
struct Ws {
    char* base;
    size_t off = 0;
    explicit Ws(void* b)
        : base(b ? reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(b) + 255) & ~uintptr_t(255))
                 : nullptr) {}
    float* take(int64_t floats) {
        off = (off + 255) & ~size_t(255);
        float* p = base ? reinterpret_cast<float*>(base + off) : nullptr;
        off += size_t(floats) * sizeof(float);
        return p;
    }
};

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

bool implicit_enabled();
int resolve_type(const cct_conv_desc* d, cct_lowering l, cct_pass pass) {
    if (l == CCT_LOWER_T1 || l == CCT_LOWER_T2 || l == CCT_LOWER_T3) return int(l);
    cct_calibration cal;
    cct_calibration_default(&cal);
    cct_lowering out = CCT_LOWER_T1;
    if (cct_select_lowering(d, &cal, int(pass), &out, nullptr) != CCT_OK) return 1;
    return int(out);
}
// Types 2 / 3 fused (CCT_TUNE_FUSED_T23): with the implicit form available (TMA im2col of x,
// d % 16 == 0) a fused Type 3 -- the GEMM on the input with the k^2 shifted products summed
// in the accumulator instead of through a materialised Rhat and a lift -- is exactly the
// implicit Type 1 kernel (one im2col box per filter tap, tap-shifted accumulation in TMEM),
// and a fused Type 2 the same with the vertical taps accumulated.
int resolve(const cct_conv_desc* d, cct_lowering l, cct_pass pass) {
    const int t = resolve_type(d, l, pass);
    if ((t == 2 || t == 3) && tuning(CCT_TUNE_FUSED_T23) && implicit_enabled() && im2col_ok(d->d, true))
        return 1;
    return t;
}

// Lowered-matrix geometry of one type.
struct Lowered {
    int64_t rows, cols, ncols;  // Dhat rows x cols, Khat^T rows (= ncols)
    int64_t ldc;                // row stride of Dhat / dDhat / W' (floats, multiple of 4)
    int64_t ldr;                // row stride of Rhat^T / dRhat^T (floats, multiple of 4)
    RowMap rm;
};

Lowered lowered_of(const Geo& g, int type) {
    Lowered L;
    L.rm = rowmap_internal(g, type);
    L.rows = g.b * L.rm.rpi;
    L.cols = lowered_cols(g, type);
    L.ncols = lowered_ncols(g, type);
    L.ldc = rup4(L.cols);
    L.ldr = rup4(L.rows);
    return L;
}

// W viewed as (ncols x cols) row-major; zero-copy when the row stride is TMA-legal.
const float* weights_view(const Lowered& L, const float* w, Ws& ws, cudaStream_t st, int64_t* ld,
                          cudaError_t* err) {
    *err = cudaSuccess;
    if (L.cols % 4 == 0 && aligned16(w)) {
        *ld = L.cols;
        return w;
    }
    float* wp = ws.take(L.ncols * L.ldc);
    *ld = L.ldc;
    if (ws.base) *err = pad_rows(w, L.ncols, L.cols, L.cols, wp, L.ldc, st);
    return wp;
}

// Implicit Type 1 lowering (TMA im2col A operand) -- on by default; the
// materialised path stays available for parity tests and small-channel layers.
// process-wide knobs (atomics: the ABI may be called from several host threads)
std::atomic<int> g_implicit{1};
bool implicit_enabled() { return g_implicit.load() != 0; }

// Type 1 with d % 16 == 0 runs forward and backward-weight on the input itself.
bool t1_implicit(const Geo& g, int type, const float* x) {
    return implicit_enabled() && type == 1 && im2col_ok(g.d, true) && x && aligned16(x) &&
           g.n * g.n * g.d * g.b < (int64_t(1) << 40) && g.b * g.m * g.m < (int64_t(1) << 31);
}

// A strided Type 1 layer whose blocked depth s^2 d is a multiple of 16 runs in
// space-to-depth form (s2d.cuh): the implicit stride-1 GEMMs on X' (CaffeNet
// conv1: 3 x 3 taps of depth 48).  CCT_TUNE_S2D = 0 keeps the materialised path.
// Whether that form is used is the cost model's call per pass (prefer_s2d): the
// entry points set the pass context (0 fwd, 1 bwd-data, 2 bwd-weight, 3 training
// step: cct_conv_fwd_cached + cct_conv_bwd, whose lowered cache must agree).
thread_local int t_pass = 3;
struct PassCtx {
    int old;
    explicit PassCtx(int p) : old(t_pass) { t_pass = p; }
    ~PassCtx() { t_pass = old; }
};

}  // namespace
namespace cct {
bool prefer_s2d(const cct_conv_desc* desc, int pass);  // cost_model.cpp
}  // namespace cct
namespace {

bool t1_s2d(const Geo& g, int type) {
    const int env = tuning(CCT_TUNE_S2D);
    if (!(env && implicit_enabled() && type == 1 && g.s > 1)) return false;
    const Geo v = s2d_geo(g);
    if (!(im2col_ok(v.d, false) && v.b * v.n * v.n * v.d < (int64_t(1) << 40) && v.b * v.n * v.n < (int64_t(1) << 31)))
        return false;
    if (env == 2) return true;  // CCT_TUNE_S2D = 2: always (profiling)
    cct_conv_desc d{};
    d.n = g.n; d.k = g.k; d.d = g.d; d.o = g.o; d.b = g.b; d.stride = g.s; d.pad = g.p;
    return prefer_s2d(&d, t_pass);
}

// Small-channel Type 1 layers with d s % 4 == 0 (CaffeNet conv1) run fused: the lowered
// matrix is gathered from staged input rows inside the GEMM (gather.cuh) -- no Dhat in
// HBM, no separate lowering.  Takes precedence over the space-to-depth form (CCT_TUNE_GATHER
// = 0 restores the earlier choices).
bool t1_gather_fwd(const Geo& g, int type) {
    return tuning(CCT_TUNE_GATHER) && implicit_enabled() && type == 1 && !im2col_ok(g.d, true) && gather_fwd_ok(g);
}
bool t1_gather_wgrad(const Geo& g, int type) {
    return tuning(CCT_TUNE_GATHER) && implicit_enabled() && type == 1 && !im2col_ok(g.d, true) && gather_wgrad_ok(g);
}
// ... and backward-data folds the horizontal overlap of dDhat in the GEMM epilogue (dgrad.cuh)
bool t1_hfold_dgrad(const Geo& g, int type) {
    return tuning(CCT_TUNE_GATHER) && implicit_enabled() && type == 1 && !im2col_ok(g.d, true) && hfold_dgrad_ok(g);
}

// planning runs (no workspace) still need non-null, aligned operand pointers so
// they follow the same decisions as the real call
const float* kPlanPtr = reinterpret_cast<const float*>(uintptr_t(256));
template <class T>
T* or_plan(T* p, const Ws& ws) {
    return ws.base ? p : const_cast<T*>(reinterpret_cast<const T*>(kPlanPtr));
}

// floats per image of the forward's lowered cache (the blocked input X' in s2d form)
int64_t cache_per_image(const Geo& g, int type) {
    if (t1_gather_fwd(g, type)) return 0;  // no Dhat: the backward gathers (or lowers) x itself
    if (t1_s2d(g, type)) {
        const Geo v = s2d_geo(g);
        return v.n * v.n * v.d;
    }
    const RowMap rm = rowmap_internal(g, type);
    return rm.rpi * rup4(lowered_cols(g, type));
}

}  // namespace
namespace cct {
bool prefer_implicit_dgrad(const cct_conv_desc* desc);  // cost_model.cpp
}  // namespace cct
namespace {

// Implicit Type 1 backward (stride 1): dy is transposed once to NHWC and
//  * backward-data is the forward convolution of dy with the rotated kernel bank
//    wr[c][k-1-i][k-1-j][o] = w[o][i][j][c] at pad k-1-p, gathered by TMA im2col
//    and written straight to dx (no dDhat, no col2im);
//  * backward-weight reads that NHWC dy as its (MN-major) B operand.
// Used when the cost model predicts it faster than the materialised form
// (prefer_implicit_dgrad, cost_model.cpp) -- always under implicit mode 2.
bool t1_implicit_bwd(const Geo& g, int type) {
    if (!(implicit_enabled() && type == 1 && g.s == 1 && g.p <= g.k - 1 && im2col_ok(g.o, false) &&
          g.b * g.n * g.n < (int64_t(1) << 31) && g.b * g.m * g.m * g.o < (int64_t(1) << 40)))
        return false;
    const int env = tuning(CCT_TUNE_IMPLICIT_BWD);  // 0 never, 2 always (profiling)
    if (env == 0) return false;
    if (env == 2) return true;
    cct_conv_desc d{};
    d.n = g.n; d.k = g.k; d.d = g.d; d.o = g.o; d.b = g.b; d.stride = g.s; d.pad = g.p;
    return prefer_implicit_dgrad(&d);
}

// Implicit backward-weight of a narrow bank (o < 128) runs swapped: dW rows = the o
// channels, columns = (tap, channel) -- B is the MN-major TMA im2col of x -- instead of
// an o-wide tile.  CCT_TUNE_WGRAD_SWAP = 0 disables it (A/B).
bool wgrad_swapped(const Geo& g) {
    const int env = tuning(CCT_TUNE_WGRAD_SWAP);
    return env != 0 && g.o < 128 && g.k * g.k * im2col_dk(g.d, true) >= 192;
}

// Implicit backward-data with a narrow kernel depth (d < 128) runs swapped, the
// pixels as the GEMM's N side (B = TMA im2col of dy): a 128-row tile with d useful
// rows beats a d-wide tile (measured narrow-tile rate ~ 0.58 of the 256-wide one at
// d = 96).  CCT_TUNE_DGRAD_SWAP: 0 never, 2 always (A/B).
bool dgrad_swapped(const Geo& g) {
    const int env = tuning(CCT_TUNE_DGRAD_SWAP);
    if (env == 0) return false;
    if (env == 2) return g.d <= 128;
    return g.d < 128;
}

// Forward of a narrow kernel bank (o < 128) in the swapped orientation: channels on the
// 128-row side, pixels as the 256-wide tile, NCHW rows written by the transposing epilogue.
// Measured on conv1 (b = 256): 0.50 ms vs 0.40 ms for the o-wide tile (materialised) and
// 0.64 vs 0.56 ms in space-to-depth form -- the NCHW row stores (one 1 KB run per channel per
// tile) cost more than the narrow MMAs -- so it is off by default; CCT_TUNE_FWD_SWAP = 1 enables it.
bool fwd_swapped(const Geo& g) {
    const int env = tuning(CCT_TUNE_FWD_SWAP);
    return env != 0 && g.o < 128 && g.b * g.m * g.m >= 4096;
}

Im2col im2col_of(const Geo& g, const float* x) {
    Im2col ic;
    ic.x = x;
    ic.b = g.b; ic.n = g.n; ic.d = g.d; ic.k = g.k; ic.s = g.s; ic.p = g.p; ic.m = g.m;
    return ic;
}

// True when Dhat of this type is the (unpadded, aligned) input itself.
bool dhat_is_input(const Geo& g, int type, const float* x) {
    return type == 3 && g.p == 0 && g.R == g.n && g.d % 4 == 0 && aligned16(x);
}

// Dhat in internal order, written to `dst` when given (the caller's lowered
// cache) else to the workspace; T3 with no padding is the input itself.
const float* dhat_of(const Geo& g, int type, const Lowered& L, const float* x, float* dst, Ws& ws,
                     cudaStream_t st, cudaError_t* err) {
    *err = cudaSuccess;
    if (dhat_is_input(g, type, x)) return x;
    float* dh = dst ? dst : ws.take(L.rows * L.ldc);
    if (ws.base) *err = lower(g, type, L.rm, x, dh, L.ldc, st);
    return dh;
}

// Run gp writing a flat output span of `span` floats at `out`.  Reductions
// longer than the accumulation-chain cap (kMaxChainKB k-blocks) are split and
// reduced in fp32 round-to-nearest (deterministic order).  In planning mode
// (ws.base == nullptr) only the workspace is reserved.
cct_status gemm_capped(GemmProblem gp, float* out, int64_t span, Ws& ws, cudaStream_t st, const char* what,
                       bool* fused = nullptr) {
    const int64_t kb = (gp.K + kBK - 1) / kBK;
    // narrow tiles (N <= 128) accumulate alternate 8-wide K steps into two sub-accumulators
    // (gemm_kernel.cuh Cfg::NACC): each TMEM chain holds half the K terms, so the accuracy cap
    // allows twice the k-blocks per tile (not for the one-accumulator A ring or the merged form)
    const int64_t cap = kMaxChainKB * ((tile_n(gp) <= 128 && tuning(CCT_TUNE_A_TMEM) < 2) ? 2 : 1);
    int splits = effective_splits(kb, int((kb + cap - 1) / cap));
    // a 2-way accuracy split of a wide-tile K-major GEMM runs as two TMEM chains of one tile
    // (no partial tiles, no reduce kernel); CCT_TUNE_CHAIN2 = 0 keeps the split-K form (A/B)
    const int chain2_env = tuning(CCT_TUNE_CHAIN2);
    if (splits == 2 && chain2_env && gp.A.major == Major::K && gp.B.major == Major::K && !gp.C.transposed &&
        gp.passes == 3 && tile_n(gp) >= 192 && tile_n(gp) <= 256) {
        splits = 1;
        gp.chain2 = 1;
    }
    // a fused epilogue (bias / ReLU) applies to final stores only: not to split partials
    if (fused) *fused = splits == 1;
    if (splits > 1) {
        gp.C.bias = nullptr;
        gp.C.relu = 0;
    }
    float* parts = splits > 1 ? ws.take(int64_t(splits) * span) : nullptr;
    gp.splits = splits;
    const size_t skb = gemm_workspace_bytes(gp);  // stream-K partial tiles
    float* sk = skb ? ws.take(int64_t(skb / 4)) : nullptr;
    if (!ws.base) return CCT_OK;
    gp.ws = sk;
    gp.ws_bytes = skb;
    gp.C.ptr = splits > 1 ? parts : out;
    gp.C.s_split = span;
    CCT_TRY(run_gemm(gp, st), what);
    if (splits > 1) CCT_TRY(splitk_reduce(parts, span, splits, 1, span, span, out, span, st), "split-K reduce");
    return CCT_OK;
}

// implicit backward-weight: A = im2col(x)^T (MN-major).  Its 32-channel boxes
// need taps padded to dk = d rounded up to 32: M = k^2 dk, and rows (tap, ch >= d)
// -- zeros read past the channel extent -- are not stored.
void wgrad_im2col(GemmProblem& gp, const Geo& g, const float* x) {
    gp.im2col = im2col_of(g, x);
    const int64_t dk = im2col_dk(g.d, true);
    gp.im2col.dk = dk;
    if (dk != g.d) {
        gp.M = g.k * g.k * dk;
        gp.C.mdiv = dk;
        gp.C.s_mq = g.d;
        gp.C.mlim = g.d;
    }
}

// Backward-weight reductions (K = b m^2 pixels) are split for accuracy and wave fill; with
// two TMEM chains per unit (CH2) the accuracy floor halves, so half as many partial tiles
// reach HBM.  Wide tiles only (two 256-column accumulators fit TMEM).  CCT_TUNE_CHAIN2 = 0: off.
int wgrad_chain2(const GemmProblem& gp) {
    const int env = tuning(CCT_TUNE_CHAIN2);
    const int bn = tile_n(gp);
    return (env && gp.passes == 3 && !gp.C.transposed && bn >= 192 && bn <= 256 &&
            gp.K > int64_t(kMaxChainKB) * kBK) ? 1 : 0;
}

// backward-weight GEMM: dW^T (cols x ncols) = Dhat^T * dRhat, reduction over rows
GemmProblem wgrad_problem(const Lowered& L, Operand a, Operand b) {
    GemmProblem gp;
    gp.M = L.cols;
    gp.N = L.ncols;
    gp.K = L.rows;
    gp.A = a;
    gp.B = b;
    return gp;
}

// ---------------------------------------------------------------------------
// the three passes; ws.base == nullptr plans sizes only
// ---------------------------------------------------------------------------

// Extension options of a forward pass (cct_conv_fwd_ex): a channel group read
// straight from a wider x (pixel stride xcs) and written into a wider y (image
// stride ycs) -- implicit Type 1 only -- and the fused bias / ReLU epilogue
// (applied by the GEMM when it writes y unsplit; `fused` reports whether it did).
struct FwdOpts {
    int64_t xcs = 0, ycs = 0;
    const float* bias = nullptr;
    int relu = 0;
    bool* fused = nullptr;
};

cct_status run_fwd_one(const Geo& g, int type, const float* x, const float* w, float* y, float* cache, Ws& ws,
                       cudaStream_t st, const FwdOpts& opts = FwdOpts{}) {
    if (opts.fused) *opts.fused = false;
    const bool strided = (opts.xcs && opts.xcs != g.d) || (opts.ycs && opts.ycs != g.o * g.m * g.m);
    if (strided && !(type == 1 && t1_implicit(g, type, x) && !t1_s2d(g, type)))
        return fail(CCT_ERR_UNSUPPORTED, "channel-group views need the implicit Type 1 path");
    if (!strided && t1_gather_fwd(g, type) && aligned16(or_plan(x, ws))) {
        float* w2 = ws.take(gather_fwd_ws_floats(g));
        if (ws.base) CCT_TRY(gather_fwd(g, x, w, y, 0, opts.bias, opts.relu, w2, st), "fused gather forward");
        if (opts.fused) *opts.fused = true;
        return CCT_OK;
    }
    if (t1_s2d(g, type)) {
        // blocked input (kept in the caller's lowered cache when given) and kernel bank
        const Geo v = s2d_geo(g);
        float* xs = cache ? cache : ws.take(v.b * v.n * v.n * v.d);
        float* wsd = ws.take(v.o * v.k * v.k * v.d);
        if (ws.base) {
            CCT_TRY(s2d_input(g, x, xs, st), "space-to-depth (x)");
            CCT_TRY(s2d_weights(g, w, wsd, st), "space-to-depth (w)");
        }
        return run_fwd_one(v, 1, or_plan(xs, ws), or_plan(wsd, ws), y, nullptr, ws, st);
    }
    const Lowered L = lowered_of(g, type);
    cudaError_t e = cudaSuccess;
    int64_t ldw;
    const float* wv = weights_view(L, w, ws, st, &ldw, &e);
    CCT_TRY(e, "pad weights");
    const bool implicit = t1_implicit(g, type, x);
    const float* dh = implicit ? nullptr : dhat_of(g, type, L, x, cache, ws, st, &e);
    CCT_TRY(e, "lower");
    const int64_t ldd = (dh == x) ? g.d : L.ldc;
    GemmProblem gp;
    gp.M = L.rows;
    gp.N = L.ncols;
    gp.K = L.cols;
    gp.A = {dh, ldd, Major::K};
    gp.B = {wv, ldw, Major::K};
    if (implicit) {
        gp.im2col = im2col_of(g, x);
        gp.im2col.cs = opts.xcs;
    }
    float* rht = nullptr;
    float* out;
    int64_t span;
    if (type == 1 && fwd_swapped(g)) {
        // narrow bank (o < 128): y^T = W * lowered^T -- channels on the 128-row side, pixels
        // as the 256-wide tile (B = Dhat rows, or TMA im2col of x), NCHW rows written through
        // the transposing epilogue (+ per-channel bias / ReLU)
        out = y;
        gp.M = g.o;
        gp.N = L.rows;
        gp.A = {wv, ldw, Major::K};
        gp.B = {dh, ldd, Major::K};
        if (implicit) gp.im2col.operand = 1;
        if (g.yl) {
            // NHWC y: lanes = channels are contiguous -- plain coalesced stores, no transposition
            gp.C.s_mr = 1;
            gp.C.s_n = g.o;
            span = g.b * g.m * g.m * g.o;
        } else {
            gp.C.transposed = 1;
            gp.C.s_mr = g.m * g.m;
            gp.C.ndiv = g.m * g.m;
            gp.C.s_nq = opts.ycs ? opts.ycs : g.o * g.m * g.m;
            gp.C.s_n = 1;
            span = (g.b - 1) * gp.C.s_nq + g.o * g.m * g.m;
        }
        gp.C.bias = opts.bias;
        gp.C.relu = opts.relu;
    } else if (type == 1) {
        // lift_t1 is a reshape: write y straight from the epilogue (+ bias / ReLU)
        out = y;
        if (g.yl) {  // NHWC: row = pixel, o consecutive channels
            gp.C.s_mr = g.o;
            gp.C.s_n = 1;
            span = g.b * g.m * g.m * g.o;
        } else {
            gp.C.mdiv = g.m * g.m;
            gp.C.s_mq = opts.ycs ? opts.ycs : g.o * g.m * g.m;
            gp.C.s_mr = 1;
            gp.C.s_n = g.m * g.m;
            span = (g.b - 1) * gp.C.s_mq + g.o * g.m * g.m;
        }
        gp.C.bias = opts.bias;
        gp.C.relu = opts.relu;
    } else if (planes_ok(g, type)) {
        // Rhat plane-major (lowering23.cu): the k^a tap planes of one (image, channel) contiguous
        span = g.b * L.ncols * L.rm.rpi;
        rht = ws.take(span);
        out = rht;
        gp.C.mdiv = L.rm.rpi;
        gp.C.s_mq = L.ncols * L.rm.rpi;
        gp.C.s_mr = 1;
        gp.C.s_n = L.rm.rpi;
    } else {
        rht = ws.take(L.ncols * L.ldr);
        out = rht;
        span = L.ncols * L.ldr;
        gp.C.s_mr = 1;
        gp.C.s_n = L.ldr;
    }
    cct_status s = gemm_capped(gp, out, span, ws, st, "gemm (fwd)", type == 1 ? opts.fused : nullptr);
    if (s != CCT_OK || !ws.base) return s;
    if (type != 1) {
        if (planes_ok(g, type)) CCT_TRY(lift_planes(g, type, rht, y, st), "lift");
        else CCT_TRY(lift(g, type, L.rm, rht, 1, L.ldr, y, st), "lift");
    }
    return CCT_OK;
}

// Backward: dRhat^T is expanded once and shared by bwd-data (dx != null) and
// bwd-weight (dw != null).  bwd-weight reads Dhat from `cache` when given (as
// left there by cct_conv_fwd_cached), else lowers x again.  The two passes run
// in stream order and reuse the same scratch region after dRhat^T.
cct_status run_bwd_implicit(const Geo& g, const float* x, const float* cache, const float* dy, const float* w,
                            float* dx, float* dw, Ws& ws, cudaStream_t st) {
    const Lowered L = lowered_of(g, 1);
    const int64_t mm = g.m * g.m, kk = g.k * g.k;
    // dy as NHWC: [b][m][m][o] = dRhat (rows x o) -- the caller's dy when its layout is NHWC
    const float* dyn = dy;
    if (!g.yl) {
        float* t = ws.take(g.b * mm * g.o);
        if (ws.base)
            CCT_TRY(transpose_batched(dy, g.o, mm, mm, g.o * mm, t, g.o, mm * g.o, g.b, kPhaseExpand, st), "dy to NHWC");
        dyn = or_plan(t, ws);
    }
    const size_t mark = ws.off;
    size_t hi = mark;
    if (dx) {
        // rotated kernel bank wr[c][(k-1-i)*k + (k-1-j)][o] = w[o][i][j][c]: one
        // (o x d) -> (d x o) transpose per tap, written in reversed tap order
        float* wr = ws.take(g.d * kk * g.o);
        if (ws.base)
            CCT_TRY(transpose_batched(w, g.o, g.d, kk * g.d, g.d, wr + (kk - 1) * g.o, kk * g.o, -g.o, kk, kPhaseOther,
                                      st),
                    "rotate weights");
        Geo v = g;  // the forward convolution that computes dx
        v.n = g.m; v.d = g.o; v.o = g.d; v.p = g.k - 1 - g.p; v.m = g.n;
        GemmProblem gp;
        gp.K = kk * g.o;
        gp.im2col = im2col_of(v, dyn);
        if (dgrad_swapped(g)) {
            // narrow d: dx^T (d x pixels) = wr (d x k^2 o) * im2col(dy)^T -- the pixels are the
            // 256-wide tile side instead of a d-wide one (lanes = channels: coalesced NHWC stores)
            gp.M = g.d;
            gp.N = g.b * g.n * g.n;
            gp.A = {wr, kk * g.o, Major::K};
            gp.B = {nullptr, 0, Major::K};
            gp.im2col.operand = 1;
            gp.C.s_mr = 1;
            gp.C.s_n = g.d;
        } else {
            gp.M = g.b * g.n * g.n;
            gp.N = g.d;
            gp.A = {nullptr, 0, Major::K};
            gp.B = {wr, kk * g.o, Major::K};
            gp.C.s_mr = g.d;
            gp.C.s_n = 1;
        }
        cct_status s = gemm_capped(gp, dx, g.b * g.n * g.n * g.d, ws, st, "gemm (bwd-data, implicit)");
        if (s != CCT_OK) return s;
        hi = std::max(hi, ws.off);
        ws.off = mark;
    }
    if (dw) {
        cudaError_t e = cudaSuccess;
        const bool implicit = t1_implicit(g, 1, x);
        const float* dh = implicit ? nullptr : cache ? cache : dhat_of(g, 1, L, x, nullptr, ws, st, &e);
        CCT_TRY(e, "lower");
        GemmProblem gp = wgrad_problem(L, {dh, L.ldc, Major::MN}, {dyn, g.o, Major::MN});
        const bool swapped = implicit && wgrad_swapped(g);
        if (swapped) {
            // narrow bank (o < 128): dW (o x k^2 d) = dy^T * im2col(x) -- channels on the 128-row
            // side, the (tap, channel) columns 192 / 256 wide (B = MN-major TMA im2col, taps
            // padded to dk; padded columns are not stored)
            const int64_t dk = im2col_dk(g.d, true);
            gp.M = g.o;
            gp.N = kk * dk;
            gp.A = {dyn, g.o, Major::MN};
            gp.B = {nullptr, 0, Major::MN};
            gp.im2col = im2col_of(g, x);
            gp.im2col.dk = dk;
            gp.im2col.operand = 2;
            gp.C.ndiv = dk;
            gp.C.s_nq = g.d;
            gp.C.nmlim = g.d;
        } else if (implicit) {
            wgrad_im2col(gp, g, x);
        }
        gp.chain2 = wgrad_chain2(gp);
        const int splits = plan_splits(gp);
        const int64_t wsize = L.ncols * L.cols;
        float* parts = splits > 1 ? ws.take(int64_t(splits) * wsize) : dw;
        if (ws.base) {
            gp.C.ptr = parts;
            gp.C.s_mr = swapped ? L.cols : 1;
            gp.C.s_n = swapped ? 1 : L.cols;
            gp.C.s_split = wsize;
            gp.splits = splits;
            CCT_TRY(run_gemm(gp, st), "gemm (bwd-weight)");
            if (splits > 1)
                CCT_TRY(splitk_reduce(parts, wsize, splits, 1, wsize, wsize, dw, wsize, st), "split-K reduce");
        }
        hi = std::max(hi, ws.off);
    }
    ws.off = hi;
    return CCT_OK;
}

cct_status run_bwd_one(const Geo& g, int type, const float* x, const float* cache, const float* dy, const float* w,
                       float* dx, float* dw, Ws& ws, cudaStream_t st) {
    if (dx && t1_hfold_dgrad(g, type) && aligned16(or_plan(dy, ws))) {  // (dx: plain stores)
        const size_t mark = ws.off;
        float* w2 = ws.take(hfold_dgrad_ws_floats(g));
        const Fork* fk = dw && tuning(CCT_TUNE_OVERLAP) ? fork_resources() : nullptr;
        if (fk) {
            // the backward-weight (x, dy -> dW; scratch above H) on the side stream from the end of
            // the backward-data GEMM, beside the vertical fold; joined back into st
            if (ws.base) {
                CCT_TRY(hfold_dgrad(g, dy, w, dx, w2, st, fk->fork), "fused backward-data");
                CCT_TRY(cudaStreamWaitEvent(fk->side, fk->fork, 0), "fork");
            }
            cct_status s = run_bwd_one(g, type, x, cache, dy, w, nullptr, dw, ws, ws.base ? fk->side : st);
            if (ws.base) {  // joined on every path, so st never runs ahead of the side stream's work
                CCT_TRY(cudaEventRecord(fk->join, fk->side), "join");
                CCT_TRY(cudaStreamWaitEvent(st, fk->join, 0), "join");
            }
            return s;
        }
        if (ws.base) CCT_TRY(hfold_dgrad(g, dy, w, dx, w2, st), "fused backward-data");
        if (!dw) return CCT_OK;
        const size_t hi = ws.off;
        ws.off = mark;  // stream order: the backward-weight may reuse the backward-data scratch
        cct_status s = run_bwd_one(g, type, x, cache, dy, w, nullptr, dw, ws, st);
        ws.off = std::max(hi, ws.off);
        return s;
    }
    if (t1_s2d(g, type)) {
        // the stride-1 backward of the blocked layer, then the depth-to-space gathers
        const Geo v = s2d_geo(g);
        const float* xs = nullptr;
        float *wsd = nullptr, *dxs = nullptr, *dws = nullptr;
        if (dw) {
            if (cache) {
                xs = cache;
            } else {
                float* t = ws.take(v.b * v.n * v.n * v.d);
                if (ws.base) CCT_TRY(s2d_input(g, x, t, st), "space-to-depth (x)");
                xs = t;
            }
            dws = ws.take(v.o * v.k * v.k * v.d);
        }
        if (dx) {
            wsd = ws.take(v.o * v.k * v.k * v.d);
            dxs = ws.take(v.b * v.n * v.n * v.d);
            if (ws.base) CCT_TRY(s2d_weights(g, w, wsd, st), "space-to-depth (w)");
        }
        cct_status s = run_bwd_one(v, 1, dw ? or_plan(xs, ws) : nullptr, nullptr, dy, dx ? or_plan(wsd, ws) : nullptr,
                                   dx ? or_plan(dxs, ws) : nullptr, dw ? or_plan(dws, ws) : nullptr, ws, st);
        if (s != CCT_OK || !ws.base) return s;
        if (dx) CCT_TRY(d2s_input(g, dxs, dx, st), "depth-to-space (dx)");
        if (dw) CCT_TRY(d2s_weights(g, dws, dw, st), "depth-to-space (dw)");
        return CCT_OK;
    }
    if (t1_implicit_bwd(g, type)) return run_bwd_implicit(g, x, cache, dy, w, dx, dw, ws, st);
    const Lowered L = lowered_of(g, type);
    cudaError_t e = cudaSuccess;
    // small-channel Type 1: backward-weight gathers Dhat from x inside the GEMM (gather.cuh)
    if (dw && t1_gather_wgrad(g, type) && aligned16(or_plan(x, ws))) {
        const size_t mark = ws.off;
        size_t hi = mark;
        if (dx) {
            cct_status s = run_bwd_one(g, type, x, cache, dy, w, dx, nullptr, ws, st);
            if (s != CCT_OK) return s;
            hi = ws.off;
            ws.off = mark;  // stream order: the backward-weight may reuse the backward-data scratch
        }
        float* w2 = ws.take(gather_wgrad_ws_floats(g));
        if (ws.base) CCT_TRY(gather_wgrad(g, x, dy, dw, w2, st), "fused gather backward-weight");
        ws.off = std::max(hi, ws.off);
        return CCT_OK;
    }
    // Type 1 with an NHWC dy: dy IS dRhat (rows x o, row-major) -- the GEMMs read it in place
    // (K-major B of backward-data, MN-major operand of backward-weight); otherwise expand dRhat^T
    const bool dy_direct = type == 1 && g.yl && g.o % 4 == 0 && aligned16(dy);
    float* drt = dy_direct ? nullptr : ws.take(L.ncols * L.ldr);
    if (ws.base && !dy_direct) CCT_TRY(expand(g, type, dy, drt, L.ldr, st), "expand");
    const Operand drt_n = dy_direct ? Operand{dy, g.o, Major::K} : Operand{drt, L.ldr, Major::MN};   // (rows, ncols)
    const Operand drt_k = dy_direct ? Operand{dy, g.o, Major::MN} : Operand{drt, L.ldr, Major::K};   // (ncols, rows)
    const size_t mark = ws.off;
    size_t hi = mark;
    if (dx) {
        int64_t ldw;
        const float* wv = weights_view(L, w, ws, st, &ldw, &e);
        CCT_TRY(e, "pad weights");
        const bool direct = (type == 3 && g.p == 0 && g.R == g.n && g.d % 4 == 0 && aligned16(dx));
        const bool slab = col2im_slab_layout(g, type);
        const int64_t S = slab_stride(g);
        const int64_t span = direct ? L.rows * g.d : slab ? g.b * g.m * g.k * S : L.rows * L.ldc;
        float* dd = direct ? dx : ws.take(span);
        const int64_t ldd = direct ? g.d : slab ? S : L.ldc;
        GemmProblem gp;
        gp.M = L.cols;
        gp.N = L.rows;
        gp.K = L.ncols;
        gp.A = {wv, ldw, Major::MN};
        gp.B = drt_n;
        if (slab) {  // column (i, j, ch) -> slab i; row (q, r, c) -> slab (q, r), run c
            gp.C.mdiv = g.k * g.d;
            gp.C.s_mq = S;
            gp.C.s_mr = 1;
            gp.C.ndiv = g.m;
            gp.C.s_nq = g.k * S;
            gp.C.s_n = g.k * g.d;
        } else {
            gp.C.s_mr = 1;
            gp.C.s_n = ldd;
        }
        cct_status s = gemm_capped(gp, dd, span, ws, st, "gemm (bwd-data)");
        if (s != CCT_OK) return s;
        if (ws.base && !direct) CCT_TRY(col2im(g, type, dd, ldd, dx, st), "col2im");
        hi = std::max(hi, ws.off);
        ws.off = mark;  // stream order: bwd-weight may reuse the bwd-data scratch
    }
    if (dw) {
        const bool implicit = t1_implicit(g, type, x);
        const float* dh = implicit ? nullptr
                          : (cache && !dhat_is_input(g, type, x)) ? cache
                                                                  : dhat_of(g, type, L, x, nullptr, ws, st, &e);
        CCT_TRY(e, "lower");
        const int64_t ldd = (dh == x) ? g.d : L.ldc;
        GemmProblem gp = wgrad_problem(L, {dh, ldd, Major::MN}, drt_k);
        // narrow kernel banks (ncols < 128, e.g. conv1 o = 96) with a materialised Dhat:
        // compute dW (ncols x cols) = dRhat^T * Dhat instead, so the wide lowered side
        // is the tile width N
        const bool swap = !implicit && L.ncols < 128 && L.cols >= 192;
        if (swap) {
            gp.M = L.ncols;
            gp.N = L.cols;
            gp.A = drt_k;
            gp.B = {dh, ldd, Major::MN};
        }
        if (implicit) wgrad_im2col(gp, g, x);
        gp.chain2 = wgrad_chain2(gp);
        const int splits = plan_splits(gp);
        const int64_t wsize = L.ncols * L.cols;
        float* parts = splits > 1 ? ws.take(int64_t(splits) * wsize) : dw;
        if (ws.base) {
            gp.C.ptr = parts;
            gp.C.s_mr = swap ? L.cols : 1;
            gp.C.s_n = swap ? 1 : L.cols;
            gp.C.s_split = wsize;
            gp.splits = splits;
            CCT_TRY(run_gemm(gp, st), "gemm (bwd-weight)");
            if (splits > 1)
                CCT_TRY(splitk_reduce(parts, wsize, splits, 1, wsize, wsize, dw, wsize, st), "split-K reduce");
        }
        hi = std::max(hi, ws.off);
    }
    ws.off = hi;
    return CCT_OK;
}

// ---------------------------------------------------------------------------
// batch chunking (the SPEC batching module's partitions):
// a pass whose scratch exceeds the workspace limit runs over image chunks that
// reuse the same scratch region in stream order.  Backward-weight partials of
// the chunks are summed in a fixed order (deterministic).
// ---------------------------------------------------------------------------
std::atomic<size_t> g_ws_limit{size_t(16) << 30};

size_t ws_limit() { return g_ws_limit.load(); }

Geo with_batch(Geo g, int64_t b) {
    g.b = b;
    return g;
}

// scratch bytes of one pass at batch b (planning run)
size_t plan_bytes(const Geo& g, int type, int pass, int64_t b) {
    Ws ws(nullptr);
    const float* dummy = reinterpret_cast<const float*>(uintptr_t(256));
    float* dout = reinterpret_cast<float*>(uintptr_t(256));
    const Geo gb = with_batch(g, b);
    if (pass == CCT_PASS_FWD) run_fwd_one(gb, type, dummy, dummy, nullptr, nullptr, ws, nullptr);
    else run_bwd_one(gb, type, dummy, nullptr, dummy, dummy, pass != CCT_PASS_BWD_WEIGHT ? dout : nullptr,
                     pass != CCT_PASS_BWD_DATA ? dout : nullptr, ws, nullptr);
    return ws.off;
}

// images per chunk so the pass fits the workspace limit (>= 1)
int64_t chunk_images(const Geo& g, int type, int pass) {
    const size_t full = plan_bytes(g, type, pass, g.b);
    if (full <= ws_limit() || g.b == 1) return g.b;
    const size_t one = plan_bytes(g, type, pass, 1), two = plan_bytes(g, type, pass, 2);
    const size_t per = two > one ? two - one : one;
    const size_t fixed = one > per ? one - per : 0;
    int64_t cb = ws_limit() > fixed ? int64_t((ws_limit() - fixed) / std::max<size_t>(per, 1)) : 1;
    // chunks start at 16-byte aligned image offsets (the TMA / bulk-copy paths need aligned x):
    // with an image size not a multiple of 4 floats (conv1: 227 x 227 x 3), whole groups of 4
    if ((g.n * g.n * g.d) % 4 != 0 && cb >= 4) cb &= ~int64_t(3);
    return std::max<int64_t>(1, std::min<int64_t>(cb, g.b));
}

cct_status run_fwd(const Geo& g, int type, const float* x, const float* w, float* y, float* cache, Ws& ws,
                   cudaStream_t st, const FwdOpts& opts = FwdOpts{}) {
    const int64_t cb = chunk_images(g, type, CCT_PASS_FWD);
    if (cb == g.b) return run_fwd_one(g, type, x, w, y, cache, ws, st, opts);
    const int64_t per_x = g.n * g.n * (opts.xcs ? opts.xcs : g.d), per_y = opts.ycs ? opts.ycs : g.o * g.m * g.m;
    const int64_t per_c = cache_per_image(g, type);
    const size_t base = ws.off;
    size_t hi = base;
    bool all_fused = true;
    for (int64_t q0 = 0; q0 < g.b; q0 += cb) {
        const Geo gc = with_batch(g, std::min(cb, g.b - q0));
        ws.off = base;
        bool f = false;
        FwdOpts oc = opts;
        oc.fused = &f;
        cct_status s = run_fwd_one(gc, type, x + q0 * per_x, w, y ? y + q0 * per_y : nullptr,
                                   cache ? cache + q0 * per_c : nullptr, ws, st, oc);
        if (s != CCT_OK) return s;
        all_fused = all_fused && f;
        hi = std::max(hi, ws.off);
        if (!ws.base) break;  // planning: one chunk is representative
    }
    if (opts.fused) *opts.fused = all_fused;
    ws.off = hi;
    return CCT_OK;
}

cct_status run_bwd(const Geo& g, int type, const float* x, const float* cache, const float* dy, const float* w,
                   float* dx, float* dw, Ws& ws, cudaStream_t st) {
    const int pass = dx && dw ? CCT_PASS_BWD : dx ? CCT_PASS_BWD_DATA : CCT_PASS_BWD_WEIGHT;
    const int64_t cb = chunk_images(g, type, pass);
    if (cb == g.b) return run_bwd_one(g, type, x, cache, dy, w, dx, dw, ws, st);
    const int64_t per_x = g.n * g.n * g.d, per_y = g.o * g.m * g.m, per_c = cache_per_image(g, type);
    const int64_t nchunks = (g.b + cb - 1) / cb;
    const int64_t wsize = g.o * g.k * g.k * g.d;
    float* parts = dw ? ws.take(nchunks * wsize) : nullptr;  // per-chunk dW, reduced at the end
    const size_t base = ws.off;
    size_t hi = base;
    int64_t c = 0;
    for (int64_t q0 = 0; q0 < g.b; q0 += cb, ++c) {
        const Geo gc = with_batch(g, std::min(cb, g.b - q0));
        ws.off = base;
        cct_status s = run_bwd_one(gc, type, x ? x + q0 * per_x : nullptr, cache ? cache + q0 * per_c : nullptr,
                                   dy + q0 * per_y, w, dx ? dx + q0 * per_x : nullptr,
                                   dw ? (parts ? parts + c * wsize : dw) : nullptr, ws, st);
        if (s != CCT_OK) return s;
        hi = std::max(hi, ws.off);
        if (!ws.base) break;
    }
    ws.off = hi;
    if (dw && ws.base) CCT_TRY(splitk_reduce(parts, wsize, int(nchunks), 1, wsize, wsize, dw, wsize, st), "chunk reduce");
    return CCT_OK;
}

// ---------------------------------------------------------------------------
// layer extension (cct_conv_*_ex): channel groups and the bias / ReLU epilogue
// (SURVEY 8(f) item 3).  Group j of G convolves input channels [j d/G, (j+1) d/G)
// with kernels [j o/G, (j+1) o/G) (KernelBank (o, k, k, d/G)).  Implicit Type 1
// reads a group's channels straight from x and writes straight into y (TMA
// im2col over a channel view, strided epilogue, fused bias / ReLU); the other
// forms gather the group into contiguous scratch and scatter the result back.
// ---------------------------------------------------------------------------
struct Ext {
    int64_t groups = 1;
    const float* bias = nullptr;
    int relu = 0;
};

Geo group_geo(const Geo& g, int64_t G) {
    Geo v = g;
    v.d = g.d / G;
    v.o = g.o / G;
    return v;
}

// the direct (no gather / scatter) grouped forward: implicit Type 1, one chain
bool group_direct(const Geo& gg, int type) {
    return type == 1 && t1_implicit(gg, type, kPlanPtr) && !t1_s2d(gg, type) &&
           gg.k * gg.k * gg.d <= int64_t(kMaxChainKB) * kBK;
}

cct_status run_fwd_ex(const Geo& g, int type, const Ext& e, const float* x, const float* w, float* y, Ws& ws,
                      cudaStream_t st) {
    const int64_t G = e.groups, mm = g.m * g.m;
    const Geo gg = group_geo(g, G);
    const int64_t dg = gg.d, og = gg.o, wsz = og * g.k * g.k * dg;
    if (G == 1 || group_direct(gg, type)) {
        const size_t mark = ws.off;
        size_t hi = mark;
        for (int64_t j = 0; j < G; ++j) {
            ws.off = mark;
            bool fused = false;
            FwdOpts o;
            o.xcs = G > 1 ? g.d : 0;
            o.ycs = G > 1 ? g.o * mm : 0;
            o.bias = e.bias ? e.bias + j * og : nullptr;
            o.relu = e.relu;
            o.fused = &fused;
            cct_status s = run_fwd(G > 1 ? gg : g, type, x + j * dg, w + j * wsz, y + j * og * mm, nullptr, ws, st, o);
            if (s != CCT_OK) return s;
            hi = std::max(hi, ws.off);
            if (ws.base && !fused && (e.bias || e.relu))
                CCT_TRY(bias_act(y + j * og * mm, o.bias, e.relu, g.b, og, mm, g.o, st), "bias / ReLU");
            if (!ws.base) break;  // planning: every group needs the same scratch
        }
        ws.off = hi;
        return CCT_OK;
    }
    float* xg = ws.take(g.b * g.n * g.n * dg);
    float* yg = ws.take(g.b * og * mm);
    const size_t mark = ws.off;
    size_t hi = mark;
    for (int64_t j = 0; j < G; ++j) {
        ws.off = mark;
        if (ws.base) CCT_TRY(copy2d(xg, dg, x + j * dg, g.d, dg, g.b * g.n * g.n, st), "gather channel group");
        cct_status s = run_fwd(gg, type, or_plan(xg, ws), w + j * wsz, or_plan(yg, ws), nullptr, ws, st);
        if (s != CCT_OK) return s;
        hi = std::max(hi, ws.off);
        if (!ws.base) break;
        CCT_TRY(copy2d(y + j * og * mm, g.o * mm, yg, og * mm, og * mm, g.b, st), "scatter channel group");
    }
    ws.off = hi;
    if (ws.base) CCT_TRY(bias_act(y, e.bias, e.relu, g.b, g.o, mm, g.o, st), "bias / ReLU");
    return CCT_OK;
}

// dy is the gradient of the layer output (after the ReLU); y that output
cct_status run_bwd_ex(const Geo& g, int type, const Ext& e, const float* x, const float* y, const float* dy,
                      const float* w, float* dx, float* dw, float* db, Ws& ws, cudaStream_t st) {
    const int64_t G = e.groups, mm = g.m * g.m;
    const float* dz = dy;
    if (e.relu || db) {
        float* z = e.relu ? ws.take(g.b * g.o * mm) : nullptr;
        float* partial = db ? ws.take(g.b * g.o) : nullptr;
        if (ws.base) CCT_TRY(relu_bias_bwd(dy, y, z, db, partial, e.relu, g.b, g.o, mm, st), "ReLU / bias backward");
        if (e.relu) dz = or_plan(z, ws);
    }
    if (!dx && !dw) return CCT_OK;
    if (G == 1) return run_bwd(g, type, x, nullptr, dz, w, dx, dw, ws, st);
    const Geo gg = group_geo(g, G);
    const int64_t dg = gg.d, og = gg.o, wsz = og * g.k * g.k * dg;
    float* zg = ws.take(g.b * og * mm);
    float* xg = dw ? ws.take(g.b * g.n * g.n * dg) : nullptr;
    float* dxg = dx ? ws.take(g.b * g.n * g.n * dg) : nullptr;
    const size_t mark = ws.off;
    size_t hi = mark;
    for (int64_t j = 0; j < G; ++j) {
        ws.off = mark;
        if (ws.base) {
            CCT_TRY(copy2d(zg, og * mm, dz + j * og * mm, g.o * mm, og * mm, g.b, st), "gather dy group");
            if (dw) CCT_TRY(copy2d(xg, dg, x + j * dg, g.d, dg, g.b * g.n * g.n, st), "gather x group");
        }
        cct_status s = run_bwd(gg, type, dw ? or_plan(xg, ws) : nullptr, nullptr, or_plan(zg, ws), w + j * wsz,
                               dx ? or_plan(dxg, ws) : nullptr, dw ? dw + j * wsz : nullptr, ws, st);
        if (s != CCT_OK) return s;
        hi = std::max(hi, ws.off);
        if (!ws.base) break;
        if (dx) CCT_TRY(copy2d(dx + j * dg, g.d, dxg, dg, dg, g.b * g.n * g.n, st), "scatter dx group");
    }
    ws.off = hi;
    return CCT_OK;
}

cct_status check_ext(const cct_conv_desc* d, const cct_conv_ext* x, Ext* e) {
    if (d->layout != CCT_LAYOUT_NCHW) return fail(CCT_ERR_UNSUPPORTED, "the _ex extension takes NCHW y / dy");
    if (x) {
        e->groups = x->groups;
        e->bias = x->bias;
        e->relu = x->relu;
    }
    if (e->groups < 1 || d->d % e->groups || d->o % e->groups)
        return fail(CCT_ERR_CONFIG, "groups must be >= 1 and divide d and o " + desc_str(d));
    if (e->relu != 0 && e->relu != 1) return fail(CCT_ERR_CONFIG, "relu must be 0 or 1");
    if (e->bias && !aligned16(e->bias)) return fail(CCT_ERR_CONFIG, "bias must be 16-byte aligned");
    return CCT_OK;
}

cct_status check_ptrs(std::initializer_list<const void*> ps) {
    for (const void* p : ps)
        if (!p) return fail(CCT_ERR_CONFIG, "null tensor pointer");
    return CCT_OK;
}

}  // namespace

extern "C" {

int cct_abi_version(void) { return CCT_ABI_VERSION; }

int cct_device_info(char* name, size_t len, int* sms) {
    int dev = 0, n = 0;
    cudaDeviceProp prop;
    const bool ok = cudaGetDeviceCount(&n) == cudaSuccess && n > 0 && cudaGetDevice(&dev) == cudaSuccess &&
                    cudaGetDeviceProperties(&prop, dev) == cudaSuccess;
    if (!ok) cudaGetLastError();  // clear the sticky "no device" error
    if (name && len) snprintf(name, len, "%s", ok ? prop.name : "none");
    if (sms) *sms = ok ? prop.multiProcessorCount : 0;
    return ok ? n : 0;
}
void cct_set_workspace_limit(size_t bytes) { g_ws_limit = bytes; }
void cct_set_implicit_lowering(int mode) { g_implicit = std::max(0, std::min(2, mode)); }
int cct_get_implicit_lowering(void) { return implicit_enabled() ? g_implicit.load() : 0; }
size_t cct_get_workspace_limit(void) { return ws_limit(); }
void cct_profile_enable(int on) { cct::profile_enable(on != 0); }
void cct_profile_read(double* ms, double* flops, double* bytes, uint64_t* launches, int reset) {
    cct::profile_read(ms, flops, bytes, launches, reset != 0);
}
const char* cct_last_error(void) { return cct::last_error(); }
uint64_t cct_launch_count(void) { return cct::launch_count(); }
void cct_reset_launch_count(void) { cct::reset_launch_count(); }

cct_status cct_conv_desc_init(cct_conv_desc* desc, int64_t n, int64_t k, int64_t d, int64_t o, int64_t b,
                              int64_t stride, int64_t pad) {
    if (!desc) return fail(CCT_ERR_CONFIG, "null conv descriptor");
    desc->n = n; desc->k = k; desc->d = d; desc->o = o; desc->b = b; desc->stride = stride; desc->pad = pad;
    desc->m = desc->R = 0;
    desc->layout = CCT_LAYOUT_NCHW;
    cct_status s = check_desc(desc);
    if (s != CCT_OK) return s;
    const Geo g = geo_of(desc);
    desc->m = g.m;
    desc->R = g.R;
    return CCT_OK;
}

cct_status cct_conv_desc_set_layout(cct_conv_desc* desc, cct_layout layout) {
    if (!desc) return fail(CCT_ERR_CONFIG, "null conv descriptor");
    if (layout != CCT_LAYOUT_NCHW && layout != CCT_LAYOUT_NHWC) return fail(CCT_ERR_CONFIG, "unknown layout");
    desc->layout = layout;
    return CCT_OK;
}

cct_status cct_workspace_size(const cct_conv_desc* desc, cct_lowering lowering, cct_pass pass, size_t* bytes) {
    cct_status s = check_desc(desc);
    if (s != CCT_OK) return s;
    if (!bytes) return fail(CCT_ERR_CONFIG, "null size pointer");
    const Geo g = geo_of(desc);
    const int type = resolve(desc, lowering, pass);
    if (int(pass) < CCT_PASS_FWD || int(pass) > CCT_PASS_BWD) return fail(CCT_ERR_CONFIG, "unknown pass");
    // dummy, 16-byte aligned non-null pointers so zero-copy decisions match the real call
    const float* dummy = reinterpret_cast<const float*>(uintptr_t(256));
    float* dout = reinterpret_cast<float*>(uintptr_t(256));
    // the size covers the pass both stand-alone and inside a training step (the
    // two may pick different forms of a strided layer, t1_s2d)
    size_t most = 0;
    for (int ctx : {int(pass) == CCT_PASS_BWD ? 3 : int(pass), 3}) {
        PassCtx pc(ctx);
        Ws ws(nullptr);
        switch (int(pass)) {
        case CCT_PASS_FWD: s = run_fwd(g, type, dummy, dummy, nullptr, nullptr, ws, nullptr); break;
        case CCT_PASS_BWD_DATA: s = run_bwd(g, type, dummy, nullptr, dummy, dummy, dout, nullptr, ws, nullptr); break;
        case CCT_PASS_BWD_WEIGHT: s = run_bwd(g, type, dummy, nullptr, dummy, dummy, nullptr, dout, ws, nullptr); break;
        default: s = run_bwd(g, type, dummy, nullptr, dummy, dummy, dout, dout, ws, nullptr); break;
        }
        if (s != CCT_OK) return s;
        most = std::max(most, ws.off);
    }
    *bytes = most + 256;
    return s;
}

static cct_status run_pass(const cct_conv_desc* desc, cct_lowering lowering, cct_pass pass, const float* a,
                           const float* b, float* out, void* wsp, size_t ws_bytes, void* stream) {
    cct_status s = check_desc(desc);
    if (s != CCT_OK) return s;
    if ((s = check_ptrs({a, b, out})) != CCT_OK) return s;
    if (!aligned16(a) || !aligned16(b) || !aligned16(out))
        return fail(CCT_ERR_CONFIG, "tensor pointers must be 16-byte aligned (cudaMalloc / torch allocations are)");
    size_t need = 0;
    if ((s = cct_workspace_size(desc, lowering, pass, &need)) != CCT_OK) return s;
    if (ws_bytes < need || !wsp) {
        std::ostringstream os;
        os << "workspace too small: need " << need << " bytes, got " << ws_bytes << " for " << desc_str(desc);
        return fail(CCT_ERR_RESOURCE, os.str());
    }
    const Geo g = geo_of(desc);
    const int type = resolve(desc, lowering, pass);
    Ws ws(wsp);
    cudaStream_t st = as_stream(stream);
    PassCtx pc{int(pass)};
    switch (pass) {
    case CCT_PASS_FWD: return run_fwd(g, type, a, b, out, nullptr, ws, st);
    case CCT_PASS_BWD_DATA: return run_bwd(g, type, nullptr, nullptr, a, b, out, nullptr, ws, st);
    default: return run_bwd(g, type, a, nullptr, b, nullptr, nullptr, out, ws, st);
    }
}

cct_status cct_conv_fwd(const cct_conv_desc* desc, cct_lowering lowering, const float* x, const float* w,
                        float* y, void* ws, size_t ws_bytes, void* stream) {
    return run_pass(desc, lowering, CCT_PASS_FWD, x, w, y, ws, ws_bytes, stream);
}

cct_status cct_conv_bwd_data(const cct_conv_desc* desc, cct_lowering lowering, const float* dy, const float* w,
                             float* dx, void* ws, size_t ws_bytes, void* stream) {
    return run_pass(desc, lowering, CCT_PASS_BWD_DATA, dy, w, dx, ws, ws_bytes, stream);
}

cct_status cct_conv_bwd_weight(const cct_conv_desc* desc, cct_lowering lowering, const float* x,
                               const float* dy, float* dw, void* ws, size_t ws_bytes, void* stream) {
    return run_pass(desc, lowering, CCT_PASS_BWD_WEIGHT, x, dy, dw, ws, ws_bytes, stream);
}

static int resolve_train(const cct_conv_desc* d, cct_lowering l) {
    // fwd_cached and bwd must agree on the type (the cache layout depends on it):
    // AUTO scores fwd + bwd together.
    return resolve(d, l, cct_pass(CCT_PASS_BWD));
}

cct_status cct_lowered_cache_size(const cct_conv_desc* desc, cct_lowering lowering, size_t* bytes) {
    cct_status s = check_desc(desc);
    if (s != CCT_OK) return s;
    if (!bytes) return fail(CCT_ERR_CONFIG, "null size pointer");
    const Geo g = geo_of(desc);
    const int type = resolve_train(desc, lowering);
    PassCtx pc(3);
    const float* aligned = reinterpret_cast<const float*>(uintptr_t(256));
    *bytes = (!t1_s2d(g, type) && (dhat_is_input(g, type, aligned) || t1_implicit(g, type, aligned)))
                 ? 0
                 : size_t(g.b * cache_per_image(g, type)) * sizeof(float);
    return CCT_OK;
}

cct_status cct_conv_fwd_cached(const cct_conv_desc* desc, cct_lowering lowering, const float* x, const float* w,
                               float* y, float* cache, size_t cache_bytes, void* wsp, size_t ws_bytes,
                               void* stream) {
    cct_status s = check_desc(desc);
    if (s != CCT_OK) return s;
    if ((s = check_ptrs({x, w, y})) != CCT_OK) return s;
    if (!aligned16(x) || !aligned16(w) || !aligned16(y) || (cache && !aligned16(cache)))
        return fail(CCT_ERR_CONFIG, "tensor pointers must be 16-byte aligned");
    const int type = resolve_train(desc, lowering);
    size_t need = 0, cneed = 0;
    cct_workspace_size(desc, cct_lowering(type), CCT_PASS_FWD, &need);
    cct_lowered_cache_size(desc, cct_lowering(type), &cneed);
    if (cache && cache_bytes < cneed) return fail(CCT_ERR_RESOURCE, "lowered cache too small for " + desc_str(desc));
    if (!wsp || ws_bytes < need) return fail(CCT_ERR_RESOURCE, "workspace too small for " + desc_str(desc));
    Ws ws(wsp);
    PassCtx pc(3);
    return run_fwd(geo_of(desc), type, x, w, y, cneed ? cache : nullptr, ws, as_stream(stream));
}

cct_status cct_conv_bwd(const cct_conv_desc* desc, cct_lowering lowering, const float* x, const float* cache,
                        const float* dy, const float* w, float* dx, float* dw, void* wsp, size_t ws_bytes,
                        void* stream) {
    cct_status s = check_desc(desc);
    if (s != CCT_OK) return s;
    if (!dy || (!dx && !dw)) return fail(CCT_ERR_CONFIG, "cct_conv_bwd needs dy and at least one of dx, dw");
    if (dx && !w) return fail(CCT_ERR_CONFIG, "bwd-data needs w");
    if (dw && !x && !cache) return fail(CCT_ERR_CONFIG, "bwd-weight needs x or a lowered cache");
    for (const void* p : {static_cast<const void*>(x), static_cast<const void*>(cache), static_cast<const void*>(dy),
                          static_cast<const void*>(w), static_cast<const void*>(dx), static_cast<const void*>(dw)})
        if (p && !aligned16(p)) return fail(CCT_ERR_CONFIG, "tensor pointers must be 16-byte aligned");
    const int type = resolve_train(desc, lowering);
    size_t need = 0;
    cct_workspace_size(desc, cct_lowering(type), CCT_PASS_BWD, &need);
    if (!wsp || ws_bytes < need) return fail(CCT_ERR_RESOURCE, "workspace too small for " + desc_str(desc));
    Ws ws(wsp);
    const Geo g = geo_of(desc);
    // a cache is only meaningful when the forward wrote one: not when Dhat is the input itself, and
    // not for the implicit forms (cct_lowered_cache_size 0: cct_conv_fwd_cached left it untouched)
    size_t cneed = 0;
    if ((s = cct_lowered_cache_size(desc, cct_lowering(type), &cneed)) != CCT_OK) return s;
    const float* c = (cache && cneed && !(x && dhat_is_input(g, type, x))) ? cache : nullptr;
    if (dw && !x && !c) return fail(CCT_ERR_CONFIG, "bwd-weight needs x for this lowering");
    PassCtx pc(3);
    return run_bwd(g, type, x, c, dy, w, dx, dw, ws, as_stream(stream));
}

// ---- layer extension: groups, bias, ReLU ------------------

static int resolve_ex(const cct_conv_desc* desc, const Ext& e, cct_lowering l, cct_pass pass) {
    cct_conv_desc gd = *desc;  // the lowering choice is the group's (each group is one such layer)
    gd.d /= e.groups;
    gd.o /= e.groups;
    return resolve(&gd, l, pass);
}

static cct_status plan_ex(const cct_conv_desc* desc, const Ext& e, int type, cct_pass pass, size_t* bytes) {
    const Geo g = geo_of(desc);
    const float* dummy = kPlanPtr;
    float* dout = const_cast<float*>(kPlanPtr);
    size_t most = 0;
    for (int ctx : {int(pass) == CCT_PASS_BWD ? 3 : int(pass), 3}) {
        PassCtx pc(ctx);
        Ws ws(nullptr);
        cct_status s;
        if (pass == CCT_PASS_FWD) s = run_fwd_ex(g, type, e, dummy, dummy, dout, ws, nullptr);
        else s = run_bwd_ex(g, type, e, dummy, dummy, dummy, dummy, pass != CCT_PASS_BWD_WEIGHT ? dout : nullptr,
                            pass != CCT_PASS_BWD_DATA ? dout : nullptr, dout, ws, nullptr);
        if (s != CCT_OK) return s;
        most = std::max(most, ws.off);
    }
    *bytes = most + 256;
    return CCT_OK;
}

cct_status cct_workspace_size_ex(const cct_conv_desc* desc, cct_lowering lowering, const cct_conv_ext* ext,
                                 cct_pass pass, size_t* bytes) {
    cct_status s = check_desc(desc);
    if (s != CCT_OK) return s;
    Ext e;
    if ((s = check_ext(desc, ext, &e)) != CCT_OK) return s;
    if (!bytes) return fail(CCT_ERR_CONFIG, "null size pointer");
    if (int(pass) < CCT_PASS_FWD || int(pass) > CCT_PASS_BWD) return fail(CCT_ERR_CONFIG, "unknown pass");
    return plan_ex(desc, e, resolve_ex(desc, e, lowering, pass), pass, bytes);
}

cct_status cct_conv_fwd_ex(const cct_conv_desc* desc, cct_lowering lowering, const cct_conv_ext* ext, const float* x,
                           const float* w, float* y, void* wsp, size_t ws_bytes, void* stream) {
    cct_status s = check_desc(desc);
    if (s != CCT_OK) return s;
    Ext e;
    if ((s = check_ext(desc, ext, &e)) != CCT_OK) return s;
    if ((s = check_ptrs({x, w, y})) != CCT_OK) return s;
    if (!aligned16(x) || !aligned16(w) || !aligned16(y))
        return fail(CCT_ERR_CONFIG, "tensor pointers must be 16-byte aligned");
    const int type = resolve_ex(desc, e, lowering, CCT_PASS_FWD);
    size_t need = 0;
    if ((s = plan_ex(desc, e, type, CCT_PASS_FWD, &need)) != CCT_OK) return s;
    if (!wsp || ws_bytes < need) return fail(CCT_ERR_RESOURCE, "workspace too small for " + desc_str(desc));
    Ws ws(wsp);
    PassCtx pc(CCT_PASS_FWD);
    return run_fwd_ex(geo_of(desc), type, e, x, w, y, ws, as_stream(stream));
}

cct_status cct_conv_bwd_ex(const cct_conv_desc* desc, cct_lowering lowering, const cct_conv_ext* ext, const float* x,
                           const float* y, const float* dy, const float* w, float* dx, float* dw, float* db,
                           void* wsp, size_t ws_bytes, void* stream) {
    cct_status s = check_desc(desc);
    if (s != CCT_OK) return s;
    Ext e;
    if ((s = check_ext(desc, ext, &e)) != CCT_OK) return s;
    if (!dy || (!dx && !dw && !db)) return fail(CCT_ERR_CONFIG, "cct_conv_bwd_ex needs dy and one of dx, dw, db");
    if (dx && !w) return fail(CCT_ERR_CONFIG, "bwd-data needs w");
    if (dw && !x) return fail(CCT_ERR_CONFIG, "bwd-weight needs x");
    if (e.relu && !y) return fail(CCT_ERR_CONFIG, "the ReLU backward needs the layer output y");
    for (const void* p : {static_cast<const void*>(x), static_cast<const void*>(y), static_cast<const void*>(dy),
                          static_cast<const void*>(w), static_cast<const void*>(dx), static_cast<const void*>(dw),
                          static_cast<const void*>(db)})
        if (p && !aligned16(p)) return fail(CCT_ERR_CONFIG, "tensor pointers must be 16-byte aligned");
    const cct_pass pass = dx && dw ? CCT_PASS_BWD : dx ? CCT_PASS_BWD_DATA : CCT_PASS_BWD_WEIGHT;
    const int type = resolve_ex(desc, e, lowering, pass);
    size_t need = 0;
    if ((s = plan_ex(desc, e, type, pass, &need)) != CCT_OK) return s;
    if (!wsp || ws_bytes < need) return fail(CCT_ERR_RESOURCE, "workspace too small for " + desc_str(desc));
    Ws ws(wsp);
    PassCtx pc{int(pass)};
    return run_bwd_ex(geo_of(desc), type, e, x, y, dy, w, dx, dw, db, ws, as_stream(stream));
}

// ---- phase-level API ---------------------------------------------------------

static cct_status phase_geo(const cct_conv_desc* desc, cct_lowering lowering, cct_row_order order, Geo* g,
                            RowMap* rm) {
    cct_status s = check_desc(desc);
    if (s != CCT_OK) return s;
    if (lowering < CCT_LOWER_T1 || lowering > CCT_LOWER_T3)
        return fail(CCT_ERR_CONFIG, "phase API needs an explicit lowering type (1, 2 or 3)");
    *g = geo_of(desc);
    if (order == CCT_ROWS_SPEC) {
        if (g->s != 1 || g->p != 0)
            return fail(CCT_ERR_UNSUPPORTED, "SPEC row order is defined for stride 1, pad 0 only (SPEC.md:85)");
        *rm = rowmap_spec(*g, int(lowering));
    } else {
        *rm = rowmap_internal(*g, int(lowering));
    }
    return CCT_OK;
}

cct_status cct_lowered_shape(const cct_conv_desc* desc, cct_lowering lowering, cct_row_order order,
                             int64_t* rows, int64_t* cols, int64_t* kcols) {
    Geo g;
    RowMap rm;
    cct_status s = phase_geo(desc, lowering, order, &g, &rm);
    if (s != CCT_OK) return s;
    if (rows) *rows = g.b * rm.rpi;
    if (cols) *cols = lowered_cols(g, int(lowering));
    if (kcols) *kcols = lowered_ncols(g, int(lowering));
    return CCT_OK;
}

cct_status cct_lower(const cct_conv_desc* desc, cct_lowering lowering, cct_row_order order, const float* x,
                     float* dhat, int64_t ld, void* stream) {
    Geo g;
    RowMap rm;
    cct_status s = phase_geo(desc, lowering, order, &g, &rm);
    if (s != CCT_OK) return s;
    if ((s = check_ptrs({x, dhat})) != CCT_OK) return s;
    if (ld < lowered_cols(g, int(lowering))) return fail(CCT_ERR_CONFIG, "ld smaller than the lowered row length");
    return cuda_status(lower(g, int(lowering), rm, x, dhat, ld, as_stream(stream)), "lower");
}

cct_status cct_lower_khat(const cct_conv_desc* desc, cct_lowering lowering, const float* w, float* khat,
                          void* stream) {
    Geo g;
    RowMap rm;
    cct_status s = phase_geo(desc, lowering, CCT_ROWS_INTERNAL, &g, &rm);
    if (s != CCT_OK) return s;
    if ((s = check_ptrs({w, khat})) != CCT_OK) return s;
    const int64_t cols = lowered_cols(g, int(lowering)), ncols = lowered_ncols(g, int(lowering));
    // KernelBank storage is Khat^T (ncols x cols); Khat is its transpose
    return cuda_status(transpose(w, ncols, cols, cols, khat, ncols, as_stream(stream)), "transpose");
}

cct_status cct_lift(const cct_conv_desc* desc, cct_lowering lowering, cct_row_order order, const float* rhat,
                    int64_t ld, float* y, void* stream) {
    Geo g;
    RowMap rm;
    cct_status s = phase_geo(desc, lowering, order, &g, &rm);
    if (s != CCT_OK) return s;
    if ((s = check_ptrs({rhat, y})) != CCT_OK) return s;
    if (ld < lowered_ncols(g, int(lowering))) return fail(CCT_ERR_CONFIG, "ld smaller than the Rhat row length");
    return cuda_status(lift(g, int(lowering), rm, rhat, ld, 1, y, as_stream(stream)), "lift");
}

// ---- GEMM (multiply replacement) ---------------------------------------------

static cct_status gemm_common(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B,
                              int64_t ldb, float* C, int64_t ldc, int split_k, void* ws, size_t ws_bytes,
                              int passes, void* stream) {
    if (M < 0 || N < 0 || K < 0) return fail(CCT_ERR_CONFIG, "negative GEMM extent");
    if (M == 0 || N == 0) return CCT_OK;
    if (!A || !B || !C) return fail(CCT_ERR_CONFIG, "null matrix pointer");
    if (lda < K || ldb < N || ldc < N) return fail(CCT_ERR_CONFIG, "leading dimension smaller than the row length");
    if (lda % 4 || ldb % 4 || !aligned16(A) || !aligned16(B))
        return fail(CCT_ERR_CONFIG, "A/B must be 16-byte aligned with lda, ldb multiples of 4 (TMA)");
    cudaStream_t st = as_stream(stream);
    if (K == 0) {
        return cuda_status(cudaMemset2DAsync(C, size_t(ldc) * 4, 0, size_t(N) * 4, size_t(M), st), "memset");
    }
    // Orientation: lanes run over N (columns of C are contiguous):
    //   C^T (N x M) = B^T (N x K) * A^T:  A' = B stored (K rows x N) -> MN-major,
    //   B' = A stored (M rows x K) -> K-major, C'(n, m) at C + m*ldc + n.
    GemmProblem gp;
    gp.M = N;
    gp.N = M;
    gp.K = K;
    gp.A = {B, ldb, Major::MN};
    gp.B = {A, lda, Major::K};
    gp.passes = passes;
    const int64_t kb = (K + kBK - 1) / kBK;
    // accuracy floor: every TMEM accumulation chain <= kMaxChainKB k-blocks (the tensor core
    // truncates its fp32 accumulation, so one long chain drifts ~linearly with K)
    const int floor_splits = effective_splits(kb, int((kb + kMaxChainKB - 1) / kMaxChainKB));
    int splits = split_k > 0 ? effective_splits(kb, std::max(split_k, floor_splits)) : plan_splits(gp);
    if (passes != 3) splits = 1;
    if (splits > 1) {
        const size_t need = size_t(splits) * size_t(M) * size_t(N) * 4;
        if (!ws || ws_bytes < need) {
            if (passes == 3 && floor_splits > 1) {
                std::ostringstream os;
                os << "gemm (" << M << " x " << N << " x " << K << "): K needs " << floor_splits
                   << " accumulation chains for fp32 accuracy; workspace of " << need << " bytes required, got "
                   << (ws ? ws_bytes : 0) << " (cct_gemm_workspace_size)";
                return fail(CCT_ERR_RESOURCE, os.str());
            }
            splits = 1;  // wave-fill splits only: run unsplit
        }
    }
    if (splits > 1) {
        float* parts = static_cast<float*>(ws);
        gp.C = {parts, INT64_MAX, 0, 1, N, M * N};
        gp.splits = splits;
        CCT_TRY(run_gemm(gp, st), "gemm");
        return cuda_status(splitk_reduce(parts, M * N, splits, M, N, N, C, ldc, st), "split-K reduce");
    }
    gp.C = {C, INT64_MAX, 0, 1, ldc, 0};
    return cuda_status(run_gemm(gp, st), "gemm");
}

cct_status cct_gemm_workspace_size(int64_t M, int64_t N, int64_t K, int split_k, size_t* bytes) {
    if (!bytes) return fail(CCT_ERR_CONFIG, "null size pointer");
    GemmProblem gp;  // same orientation as gemm_common
    gp.M = N;
    gp.N = M;
    gp.K = K;
    gp.A.major = Major::MN;
    gp.B.major = Major::K;
    const int64_t kb = (K + kBK - 1) / kBK;
    const int floor_splits = effective_splits(kb, int((kb + kMaxChainKB - 1) / kMaxChainKB));
    const int splits = split_k > 0 ? effective_splits(kb, std::max(split_k, floor_splits)) : plan_splits(gp);
    *bytes = splits > 1 ? size_t(splits) * size_t(M) * size_t(N) * 4 : 0;
    return CCT_OK;
}

cct_status cct_gemm(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B, int64_t ldb,
                    float* C, int64_t ldc, int split_k, void* ws, size_t ws_bytes, void* stream) {
    return gemm_common(M, N, K, A, lda, B, ldb, C, ldc, split_k, ws, ws_bytes, 3, stream);
}

cct_status cct_gemm_passes(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B,
                           int64_t ldb, float* C, int64_t ldc, int passes, void* stream) {
    if (passes != 1 && passes != 3) return fail(CCT_ERR_CONFIG, "passes must be 1 or 3");
    return gemm_common(M, N, K, A, lda, B, ldb, C, ldc, 1, nullptr, 0, passes, stream);
}

cct_status cct_debug_gemm(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, int a_major,
                          const float* B, int64_t ldb, int b_major, float* C, int64_t ldc_m, int64_t ldc_n,
                          int passes, int bn, void* stream) {
    if (M <= 0 || N <= 0 || K <= 0 || !A || !B || !C) return fail(CCT_ERR_CONFIG, "bad debug gemm arguments");
    if (lda % 4 || ldb % 4 || !aligned16(A) || !aligned16(B)) return fail(CCT_ERR_CONFIG, "TMA alignment");
    GemmProblem gp;
    gp.M = M;
    gp.N = N;
    gp.K = K;
    gp.A = {A, lda, a_major ? Major::MN : Major::K};
    gp.B = {B, ldb, b_major ? Major::MN : Major::K};
    gp.C = {C, INT64_MAX, 0, ldc_m, ldc_n, 0};
    gp.C.transposed = (passes & 0x100) ? 1 : 0;  // diagnostic: transposing epilogue
    gp.passes = passes & 0xFF;
    gp.bn = bn;
    return cuda_status(run_gemm(gp, as_stream(stream)), "gemm");
}

}  // extern "C"
