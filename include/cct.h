/*
 * cct.h -- C ABI of the B200-native Caffe con Troll convolution hot path.
 *
 * This is the drop-in boundary.  The reference has no FFI: its operator API is
 * the C++ `convlow` namespace.  Each entry point below names
 * the reference interface it replaces (file:line under /root/reference).  The
 * C++ `convlow` mirror in include/convlow/*.hpp is implemented on top of this
 * ABI, so a caller of the reference API switches by relinking.
 *
 * Conventions
 *   - Plain pointers and sizes only; every tensor pointer is a DEVICE pointer
 *     (cudaMalloc'd or torch-owned) unless the name ends in `_host`.
 *   - The caller owns all device memory.  Scratch space is sized by
 *     cct_workspace_size() and passed in; no hidden allocations on the hot path.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Calls are asynchronous w.r.t. the host; no host sync inside.
 *   - Status codes: CCT_ERR_CONFIG maps to convlow::config_error,
 *     CCT_ERR_RESOURCE / CCT_ERR_CUDA to convlow::resource_error
 *     (common.hpp:17-24).  cct_last_error() returns a thread-local message
 *     naming the offending shapes, like the reference messages
 *     (tensor.cpp:23-30, gemm.cpp:19-34).
 *   - Layouts are the reference containers':
 *       x, dx : DataBatch  = b images of Tensor3 HWC, depth-minor  (tensor.hpp:28-35, 105-122)
 *       w, dw : KernelBank = (o, k, k, d) depth-minor              (tensor.hpp:70-75)
 *       y, dy : OutputBatch = NCHW ((q*o+j)*m+r)*m+c               (tensor.hpp:135-150)
 *   - Arithmetic is fp32 in / fp32 out; GEMMs run on tcgen05 tensor cores with
 *     3xTF32 split emulation (relative L2 <= 1e-4 against the fp64-accumulated
 *     reference).  No CPU fallback exists: without an sm_100
 *     device every compute entry point returns CCT_ERR_CUDA.
 */
#ifndef CCT_H
#define CCT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CCT_ABI_VERSION 1

#if defined(__GNUC__)
#define CCT_API __attribute__((visibility("default")))
#else
#define CCT_API
#endif

typedef enum {
    CCT_OK = 0,
    CCT_ERR_CONFIG = 1,      /* bad shape / argument        -> convlow::config_error   */
    CCT_ERR_RESOURCE = 2,    /* workspace too small, OOM    -> convlow::resource_error */
    CCT_ERR_CUDA = 3,        /* CUDA runtime / no device    -> convlow::resource_error */
    CCT_ERR_UNSUPPORTED = 4  /* valid but not implemented   -> convlow::config_error   */
} cct_status;

/* LoweringStrategy plus AUTO (cost-model choice). */
typedef enum {
    CCT_LOWER_AUTO = 0,
    CCT_LOWER_T1 = 1, /* Type 1: expensive lowering (im2col)  */
    CCT_LOWER_T2 = 2, /* Type 2: balanced                      */
    CCT_LOWER_T3 = 3  /* Type 3: expensive lifting             */
} cct_lowering;

/* CCT_PASS_BWD = bwd-data + bwd-weight in one call (cct_conv_bwd). */
typedef enum { CCT_PASS_FWD = 0, CCT_PASS_BWD_DATA = 1, CCT_PASS_BWD_WEIGHT = 2, CCT_PASS_BWD = 3 } cct_pass;

/* Row order of a lowered matrix returned by cct_lower / consumed by cct_lift.
 * SPEC: the reference's c*m+r (T1) / c*n+r (T2, T3) order with n^2 rows per
 * image for T2/T3 and zero-filled rows; stride 1,
 * pad 0 only.  INTERNAL: the row-major compact order the fast path uses
 * (SURVEY Appendix A), any stride / pad. */
typedef enum { CCT_ROWS_SPEC = 0, CCT_ROWS_INTERNAL = 1 } cct_row_order;

/* Layout of the layer output y and its gradient dy.  NCHW is the reference's
 * OutputBatch ((q*o+j)*m+r)*m+c (tensor.hpp:135-150) and the default; NHWC
 * ((q*m+r)*m+c)*o+j is the DataBatch order of the NEXT layer's input
 * (tensor.hpp:28-35), so layers chain without a re-layout, and the implicit
 * backward reads dy as is (no transpose). */
typedef enum { CCT_LAYOUT_NCHW = 0, CCT_LAYOUT_NHWC = 1 } cct_layout;

/* LayerConfig (tensor.hpp:15-26) extended with stride and zero padding
 * (defaults 1 / 0 keep the reference semantics).  m = (n + 2p - k)/s + 1. */
typedef struct {
    int64_t n, k, d, o, b, stride, pad;
    int64_t m;      /* derived output side                        */
    int64_t R;      /* derived padded extent actually touched: s(m-1)+k */
    int64_t layout; /* cct_layout of y / dy; cct_conv_desc_init sets NCHW */
} cct_conv_desc;

/* Replaces LayerConfig::validate (tensor.cpp:23-30) / layer_of (tensor.cpp:66-75):
 * CCT_ERR_CONFIG unless 1 <= k <= n + 2 pad, d, o, b >= 1, stride >= 1, pad >= 0. */
CCT_API cct_status cct_conv_desc_init(cct_conv_desc* desc, int64_t n, int64_t k, int64_t d, int64_t o,
                              int64_t b, int64_t stride, int64_t pad);
/* y / dy layout of every pass of this layer (SURVEY 8(b) y_layout): every entry point
 * honours it except the _ex extension and the exact (oracle) entry points, which
 * return CCT_ERR_UNSUPPORTED for NHWC. */
CCT_API cct_status cct_conv_desc_set_layout(cct_conv_desc* desc, cct_layout layout);

/* Scratch bytes one call of (lowering, pass) needs.  AUTO resolves through
 * cct_select_lowering with the default calibration. */
CCT_API cct_status cct_workspace_size(const cct_conv_desc* desc, cct_lowering lowering, cct_pass pass,
                              size_t* bytes);

/* convolve_lowered: y = lift(multiply(lower(x, w))).
 * x (b,n,n,d) NHWC, w (o,k,k,d), y (b,o,m,m) NCHW. */
CCT_API cct_status cct_conv_fwd(const cct_conv_desc* desc, cct_lowering lowering, const float* x,
                        const float* w, float* y, void* ws, size_t ws_bytes, void* stream);

/* Backward-data (north_star; absent from the reference): dx = d(sum(y*dy))/dx. */
CCT_API cct_status cct_conv_bwd_data(const cct_conv_desc* desc, cct_lowering lowering, const float* dy,
                             const float* w, float* dx, void* ws, size_t ws_bytes, void* stream);

/* Backward-weight (north_star; absent from the reference): dw = d(sum(y*dy))/dw.
 * Deterministic (fixed split-K reduction order). */
CCT_API cct_status cct_conv_bwd_weight(const cct_conv_desc* desc, cct_lowering lowering, const float* x,
                               const float* dy, float* dw, void* ws, size_t ws_bytes,
                               void* stream);

/* Workspace limit (bytes; default 16 GiB).  A pass whose
 * scratch would exceed it runs over batch chunks that reuse one scratch region
 * (the SPEC batching module's partitions), e.g. Type 3 on
 * conv1, whose Rhat is 2.4 GB per image.  cct_workspace_size() reports the
 * chunked size. */
CCT_API void cct_set_workspace_limit(size_t bytes);
CCT_API size_t cct_get_workspace_limit(void);

/* Implicit Type 1 lowering (the paper's "fusion").
 * mode 1 (default): for Type 1 layers with d % 16 == 0 the
 *   forward and backward-weight GEMMs read their lowered operand straight from
 *   x through TMA im2col tiles -- Dhat never exists in HBM (the forward is
 *   bit-identical to the materialised path).  At stride 1 with o % 16 == 0,
 *   backward-data runs as the forward convolution of dy (transposed to NHWC)
 *   with the rotated kernel bank, written straight to dx (no dDhat, no col2im;
 *   swapped, pixels as the wide tile side, when d < 128), whenever the cost
 *   model predicts that faster.  A strided layer with s^2 d % 16 == 0 may run
 *   as the stride-1 convolution of its space-to-depth blocked input (cost
 *   model, per pass); the lowered cache then holds the blocked input.
 * mode 2: every implicit form whenever possible (tests).
 * mode 0: everything materialised. */
CCT_API void cct_set_implicit_lowering(int mode);
CCT_API int cct_get_implicit_lowering(void);

/* Tuning switches.  Process-wide and explicit: the library reads no environment
 * variables, so results and kernel choices depend only on calls made through
 * this ABI.  Each key selects between measured variants of the same computation
 * (every value stays within the parity tolerance; the defaults are the forms
 * measured fastest on B200).  cct_set_tuning returns
 * CCT_ERR_CONFIG for an unknown key or an out-of-range value. */
typedef enum {
    CCT_TUNE_SPLIT_PRODUCER = 0, /* 1: A and B TMA tiles issued by two producer threads (default 0:    */
                                 /* with warp-uniform issue one producer warp is 0.4 % faster, measured) */
    CCT_TUNE_A_TMEM = 1,         /* N <= 96 tiles: 0 A from smem, 1 A in TMEM (default), 2 deeper A ring, */
                                 /* 3 A in TMEM + merged N = 2 BN product (single CTAs, K-major B)       */
    CCT_TUNE_A_TMEM_WIDE = 2,    /* 1 (default): 192/256/384-wide CTA-pair tiles keep A in TMEM          */
    CCT_TUNE_CTA_PAIRS = 3,      /* 0 auto (default), 1 single CTAs only, 2 CTA pairs whenever legal     */
    CCT_TUNE_BN384 = 4,          /* 1: one 256 + 128 composite tile for N = 384 (default 0: two 192-wide */
                                 /* tiles, which also take the two-chain form; 0.8 % faster on the step)  */
    CCT_TUNE_STREAMK = 5,        /* 1 (default): stream-K for GEMMs whose last wave would idle           */
    CCT_TUNE_CHAIN2 = 6,         /* 1 (default): two TMEM accumulation chains instead of 2-way split-K   */
    CCT_TUNE_S2D = 7,            /* strided Type 1: 0 never space-to-depth, 1 cost model (default), 2 always */
    CCT_TUNE_IMPLICIT_BWD = 8,   /* implicit Type 1 backward-data: 0 never, 1 cost model (default), 2 always */
    CCT_TUNE_WGRAD_SWAP = 9,     /* 1 (default): swapped implicit backward-weight for o < 128            */
    CCT_TUNE_DGRAD_SWAP = 10,    /* swapped implicit backward-data: 0 never (default), 1 d < 128, 2 d <= 128 */
    CCT_TUNE_FWD_SWAP = 11,      /* 1: swapped forward for o < 128 (default 0: measured slower)          */
    CCT_TUNE_TRACE_PHASES = 12,  /* 1: one stderr line per kernel launch (diagnostics)                   */
    CCT_TUNE_GATHER = 13,        /* 1 (default): fused small-channel Type 1 (d s % 4 == 0, e.g. conv1):  */
                                 /* Dhat gathered from staged input rows inside the GEMM, never in HBM;  */
                                 /* 2: same, forward without the merged N = 2 NP product (A/B)           */
                                 /* 3: same, forward tiles of whole output rows, 3 row buffers (A/B:     */
                                 /*    bitwise equal, 10 % slower on conv1: 16 % more 128-row tiles)     */
    CCT_TUNE_FUSED_T23 = 14,     /* 1: Types 2 / 3 run fused when the layer has the implicit (TMA        */
                                 /* im2col) form: one im2col box per filter tap, the per-tap products    */
                                 /* accumulated in TMEM (tap-shifted accumulation), so Rhat is never     */
                                 /* materialised -- the implicit Type 1 kernel.  0 (default): the        */
                                 /* materialised paper forms, kept as the measured baselines             */
    CCT_TUNE_OVERLAP = 15,       /* 1 (default): inside one cct_conv_bwd call, the backward-weight of a  */
                                 /* fused small-channel layer runs on a library-owned high-priority     */
                                 /* side stream beside the backward-data's vertical fold (event fork /  */
                                 /* join; the call's stream still orders everything).  0: one stream    */
    CCT_TUNE_COUNT = 16
} cct_tuning;
CCT_API cct_status cct_set_tuning(cct_tuning key, int value);
CCT_API int cct_get_tuning(cct_tuning key); /* -1 for an unknown key */
CCT_API void cct_reset_tuning(void);        /* every key back to its default */

/* Training-step entry points (the lowered-matrix cache).
 * cct_conv_fwd_cached leaves the data-side matrix Dhat of the forward pass in a
 * caller buffer of cct_lowered_cache_size() bytes (0 when Dhat is the input
 * itself: Type 3, no padding); cct_conv_bwd then runs bwd-data (dx != NULL)
 * and bwd-weight (dw != NULL) in one call, expanding dy once and reading Dhat
 * from the cache instead of lowering x again.  x may be NULL when a cache is
 * given.  AUTO resolves with the fwd+bwd score so both calls pick the same
 * type.  Workspace: cct_workspace_size(..., CCT_PASS_FWD / CCT_PASS_BWD). */
CCT_API cct_status cct_lowered_cache_size(const cct_conv_desc* desc, cct_lowering lowering, size_t* bytes);
CCT_API cct_status cct_conv_fwd_cached(const cct_conv_desc* desc, cct_lowering lowering, const float* x,
                                       const float* w, float* y, float* cache, size_t cache_bytes, void* ws,
                                       size_t ws_bytes, void* stream);
CCT_API cct_status cct_conv_bwd(const cct_conv_desc* desc, cct_lowering lowering, const float* x,
                                const float* cache, const float* dy, const float* w, float* dx, float* dw,
                                void* ws, size_t ws_bytes, void* stream);

/* Layer extension (the reference SPEC puts groups out of
 * scope): grouped convolution as in bvlc_reference_caffenet
 * (group = 2 on conv2/4/5) and the bias + ReLU epilogue
 * around the layer.  desc->d and desc->o are the TOTAL channel counts; w is
 * (o, k, k, d / groups), output channel j reads input-channel group
 * j / (o / groups); y = relu ? max(conv + bias, 0) : conv + bias (bias may be
 * NULL).  The lowering type (AUTO: the cost model's choice for one group) is
 * applied per group.  Implicit Type 1 groups run straight on x / y (TMA im2col
 * over a channel view, strided epilogue with the bias / ReLU fused); other forms
 * gather each group into scratch.  NULL ext = { 1, NULL, 0 }. */
typedef struct {
    int64_t groups;
    const float* bias; /* (o) device pointer or NULL */
    int relu;          /* 0 or 1 */
} cct_conv_ext;

CCT_API cct_status cct_workspace_size_ex(const cct_conv_desc* desc, cct_lowering lowering, const cct_conv_ext* ext,
                                         cct_pass pass, size_t* bytes);
CCT_API cct_status cct_conv_fwd_ex(const cct_conv_desc* desc, cct_lowering lowering, const cct_conv_ext* ext,
                                   const float* x, const float* w, float* y, void* ws, size_t ws_bytes, void* stream);
/* dy: gradient of the layer output y (post-activation; y is needed when relu).
 * Any of dx, dw, db (bias gradient, (o)) may be NULL.  Deterministic. */
CCT_API cct_status cct_conv_bwd_ex(const cct_conv_desc* desc, cct_lowering lowering, const cct_conv_ext* ext,
                                   const float* x, const float* y, const float* dy, const float* w, float* dx,
                                   float* dw, float* db, void* ws, size_t ws_bytes, void* stream);

/* Phase-level API for PhaseTimings and the bit-exact lowering parity.
 * lower: dhat gets the data-side matrix with row stride ld
 * (floats, >= cols).  Shapes: cct_lowered_shape().  The kernel side never
 * needs lowering: KernelBank storage already is Khat^T for every type
 * (SURVEY 0.6); cct_lower_khat materialises the SPEC's Khat for parity. */
CCT_API cct_status cct_lowered_shape(const cct_conv_desc* desc, cct_lowering lowering,
                             cct_row_order order, int64_t* dhat_rows, int64_t* dhat_cols,
                             int64_t* khat_cols);
CCT_API cct_status cct_lower(const cct_conv_desc* desc, cct_lowering lowering, cct_row_order order,
                     const float* x, float* dhat, int64_t ld, void* stream);
CCT_API cct_status cct_lower_khat(const cct_conv_desc* desc, cct_lowering lowering, const float* w,
                          float* khat, void* stream);
/* lift: rhat row-major (rows x khat_cols, row stride ld) -> y NCHW. */
CCT_API cct_status cct_lift(const cct_conv_desc* desc, cct_lowering lowering, cct_row_order order,
                    const float* rhat, int64_t ld, float* y, void* stream);

/* multiply (gemm.cpp:93-122) replacement: C(MxN) = A(MxK) * B(KxN), all
 * row-major fp32 device matrices with leading dimensions lda/ldb/ldc in
 * floats.  lda and ldb must be multiples of 4 and A, B 16-byte aligned (TMA);
 * the C++ wrapper pads on upload.  split_k <= 0 chooses automatically; ws may
 * be NULL when split_k == 1 (see cct_gemm_workspace_size). */
CCT_API cct_status cct_gemm(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                    const float* B, int64_t ldb, float* C, int64_t ldc, int split_k, void* ws,
                    size_t ws_bytes, void* stream);
CCT_API cct_status cct_gemm_workspace_size(int64_t M, int64_t N, int64_t K, int split_k, size_t* bytes);

/* Diagnostic single-product tensor-core GEMM (passes = 1: big*big only,
 * i.e. plain TF32) used to characterise how the tensor core consumes fp32
 * operands; not used by the convolution path. */
CCT_API cct_status cct_gemm_passes(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                           const float* B, int64_t ldb, float* C, int64_t ldc, int passes,
                           void* stream);

/* The reference's ORACLE entry points on the device (not the hot path):
 * direct_convolve (tensor.cpp:77-106) and multiply_reference (gemm.cpp:124-141)
 * with their exact arithmetic -- fp64 accumulator in the reference loop order,
 * explicitly rounded multiply and add -- so results are bit-identical to the
 * reference.  The conv variant accepts stride / pad like the oracle. */
CCT_API cct_status cct_direct_conv_fwd_exact(const cct_conv_desc* desc, const float* x, const float* w, float* y,
                                             void* stream);
CCT_API cct_status cct_gemm_exact(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B,
                                  int64_t ldb, float* C, int64_t ldc, void* stream);

/* Diagnostic: one raw kernel launch with explicit operand storage.
 * a_major/b_major: 0 = K-major (rows = M|N, cols = K), 1 = MN-major (rows = K).
 * C(m, n) at C + m*ldc_m + n*ldc_n.  bn = 0 chooses the tile width. */
CCT_API cct_status cct_debug_gemm(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                                  int a_major, const float* B, int64_t ldb, int b_major, float* C,
                                  int64_t ldc_m, int64_t ldc_n, int passes, int bn, void* stream);

/* ---- cost model / automatic lowering optimizer ---------- */

/* CostEstimate with exact counts plus the
 * B200 model time. */
typedef struct {
    uint64_t lower_elements_written;
    uint64_t gemm_flops;       /* executed (lowered-shape) flops              */
    uint64_t lift_adds;
    uint64_t lowered_bytes;    /* bytes of Dhat                               */
    uint64_t hbm_bytes;        /* modelled HBM traffic of lower+gemm+lift     */
    double total_score;        /* alpha*(lower + lift) + beta*flops (SPEC)    */
    double model_seconds;      /* calibrated B200 time estimate (this build)  */
} cct_cost_estimate;

/* Calibration: alpha/beta of the SPEC score and the measured
 * B200 rates the model time uses.  cct_calibration_default() fills the values
 * measured on this build's B200 box. */
typedef struct {
    double alpha;            /* seconds per element moved (1 / copy rate)      */
    double beta;             /* seconds per flop (1 / GEMM rate)               */
    double hbm_bytes_per_s;  /* sustained lowering/lift kernel bandwidth       */
    double gemm_flops_per_s; /* sustained 3xTF32 algorithmic GEMM rate         */
    double launch_s;         /* per-kernel fixed cost                          */
} cct_calibration;

CCT_API void cct_calibration_default(cct_calibration* cal);

/* select_strategy: argmin of the model over T1/T2/T3 for
 * `pass` (CCT_PASS_FWD scores fwd only; passing 3 scores fwd+bwd).  Ties break
 * T1 < T2 < T3.  est may be NULL or point at 3 entries. */
CCT_API cct_status cct_select_lowering(const cct_conv_desc* desc, const cct_calibration* cal, int pass,
                               cct_lowering* out, cct_cost_estimate* est);
CCT_API cct_status cct_estimate(const cct_conv_desc* desc, cct_lowering lowering, const cct_calibration* cal,
                        int pass, cct_cost_estimate* est);

/* ---- phase timings (PhaseTimings) ------------------------
 * When enabled, each kernel launch is bracketed by CUDA events on its stream.
 * cct_profile_read synchronises and returns, per phase, the accumulated device
 * milliseconds, algorithmic flops (GEMM), algorithmic bytes (HBM kernels) and
 * launch counts.  Phases: 0 lower, 1 gemm, 2 lift, 3 expand, 4 col2im,
 * 5 split-K reduce, 6 other.  Arrays must hold CCT_NUM_PHASES entries. */
#define CCT_NUM_PHASES 7
CCT_API void cct_profile_enable(int on);
CCT_API void cct_profile_read(double* ms, double* flops, double* bytes, uint64_t* launches, int reset);

/* ---- misc ------------------------------------------------------------- */
CCT_API const char* cct_last_error(void);
CCT_API int cct_abi_version(void);
/* name of the current CUDA device and its SM count (0 and "none" without a
 * device): the machine descriptor of convbench records */
CCT_API int cct_device_info(char* name, size_t len, int* sms);
/* number of CUDA kernels this library launched on the calling host thread
 * since the last reset (the bench's gpu_launches evidence) */
CCT_API uint64_t cct_launch_count(void);
CCT_API void cct_reset_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* CCT_H */
