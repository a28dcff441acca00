/*
 * cct_oracle.h -- CPU restatement of the Caffe con Troll convolution hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the B200
 * path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it.  The product library (libcct.so) never
 * links, loads or calls anything under oracle/.
 *
 * Every function cites the reference file:line (under /root/reference) whose
 * behaviour it restates.  Parity is pinned in tests/ against (a) the SPEC
 * known-answer examples and (b) golden vectors produced by the reference's own
 * tensor.cpp / gemm.cpp compiled from /root/reference (oracle/_ref, see
 * oracle/Makefile and tests/golden/make_golden.py).
 *
 * Layouts (identical to the reference containers):
 *   x  : DataBatch as b contiguous Tensor3, HWC depth-minor  (tensor.hpp:28-35)
 *   w  : KernelBank (o,k,k,d) depth-minor                      (tensor.hpp:70-75)
 *   y  : OutputBatch NCHW ((q*o+j)*m+r)*m+c                    (tensor.hpp:135-150)
 *   dy : same layout as y;  dx : same as x;  dw : same as w.
 * Matrices are row-major like convlow::Mat (gemm.hpp:11-37).
 */
#ifndef CCT_ORACLE_H
#define CCT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- RNG: std::mt19937_64 + std::uniform_real_distribution<float>(-1, 1),
 *      exactly as Tensor3::random / KernelBank::random (tensor.cpp:32-45). */
typedef struct {
    uint64_t mt[312];
    int idx;
} orc_rng;

void orc_rng_seed(orc_rng* g, uint64_t seed);
uint64_t orc_rng_next(orc_rng* g);
void orc_rng_uniform(orc_rng* g, float* out, size_t count);
/* fresh generator seeded with `seed`, `skip` draws discarded, then `count` values */
void orc_uniform_fill(uint64_t seed, uint64_t skip, float* out, size_t count);

/* ---- Eq. 1 direct convolution oracle (tensor.cpp:77-118).  Returns 0 or -1. */
int orc_direct_convolve_batch(const float* x, long b, long n, long d,
                              const float* w, long k, long o, float* y);

/* Generalised to stride s / zero padding p (builder
 * extension).  Bit-identical to running direct_convolve on the zero-padded
 * input and subsampling, and to the dgrad / wgrad adapters of SURVEY 8(c)
 * (same double accumulator, same loop order). m = (n + 2p - k)/s + 1. */
int orc_conv_fwd(const float* x, const float* w, float* y,
                 long b, long n, long d, long k, long o, long s, long p);
int orc_conv_bwd_data(const float* dy, const float* w, float* dx,
                      long b, long n, long d, long k, long o, long s, long p);
int orc_conv_bwd_weight(const float* x, const float* dy, float* dw,
                        long b, long n, long d, long k, long o, long s, long p);

/* ---- GEMM: multiply_reference (gemm.cpp:124-141): double accumulator in
 * ascending k, one rounding to float per element.  C = A(MxK) * B(KxN). */
void orc_multiply(const float* A, const float* B, float* C, long M, long K, long N);

/* Generic row-major GEMM with transposes; same double/ascending-k rule.
 * C(MxN) = op(A) op(B); op(A) is MxK, op(B) is KxN. */
void orc_gemm(int transA, int transB, long M, long N, long K,
              const float* A, long lda, const float* B, long ldb,
              float* C, long ldc);

/* A pluggable GEMM (same signature as orc_gemm) used by the lowered paths,
 * so the reference's own multiply (gemm.cpp:93) can be substituted. */
typedef void (*orc_gemm_fn)(void* ctx, int transA, int transB, long M, long N, long K,
                            const float* A, long lda, const float* B, long ldb,
                            float* C, long ldc);

/* ---- SPEC lowering / lifting, stride 1, no padding.
 * type in {1,2,3}.  Shapes:
 *   T1: Dhat (b*m^2) x (k^2 d),  Khat (k^2 d) x o
 *   T2: Dhat (b*n^2) x (k d),    Khat (k d) x (k o)
 *   T3: Dhat (b*n^2) x d,        Khat d x (k^2 o)
 * Row order inside an image block is the SPEC's column-major c*m+r / c*n+r. */
int orc_lowered_shape(int type, long b, long n, long d, long k, long o,
                      long* dhat_rows, long* dhat_cols, long* khat_cols);
int orc_lower(int type, const float* x, const float* w, long b, long n, long d,
              long k, long o, float* dhat, float* khat);
int orc_lift(int type, const float* rhat, long b, long n, long d, long k, long o,
             float* y);
/* lift(multiply(lower(...))) -- convolve_lowered. */
int orc_convolve_lowered(int type, const float* x, const float* w, long b, long n,
                         long d, long k, long o, float* y);
/* exact per-phase counts (cost model) */
void orc_estimate(int type, long b, long n, long d, long k, long o,
                  uint64_t* lower_elements, uint64_t* gemm_flops, uint64_t* lift_adds);

/* ---- Appendix A generalised lowered paths (stride/pad, fwd/dgrad/wgrad),
 * internal row-major pixel order.  These are the CPU restatement of the
 * whole lowered hot path; with gemm=NULL they use orc_gemm.  ws may be NULL
 * (allocated internally).  Used as the timed CPU baseline with the
 * reference's multiply plugged in (oracle/ref_shim.cpp). */
int orc_lowered_fwd(int type, const float* x, const float* w, float* y,
                    long b, long n, long d, long k, long o, long s, long p,
                    orc_gemm_fn gemm, void* ctx);
int orc_lowered_bwd_data(int type, const float* dy, const float* w, float* dx,
                         long b, long n, long d, long k, long o, long s, long p,
                         orc_gemm_fn gemm, void* ctx);
int orc_lowered_bwd_weight(int type, const float* x, const float* dy, float* dw,
                           long b, long n, long d, long k, long o, long s, long p,
                           orc_gemm_fn gemm, void* ctx);

/* Appendix A internal lowering (row-major pixel order, padded input Xp):
 *   T1 rows (q,r,c) x cols (i,j,ch)   : b*m^2 x k^2 d
 *   T2 rows (q,y,c) x cols (j,ch)     : b*R*m x k d     (y in [0,R))
 *   T3 rows (q,y,x) x cols ch         : b*R*R x d
 * with R = s(m-1)+k.  ld = row stride of the output (>= cols). */
int orc_lower_internal(int type, const float* x, long b, long n, long d, long k,
                       long s, long p, float* dhat, long ld);

#ifdef __cplusplus
}
#endif
#endif
