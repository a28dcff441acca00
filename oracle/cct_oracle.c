/*
 * cct_oracle.c -- CPU restatement of the CcT convolution hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see cct_oracle.h).  Compiled with the
 * reference's own flags (-O3 -ffp-contract=off, proj/CMakeLists.txt:15-17)
 * so every double accumulation rounds exactly like the reference.
 */
#include "cct_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* RNG: restates std::mt19937_64 (libstdc++) and                            */
/* std::uniform_real_distribution<float>(-1,1) as used by Tensor3::random /  */
/* KernelBank::random / Mat::random (tensor.cpp:32-45, gemm.cpp:82-87).      */
/* ------------------------------------------------------------------------ */
#define MT_N 312
#define MT_M 156

void orc_rng_seed(orc_rng* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = MT_N;
}

static void mt_regen(orc_rng* g) {
    const uint64_t upper = ~0ULL << 31, lower = ~upper, a = 0xB5026F5AA96619E9ULL;
    int k;
    for (k = 0; k < MT_N - MT_M; ++k) {
        uint64_t y = (g->mt[k] & upper) | (g->mt[k + 1] & lower);
        g->mt[k] = g->mt[k + MT_M] ^ (y >> 1) ^ ((y & 1ULL) ? a : 0ULL);
    }
    for (; k < MT_N - 1; ++k) {
        uint64_t y = (g->mt[k] & upper) | (g->mt[k + 1] & lower);
        g->mt[k] = g->mt[k + (MT_M - MT_N)] ^ (y >> 1) ^ ((y & 1ULL) ? a : 0ULL);
    }
    uint64_t y = (g->mt[MT_N - 1] & upper) | (g->mt[0] & lower);
    g->mt[MT_N - 1] = g->mt[MT_M - 1] ^ (y >> 1) ^ ((y & 1ULL) ? a : 0ULL);
    g->idx = 0;
}

uint64_t orc_rng_next(orc_rng* g) {
    if (g->idx >= MT_N) mt_regen(g);
    uint64_t z = g->mt[g->idx++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= (z >> 43);
    return z;
}

/* generate_canonical<float, 24>(mt19937_64) then a + (b - a) * u. */
static float canonical_to_uniform(uint64_t z) {
    volatile float sum = (float)z;                 /* round-to-nearest u64 -> float */
    volatile float tmp = 18446744073709551616.0f;  /* float(2^64) */
    float ret = sum / tmp;
    if (ret >= 1.0f) ret = nextafterf(1.0f, 0.0f);
    volatile float scaled = ret * 2.0f;            /* (b - a) = 2, no contraction */
    return scaled + -1.0f;
}

void orc_rng_uniform(orc_rng* g, float* out, size_t count) {
    for (size_t i = 0; i < count; ++i) out[i] = canonical_to_uniform(orc_rng_next(g));
}

void orc_uniform_fill(uint64_t seed, uint64_t skip, float* out, size_t count) {
    orc_rng g;
    orc_rng_seed(&g, seed);
    for (uint64_t i = 0; i < skip; ++i) (void)orc_rng_next(&g);
    orc_rng_uniform(&g, out, count);
}

/* ------------------------------------------------------------------------ */
/* Direct convolution (Eq. 1)                                               */
/* ------------------------------------------------------------------------ */

/* Restates direct_convolve (tensor.cpp:77-106) over a batch
 * (direct_convolve_batch, tensor.cpp:108-118): for every (q, j, r, c) the
 * double accumulator runs i -> c' -> r' (tensor.cpp:94-101). */
int orc_direct_convolve_batch(const float* x, long b, long n, long d,
                              const float* w, long k, long o, float* y) {
    if (k < 1 || k > n || d < 1 || o < 1 || b < 1) return -1; /* LayerConfig::validate */
    return orc_conv_fwd(x, w, y, b, n, d, k, o, 1, 0);
}

static inline long out_side(long n, long k, long s, long p) { return (n + 2 * p - k) / s + 1; }

/* Forward with stride/pad: identical arithmetic to direct_convolve applied to
 * the zero-padded input and sampled at (s r, s c).  Padding taps contribute
 * +-0.0 products, which leave the accumulator unchanged, so they are skipped. */
int orc_conv_fwd(const float* x, const float* w, float* y,
                 long b, long n, long d, long k, long o, long s, long p) {
    if (k < 1 || d < 1 || o < 1 || b < 1 || s < 1 || p < 0 || k > n + 2 * p) return -1;
    const long m = out_side(n, k, s, p);
    for (long q = 0; q < b; ++q) {
        const float* xq = x + (size_t)q * n * n * d;
        for (long j = 0; j < o; ++j) {
            const float* wj = w + (size_t)j * k * k * d;
            float* yp = y + ((size_t)q * o + j) * m * m;
            for (long r = 0; r < m; ++r)
                for (long c = 0; c < m; ++c) {
                    double acc = 0.0;
                    for (long i = 0; i < d; ++i)
                        for (long cp = 0; cp < k; ++cp) {
                            const long xc = s * c + cp - p;
                            if (xc < 0 || xc >= n) continue;
                            for (long rp = 0; rp < k; ++rp) {
                                const long xr = s * r + rp - p;
                                if (xr < 0 || xr >= n) continue;
                                acc += (double)xq[((size_t)xr * n + xc) * d + i] *
                                       (double)wj[((size_t)rp * k + cp) * d + i];
                            }
                        }
                    yp[r * m + c] = (float)acc;
                }
        }
    }
    return 0;
}

/* Backward-data.  Restates the SURVEY 8(c) adapter over direct_convolve
 * (tensor.cpp:77-106): canvas = dY dilated by s at offset k-1, kernel
 * Kr[i',j',oj] = W[oj, k-1-i', k-1-j', ch]; direct_convolve's loop order
 * (depth oj -> column j' -> row i') is kept, so the result is bit-identical. */
int orc_conv_bwd_data(const float* dy, const float* w, float* dx,
                      long b, long n, long d, long k, long o, long s, long p) {
    if (k < 1 || d < 1 || o < 1 || b < 1 || s < 1 || p < 0 || k > n + 2 * p) return -1;
    const long m = out_side(n, k, s, p);
    for (long q = 0; q < b; ++q)
        for (long yy = 0; yy < n; ++yy)
            for (long xx = 0; xx < n; ++xx)
                for (long ch = 0; ch < d; ++ch) {
                    const long yp = yy + p, xp = xx + p; /* padded coordinates */
                    double acc = 0.0;
                    for (long oj = 0; oj < o; ++oj) {
                        const float* dyp = dy + ((size_t)q * o + oj) * m * m;
                        for (long jj = 0; jj < k; ++jj) {          /* j' */
                            const long j = k - 1 - jj;
                            const long tx = xp - j;
                            if (tx < 0 || tx % s) continue;
                            const long c = tx / s;
                            if (c >= m) continue;
                            for (long ii = 0; ii < k; ++ii) {      /* i' */
                                const long i = k - 1 - ii;
                                const long ty = yp - i;
                                if (ty < 0 || ty % s) continue;
                                const long r = ty / s;
                                if (r >= m) continue;
                                acc += (double)dyp[r * m + c] *
                                       (double)w[(((size_t)oj * k + i) * k + j) * d + ch];
                            }
                        }
                    }
                    dx[(((size_t)q * n + yy) * n + xx) * d + ch] = (float)acc;
                }
    return 0;
}

/* Backward-weight.  Restates the SURVEY 8(c) adapter: for each ch, data
 * D'[y,x,q] = Xp[q,y,x,ch]; kernel K' = dY[:,oj] dilated by s; output
 * (i,j) of direct_convolve(D', K') accumulates depth q -> column c -> row r. */
int orc_conv_bwd_weight(const float* x, const float* dy, float* dw,
                        long b, long n, long d, long k, long o, long s, long p) {
    if (k < 1 || d < 1 || o < 1 || b < 1 || s < 1 || p < 0 || k > n + 2 * p) return -1;
    const long m = out_side(n, k, s, p);
    for (long oj = 0; oj < o; ++oj)
        for (long i = 0; i < k; ++i)
            for (long j = 0; j < k; ++j)
                for (long ch = 0; ch < d; ++ch) {
                    double acc = 0.0;
                    for (long q = 0; q < b; ++q) {
                        const float* xq = x + (size_t)q * n * n * d;
                        const float* dyp = dy + ((size_t)q * o + oj) * m * m;
                        for (long c = 0; c < m; ++c) {
                            const long xc = j + s * c - p;
                            if (xc < 0 || xc >= n) continue;
                            for (long r = 0; r < m; ++r) {
                                const long xr = i + s * r - p;
                                if (xr < 0 || xr >= n) continue;
                                acc += (double)xq[((size_t)xr * n + xc) * d + ch] *
                                       (double)dyp[r * m + c];
                            }
                        }
                    }
                    dw[(((size_t)oj * k + i) * k + j) * d + ch] = (float)acc;
                }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* GEMM                                                                     */
/* ------------------------------------------------------------------------ */

/* multiply_reference (gemm.cpp:124-141). */
void orc_multiply(const float* A, const float* B, float* C, long M, long K, long N) {
    orc_gemm(0, 0, M, N, K, A, K, B, N, C, N);
}

void orc_gemm(int transA, int transB, long M, long N, long K,
              const float* A, long lda, const float* B, long ldb,
              float* C, long ldc) {
    for (long i = 0; i < M; ++i)
        for (long j = 0; j < N; ++j) {
            double acc = 0.0;
            for (long t = 0; t < K; ++t) {
                const float a = transA ? A[(size_t)t * lda + i] : A[(size_t)i * lda + t];
                const float bb = transB ? B[(size_t)j * ldb + t] : B[(size_t)t * ldb + j];
                acc += (double)a * (double)bb;
            }
            C[(size_t)i * ldc + j] = (float)acc;
        }
}

static void default_gemm(void* ctx, int ta, int tb, long M, long N, long K,
                         const float* A, long lda, const float* B, long ldb,
                         float* C, long ldc) {
    (void)ctx;
    orc_gemm(ta, tb, M, N, K, A, lda, B, ldb, C, ldc);
}

/* ------------------------------------------------------------------------ */
/* SPEC lowering / lifting (stride 1, no padding)                           */
/* ------------------------------------------------------------------------ */

int orc_lowered_shape(int type, long b, long n, long d, long k, long o,
                      long* rows, long* cols, long* kcols) {
    if (k < 1 || k > n || d < 1 || o < 1 || b < 1) return -1;
    const long m = n - k + 1;
    switch (type) { /* LoweredMatrices invariants */
    case 1: *rows = b * m * m; *cols = k * k * d; *kcols = o; return 0;
    case 2: *rows = b * n * n; *cols = k * d; *kcols = k * o; return 0;
    case 3: *rows = b * n * n; *cols = d; *kcols = k * k * o; return 0;
    default: return -1;
    }
}

/* lower.  Image q occupies a contiguous
 * row block; vec ordering is depth-minor;
 * Type 2 rows whose window leaves the image are zero-filled. */
int orc_lower(int type, const float* x, const float* w, long b, long n, long d,
              long k, long o, float* dhat, float* khat) {
    long rows, cols, kcols;
    if (orc_lowered_shape(type, b, n, d, k, o, &rows, &cols, &kcols)) return -1;
    const long m = n - k + 1;
    memset(dhat, 0, sizeof(float) * (size_t)rows * cols);
    for (long q = 0; q < b; ++q) {
        const float* xq = x + (size_t)q * n * n * d;
        if (type == 1) {
            for (long c = 0; c < m; ++c)
                for (long r = 0; r < m; ++r) {
                    float* row = dhat + ((size_t)q * m * m + c * m + r) * cols;
                    for (long rp = 0; rp < k; ++rp)
                        for (long cp = 0; cp < k; ++cp)
                            for (long i = 0; i < d; ++i)
                                row[(rp * k + cp) * d + i] = xq[((r + rp) * n + c + cp) * d + i];
                }
        } else if (type == 2) {
            for (long c = 0; c + k - 1 <= n - 1; ++c)
                for (long r = 0; r < n; ++r) {
                    float* row = dhat + ((size_t)q * n * n + c * n + r) * cols;
                    for (long cp = 0; cp < k; ++cp)
                        for (long i = 0; i < d; ++i)
                            row[cp * d + i] = xq[(r * n + c + cp) * d + i];
                }
        } else {
            for (long c = 0; c < n; ++c)
                for (long r = 0; r < n; ++r) {
                    float* row = dhat + ((size_t)q * n * n + c * n + r) * cols;
                    for (long i = 0; i < d; ++i) row[i] = xq[(r * n + c) * d + i];
                }
        }
    }
    /* Khat: kernels are column blocks in kernel order. */
    for (long j = 0; j < o; ++j)
        for (long rp = 0; rp < k; ++rp)
            for (long cp = 0; cp < k; ++cp)
                for (long i = 0; i < d; ++i) {
                    const float v = w[((j * k + rp) * k + cp) * d + i];
                    if (type == 1) khat[((rp * k + cp) * d + i) * kcols + j] = v;
                    else if (type == 2) khat[(cp * d + i) * kcols + j * k + rp] = v;
                    else khat[i * kcols + j * k * k + rp * k + cp] = v;
                }
    (void)m;
    return 0;
}

/* lift: Type 1 reshape, Type 2 sums k
 * entries, Type 3 sums k^2 entries (double accumulator, ascending taps). */
int orc_lift(int type, const float* rhat, long b, long n, long d, long k, long o,
             float* y) {
    long rows, cols, kcols;
    if (orc_lowered_shape(type, b, n, d, k, o, &rows, &cols, &kcols)) return -1;
    const long m = n - k + 1;
    for (long q = 0; q < b; ++q)
        for (long j = 0; j < o; ++j)
            for (long r = 0; r < m; ++r)
                for (long c = 0; c < m; ++c) {
                    float v;
                    if (type == 1) {
                        v = rhat[((size_t)q * m * m + c * m + r) * kcols + j];
                    } else if (type == 2) {
                        double acc = 0.0;
                        for (long t = 0; t < k; ++t)
                            acc += (double)rhat[((size_t)q * n * n + c * n + r + t) * kcols + j * k + t];
                        v = (float)acc;
                    } else {
                        double acc = 0.0;
                        for (long ti = 0; ti < k; ++ti)
                            for (long tj = 0; tj < k; ++tj)
                                acc += (double)rhat[((size_t)q * n * n + (c + tj) * n + r + ti) * kcols +
                                                    j * k * k + ti * k + tj];
                        v = (float)acc;
                    }
                    y[(((size_t)q * o + j) * m + r) * m + c] = v;
                }
    return 0;
}

int orc_convolve_lowered(int type, const float* x, const float* w, long b, long n,
                         long d, long k, long o, float* y) {
    long rows, cols, kcols;
    if (orc_lowered_shape(type, b, n, d, k, o, &rows, &cols, &kcols)) return -1;
    float* dhat = (float*)malloc(sizeof(float) * (size_t)rows * cols);
    float* khat = (float*)malloc(sizeof(float) * (size_t)cols * kcols);
    float* rhat = (float*)malloc(sizeof(float) * (size_t)rows * kcols);
    int rc = -1;
    if (dhat && khat && rhat) {
        orc_lower(type, x, w, b, n, d, k, o, dhat, khat);
        orc_multiply(dhat, khat, rhat, rows, cols, kcols);
        rc = orc_lift(type, rhat, b, n, d, k, o, y);
    }
    free(dhat); free(khat); free(rhat);
    return rc;
}

/* estimate: exact counts. */
void orc_estimate(int type, long b, long n, long d, long k, long o,
                  uint64_t* lower_elements, uint64_t* gemm_flops, uint64_t* lift_adds) {
    const uint64_t m = (uint64_t)(n - k + 1), B = (uint64_t)b, N = (uint64_t)n,
                   D = (uint64_t)d, K = (uint64_t)k, O = (uint64_t)o;
    long rows = 0, cols = 0, kcols = 0;
    orc_lowered_shape(type, b, n, d, k, o, &rows, &cols, &kcols);
    *gemm_flops = 2ULL * (uint64_t)rows * (uint64_t)cols * (uint64_t)kcols;
    if (type == 1) { *lower_elements = B * m * m * K * K * D; *lift_adds = 0; }
    else if (type == 2) { *lower_elements = B * N * N * K * D; *lift_adds = B * m * m * (K - 1) * O; }
    else { *lower_elements = B * N * N * D; *lift_adds = B * m * m * (K * K - 1) * O; }
}

/* ------------------------------------------------------------------------ */
/* Appendix A: generalised lowered paths (stride s, pad p, fwd/dgrad/wgrad)  */
/* ------------------------------------------------------------------------ */

typedef struct {
    long b, n, d, k, o, s, p, m, R, N;
} geo;

static int make_geo(geo* g, long b, long n, long d, long k, long o, long s, long p) {
    if (k < 1 || d < 1 || o < 1 || b < 1 || s < 1 || p < 0 || k > n + 2 * p) return -1;
    g->b = b; g->n = n; g->d = d; g->k = k; g->o = o; g->s = s; g->p = p;
    g->N = n + 2 * p;
    g->m = (g->N - k) / s + 1;
    g->R = s * (g->m - 1) + k;
    return 0;
}

static inline float xp_at(const geo* g, const float* x, long q, long y, long xx, long ch) {
    const long yy = y - g->p, xc = xx - g->p;
    if (yy < 0 || yy >= g->n || xc < 0 || xc >= g->n) return 0.0f;
    return x[(((size_t)q * g->n + yy) * g->n + xc) * g->d + ch];
}

static void lowered_dims(int type, const geo* g, long* rows, long* cols, long* nco) {
    if (type == 1) { *rows = g->b * g->m * g->m; *cols = g->k * g->k * g->d; *nco = g->o; }
    else if (type == 2) { *rows = g->b * g->R * g->m; *cols = g->k * g->d; *nco = g->k * g->o; }
    else { *rows = g->b * g->R * g->R; *cols = g->d; *nco = g->k * g->k * g->o; }
}

static void lower_internal_geo(int type, const geo* g, const float* x, float* dh, long ld) {
    const long b = g->b, d = g->d, k = g->k, m = g->m, R = g->R, s = g->s;
    if (type == 1) {
        for (long q = 0; q < b; ++q)
            for (long r = 0; r < m; ++r)
                for (long c = 0; c < m; ++c) {
                    float* row = dh + ((size_t)(q * m + r) * m + c) * ld;
                    for (long i = 0; i < k; ++i)
                        for (long j = 0; j < k; ++j)
                            for (long ch = 0; ch < d; ++ch)
                                row[(i * k + j) * d + ch] = xp_at(g, x, q, s * r + i, s * c + j, ch);
                }
    } else if (type == 2) {
        for (long q = 0; q < b; ++q)
            for (long y = 0; y < R; ++y)
                for (long c = 0; c < m; ++c) {
                    float* row = dh + ((size_t)(q * R + y) * m + c) * ld;
                    for (long j = 0; j < k; ++j)
                        for (long ch = 0; ch < d; ++ch)
                            row[j * d + ch] = xp_at(g, x, q, y, s * c + j, ch);
                }
    } else {
        for (long q = 0; q < b; ++q)
            for (long y = 0; y < R; ++y)
                for (long xx = 0; xx < R; ++xx) {
                    float* row = dh + ((size_t)(q * R + y) * R + xx) * ld;
                    for (long ch = 0; ch < d; ++ch) row[ch] = xp_at(g, x, q, y, xx, ch);
                }
    }
}

int orc_lower_internal(int type, const float* x, long b, long n, long d, long k,
                       long s, long p, float* dhat, long ld) {
    geo g;
    if (make_geo(&g, b, n, d, k, 1, s, p) || type < 1 || type > 3) return -1;
    lower_internal_geo(type, &g, x, dhat, ld);
    return 0;
}

int orc_lowered_fwd(int type, const float* x, const float* w, float* y,
                    long b, long n, long d, long k, long o, long s, long p,
                    orc_gemm_fn gemm, void* ctx) {
    geo g;
    if (make_geo(&g, b, n, d, k, o, s, p) || type < 1 || type > 3) return -1;
    if (!gemm) gemm = default_gemm;
    long rows, cols, nco;
    lowered_dims(type, &g, &rows, &cols, &nco);
    float* dh = (float*)malloc(sizeof(float) * (size_t)rows * cols);
    float* rh = (float*)malloc(sizeof(float) * (size_t)rows * nco);
    if (!dh || !rh) { free(dh); free(rh); return -1; }
    lower_internal_geo(type, &g, x, dh, cols);
    /* Rhat = Dhat * Khat, Khat^T = W viewed (nco x cols) row-major */
    gemm(ctx, 0, 1, rows, nco, cols, dh, cols, w, cols, rh, nco);
    const long m = g.m, R = g.R;
    for (long q = 0; q < b; ++q)
        for (long oj = 0; oj < o; ++oj)
            for (long r = 0; r < m; ++r)
                for (long c = 0; c < m; ++c) {
                    float v;
                    if (type == 1) {
                        v = rh[((size_t)(q * m + r) * m + c) * nco + oj];
                    } else if (type == 2) {
                        double acc = 0.0;
                        for (long i = 0; i < k; ++i)
                            acc += (double)rh[((size_t)(q * R + s * r + i) * m + c) * nco + oj * k + i];
                        v = (float)acc;
                    } else {
                        double acc = 0.0;
                        for (long i = 0; i < k; ++i)
                            for (long j = 0; j < k; ++j)
                                acc += (double)rh[((size_t)(q * R + s * r + i) * R + s * c + j) * nco +
                                                  (oj * k + i) * k + j];
                        v = (float)acc;
                    }
                    y[(((size_t)q * o + oj) * m + r) * m + c] = v;
                }
    free(dh); free(rh);
    return 0;
}

/* dRhat = expand_t(dY): adjoint of lift (zeros where lift does not read). */
static void expand_geo(int type, const geo* g, const float* dy, float* dr, long nco) {
    const long b = g->b, o = g->o, k = g->k, m = g->m, R = g->R, s = g->s;
    long rows, cols, nc;
    lowered_dims(type, g, &rows, &cols, &nc);
    if (type != 1) memset(dr, 0, sizeof(float) * (size_t)rows * nco);
    for (long q = 0; q < b; ++q)
        for (long oj = 0; oj < o; ++oj)
            for (long r = 0; r < m; ++r)
                for (long c = 0; c < m; ++c) {
                    const float v = dy[(((size_t)q * o + oj) * m + r) * m + c];
                    if (type == 1) {
                        dr[((size_t)(q * m + r) * m + c) * nco + oj] = v;
                    } else if (type == 2) {
                        for (long i = 0; i < k; ++i)
                            dr[((size_t)(q * R + s * r + i) * m + c) * nco + oj * k + i] = v;
                    } else {
                        for (long i = 0; i < k; ++i)
                            for (long j = 0; j < k; ++j)
                                dr[((size_t)(q * R + s * r + i) * R + s * c + j) * nco + (oj * k + i) * k + j] = v;
                    }
                }
}

int orc_lowered_bwd_data(int type, const float* dy, const float* w, float* dx,
                         long b, long n, long d, long k, long o, long s, long p,
                         orc_gemm_fn gemm, void* ctx) {
    geo g;
    if (make_geo(&g, b, n, d, k, o, s, p) || type < 1 || type > 3) return -1;
    if (!gemm) gemm = default_gemm;
    long rows, cols, nco;
    lowered_dims(type, &g, &rows, &cols, &nco);
    float* dr = (float*)malloc(sizeof(float) * (size_t)rows * nco);
    float* dd = (float*)malloc(sizeof(float) * (size_t)rows * cols);
    if (!dr || !dd) { free(dr); free(dd); return -1; }
    expand_geo(type, &g, dy, dr, nco);
    /* dDhat = dRhat * Khat^T, Khat^T = W viewed (nco x cols) */
    gemm(ctx, 0, 0, rows, cols, nco, dr, nco, w, cols, dd, cols);
    /* col2im_t (adjoint of lower_t): gather form, ascending taps, double acc */
    const long m = g.m, R = g.R;
    for (long q = 0; q < b; ++q)
        for (long yy = 0; yy < n; ++yy)
            for (long xx = 0; xx < n; ++xx)
                for (long ch = 0; ch < d; ++ch) {
                    const long py = yy + p, px = xx + p;
                    double acc = 0.0;
                    if (type == 3) {
                        if (py < R && px < R) acc = dd[((size_t)(q * R + py) * R + px) * cols + ch];
                    } else if (type == 2) {
                        if (py < R)
                            for (long j = 0; j < k; ++j) {
                                const long t = px - j;
                                if (t < 0 || t % s || t / s >= m) continue;
                                acc += (double)dd[((size_t)(q * R + py) * m + t / s) * cols + j * d + ch];
                            }
                    } else {
                        for (long i = 0; i < k; ++i) {
                            const long ty = py - i;
                            if (ty < 0 || ty % s || ty / s >= m) continue;
                            for (long j = 0; j < k; ++j) {
                                const long tx = px - j;
                                if (tx < 0 || tx % s || tx / s >= m) continue;
                                acc += (double)dd[((size_t)(q * m + ty / s) * m + tx / s) * cols + (i * k + j) * d + ch];
                            }
                        }
                    }
                    dx[(((size_t)q * n + yy) * n + xx) * d + ch] = (float)acc;
                }
    free(dr); free(dd);
    return 0;
}

int orc_lowered_bwd_weight(int type, const float* x, const float* dy, float* dw,
                           long b, long n, long d, long k, long o, long s, long p,
                           orc_gemm_fn gemm, void* ctx) {
    geo g;
    if (make_geo(&g, b, n, d, k, o, s, p) || type < 1 || type > 3) return -1;
    if (!gemm) gemm = default_gemm;
    long rows, cols, nco;
    lowered_dims(type, &g, &rows, &cols, &nco);
    float* dh = (float*)malloc(sizeof(float) * (size_t)rows * cols);
    float* dr = (float*)malloc(sizeof(float) * (size_t)rows * nco);
    if (!dh || !dr) { free(dh); free(dr); return -1; }
    lower_internal_geo(type, &g, x, dh, cols);
    expand_geo(type, &g, dy, dr, nco);
    /* dKhat^T (nco x cols) = dRhat^T * Dhat  ==  dW viewed (o k^a) x (k^b d) */
    gemm(ctx, 1, 0, nco, cols, rows, dr, nco, dh, cols, dw, cols);
    free(dh); free(dr);
    return 0;
}
