// ref_shim.cpp -- C entry points over the REFERENCE's own tensor.cpp / gemm.cpp.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with
// /root/reference/proj/src/{tensor,gemm}.cpp (unmodified, read in place) into
// oracle/_ref/libcctref.so (git-ignored).  Used to
//   * generate golden vectors (tests/golden/make_golden.py),
//   * pin the C restatement (oracle/cct_oracle.c) against the reference, and
//   * time the reference CPU path (bench.py --impl reference / cpu_baseline):
//     restated lowering/lifting around the
//     reference's own threaded multiply (gemm.cpp:93-122).
#include <convlow/gemm.hpp>
#include <convlow/tensor.hpp>

#include <cstring>
#include <exception>
#include <random>
#include <vector>

#include "cct_oracle.h"

using namespace convlow;

namespace {

DataBatch make_batch(const float* x, long b, long n, long d) {
    std::vector<Tensor3> imgs;
    imgs.reserve(size_t(b));
    for (long q = 0; q < b; ++q) {
        Tensor3 t(static_cast<size_t>(n), static_cast<size_t>(d));
        std::memcpy(t.values().data(), x + size_t(q) * n * n * d, sizeof(float) * n * n * d);
        imgs.push_back(std::move(t));
    }
    return DataBatch(std::move(imgs));
}

KernelBank make_bank(const float* w, long k, long d, long o) {
    KernelBank bk(static_cast<size_t>(k), static_cast<size_t>(d), static_cast<size_t>(o));
    for (long j = 0; j < o; ++j)
        for (long r = 0; r < k; ++r)
            for (long c = 0; c < k; ++c)
                for (long i = 0; i < d; ++i) bk.at(j, r, c, i) = w[((j * k + r) * k + c) * d + i];
    return bk;
}

struct RefGemmCtx {
    std::size_t threads;
};

// op(A) op(B) through the reference multiply (gemm.cpp:93).  Transposed
// operands are materialised first (the reference Mat is row-major only).
void ref_gemm_cb(void* ctx, int ta, int tb, long M, long N, long K, const float* A, long lda,
                 const float* B, long ldb, float* C, long ldc) {
    Mat a(static_cast<size_t>(M), static_cast<size_t>(K));
    Mat bm(static_cast<size_t>(K), static_cast<size_t>(N));
    for (long i = 0; i < M; ++i)
        for (long t = 0; t < K; ++t) a.at(i, t) = ta ? A[size_t(t) * lda + i] : A[size_t(i) * lda + t];
    for (long t = 0; t < K; ++t)
        for (long j = 0; j < N; ++j) bm.at(t, j) = tb ? B[size_t(j) * ldb + t] : B[size_t(t) * ldb + j];
    GemmConfig cfg;
    cfg.threads = static_cast<RefGemmCtx*>(ctx)->threads;
    Mat c = multiply(a, bm, cfg);
    for (long i = 0; i < M; ++i) std::memcpy(C + size_t(i) * ldc, c.row(size_t(i)), sizeof(float) * N);
}

}  // namespace

extern "C" {

// rng(seed); batch = DataBatch::random(b,n,d,rng); bank = KernelBank::random(k,d,o,rng)
// (tensor.cpp:58-64, 39-45) -- the convention every test fixture uses.
int ref_random_problem(unsigned long long seed, long b, long n, long d, long k, long o, float* x,
                       float* w) {
    try {
        std::mt19937_64 rng(seed);
        DataBatch batch = DataBatch::random(size_t(b), size_t(n), size_t(d), rng);
        KernelBank bank = KernelBank::random(size_t(k), size_t(d), size_t(o), rng);
        for (long q = 0; q < b; ++q)
            std::memcpy(x + size_t(q) * n * n * d, batch[size_t(q)].values().data(),
                        sizeof(float) * n * n * d);
        for (long j = 0; j < o; ++j)
            for (long r = 0; r < k; ++r)
                for (long c = 0; c < k; ++c)
                    for (long i = 0; i < d; ++i) w[((j * k + r) * k + c) * d + i] = bank.at(j, r, c, i);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// Mat::random (gemm.cpp:82-87) from rng(seed)
int ref_random_mat(unsigned long long seed, long rows, long cols, float* out) {
    std::mt19937_64 rng(seed);
    Mat m = Mat::random(size_t(rows), size_t(cols), rng);
    std::memcpy(out, m.values().data(), sizeof(float) * rows * cols);
    return 0;
}

// direct_convolve_batch (tensor.cpp:108-118), unmodified reference oracle.
int ref_direct_convolve_batch(const float* x, long b, long n, long d, const float* w, long k,
                              long o, float* y) {
    try {
        OutputBatch out = direct_convolve_batch(make_batch(x, b, n, d), make_bank(w, k, d, o));
        std::memcpy(y, out.values().data(), sizeof(float) * out.size());
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// Forward with stride/pad through direct_convolve: zero-embed n -> n+2p
// (translation consistency), convolve at stride 1, subsample.
int ref_conv_fwd_adapter(const float* x, const float* w, float* y, long b, long n, long d, long k,
                         long o, long s, long p) {
    try {
        const long N = n + 2 * p, M1 = N - k + 1, m = (N - k) / s + 1;
        std::vector<float> xp(size_t(b) * N * N * d, 0.0f);
        for (long q = 0; q < b; ++q)
            for (long r = 0; r < n; ++r)
                std::memcpy(&xp[((size_t(q) * N + r + p) * N + p) * d], x + (size_t(q) * n + r) * n * d,
                            sizeof(float) * n * d);
        OutputBatch full = direct_convolve_batch(make_batch(xp.data(), b, N, d), make_bank(w, k, d, o));
        for (long q = 0; q < b; ++q)
            for (long j = 0; j < o; ++j)
                for (long r = 0; r < m; ++r)
                    for (long c = 0; c < m; ++c)
                        y[((size_t(q) * o + j) * m + r) * m + c] = full.at(q, j, s * r, s * c);
        (void)M1;
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// Backward-data through direct_convolve: canvas T of side N+k-1,
// depth o, dY dilated by s at offset k-1; per input channel ch a KernelBank of
// depth o with Kr[i',j',oj] = W[oj,k-1-i',k-1-j',ch]; crop the padding.
int ref_conv_bwd_data_adapter(const float* dy, const float* w, float* dx, long b, long n, long d,
                              long k, long o, long s, long p) {
    try {
        const long N = n + 2 * p, m = (N - k) / s + 1, T = N + k - 1;
        KernelBank kr{size_t(k), size_t(o), size_t(d)};
        for (long ch = 0; ch < d; ++ch)
            for (long ii = 0; ii < k; ++ii)
                for (long jj = 0; jj < k; ++jj)
                    for (long oj = 0; oj < o; ++oj)
                        kr.at(ch, ii, jj, oj) = w[((oj * k + (k - 1 - ii)) * k + (k - 1 - jj)) * d + ch];
        for (long q = 0; q < b; ++q) {
            Tensor3 canvas{size_t(T), size_t(o)};
            for (long oj = 0; oj < o; ++oj)
                for (long r = 0; r < m; ++r)
                    for (long c = 0; c < m; ++c)
                        canvas.at(k - 1 + s * r, k - 1 + s * c, oj) = dy[((size_t(q) * o + oj) * m + r) * m + c];
            for (long ch = 0; ch < d; ++ch) {
                OutputPlane pl = direct_convolve(canvas, kr, size_t(ch));  // N x N
                for (long yy = 0; yy < n; ++yy)
                    for (long xx = 0; xx < n; ++xx)
                        dx[((size_t(q) * n + yy) * n + xx) * d + ch] = pl.at(yy + p, xx + p);
            }
        }
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// Backward-weight through direct_convolve: for each ch,
// D'[y,x,q] = Xp[q,y,x,ch] (side N, depth b); for each oj the kernel is
// dY[:,oj] dilated by s (side s(m-1)+1, depth b); keep the top-left k x k.
int ref_conv_bwd_weight_adapter(const float* x, const float* dy, float* dw, long b, long n, long d,
                                long k, long o, long s, long p) {
    try {
        const long N = n + 2 * p, m = (N - k) / s + 1, ks = s * (m - 1) + 1;
        KernelBank kd{size_t(ks), size_t(b), size_t(o)};
        for (long oj = 0; oj < o; ++oj)
            for (long r = 0; r < m; ++r)
                for (long c = 0; c < m; ++c)
                    for (long q = 0; q < b; ++q)
                        kd.at(oj, s * r, s * c, q) = dy[((size_t(q) * o + oj) * m + r) * m + c];
        for (long ch = 0; ch < d; ++ch) {
            Tensor3 dp{size_t(N), size_t(b)};
            for (long q = 0; q < b; ++q)
                for (long yy = 0; yy < n; ++yy)
                    for (long xx = 0; xx < n; ++xx)
                        dp.at(yy + p, xx + p, q) = x[((size_t(q) * n + yy) * n + xx) * d + ch];
            for (long oj = 0; oj < o; ++oj) {
                OutputPlane pl = direct_convolve(dp, kd, size_t(oj));
                for (long i = 0; i < k; ++i)
                    for (long j = 0; j < k; ++j) dw[((size_t(oj) * k + i) * k + j) * d + ch] = pl.at(i, j);
            }
        }
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// multiply (gemm.cpp:93-122) and multiply_reference (gemm.cpp:124-141).
int ref_multiply(const float* A, const float* B, float* C, long M, long K, long N, long threads) {
    try {
        Mat a(static_cast<size_t>(M), static_cast<size_t>(K));
    Mat bm(static_cast<size_t>(K), static_cast<size_t>(N));
        std::memcpy(a.values().data(), A, sizeof(float) * M * K);
        std::memcpy(bm.values().data(), B, sizeof(float) * K * N);
        GemmConfig cfg;
        cfg.threads = size_t(threads);
        Mat c = multiply(a, bm, cfg);
        std::memcpy(C, c.values().data(), sizeof(float) * M * N);
        return 0;
    } catch (const config_error&) {
        return 1;
    } catch (const std::exception&) {
        return 2;
    }
}

int ref_multiply_reference(const float* A, const float* B, float* C, long M, long K, long N) {
    try {
        Mat a(static_cast<size_t>(M), static_cast<size_t>(K));
    Mat bm(static_cast<size_t>(K), static_cast<size_t>(N));
        std::memcpy(a.values().data(), A, sizeof(float) * M * K);
        std::memcpy(bm.values().data(), B, sizeof(float) * K * N);
        Mat c = multiply_reference(a, bm);
        std::memcpy(C, c.values().data(), sizeof(float) * M * N);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// The reference CPU lowered path: restated lower/lift around the reference's
// threaded multiply.  pass: 0 fwd, 1 bwd-data, 2 bwd-weight.
int ref_lowered(int pass, int type, long threads, const float* in0, const float* in1, float* out,
                long b, long n, long d, long k, long o, long s, long p) {
    try {
        RefGemmCtx ctx{size_t(threads)};
        if (pass == 0) return orc_lowered_fwd(type, in0, in1, out, b, n, d, k, o, s, p, ref_gemm_cb, &ctx);
        if (pass == 1)
            return orc_lowered_bwd_data(type, in0, in1, out, b, n, d, k, o, s, p, ref_gemm_cb, &ctx);
        return orc_lowered_bwd_weight(type, in0, in1, out, b, n, d, k, o, s, p, ref_gemm_cb, &ctx);
    } catch (const std::exception&) {
        return -2;
    }
}

// gemm_throughput_probe (gemm.cpp:143-179) / memcpy_bandwidth_probe (gemm.cpp:181-200)
double ref_gemm_throughput_probe(long rows, long inner, long cols, long threads, int reps) {
    try {
        GemmConfig cfg;
        cfg.threads = size_t(threads);
        return gemm_throughput_probe(size_t(rows), size_t(inner), size_t(cols), cfg, reps).flops_per_s;
    } catch (const std::exception&) {
        return -1.0;
    }
}

double ref_memcpy_bandwidth_probe(long bytes, int reps) {
    try {
        return memcpy_bandwidth_probe(size_t(bytes), reps);
    } catch (const std::exception&) {
        return -1.0;
    }
}

}  // extern "C"
