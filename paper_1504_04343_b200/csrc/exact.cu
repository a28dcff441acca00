// exact.cu -- the reference's ORACLE entry points on the device, bit-identical.
//
// direct_convolve (tensor.cpp:77-106) and multiply_reference (gemm.cpp:124-141)
// are part of the convlow API a drop-in must provide.  They are not the hot path
// (that is lowering + the tcgen05 GEMM); they are the reference's ground truth,
// kept exact: one thread per output, a double accumulator updated in the
// reference's loop order with explicitly rounded multiply and add (__dmul_rn /
// __dadd_rn: no FMA contraction, matching -ffp-contract=off), one rounding to
// float at the end.
#include "cct.h"
#include "common.cuh"

namespace cct {
namespace {

__global__ void direct_conv_exact_kernel(const float* __restrict__ x, const float* __restrict__ w,
                                         float* __restrict__ y, int64_t b, int n, int d, int k, int o, int s, int p,
                                         int m) {
    const int64_t total = b * o * int64_t(m) * m;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(e % m);
        int64_t t = e / m;
        const int r = int(t % m);
        t /= m;
        const int j = int(t % o);
        const int64_t q = t / o;
        const float* xq = x + q * int64_t(n) * n * d;
        const float* wj = w + int64_t(j) * k * k * d;
        double acc = 0.0;
        // loop order i -> c' -> r' (tensor.cpp:94-101); padding taps contribute
        // +-0.0 in the reference's zero-embedded formulation and are skipped
        for (int i = 0; i < d; ++i)
            for (int cp = 0; cp < k; ++cp) {
                const int xc = s * c + cp - p;
                if (xc < 0 || xc >= n) continue;
                for (int rp = 0; rp < k; ++rp) {
                    const int xr = s * r + rp - p;
                    if (xr < 0 || xr >= n) continue;
                    acc = __dadd_rn(acc, __dmul_rn(double(xq[(int64_t(xr) * n + xc) * d + i]),
                                                   double(wj[(int64_t(rp) * k + cp) * d + i])));
                }
            }
        y[e] = float(acc);
    }
}

__global__ void gemm_exact_kernel(int64_t M, int64_t N, int64_t K, const float* __restrict__ A, int64_t lda,
                                  const float* __restrict__ B, int64_t ldb, float* __restrict__ C, int64_t ldc) {
    const int64_t total = M * N;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = e / N, j = e - i * N;
        double acc = 0.0;
        for (int64_t t = 0; t < K; ++t)
            acc = __dadd_rn(acc, __dmul_rn(double(A[i * lda + t]), double(B[t * ldb + j])));
        C[i * ldc + j] = float(acc);
    }
}

}  // namespace
}  // namespace cct

using namespace cct;

extern "C" {

cct_status cct_direct_conv_fwd_exact(const cct_conv_desc* desc, const float* x, const float* w, float* y,
                                     void* stream) {
    cct_conv_desc d;
    if (!desc) return CCT_ERR_CONFIG;
    if (desc->layout != CCT_LAYOUT_NCHW) return CCT_ERR_UNSUPPORTED;  // the oracle entry point writes OutputBatch
    cct_status st = cct_conv_desc_init(&d, desc->n, desc->k, desc->d, desc->o, desc->b, desc->stride, desc->pad);
    if (st != CCT_OK) return st;
    if (!x || !w || !y) return CCT_ERR_CONFIG;
    const int64_t total = d.b * d.o * d.m * d.m;
    direct_conv_exact_kernel<<<grid_for(total, 256, 16), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        x, w, y, d.b, int(d.n), int(d.d), int(d.k), int(d.o), int(d.stride), int(d.pad), int(d.m));
    note_launch();
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string("direct convolution: ") + cudaGetErrorString(e));
        return CCT_ERR_CUDA;
    }
    return CCT_OK;
}

cct_status cct_gemm_exact(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B, int64_t ldb,
                          float* C, int64_t ldc, void* stream) {
    if (M < 0 || N < 0 || K < 0 || lda < K || ldb < N || ldc < N) {
        set_error("invalid exact gemm arguments");
        return CCT_ERR_CONFIG;
    }
    if (M == 0 || N == 0) return CCT_OK;
    if (!A || !B || !C) return CCT_ERR_CONFIG;
    gemm_exact_kernel<<<grid_for(M * N, 256, 16), 256, 0, static_cast<cudaStream_t>(stream)>>>(M, N, K, A, lda, B, ldb,
                                                                                              C, ldc);
    note_launch();
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string("exact gemm: ") + cudaGetErrorString(e));
        return CCT_ERR_CUDA;
    }
    return CCT_OK;
}

}  // extern "C"
