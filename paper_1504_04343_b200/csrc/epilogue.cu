// epilogue.cu -- bias / ReLU kernels around the convolution (see epilogue.cuh).
#include <algorithm>

#include "common.cuh"
#include "epilogue.cuh"

namespace cct {

namespace {

constexpr int kThreads = 256;

__global__ void bias_act_kernel(float* __restrict__ y, const float* __restrict__ bias, int relu, int64_t planes,
                                int o, int mm, int64_t ostride) {
    for (int64_t pl = blockIdx.x; pl < planes; pl += gridDim.x) {
        const int64_t q = pl / o;
        const int j = int(pl - q * o);
        const float bv = bias ? __ldg(bias + j) : 0.f;
        float* p = y + (q * ostride + j) * mm;
        for (int i = threadIdx.x; i < mm; i += blockDim.x) {
            float v = p[i] + bv;
            p[i] = relu ? fmaxf(v, 0.f) : v;
        }
    }
}

// one block per (image, channel) plane: mask, store, block-reduce the plane sum
__global__ void relu_bias_bwd_kernel(const float* __restrict__ dy, const float* __restrict__ y, float* __restrict__ dz,
                                     float* __restrict__ partial, int relu, int64_t planes, int mm) {
    __shared__ float red[kThreads / 32];
    for (int64_t pl = blockIdx.x; pl < planes; pl += gridDim.x) {
        const float* g = dy + pl * mm;
        const float* a = y ? y + pl * mm : nullptr;
        float* z = dz + pl * mm;
        float sum = 0.f;
        for (int i = threadIdx.x; i < mm; i += blockDim.x) {
            float v = __ldg(g + i);
            if (relu) {
                v = (__ldg(a + i) > 0.f) ? v : 0.f;
                z[i] = v;
            }
            sum += v;
        }
        if (partial) {
#pragma unroll
            for (int off = 16; off; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
            if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
            __syncthreads();
            if (threadIdx.x == 0) {
                float t = 0.f;
                for (int w = 0; w < kThreads / 32; ++w) t += red[w];
                partial[pl] = t;
            }
            __syncthreads();
        }
    }
}

// db[j] = sum_q partial[q][j] in image order (deterministic)
__global__ void bias_grad_kernel(const float* __restrict__ partial, float* __restrict__ db, int64_t b, int o) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= o) return;
    float t = 0.f;
    for (int64_t q = 0; q < b; ++q) t += partial[q * o + j];
    db[j] = t;
}

}  // namespace

cudaError_t bias_act(float* y, const float* bias, int relu, int64_t b, int64_t o, int64_t mm, int64_t ostride,
                     cudaStream_t st) {
    if (!bias && !relu) return cudaSuccess;
    PhaseScope ps(kPhaseOther, st, 0, 8.0 * double(b * o * mm));
    const int64_t planes = b * o;
    bias_act_kernel<<<int(std::min<int64_t>(planes, int64_t(num_sms()) * 16)), kThreads, 0, st>>>(
        y, bias, relu, planes, int(o), int(mm), ostride);
    note_launch();
    return cudaGetLastError();
}

cudaError_t relu_bias_bwd(const float* dy, const float* y, float* dz, float* db, float* partial, int relu, int64_t b,
                          int64_t o, int64_t mm, cudaStream_t st) {
    if (!relu && !db) return cudaSuccess;
    {
        PhaseScope ps(kPhaseExpand, st, 0, 4.0 * double(b * o * mm) * (relu ? 3.0 : 1.0));
        const int64_t planes = b * o;
        relu_bias_bwd_kernel<<<int(std::min<int64_t>(planes, int64_t(num_sms()) * 16)), kThreads, 0, st>>>(
            dy, y, dz, db ? partial : nullptr, relu, planes, int(mm));
        note_launch();
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (db) {
        PhaseScope ps(kPhaseReduce, st, 0, 4.0 * double(b * o + o));
        bias_grad_kernel<<<int(cdiv(o, 128)), 128, 0, st>>>(partial, db, b, int(o));
        note_launch();
        return cudaGetLastError();
    }
    return cudaSuccess;
}

cudaError_t copy2d(float* dst, int64_t dpitch, const float* src, int64_t spitch, int64_t width, int64_t rows,
                   cudaStream_t st) {
    PhaseScope ps(kPhaseOther, st, 0, 8.0 * double(width * rows));
    return cudaMemcpy2DAsync(dst, size_t(dpitch) * 4, src, size_t(spitch) * 4, size_t(width) * 4, size_t(rows),
                             cudaMemcpyDeviceToDevice, st);
}

}  // namespace cct
