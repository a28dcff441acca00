// reduce.cu -- deterministic split-K reduction for the backward-weight GEMMs.
// Each output element sums its split partials in ascending split order, so the
// result is run-to-run bit-identical (no atomics).
#include <algorithm>

#include "common.cuh"
#include "reduce.cuh"

namespace cct {

namespace {
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int64_t sstride, int splits,
                                     int64_t rows, int64_t cols, int64_t ldi, float* __restrict__ out,
                                     int64_t ldo) {
    const int64_t total = rows * cols;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / cols, c = e - r * cols;
        const float* p = part + r * ldi + c;
        float acc = 0.f;
        for (int s = 0; s < splits; ++s) acc += p[int64_t(s) * sstride];
        out[r * ldo + c] = acc;
    }
}
// contiguous partials and output (ldi == ldo == cols), float4 columns: no index division
__global__ void splitk_reduce_flat4_kernel(const float4* __restrict__ part, int64_t sstride4, int splits, int64_t n4,
                                           float4* __restrict__ out) {
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n4; e += int64_t(gridDim.x) * blockDim.x) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int s = 0; s < splits; ++s) {
            const float4 v = part[int64_t(s) * sstride4 + e];
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        out[e] = acc;
    }
}
}  // namespace

// first level of a two-level reduce: group g sums splits [g*G, min((g+1)*G, S))
// into tmp[g] (ascending order), so the final result is a fixed-order sum.  V4: float4
// columns (n and the split stride multiples of 4, 16-byte aligned partials).
template <bool V4>
__global__ void splitk_group_kernel(const float* part, int64_t sstride, int splits, int group, int64_t n,
                                    float* tmp) {
    const int g = blockIdx.y;
    const int s0 = g * group, s1 = min(splits, s0 + group);
    if constexpr (V4) {
        const float4* p4 = reinterpret_cast<const float4*>(part);
        float4* t4 = reinterpret_cast<float4*>(tmp);
        const int64_t n4 = n / 4, ss4 = sstride / 4;
        for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n4;
             e += int64_t(gridDim.x) * blockDim.x) {
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
            for (int s = s0; s < s1; ++s) {
                const float4 v = p4[int64_t(s) * ss4 + e];
                acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
            }
            t4[int64_t(s0) * ss4 + e] = acc;  // in place: the group's first slice
        }
    } else {
        for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
             e += int64_t(gridDim.x) * blockDim.x) {
            float acc = 0.f;
#pragma unroll 4
            for (int s = s0; s < s1; ++s) acc += part[int64_t(s) * sstride + e];
            tmp[int64_t(s0) * sstride + e] = acc;  // in place: the group's first slice
        }
    }
}

cudaError_t splitk_reduce(const float* part, int64_t split_stride, int splits, int64_t rows,
                          int64_t cols, int64_t ld_in, float* out, int64_t ld_out, cudaStream_t st) {
    const int threads = 256;
    PhaseScope ps(kPhaseReduce, st, 0, 4.0 * double(rows * cols) * double(splits + 1));
    // Many partials (long-K backward-weight): two fixed-order levels, the first
    // in place over groups of 16 slices, so thousands of threads stream instead
    // of each summing hundreds of dependent loads.
    constexpr int kGroup = 16;
    if (splits > kGroup && ld_in == cols) {
        const int64_t n = rows * cols;
        const int ngroups = (splits + kGroup - 1) / kGroup;
        const int gx = std::max(1, int(std::min<int64_t>(cdiv(n, threads), int64_t(num_sms()) * 16 / ngroups + 1)));
        const bool v4 = n % 4 == 0 && split_stride % 4 == 0 && (reinterpret_cast<uintptr_t>(part) & 15) == 0;
        if (v4)
            splitk_group_kernel<true><<<dim3(std::max(1, gx / 4), ngroups), threads, 0, st>>>(
                part, split_stride, splits, kGroup, n, const_cast<float*>(part));
        else
            splitk_group_kernel<false><<<dim3(gx, ngroups), threads, 0, st>>>(part, split_stride, splits, kGroup, n,
                                                                              const_cast<float*>(part));
        note_launch();
        split_stride *= kGroup;
        splits = ngroups;
    }
    const int64_t n = rows * cols;
    if ((rows == 1 || (ld_in == cols && ld_out == cols)) && n % 4 == 0 && split_stride % 4 == 0 &&
        ((reinterpret_cast<uintptr_t>(part) | reinterpret_cast<uintptr_t>(out)) & 15) == 0) {
        splitk_reduce_flat4_kernel<<<grid_for(n / 4, threads), threads, 0, st>>>(
            reinterpret_cast<const float4*>(part), split_stride / 4, splits, n / 4, reinterpret_cast<float4*>(out));
    } else {
        splitk_reduce_kernel<<<grid_for(rows * cols, threads), threads, 0, st>>>(
            part, split_stride, splits, rows, cols, ld_in, out, ld_out);
    }
    note_launch();
    return cudaGetLastError();
}

}  // namespace cct
