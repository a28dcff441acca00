// m64_probe.cu -- diagnostic: tcgen05.mma kind::tf32 with M = 64 vs M = 128 (cta_group::1).
// (1) where the M = 64 accumulator rows land in TMEM, (2) cycles per MMA back to back.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../paper_1504_04343_b200/csrc m64_probe.cu
#include <cstdio>
#include <cstdint>

#include "ptx.cuh"

using namespace cct;

__device__ __forceinline__ uint32_t sw64(int r, int k) {  // K-major SWIZZLE_64B element address (bytes)
    const int c = k >> 2;
    return uint32_t(r * 64 + ((c ^ ((r >> 1) & 3)) << 4) + (k & 3) * 4);
}

__global__ void probe(float* out, long long* cyc, int M, int N, int reps, int alt = 1) {
    __shared__ __align__(1024) uint8_t a_s[128 * 64];
    __shared__ __align__(1024) uint8_t b_s[256 * 64];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 128 * 16; i += blockDim.x) {
        const int r = i / 16, k = i % 16;
        *reinterpret_cast<float*>(a_s + sw64(r, k)) = (k == 0) ? float(r + 1) : 0.f;
    }
    for (int i = tid; i < 256 * 16; i += blockDim.x) {
        const int n = i / 16, k = i % 16;
        *reinterpret_cast<float*>(b_s + sw64(n, k)) = (k == 0) ? 1.f : 0.f;
    }
    if (tid == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_barrier_init();
    }
    ptx::fence_proxy_async_smem();
    __syncthreads();
    if (warp == 0) ptx::tmem_alloc<512, 1>(&tslot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tslot;
    const uint32_t idesc = ptx::idesc_tf32(uint32_t(M), uint32_t(N), 0, 0);
    const uint64_t ad = ptx::smem_desc(ptx::smem_u32(a_s), 16, 512, 4);
    const uint64_t bd = ptx::smem_desc(ptx::smem_u32(b_s), 16, 512, 4);
    if (tid == 0) {
        // one MMA to map rows, then `reps` accumulating MMAs timed
        ptx::mma_tf32(tmem, ad, bd, idesc, 0u);
        ptx::mma_commit(&bar);
    }
    ptx::mbar_wait(&bar, 0);
    ptx::tc_fence_after();
    uint32_t v[32];
    ptx::tmem_ld_32x32b_x32(tmem + (uint32_t(warp * 32) << 16), v);
    ptx::tmem_ld_wait();
    for (int j = 0; j < 4; ++j) out[(warp * 32 + lane) * 4 + j] = __uint_as_float(v[j]);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (tid == 0) {
        const long long t0 = clock64();
        for (int i = 0; i < reps; ++i) ptx::mma_tf32(tmem + (alt ? 256 * (i & 1) : 0), ad, bd, idesc, 1u);
        ptx::mma_commit(&bar);
        ptx::mbar_wait(&bar, 1);
        cyc[0] = clock64() - t0;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<512, 1>(tmem);
}

int main() {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 128 * 4 * 4);
    cudaMalloc(&cyc, 8);
    for (int M : {128, 64}) {
        cudaMemset(out, 0, 128 * 4 * 4);
        probe<<<1, 128>>>(out, cyc, M, 256, 2000);
        cudaError_t e = cudaDeviceSynchronize();
        float h[128 * 4];
        long long c = 0;
        cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("M=%d err=%s cycles/MMA (N=256, K=8) = %.1f\n  lane -> D[.,0]: ", M, cudaGetErrorString(e),
               double(c) / 2000.0);
        for (int l = 0; l < 128; l += 8) printf("%d:%g ", l, h[l * 4]);
        printf("\n");
    }
    for (int N : {64, 128, 192, 256}) {
        for (int M : {128, 64}) {
            probe<<<1, 128>>>(out, cyc, M, N, 2000);
            cudaDeviceSynchronize();
            long long c = 0;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("M=%3d N=%3d: %.1f cycles per MMA\n", M, N, double(c) / 2000.0);
        }
    }
    for (int N : {128, 256}) {
        for (int alt : {0, 1}) {
            probe<<<1, 128>>>(out, cyc, 128, N, 2000, alt);
            cudaDeviceSynchronize();
            long long c = 0;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("M=128 N=%3d %s accumulator: %.1f cycles per MMA\n", N, alt ? "alternating" : "same", double(c) / 2000.0);
        }
    }
    return 0;
}
