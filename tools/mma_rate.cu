// mma_rate.cu -- diagnostic: tcgen05.mma kind::tf32 throughput on all SMs (event-timed), A
// from shared memory vs from TMEM, per tile width N.  Per "k-block": 6 MMAs (M = 128, K = 8),
// commit to a 4-deep barrier ring, the issuing thread waits for k-block kb - 4 (bounded queue).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../paper_1504_04343_b200/csrc mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <vector>

#include "ptx.cuh"

using namespace cct;

template <int N, bool ATM, int ROT, int NACC, bool BMN = false>
__global__ void __launch_bounds__(128, 1) probe(int kblocks) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = sm_raw + ((1024u - (ptx::smem_u32(sm_raw) & 1023u)) & 1023u);
    uint8_t* a = sm;                  // ROT x 2 x 128 x 64 B (big | small)
    uint8_t* b = sm + 16384 * ROT;    // 2 x N x 64 B
    uint64_t* bar = reinterpret_cast<uint64_t*>(b + 2 * N * 64);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 4);
    for (int i = threadIdx.x; i < (16384 * ROT + 2 * N * 64) / 4; i += 128) reinterpret_cast<float*>(sm)[i] = 0.25f;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 4; ++s) ptx::mbar_init(&bar[s], 1);
        ptx::fence_barrier_init();
    }
    ptx::fence_proxy_async_smem();
    if ((threadIdx.x >> 5) == 2) ptx::tmem_alloc<512, 1>(tslot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = ptx::idesc_tf32(128, N, 0, BMN ? 1 : 0);
        const uint32_t as = ptx::smem_u32(a), bs = ptx::smem_u32(b);
        uint32_t ph[4] = {0, 0, 0, 0};
        for (int kb = 0; kb < kblocks; ++kb) {
            const int s = kb & 3;
            if (kb >= 4) { ptx::mbar_wait(&bar[s], ph[s]); ph[s] ^= 1; }
            ptx::tc_fence_after();
#pragma unroll
            for (int prod = 0; prod < 3; ++prod)
#pragma unroll
                for (int kk = 0; kk < 2; ++kk) {
                    const uint64_t bd = BMN ? ptx::smem_desc(bs + (prod == 1 ? N * 64 : 0) + kk * 1024, 2048, 512, 1)
                                             : ptx::smem_desc(bs + (prod == 1 ? N * 64 : 0) + kk * 32, 16, 512, 4);
                    const uint32_t acc = (kb | prod | (NACC == 1 ? kk : 0)) ? 1u : 0u;
                    const uint32_t d = tmem + (NACC == 2 ? kk * N : 0);
                    const int slot = kb % ROT;
                    if constexpr (ATM) {
                        const uint32_t at = tmem + NACC * N + slot * 32;
                        ptx::mma_tf32_ts(d, at + (prod == 0 ? 16 : 0) + kk * 8, bd, idesc, acc);
                    } else {
                        ptx::mma_tf32(d, ptx::smem_desc(as + slot * 16384 + (prod == 0 ? 8192 : 0) + kk * 32, 16, 512, 4), bd,
                                      idesc, acc);
                    }
                }
            ptx::mma_commit(&bar[s]);
        }
        for (int kb = kblocks; kb < kblocks + 4; ++kb) {
            const int s = kb & 3;
            ptx::mbar_wait(&bar[s], ph[s]);
            ph[s] ^= 1;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if ((threadIdx.x >> 5) == 2) ptx::tmem_dealloc<512, 1>(tmem);
}

template <int N, bool ATM, int ROT, int NACC, bool BMN = false>
void run(int sms) {
    const int smem = 16384 * ROT + 2 * N * 64 + 2048;
    cudaFuncSetAttribute(probe<N, ATM, ROT, NACC, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int kb = 20000;
    probe<N, ATM, ROT, NACC, BMN><<<sms, 128, smem>>>(100);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<N, ATM, ROT, NACC, BMN><<<sms, 128, smem>>>(kb);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ns = ms * 1e6 / kb;
    printf("N=%3d B_%s A_%s rot=%d nacc=%d: %6.1f ns per k-block (6 MMAs) = %5.1f cycles @1.965 GHz, %6.1f TF/s tf32  %s\n", N, BMN ? "MN" : "K ",
           ATM ? "TMEM" : "SMEM", ROT, NACC, ns, ns * 1.965, 6.0 * 2 * 128 * N * 8 * sms / ns / 1e3, cudaGetErrorString(e));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<96, true, 8, 1, false>(sms); run<96, true, 8, 1, true>(sms);
    run<96, false, 4, 1, false>(sms); run<96, false, 4, 1, true>(sms);
    run<128, true, 8, 1, true>(sms); run<64, true, 8, 1, true>(sms); run<256, true, 4, 1, true>(sms);
    run<96, false, 1, 1>(sms); run<96, true, 1, 1>(sms);
    run<96, false, 4, 1>(sms); run<96, true, 8, 1>(sms);
    run<96, false, 4, 2>(sms); run<96, true, 8, 2>(sms);
    run<128, false, 4, 1>(sms); run<128, true, 8, 1>(sms);
    run<128, false, 4, 2>(sms); run<128, true, 4, 2>(sms);
    run<192, false, 4, 1>(sms); run<192, true, 4, 1>(sms);
    run<256, false, 4, 1>(sms); run<256, true, 4, 1>(sms);
    return 0;
}
