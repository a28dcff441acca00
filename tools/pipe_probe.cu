// pipe_probe.cu -- diagnostic: cycles per 16-wide k-block of the 3xTF32 MMA pipeline
// (6 tcgen05.mma kind::tf32 per k-block, M = 128) on all SMs at once, isolating the
// A-operand handoff from everything else (no TMA, no HBM):
//   mode 0: MMA issue only (operands static in smem / TMEM, commit per k-block)
//   mode 1: + A ring: 4 "gather" warps per group (2 groups, alternate k-blocks) write
//           the k-block's A big / small (tcgen05.st to a TMEM slot, or st.shared) and
//           arrive on tdone; the MMA thread waits tdone and commits to empty
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../paper_1504_04343_b200/csrc pipe_probe.cu
#include <cstdio>
#include <cstdint>

#include "ptx.cuh"

using namespace cct;

template <int N, int ATM, int SLOTS, int NACC>
__global__ void __launch_bounds__(384, 1) probe(long long* cyc, int kblocks, int mode) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = sm_raw + ((1024u - (ptx::smem_u32(sm_raw) & 1023u)) & 1023u);
    uint8_t* b_big = sm;                    // N x 16 fp32, K-major SW64
    uint8_t* b_sml = b_big + N * 64;
    uint8_t* a_ring = b_sml + N * 64;       // SLOTS x (big 8 KB | small 8 KB) when !ATM
    uint64_t* tdone = reinterpret_cast<uint64_t*>(a_ring + (ATM ? 0 : SLOTS * 16384));
    uint64_t* empty = tdone + SLOTS;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(empty + SLOTS);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < N * 32; i += blockDim.x) reinterpret_cast<float*>(b_big)[i] = 0.001f * (i & 7);
    if (!ATM)
        for (int i = tid; i < SLOTS * 4096; i += blockDim.x) reinterpret_cast<float*>(a_ring)[i] = 0.5f;
    if (tid == 0) {
        for (int s = 0; s < SLOTS; ++s) {
            ptx::mbar_init(&tdone[s], 4);  // one arrive per warp of the group
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::fence_barrier_init();
    }
    ptx::fence_proxy_async_smem();
    __syncthreads();
    if (warp == 2) ptx::tmem_alloc<512, 1>(tslot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    constexpr uint32_t A_COL = uint32_t(NACC * N);
    const uint32_t idesc = ptx::idesc_tf32(128, N, 0, 0);
    if (warp == 1 && lane == 0) {
        const long long t0 = clock64();
        int s = 0;
        uint32_t ph = 0;
        for (int kb = 0; kb < kblocks; ++kb) {
            if (mode == 1) ptx::mbar_wait(&tdone[s], ph);
            else if (kb >= SLOTS) ptx::mbar_wait(&empty[s], ph ^ 1);
            ptx::tc_fence_after();
            const uint32_t first = kb ? 1u : 0u;
            if constexpr (ATM) {
                const uint32_t ab = tmem + A_COL + uint32_t(s) * 32, as = ab + 16;
#pragma unroll
                for (int kk = 0; kk < 2; ++kk)
                    ptx::mma_tf32_ts(tmem + kk * (NACC - 1) * N, as + kk * 8,
                                     ptx::smem_desc(ptx::smem_u32(b_big) + kk * 32, 16, 512, 4), idesc, first);
#pragma unroll
                for (int kk = 0; kk < 2; ++kk)
                    ptx::mma_tf32_ts(tmem + kk * (NACC - 1) * N, ab + kk * 8,
                                     ptx::smem_desc(ptx::smem_u32(b_sml) + kk * 32, 16, 512, 4), idesc, 1u);
#pragma unroll
                for (int kk = 0; kk < 2; ++kk)
                    ptx::mma_tf32_ts(tmem + kk * (NACC - 1) * N, ab + kk * 8,
                                     ptx::smem_desc(ptx::smem_u32(b_big) + kk * 32, 16, 512, 4), idesc, 1u);
            } else {
                const uint32_t ab = ptx::smem_u32(a_ring) + s * 16384, as = ab + 8192;
#pragma unroll
                for (int kk = 0; kk < 2; ++kk)
                    ptx::mma_tf32(tmem + kk * (NACC - 1) * N, ptx::smem_desc(as + kk * 32, 16, 512, 4),
                                  ptx::smem_desc(ptx::smem_u32(b_big) + kk * 32, 16, 512, 4), idesc, first);
#pragma unroll
                for (int kk = 0; kk < 2; ++kk)
                    ptx::mma_tf32(tmem + kk * (NACC - 1) * N, ptx::smem_desc(ab + kk * 32, 16, 512, 4),
                                  ptx::smem_desc(ptx::smem_u32(b_sml) + kk * 32, 16, 512, 4), idesc, 1u);
#pragma unroll
                for (int kk = 0; kk < 2; ++kk)
                    ptx::mma_tf32(tmem + kk * (NACC - 1) * N, ptx::smem_desc(ab + kk * 32, 16, 512, 4),
                                  ptx::smem_desc(ptx::smem_u32(b_big) + kk * 32, 16, 512, 4), idesc, 1u);
            }
            ptx::mma_commit(&empty[s]);
            if (++s == SLOTS) { s = 0; ph ^= 1; }
        }
        // drain: wait for the last commit
        const int last = (kblocks - 1) % SLOTS;
        const uint32_t lph = uint32_t(((kblocks - 1) / SLOTS) & 1);
        ptx::mbar_wait(&empty[last], lph);
        cyc[blockIdx.x] = clock64() - t0;
    } else if (warp >= 4 && warp < 12 && mode == 1) {
        const int g = (warp - 4) >> 2;  // group: k-blocks kb % 2 == g
        const int q = warp & 3;
        int s = 0;
        uint32_t eph = 0;  // per-slot phase bits of empty
        for (int kb = 0; kb < kblocks; ++kb) {
            const int slot = s;
            if (++s == SLOTS) s = 0;
            if ((kb & 1) != g) continue;
            if (kb >= SLOTS) {
                ptx::mbar_wait(&empty[slot], ((kb / SLOTS) - 1) & 1);
            }
            (void)eph;
            if constexpr (ATM) {
                uint32_t v[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(0.25f + 0.001f * (j ^ lane));
                ptx::tmem_st_32x32b_x32(tmem + (uint32_t(q * 32) << 16) + A_COL + uint32_t(slot) * 32, v);
                ptx::tmem_st_wait();
                ptx::tc_fence_before();
            } else {
                const uint32_t base = ptx::smem_u32(a_ring) + slot * 16384 + (q * 32 + lane) * 64;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    ptx::sts128(base + c * 16, make_float4(0.5f, 0.25f, 0.125f, 1.f));
                    ptx::sts128(base + 8192 + c * 16, make_float4(0.5f, 0.25f, 0.125f, 1.f));
                }
                ptx::fence_proxy_async_smem();
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tdone[slot]);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) ptx::tmem_dealloc<512, 1>(tmem);
}

template <int N, int ATM, int SLOTS, int NACC>
void run(int mode, long long* d, int sms) {
    const int smem = 1024 + 2 * N * 64 + (ATM ? 0 : SLOTS * 16384) + 1024;
    auto k = probe<N, ATM, SLOTS, NACC>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int kb = 20000;
    k<<<sms, 384, smem>>>(d, 100, mode);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<sms, 384, smem>>>(d, kb, mode);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[160];
    cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
    long long mx = 0, mn = 1LL << 62;
    for (int i = 0; i < sms; ++i) { mx = h[i] > mx ? h[i] : mx; mn = h[i] < mn ? h[i] : mn; }
    printf("N=%3d A_%s slots=%2d nacc=%d mode=%d (%s): %7.1f ns per k-block (event)  [%7.1f .. %7.1f clk] %s\n", N,
           ATM ? "TMEM" : "SMEM", SLOTS, NACC, mode, mode ? "A ring" : "MMA only", ms * 1e6 / kb, double(mn) / kb,
           double(mx) / kb, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    long long* d;
    cudaMalloc(&d, 160 * 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int mode : {0, 1}) {
        run<96, 1, 8, 1>(mode, d, sms);
        run<96, 1, 4, 1>(mode, d, sms);
        run<96, 0, 8, 1>(mode, d, sms);
        run<96, 0, 4, 1>(mode, d, sms);
        run<128, 1, 8, 1>(mode, d, sms);
        run<256, 0, 4, 1>(mode, d, sms);
    }
    return 0;
}
