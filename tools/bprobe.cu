// bprobe.cu -- diagnostic: does streaming the (shared) kernel-bank tile through TMA every
// k-block limit a narrow tcgen05 GEMM?  148 CTAs, A static in TMEM, per k-block 6 MMAs
// (M = 128, N = 96) with B (big | small, 2 x 96 x 16 fp32) loaded by TMA into a ring:
//   mode 0: B static in smem (no TMA)       mode 1: every CTA reads the SAME bank (hot lines)
//   mode 2: every CTA reads its OWN copy     mode 3: like 1, cluster of 4 with TMA multicast
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../paper_1504_04343_b200/csrc bprobe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#include "ptx.cuh"

using namespace cct;
constexpr int NP = 96, KP = 400, STAGES = 8;
constexpr uint32_t BB = NP * 16 * 4;

__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(ptx::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(ptx::smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
        : "memory");
}

__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap tm, long long* cyc, int kblocks,
                                                int mode, int csize) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = sm_raw + ((1024u - (ptx::smem_u32(sm_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * 2 * BB);
    uint64_t* empty = full + STAGES;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(empty + STAGES);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = mode == 3 ? ptx::cluster_rank() : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], mode == 3 ? csize : 1);  // multicast: every CTA's MMA frees the stage
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<512, 1>(tslot);
    ptx::tc_fence_before();
    if (mode == 3) ptx::cluster_sync(); else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    const int row0 = mode == 2 ? int(blockIdx.x) * 2 * NP : 0;
    if (warp == 0 && lane == 0 && mode != 0) {
        int st = 0; uint32_t ph = 0;
        for (int kb = 0; kb < kblocks; ++kb) {
            ptx::mbar_wait(&empty[st], ph ^ 1);
            ptx::mbar_arrive_expect_tx(&full[st], 2 * BB);
            const int kc = (kb % (KP / 16)) * 16;
            uint8_t* dst = sm + st * 2 * BB;
            if (mode == 3) {
                // this CTA loads 1/csize of the rows... simpler: rank r issues the big/small halves of
                // stage kb when kb % csize == r, multicast to all
                if (int(kb % csize) == int(crank)) {
                    tma_load_2d_mc(dst, &tm, &full[st], kc, row0, uint16_t((1 << csize) - 1));
                    tma_load_2d_mc(dst + BB, &tm, &full[st], kc, row0 + NP, uint16_t((1 << csize) - 1));
                }
            } else {
                ptx::tma_load_2d(dst, &tm, &full[st], kc, row0);
                ptx::tma_load_2d(dst + BB, &tm, &full[st], kc, row0 + NP);
            }
            if (++st == STAGES) { st = 0; ph ^= 1; }
        }
    } else if (warp == 1 && lane == 0) {
        const uint32_t idesc = ptx::idesc_tf32(128, NP, 0, 0);
        const long long t0 = clock64();
        int st = 0; uint32_t ph = 0;
        for (int kb = 0; kb < kblocks; ++kb) {
            if (mode != 0) ptx::mbar_wait(&full[st], ph);
            ptx::tc_fence_after();
            const uint32_t bb = ptx::smem_u32(sm) + (mode ? st : 0) * 2 * BB, bs = bb + BB;
            const uint32_t ab = tmem + 2 * NP + (kb & 7) * 32, as = ab + 16;
            for (int kk = 0; kk < 2; ++kk) ptx::mma_tf32_ts(tmem, as + kk * 8, ptx::smem_desc(bb + kk * 32, 16, 512, 4), idesc, (kb | kk) ? 1u : 0u);
            for (int kk = 0; kk < 2; ++kk) ptx::mma_tf32_ts(tmem, ab + kk * 8, ptx::smem_desc(bs + kk * 32, 16, 512, 4), idesc, 1u);
            for (int kk = 0; kk < 2; ++kk) ptx::mma_tf32_ts(tmem, ab + kk * 8, ptx::smem_desc(bb + kk * 32, 16, 512, 4), idesc, 1u);
            if (mode == 3) {
                for (int r = 0; r < csize; ++r) {  // free the stage in every CTA of the cluster
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                                 ::"r"(ptx::smem_u32(&empty[st])), "h"(uint16_t(1 << r)) : "memory");
                }
            } else {
                ptx::mma_commit(&empty[st]);
            }
            if (++st == STAGES) { st = 0; ph ^= 1; }
        }
        uint64_t fin;
        asm volatile("{}" ::: "memory");
        ptx::mma_commit(&full[0]);  // reuse: wait for completion via a fresh barrier-ish spin
        (void)fin;
        cyc[blockIdx.x] = clock64() - t0;
    }
    ptx::tc_fence_before();
    if (mode == 3) ptx::cluster_sync(); else __syncthreads();
    if (warp == 2) ptx::tmem_dealloc<512, 1>(tmem);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t per = size_t(2) * NP * KP;
    float* w;
    cudaMalloc(&w, per * sms * 4);
    std::vector<float> h(per * sms, 0.01f);
    cudaMemcpy(w, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    long long* cyc;
    cudaMalloc(&cyc, sms * 8);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[2] = {KP, cuuint64_t(2 * NP * sms)};
    cuuint64_t str[1] = {KP * 4};
    cuuint32_t box[2] = {16, NP}, es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = STAGES * 2 * BB + 1024 + 512;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int kb = 8000;
    for (int mode : {0, 1, 2, 3}) {
        for (int cs : {2, 4}) {
            if (mode != 3 && cs == 4) continue;
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(mode == 3 ? sms / cs * cs : sms);
            cfg.blockDim = dim3(128);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = mode == 3 ? cs : 1;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            cudaError_t e = cudaLaunchKernelEx(&cfg, probe, tm, cyc, kb, mode, cs);
            cudaEventRecord(e1);
            cudaError_t e2 = cudaDeviceSynchronize();
            float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
            std::vector<long long> c(sms);
            cudaMemcpy(c.data(), cyc, sms * 8, cudaMemcpyDeviceToHost);
            long long mx = 0; for (auto v : c) mx = v > mx ? v : mx;
            printf("mode %d csize %d: %.1f issue-cycles/kblock (max over CTAs), %.1f us total -> %.1f ns/kblock  %s %s\n",
                   mode, mode == 3 ? cs : 1, double(mx) / kb, ms * 1e3, ms * 1e6 / kb, cudaGetErrorString(e), cudaGetErrorString(e2));
        }
    }
    return 0;
}
