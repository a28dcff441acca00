// dgrad.cu -- fused backward-data of small-channel strided Type 1 layers (see dgrad.cuh).
//
// GEMM (per tile = 4 x (32 - (NF - 1)) consecutive output pixels of the flattened (image, row,
// column) order; TMEM lane quadrant w holds pixels [P0 + w (32 - (NF - 1)) - (NF - 1), + 32), so
// its first NF - 1 lanes repeat the previous quadrant's last pixels -- the horizontal fold then
// needs only warp shuffles -- and do not store):
//   D (pixels x lowered columns of a filter-row group) = dy tile (pixels x o) * Khat^T group,
//   3xTF32 on tcgen05 (A_small B_big + A_big B_small + A_big B_big), fp32 accumulate in TMEM.
// The lowered columns of filter row i sit at [i KDP, i KDP + k d) of its group (KDP = k d
// rounded to 4); groups of filter rows keep N <= 256 and two accumulator buffers in TMEM.
// The group's Khat^T (both halves, all o) stays resident in shared memory while the CTA walks
// its tiles; the raw dy tiles stream through a 6-deep TMA ring (DRAM latency) and the transform
// warps put their big / small halves into TMEM, where the MMA reads its A operand.
//   warp 0        TMA producer (elected lane): group bank [bbar / bempty], raw dy k-blocks [afull / aempty]
//   warp 1        MMA issuer (elected lane of a warp-uniform loop)
//   warp 2        TMEM allocator
//   warps 4-7,    epilogue, two halves (filter rows il = half mod 2 of the group): per filter row,
//   12-15         tcgen05.ld of the row's k d columns (the next row's load in flight), horizontal
//                 fold (warp shuffles; the two pixels before lane 0 through shared memory), stores
//                 of the pixel's own s d floats of H[q][r][i][:] (float4), the tail at a row's end
//   warps 8-11    dy transform: raw tile row (thread = pixel) -> big | small -> TMEM A slot [sfull / sempty]
// Then vfold_kernel: dx[q][y][x] = sum over (r, i) with s r + i = y + p of H[q][r][i][x + p d].
#include <cudaTypedefs.h>

#include <algorithm>

#include "common.cuh"
#include "dgrad.cuh"
#include "ptx.cuh"

namespace cct {
namespace hf {

constexpr int kTileM = 128;
constexpr int kKB = 16;
constexpr int kThreads = 512;
constexpr int kRA = 6;                // dy k-block ring (raw tiles in smem; deep enough for DRAM latency)
constexpr int kSmemMax = 227 * 1024;
constexpr int kMaxGroups = 4;
constexpr uint32_t kABytes = kTileM * kKB * 4;  // one raw dy k-block (128 pixels x 16 channels)

struct Params {
    float* H;                   // [q][r][i][XP]
    int b, m, k, o, XP;
    int ov, wpix, npix, tiles;  // repeated lanes per quadrant (NF - 1), new pixels per quadrant, pixels, tiles
    int ngroups, fr, kb;        // filter-row groups, rows per group, k-blocks over o
    int nmax;                   // B rows reserved per (k-block, half) in smem
    int npad[kMaxGroups];       // N of each group (multiple of 32)
    int brow0[kMaxGroups];      // first prepared-bank row of each group ([big | small] rows)
    int dbg;                    // 0 in the product; tools/hfold_probe.cu drops stages to find the bound
};

struct Layout {
    uint32_t b, a, bars, total;
};
__host__ __device__ inline Layout layout(int nmax, int kb) {
    Layout L;
    L.b = 0;
    L.a = uint32_t(kb) * 2u * uint32_t(nmax) * 64u;
    L.bars = L.a + kRA * kABytes;
    L.total = L.bars + uint32_t(2 * kRA + 4 + 4 + 4) * 8u + 16u;
    return L;
}
// TMEM A slots (big | small halves of one dy k-block) after the two accumulator buffers
__host__ __device__ inline int a_slots(int nmax) { return std::min(4, (512 - 2 * nmax) / 32); }

template <int KD, int SD>
__global__ void __launch_bounds__(kThreads, 1)
    conv_dgrad_hfold_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                            const Params p) {
    constexpr int KDP = (KD + 3) & ~3;
    constexpr int NF = (KD + SD - 1) / SD;  // pixels meeting in one float
    static_assert(NF >= 1 && NF <= 3 && KDP <= 36 && SD % 4 == 0, "fold geometry");
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const Layout L = layout(p.nmax, p.kb);
    // afull / aempty: raw dy stage (TMA bytes / the transform has read it); sfull / sempty: TMEM
    // A slot (transform wrote big | small / MMA commit); bbar / bempty: group bank; tfull / tempty
    uint64_t* afull = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* aempty = afull + kRA;
    uint64_t* sfull = aempty + kRA;
    uint64_t* sempty = sfull + 4;
    uint64_t* bbar = sempty + 4;
    uint64_t* bempty = bbar + 1;
    uint64_t* tfull = bempty + 1;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    const int RS = a_slots(p.nmax);
    const uint32_t A_COL = uint32_t(2 * p.nmax);

    const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
        for (int s = 0; s < kRA; ++s) {
            ptx::mbar_init(&afull[s], 1);
            ptx::mbar_init(&aempty[s], 4);
        }
        for (int s = 0; s < RS; ++s) {
            ptx::mbar_init(&sfull[s], 4);
            ptx::mbar_init(&sempty[s], 1);
        }
        ptx::mbar_init(bbar, 1);
        ptx::mbar_init(bempty, 1);
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], 8);  // both epilogue halves
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<512, 1>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int mm = p.m * p.m;
    const uint32_t bslot = uint32_t(p.nmax) * 64u;  // bytes of one (k-block, half) of the bank

    if (warp == 0) {
        // ===================== producer =====================
        int as = 0;
        uint32_t aph = 0;
        for (int g = 0; g < p.ngroups; ++g) {
            // the group's bank, once the previous group's MMAs are done with the region
            ptx::mbar_wait_sleep(bempty, (g & 1) ^ 1);
            if (ptx::elect_one()) {
                ptx::mbar_arrive_expect_tx(bbar, uint32_t(p.kb) * 2u * uint32_t(p.npad[g]) * 64u);
                for (int kb = 0; kb < p.kb; ++kb)
                    for (int h = 0; h < 2; ++h)
                        for (int r32 = 0; r32 < p.npad[g]; r32 += 32)
                            ptx::tma_load_2d(smem + L.b + (uint32_t(kb) * 2u + uint32_t(h)) * bslot + uint32_t(r32) * 64u,
                                             &tmB, bbar, kb * kKB, p.brow0[g] + h * p.npad[g] + r32);
            }
            __syncwarp();
            for (int T = blockIdx.x; T < p.tiles; T += gridDim.x) {
                const int pix = T * 4 * p.wpix - p.ov;  // may start before pixel 0: TMA zero-fills
                for (int kb = 0; kb < p.kb; ++kb) {
                    ptx::mbar_wait_sleep(&aempty[as], aph ^ 1);
                    if (ptx::elect_one()) {
                        ptx::mbar_arrive_expect_tx(&afull[as], kABytes);
#pragma unroll
                        for (int w = 0; w < 4; ++w)
                            ptx::tma_load_2d(smem + L.a + uint32_t(as) * kABytes + uint32_t(w) * (kABytes / 4), &tmA,
                                             &afull[as], kb * kKB, pix + w * p.wpix);
                    }
                    __syncwarp();
                    if (++as == kRA) { as = 0; aph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer: A (dy big | small) from TMEM, B resident in smem =====================
        const uint32_t b_u = ptx::smem_u32(smem + L.b);
        int ss = 0;
        uint32_t sph = 0;
        int lt = 0;
        for (int g = 0; g < p.ngroups; ++g) {
            const uint32_t idesc = ptx::idesc_tf32(kTileM, uint32_t(p.npad[g]), 0, 0);
            ptx::mbar_wait(bbar, g & 1);
            for (int T = blockIdx.x; T < p.tiles; T += gridDim.x, ++lt) {
                const int acc = lt & 1;
                ptx::mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
                ptx::tc_fence_after();
                const uint32_t d0 = tmem + uint32_t(acc * p.nmax);
                for (int kb = 0; kb < p.kb; ++kb) {
                    ptx::mbar_wait(&sfull[ss], sph);
                    ptx::tc_fence_after();
                    const uint32_t abig = tmem + A_COL + uint32_t(ss) * 32, asml = abig + kKB;
                    const uint32_t bbig = b_u + uint32_t(kb) * 2u * bslot, bsml = bbig + bslot;
                    if (ptx::elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < 2; ++kk) {
                            if (p.dbg & 4) break;
                            const uint64_t bb = ptx::smem_desc(bbig + kk * 32, 16, 512, 4);
                            const uint64_t bs = ptx::smem_desc(bsml + kk * 32, 16, 512, 4);
                            ptx::mma_tf32_ts(d0, asml + kk * 8, bb, idesc, (kb | kk) ? 1u : 0u);  // small products first
                            ptx::mma_tf32_ts(d0, abig + kk * 8, bs, idesc, 1u);
                            ptx::mma_tf32_ts(d0, abig + kk * 8, bb, idesc, 1u);
                        }
                        ptx::mma_commit(&sempty[ss]);
                    }
                    __syncwarp();
                    if (++ss == RS) { ss = 0; sph ^= 1; }
                }
                if (ptx::elect_one()) ptx::mma_commit(&tfull[acc]);
                __syncwarp();
            }
            // the bank region is free once this group's last MMAs completed
            if (ptx::elect_one()) ptx::mma_commit(bempty);
            __syncwarp();
        }
    } else if ((warp >= 4 && warp < 8) || warp >= 12) {
        // ===================== epilogue: horizontal fold into H =====================
        const int qd = warp & 3;
        const int half = warp >= 12 ? 1 : 0;  // filter rows il = half, half + 2, ...
        int lt = 0;
        for (int g = 0; g < p.ngroups; ++g) {
            const int i0 = g * p.fr, nrow = min(p.fr, p.k - i0);
            for (int T = blockIdx.x; T < p.tiles; T += gridDim.x, ++lt) {
                const int acc = lt & 1;
                const int P = T * 4 * p.wpix + qd * p.wpix + lane - p.ov;  // this lane's pixel
                const int q = P / mm, rr = P - q * mm, r = rr / p.m, cc = rr - r * p.m;
                const bool ok = lane >= p.ov && P < p.npix;
                ptx::mbar_wait_sleep(&tfull[acc], (lt >> 1) & 1);
                ptx::tc_fence_after();
                if (p.dbg & 1) {
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
                    continue;
                }
                const uint32_t tc0 = tmem + (uint32_t(qd * 32) << 16) + uint32_t(acc * p.nmax);
                uint32_t u[32], t4[4];
                if (half < nrow) {
                    ptx::tmem_ld_32x32b_x32(tc0 + uint32_t(half * KDP), u);
                    if constexpr (KDP > 32) ptx::tmem_ld_32x32b_x4(tc0 + uint32_t(half * KDP + 32), t4);
                }
                for (int il = half; il < nrow; il += 2) {
                    ptx::tmem_ld_wait();
                    if (p.dbg & 8) {
                        if (il + 2 < nrow) {
                            ptx::tmem_ld_32x32b_x32(tc0 + uint32_t((il + 2) * KDP), u);
                            if constexpr (KDP > 32) ptx::tmem_ld_32x32b_x4(tc0 + uint32_t((il + 2) * KDP + 32), t4);
                        }
                        continue;
                    }
                    float v[KDP];
#pragma unroll
                    for (int e = 0; e < KDP; ++e) v[e] = __uint_as_float(e < 32 ? u[e] : t4[e - 32]);
                    if (il + 2 < nrow) {  // next row of this half in flight while this one is folded
                        ptx::tmem_ld_32x32b_x32(tc0 + uint32_t((il + 2) * KDP), u);
                        if constexpr (KDP > 32) ptx::tmem_ld_32x32b_x4(tc0 + uint32_t((il + 2) * KDP + 32), t4);
                    }
                    float out[KD];
#pragma unroll
                    for (int e = 0; e < KD; ++e) out[e] = v[e];
#pragma unroll
                    for (int f = 1; f < NF; ++f) {
#pragma unroll
                        for (int e = 0; e + f * SD < KD; ++e) {
                            // lanes < f read garbage: they are repeated lanes (lane < ov), not stored
                            const float pv = __shfl_up_sync(0xffffffffu, v[e + f * SD], f);
                            out[e] += cc >= f ? pv : 0.f;
                        }
                    }
                    if (ok && !(p.dbg & 16)) {
                        float* hrow = p.H + (int64_t(q * p.m + r) * p.k + (i0 + il)) * p.XP + SD * cc;
#pragma unroll
                        for (int e = 0; e < SD; e += 4)
                            *reinterpret_cast<float4*>(hrow + e) = make_float4(out[e], out[e + 1], out[e + 2], out[e + 3]);
                        if (cc == p.m - 1) {
#pragma unroll
                            for (int e = SD; e < KD; ++e) hrow[e] = out[e];
                        }
                    }
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
            }
        }
    } else if (warp >= 8 && warp < 12) {
        // ===================== dy transform: raw smem tile -> big | small in a TMEM A slot =====================
        const uint32_t a_u = ptx::smem_u32(smem + L.a);
        const int r = (warp & 3) * 32 + lane;  // this thread's pixel row of the tile (its TMEM lane)
        int as = 0, ss = 0;
        uint32_t aph = 0, sph = 0;
        for (int g = 0; g < p.ngroups; ++g)
            for (int T = blockIdx.x; T < p.tiles; T += gridDim.x)
                for (int kb = 0; kb < p.kb; ++kb) {
                    ptx::mbar_wait_sleep(&afull[as], aph);
                    if (p.dbg & 2) {
                        ptx::mbar_wait(&sempty[ss], sph ^ 1);
                        __syncwarp();
                        if (lane == 0) {
                            ptx::mbar_arrive(&sfull[ss]);
                            ptx::mbar_arrive(&aempty[as]);
                        }
                        if (++as == kRA) { as = 0; aph ^= 1; }
                        if (++ss == RS) { ss = 0; sph ^= 1; }
                        continue;
                    }
                    const uint32_t raw = a_u + uint32_t(as) * kABytes;
                    // row r of the K-major SWIZZLE_64B tile: 16-byte chunk c at (c ^ (r / 2 % 4))
                    float4 x[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c) x[c] = ptx::lds128(raw + uint32_t(r) * 64u + uint32_t((c ^ ((r >> 1) & 3)) << 4));
                    uint32_t v[32];
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const float f[4] = {x[c].x, x[c].y, x[c].z, x[c].w};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const uint32_t big = __float_as_uint(f[u]) & 0xFFFFE000u;
                            v[4 * c + u] = big;
                            v[kKB + 4 * c + u] = __float_as_uint(f[u] - __uint_as_float(big));
                        }
                    }
                    ptx::mbar_wait(&sempty[ss], sph ^ 1);
                    ptx::tc_fence_after();
                    ptx::tmem_st_32x32b_x32(tmem + (uint32_t((warp & 3) * 32) << 16) + A_COL + uint32_t(ss) * 32, v);
                    ptx::tmem_st_wait();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        ptx::mbar_arrive(&sfull[ss]);
                        // the raw stage is released only here: an arrive right after the ld.shared
                        // (before the TMEM store) corrupted tiles at b >= 8 (measured, tools/hfold_diag.py)
                        ptx::mbar_arrive(&aempty[as]);
                    }
                    if (++as == kRA) { as = 0; aph ^= 1; }
                    if (++ss == RS) { ss = 0; sph ^= 1; }
                }
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512, 1>(tmem);
    }
}

// dx[q][y][x] = sum_{r: 0 <= y + p - s r < k, 0 <= r < m} H[q][r][y + p - s r][x + p d]  (r ascending)
// (H columns >= XW, the padded input columns no filter window reaches, are zero).  One block per
// dx row (blockIdx.x = q n + y: no per-element divisions), a thread per 4 columns: the <= NF
// (= ceil(k / s) <= 3) H rows' float4 loads issued together, then the sum in r order.
__global__ void vfold_kernel(const float* __restrict__ H, float* __restrict__ dx, int n, int d, int k, int s, int p,
                             int m, int XP, int XW) {
    const int row = blockIdx.x, q = row / n, y = row - q * n;
    const int nd = n * d, yp = y + p;
    const int rlo = max(0, (yp - k + s) / s), rhi = min(m - 1, yp / s);
    for (int x = int(threadIdx.x) * 4; x < nd; x += int(blockDim.x) * 4) {
        const int xp = x + p * d;
        float4 h[3];
    #pragma unroll
        for (int j = 0; j < 3; ++j) {
            h[j] = make_float4(0.f, 0.f, 0.f, 0.f);
            const int r = rlo + j;
            if (r <= rhi && xp < XW) {
                const float* hp = H + (int64_t(q * m + r) * k + (yp - s * r)) * XP + xp;
                if (((p * d) & 3) == 0) {
                    h[j] = __ldg(reinterpret_cast<const float4*>(hp));
                } else {  // unaligned padded column offset (row pitch XP >= XW + 3 keeps hp[3] in bounds)
                    h[j] = make_float4(__ldg(hp), __ldg(hp + 1), __ldg(hp + 2), __ldg(hp + 3));
                }
            }
        }
        const float av[4] = {(h[0].x + h[1].x) + h[2].x, (h[0].y + h[1].y) + h[2].y, (h[0].z + h[1].z) + h[2].z,
                             (h[0].w + h[1].w) + h[2].w};
        float* o = dx + int64_t(row) * nd + x;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (x + u < nd) o[u] = xp + u < XW ? av[u] : 0.f;
    }
}

// Khat^T groups: rows [brow0_g, +npad_g) = big, [+npad_g, +2 npad_g) = small; row lr of a group
// half = (filter row i0 + lr / KDP, run element lr % KDP); columns = o (K, zero-padded to kp)
__global__ void prep_hfold_bank_kernel(const float* __restrict__ w, float* __restrict__ bp, int rows, int kp, int o,
                                       int k, int kd, int kdp, int fr, Params gp) {
    const int64_t total = int64_t(rows) * kp;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int row = int(idx / kp), oc = int(idx - int64_t(row) * kp);
        int g = 0;
        while (g + 1 < gp.ngroups && row >= gp.brow0[g + 1]) ++g;
        const int hr = row - gp.brow0[g];
        const bool small = hr >= gp.npad[g];
        const int lr = small ? hr - gp.npad[g] : hr;
        const int il = lr / kdp, e = lr - il * kdp, i = g * fr + il;
        float v = 0.f;
        if (il < fr && i < k && e < kd && oc < o) {
            v = w[(int64_t(oc) * k + i) * kd + e];
            if (small) v -= __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
        }
        bp[idx] = v;
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult qr;
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qr) == cudaSuccess &&
            qr == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

// K-major 2D map (rows x cols fp32, row stride ld floats): box 16 columns x box_rows rows, SWIZZLE_64B
bool kmajor_map(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
    auto enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(ld) * 4};
    cuuint32_t box[2] = {cuuint32_t(kKB), cuuint32_t(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct Plan {
    Params p{};
    int kdp = 0, kp = 0, rows = 0, grid = 0;
    uint32_t smem = 0;
    bool ok = false;
};

int g_probe_dbg = 0;  // Params::dbg of every launch (set only by tools/hfold_probe.cu)

Plan plan(const Geo& g) {
    Plan P;
    const int64_t kd = g.k * g.d, sd = g.s * g.d;
    // instantiated fold geometries (k d, s d): CaffeNet / AlexNet conv1 (33, 12), test shapes
    const bool geo_ok = (kd == 33 && sd == 12) || (kd == 20 && sd == 8) || (kd == 28 && sd == 16);
    if (!geo_ok || g.m < 2 || g.o < 1 || g.o > 96 || g.o % 4 != 0 || g.k > 32) return P;
    if (g.b * g.m * g.m >= (int64_t(1) << 31) - kTileM || g.b * g.n * g.n * g.d >= (int64_t(1) << 40)) return P;
    P.kdp = int((kd + 3) & ~int64_t(3));
    Params& p = P.p;
    p.b = int(g.b); p.m = int(g.m); p.k = int(g.k); p.o = int(g.o);
    p.XP = int((sd * (g.m - 1) + kd + 3 + 3) & ~int64_t(3));  // >= XW + 3: vfold's 4-float reads
    p.ov = int((kd + sd - 1) / sd) - 1;
    p.wpix = 32 - p.ov;
    p.npix = int(g.b * g.m * g.m);
    p.tiles = (p.npix + 4 * p.wpix - 1) / (4 * p.wpix);
    p.kb = (p.o + kKB - 1) / kKB;
    P.kp = p.kb * kKB;
    // filter-row groups: N = rows x KDP <= 256 (multiple of 32), balanced
    const int maxfr = 256 / P.kdp;
    p.ngroups = (p.k + maxfr - 1) / maxfr;
    if (p.ngroups > kMaxGroups) return P;
    p.fr = (p.k + p.ngroups - 1) / p.ngroups;
    p.nmax = 0;
    int row = 0;
    for (int gi = 0; gi < p.ngroups; ++gi) {
        const int nrow = std::min(p.fr, p.k - gi * p.fr);
        p.npad[gi] = (nrow * P.kdp + 31) / 32 * 32;
        p.brow0[gi] = row;
        row += 2 * p.npad[gi];
        p.nmax = std::max(p.nmax, p.npad[gi]);
    }
    if (a_slots(p.nmax) < 2) return P;
    P.rows = row;
    const Layout L = layout(p.nmax, p.kb);
    if (L.total + 1024 > uint32_t(kSmemMax)) return P;
    P.smem = L.total + 1024;
    P.grid = std::min(num_sms(), p.tiles);
    P.ok = true;
    return P;
}

}  // namespace hf

using namespace hf;

bool hfold_dgrad_ok(const Geo& g) { return hf::plan(g).ok; }

int64_t hfold_dgrad_ws_floats(const Geo& g) {
    const Plan P = hf::plan(g);
    if (!P.ok) return 0;
    const int64_t h = int64_t(P.p.b) * P.p.m * P.p.k * P.p.XP;
    const int64_t nhwc = g.yl ? 0 : (g.b * g.m * g.m * g.o + 3) / 4 * 4;
    return h + int64_t(P.rows) * P.kp + nhwc;
}

cudaError_t hfold_dgrad(const Geo& g, const float* dy, const float* w, float* dx, float* ws, cudaStream_t st,
                        cudaEvent_t gemm_done) {
    Plan P = hf::plan(g);
    if (!P.ok) return cudaErrorInvalidValue;
    Params& p = P.p;
    p.dbg = g_probe_dbg;
    const int64_t mm = g.m * g.m;
    float* H = ws;
    float* bp = H + int64_t(p.b) * p.m * p.k * p.XP;
    const float* dyn = dy;
    if (!g.yl) {  // NCHW dy -> NHWC (pixels x o): the K-major A operand
        float* t = bp + int64_t(P.rows) * P.kp;
        cudaError_t e = transpose_batched(dy, g.o, mm, mm, g.o * mm, t, g.o, mm * g.o, g.b, kPhaseExpand, st);
        if (e != cudaSuccess) return e;
        dyn = t;
    }
    p.H = H;
    {
        const int64_t total = int64_t(P.rows) * P.kp;
        prep_hfold_bank_kernel<<<grid_for(total, 256), 256, 0, st>>>(w, bp, P.rows, P.kp, p.o, p.k, int(g.k * g.d),
                                                                     P.kdp, p.fr, p);
        note_launch();
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    CUtensorMap ta, tb;
    if (!kmajor_map(&ta, dyn, g.b * mm, g.o, g.o, 32) || !kmajor_map(&tb, bp, P.rows, P.kp, P.kp, 32))
        return cudaErrorInvalidValue;
    {
        PhaseScope ps(kPhaseGemm, st, 2.0 * double(g.b) * double(mm) * double(g.k * g.k * g.d) * double(g.o), 0);
        cudaError_t e = cudaSuccess;
        auto go = [&](auto kern) {
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(P.smem));
            if (e == cudaSuccess) {
                kern<<<P.grid, kThreads, P.smem, st>>>(ta, tb, p);
                note_launch();
                e = cudaGetLastError();
            }
        };
        const int64_t kd = g.k * g.d, sd = g.s * g.d;
        if (kd == 33 && sd == 12) go(conv_dgrad_hfold_kernel<33, 12>);
        else if (kd == 20 && sd == 8) go(conv_dgrad_hfold_kernel<20, 8>);
        else go(conv_dgrad_hfold_kernel<28, 16>);
        if (e != cudaSuccess) return e;
    }
    if (gemm_done) {
        cudaError_t e = cudaEventRecord(gemm_done, st);
        if (e != cudaSuccess) return e;
    }
    {
        PhaseScope ps(kPhaseCol2im, st, 0, 4.0 * (double(p.b) * p.m * p.k * p.XP + double(g.b) * g.n * g.n * g.d));
        const int rows = int(g.b * g.n);
        const int xw = int(g.s * g.d * (g.m - 1) + g.k * g.d);
        // the fold may run beside a persistent max-shared-memory kernel: keep the SM's carve-out there
        static const cudaError_t carve =
            cudaFuncSetAttribute(vfold_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        (void)carve;
        const int threads = int(std::min<int64_t>(1024, (g.n * g.d + 127) / 128 * 32));
        vfold_kernel<<<rows, threads, 0, st>>>(H, dx, int(g.n), int(g.d), int(g.k), int(g.s), int(g.p), p.m, p.XP, xw);
        note_launch();
    }
    return cudaGetLastError();
}

}  // namespace cct
