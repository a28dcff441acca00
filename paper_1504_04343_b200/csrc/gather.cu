// gather.cu -- fused small-channel Type 1 convolution: forward and backward-weight
// without a materialised Dhat (see gather.cuh).
//
// Forward, one CTA per SM, persistent over 128-pixel tiles (a tile never crosses an
// image), 768 threads:
//   warp 0        TMA producer (elected lane): kernel-bank k-blocks ([small | big] halves,
//                 prepared once per call) -> smem ring stage  [bfull / bempty]
//   warp 1        MMA issuer (elected lane of a warp-uniform loop): per 16-wide k-block 4
//                 (NP <= 96, merged N = 2 NP product, see FwdCfg) or 6 tcgen05.mma.kind::tf32,
//                 A (the k-block of Dhat) from TMEM, B from smem
//   warp 2        TMEM allocator, then the staging producer (one lane): the input rows a
//                 tile touches -> a double-buffered row stage (1D bulk copies)  [xfull / xempty]
//   warps 4-7     epilogue: tcgen05.ld -> y (NCHW: lanes = consecutive pixels, coalesced)
//   warps 8-23    four gather groups (k-block gi -> group gi % 4): 128 pixels x 16 lowered columns
//                 from the staged rows -> big / small -> tcgen05.st into TMEM A slot  [afull / aempty]
// The bank ring (smem-sized) and the A slot ring (TMEM-sized) are independent; the MMA issuer
// waits one barrier of each per k-block and commits both.
// Lowered column order (this kernel's own; the kernel bank is repacked to match): filter
// row i owns the window of columns [i segw, (i + 1) segw), its k d run placed at the shift
// that makes every 4-column group of a k-block one aligned float4 of a staged row (the
// float4 phase of an image's rows is uniform over the image since s d % 4 == 0): one
// ld.shared.v4 per 4 lowered elements, no realignment (see variant_of).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>

#include "cct.h"
#include "common.cuh"
#include "gather.cuh"
#include "ptx.cuh"
#include "reduce.cuh"

// A/B builds (tools/build_variant.sh) override this default; the product is built with the measured best
#ifndef CCT_FWD_PACE_NS
#define CCT_FWD_PACE_NS 600
#endif
#ifndef CCT_FWD_MAX_STAGES  // kernel-bank ring depth cap of the forward (A/B diagnostics)
#define CCT_FWD_MAX_STAGES 12
#endif

namespace cct {
namespace gth {

constexpr int kGatherGroups = 4;            // gather groups of 4 warps, k-block gi -> group gi % 4
constexpr int kThreads = 256 + 128 * kGatherGroups;
constexpr int kTileM = 128;
constexpr int kKB = 16;                   // k-block width (fp32 columns)
constexpr int kSmemMax = 227 * 1024;      // opt-in dynamic shared memory per CTA
constexpr int kMaxKGroups = 512;          // k-block groups of 4 columns in the table (K <= 2048)

struct FwdParams {
    const float* x;
    float* y;
    const float* bias;
    int64_t y_sq, y_so, y_sp;  // y offset of (image q, channel o, pixel P)
    int64_t x_total;           // floats in x (multiple of 4)
    int b, n, d, k, s, p, m, o;
    int seg, segw, kb_tile;    // lowered run per filter row, its window width, k-blocks per tile
    int nvar;                  // kernel-bank variants (float4 phase of the image's rows, 1 or 4)
    int tpi, tpx, tiles;       // tiles per image, pixels per tile, total tiles
    int xb;                    // row-stage buffers
    int pitch, lmargin;        // staged row slot: floats, and floats before the row data
    int xr;                    // row slots per stage buffer
    int stages;                // kernel-bank ring depth (smem)
    int aslots;                // A slot ring depth (TMEM)
    int relu;
    int dbg;                   // 0 in the product; tools/gather_probe.cu drops stages to find the bound
    unsigned long long* trace; // null in the product; tools/gather_probe.cu: CTA 0 event clocks
    int pace_ns;               // epilogue pause between 32-column TMEM chunks
};

// MERGE (NP <= 96): the two products that share A_big run as ONE N = 2 NP MMA over the
// stage's [small | big] bank rows into two accumulator halves, D[0, NP) = A_big B_small and
// D[NP, 2 NP) = A_big B_big + A_small B_big, summed by the epilogue: 4 MMAs per k-block
// instead of 6 (measured, tools/mma_rate.cu: an M = 128, K = 8 tf32 MMA costs ~77 cycles
// at any N <= 128 and ~103 at N = 192).
template <int NP, bool MG>
struct FwdCfg {
    static constexpr bool MERGE = MG && NP <= 96;
    static constexpr int ACC_COLS = MERGE ? 2 * NP : NP;               // one accumulator buffer
    static constexpr int A_COL = 2 * ACC_COLS;                         // double-buffered accumulators first
    static constexpr uint32_t B_BYTES = NP * kKB * 4;                 // one half of a ring stage
    static_assert(NP % 16 == 0 && NP <= 192, "tile width");
};
__host__ __device__ constexpr int acc_cols(int np, bool mg) { return (mg && np <= 96) ? 2 * np : np; }
__host__ __device__ constexpr int max_aslots(int np, bool mg) {
    return (512 - 2 * acc_cols(np, mg)) / 32 > 8 ? 8 : (512 - 2 * acc_cols(np, mg)) / 32;
}

// dynamic smem layout (bytes): [ring stages][row stage x2][zero row][k tables][barriers]
struct FwdLayout {
    uint32_t ring, stage, zero, ktab, bars, total;
};
__host__ __device__ inline FwdLayout fwd_layout(int np, int stages, int aslots, int xr, int pitch, int kgroups,
                                                int xb) {
    FwdLayout L;
    L.ring = 0;
    L.stage = uint32_t(stages) * 2u * uint32_t(np) * kKB * 4u;
    L.zero = L.stage + uint32_t(xb) * uint32_t(xr) * uint32_t(pitch) * 4u;
    L.ktab = L.zero + uint32_t(pitch) * 4u;
    L.bars = (L.ktab + 2u * 4u * uint32_t(kgroups) * 4u + 15u) & ~15u;  // ktab + etab, 4 variants
    L.total = L.bars + uint32_t(2 * stages + 2 * aslots + 2 * xb + 4) * 8u + 16u;
    return L;
}

// Rows of image q start at float offset q n n d + y n d: their float4 phase is the same for
// every output row of an image (s d % 4 == 0), (q n n d + (i - p) n d) mod 4 for filter row i.
// The kernel bank is prepared in one variant per phase q n n d mod 4, each filter row's run
// shifted inside its window so that every 4-column group is an aligned float4 of the stage.
__host__ __device__ inline int variant_of(const FwdParams& p, int q) {
    return p.nvar == 1 ? 0 : int((int64_t(q) * p.n * p.n * p.d) & 3);
}
// shift of filter row i's run inside its window, for variant phi
__host__ __device__ inline int run_shift(int phi, int i, int n, int d, int pad) {
    const int64_t delta = (int64_t(phi) + int64_t(i - pad) * n * d) & 3;  // row phase
    return int((delta - int64_t(pad) * d) & 3);
}

struct TileGeo {
    int q, P0, P1, ra, y0, nrows;
};
__device__ __forceinline__ TileGeo tile_geo(const FwdParams& p, int T) {
    TileGeo t;
    t.q = T / p.tpi;
    t.P0 = (T - t.q * p.tpi) * p.tpx;
    t.P1 = min(t.P0 + p.tpx, p.m * p.m);
    t.ra = t.P0 / p.m;
    const int rb = (t.P1 - 1) / p.m;
    t.y0 = p.s * t.ra - p.p;
    t.nrows = p.s * (rb - t.ra) + p.k;
    return t;
}

template <int NP, bool MG>
__global__ void __launch_bounds__(kThreads, 1)
    conv_fwd_gather_kernel(const __grid_constant__ CUtensorMap tmB, const FwdParams p) {
    using C_ = FwdCfg<NP, MG>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int ngroups_k = p.kb_tile * 4;
    const int RB = p.stages, RA = p.aslots;  // kernel-bank ring (smem), A slot ring (TMEM)
    const FwdLayout L = fwd_layout(NP, RB, RA, p.xr, p.pitch, ngroups_k, p.xb);
    float* zero_row = reinterpret_cast<float*>(smem + L.zero);
    int* ktab = reinterpret_cast<int*>(smem + L.ktab);   // [variant][group]: row | zero mask | byte offset
    int* etab = ktab + 4 * ngroups_k;                      // [variant][group]: run element of the group's column 0
    // bfull / bempty: kernel-bank stage (TMA bytes / MMA commit); afull / aempty: A slot
    // (the 4 gather warps of the k-block / MMA commit)
    uint64_t* bfull = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* bempty = bfull + RB;
    uint64_t* afull = bempty + RB;
    uint64_t* aempty = afull + RA;
    uint64_t* xfull = aempty + RA;
    uint64_t* xempty = xfull + p.xb;
    uint64_t* tfull = xempty + p.xb;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const bool spin = (p.dbg & 64) != 0;
    // probe trace: [role][tile][event] clock64 of CTA 0 (role 0 MMA, 1 gather group 0, 2 epilogue,
    // 3 row producer, 4 bank producer)
    unsigned long long* const trc = (p.trace && blockIdx.x == 0) ? p.trace : nullptr;
#define FTR(role, lt, ev) \
    do { if (trc && lane == 0 && (lt) < 64) trc[(size_t(role) * 64 + (lt)) * 32 + (ev)] = clock64(); } while (0)
    auto fwait = [spin](uint64_t* bar, uint32_t par) {
        if (spin) ptx::mbar_wait(bar, par);
        else ptx::mbar_wait_sleep(bar, par);
    };
    // zero the stage buffers (their margins are never written by the row copies) and the
    // zero row; build the k-block tables: group g of k-block kb -> (filter row, offset)
    {
        float4* z = reinterpret_cast<float4*>(smem + L.stage);
        const int n4 = int((L.ktab - L.stage) / 16);
        for (int i = threadIdx.x; i < n4; i += kThreads) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int idx = threadIdx.x; idx < p.nvar * ngroups_k; idx += kThreads) {
            const int phi = idx / ngroups_k, gx = idx - phi * ngroups_k;
            const int kc = gx * 4;
            int i = kc / p.segw;
            const int u0 = kc - i * p.segw;  // window column of the group's first element
            int zmask = 0xF, boff = 0, e0 = 0;
            if (i < p.k) {
                const int sh = run_shift(phi, i, p.n, p.d, p.p);
                const int delta = int((int64_t(phi) + int64_t(i - p.p) * p.n * p.d) & 3);
                e0 = u0 - sh;
                zmask = 0;
                for (int u = 0; u < 4; ++u)
                    if (e0 + u < 0 || e0 + u >= p.seg) zmask |= 1 << u;
                boff = 4 * (p.lmargin + delta + e0);  // + 4 * col0 * d (per pixel) + the row slot
            } else {
                i = p.k;  // K padding: reads (and masks) the zero row, at an aligned offset
                boff = 4 * (p.lmargin + ((p.p * p.d) & 3));
            }
            ktab[idx] = i | (zmask << 8) | (boff << 16);
            etab[idx] = e0;
        }
    }
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmB);
        for (int s = 0; s < RB; ++s) {
            ptx::mbar_init(&bfull[s], 1);
            ptx::mbar_init(&bempty[s], 1);
        }
        for (int s = 0; s < RA; ++s) {
            ptx::mbar_init(&afull[s], 4);
            ptx::mbar_init(&aempty[s], 1);
        }
        for (int a = 0; a < p.xb; ++a) {
            ptx::mbar_init(&xfull[a], 1);
            ptx::mbar_init(&xempty[a], 4 * kGatherGroups);  // every gather warp
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], 4);  // epilogue warps
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<512, 1>(tmem_slot);
    ptx::fence_proxy_async_smem();  // zeroed stage buffers -> later bulk-copy writes are ordered after
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int nd = p.n * p.d;

    if (warp == 0) {
        // ===================== kernel-bank producer (warp-uniform loop, elected issue) =====================
        {
            int st = 0, lbt = 0;
            uint32_t ph = 0;
            for (int T = blockIdx.x; T < p.tiles; T += gridDim.x, ++lbt) {
                const int row0 = variant_of(p, T / p.tpi) * 2 * p.o;  // this image's bank variant
                for (int kb = 0; kb < p.kb_tile; ++kb) {
                    fwait(&bempty[st], ph ^ 1);
                    FTR(4, lbt, 1 + kb);
                    if (ptx::elect_one()) {
                        if (p.dbg & 16) {
                            ptx::mbar_arrive(&bfull[st]);
                        } else {
                        ptx::mbar_arrive_expect_tx(&bfull[st], 2 * C_::B_BYTES);
                        uint8_t* dst = smem + L.ring + uint32_t(st) * 2 * C_::B_BYTES;
                        ptx::tma_load_2d(dst, &tmB, &bfull[st], kb * kKB, row0);                      // small
                        ptx::tma_load_2d(dst + C_::B_BYTES, &tmB, &bfull[st], kb * kKB, row0 + p.o);  // big
                        }
                    }
                    __syncwarp();
                    if (++st == RB) { st = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        // the whole warp runs the loop (warp-uniform operands), one elected lane issues
        {
            constexpr uint32_t idesc = ptx::idesc_tf32(kTileM, NP, 0, 0);
            constexpr uint32_t idesc2 = ptx::idesc_tf32(kTileM, C_::MERGE ? 2 * NP : NP, 0, 0);
            const uint32_t ring_u = ptx::smem_u32(smem + L.ring);
            int bs = 0, as = 0;
            uint32_t bph = 0, aph = 0;
            int lt = 0;
            for (int T = blockIdx.x; T < p.tiles; T += gridDim.x, ++lt) {
                const int acc = lt & 1;
                ptx::mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
                FTR(0, lt, 0);
                ptx::tc_fence_after();
                const uint32_t d0 = tmem + uint32_t(acc * C_::ACC_COLS);
                for (int kb = 0; kb < p.kb_tile; ++kb) {
                    ptx::mbar_wait(&bfull[bs], bph);
                    FTR(5, lt, 1 + kb);
                    ptx::mbar_wait(&afull[as], aph);
                    FTR(0, lt, 1 + kb);
                    ptx::tc_fence_after();
                    const uint32_t bsml = ring_u + uint32_t(bs) * 2 * C_::B_BYTES;  // [small | big] rows
                    const uint32_t bbig = bsml + C_::B_BYTES;
                    const uint32_t abig = tmem + uint32_t(C_::A_COL) + uint32_t(as) * 32, asml = abig + kKB;
                    const uint32_t first = kb ? 1u : 0u;
                    if (ptx::elect_one()) {
                        if (p.dbg & 4) {
                        } else if constexpr (C_::MERGE) {
#pragma unroll
                            for (int kk = 0; kk < 2; ++kk) {
                                // [A_big B_small | A_big B_big] (the first MMA of a tile clears both halves)
                                ptx::mma_tf32_ts(d0, abig + kk * 8, ptx::smem_desc(bsml + kk * 32, 16, 512, 4), idesc2,
                                                 kk ? 1u : first);
                                ptx::mma_tf32_ts(d0 + NP, asml + kk * 8, ptx::smem_desc(bbig + kk * 32, 16, 512, 4),
                                                 idesc, 1u);
                            }
                        } else {
                            // small products first, big * big last
#pragma unroll
                            for (int kk = 0; kk < 2; ++kk)
                                ptx::mma_tf32_ts(d0, asml + kk * 8, ptx::smem_desc(bbig + kk * 32, 16, 512, 4), idesc,
                                                 kk ? 1u : first);
#pragma unroll
                            for (int kk = 0; kk < 2; ++kk)
                                ptx::mma_tf32_ts(d0, abig + kk * 8, ptx::smem_desc(bsml + kk * 32, 16, 512, 4), idesc, 1u);
#pragma unroll
                            for (int kk = 0; kk < 2; ++kk)
                                ptx::mma_tf32_ts(d0, abig + kk * 8, ptx::smem_desc(bbig + kk * 32, 16, 512, 4), idesc, 1u);
                        }
                        if (p.dbg & 32) {  // probe: plain arrives instead of tcgen05.commit
                            ptx::mbar_arrive(&bempty[bs]);
                            ptx::mbar_arrive(&aempty[as]);
                        } else {
                            ptx::mma_commit(&bempty[bs]);
                            ptx::mma_commit(&aempty[as]);
                        }
                    }
                    __syncwarp();
                    if (++bs == RB) { bs = 0; bph ^= 1; }
                    if (++as == RA) { as = 0; aph ^= 1; }
                }
                FTR(0, lt, 30);
                if (ptx::elect_one()) ptx::mma_commit(&tfull[acc]);
                __syncwarp();
            }
        }
    } else if (warp == 2) {
        // ===================== row-stage producer =====================
        if (lane == 0) {
            int lt = 0;
            for (int T = blockIdx.x; T < p.tiles; T += gridDim.x, ++lt) {
                const int buf = lt % p.xb;
                fwait(&xempty[buf], ((lt / p.xb) & 1) ^ 1);
                FTR(3, lt, 0);
                const TileGeo tg = tile_geo(p, T);
                float* sb = reinterpret_cast<float*>(smem + L.stage) + int64_t(buf) * p.xr * p.pitch;
                uint32_t bytes = 0;
                // total bytes first (the barrier is armed before any copy is issued); the last
                // 1-3 floats of x (when its size is not a multiple of 4) are stored directly
                for (int rho = 0; rho < tg.nrows; ++rho) {
                    const int yy = tg.y0 + rho;
                    if (yy < 0 || yy >= p.n) continue;
                    const int64_t off = (int64_t(tg.q) * p.n + yy) * nd;
                    const int64_t a0 = off & ~int64_t(3);
                    int64_t nfl = ((off - a0) + nd + 3) & ~int64_t(3);
                    if (a0 + nfl > p.x_total) {
                        nfl = (p.x_total - a0) & ~int64_t(3);
                        for (int64_t u = a0 + nfl; u < p.x_total; ++u)
                            sb[int64_t(rho) * p.pitch + p.lmargin + (u - a0)] = __ldg(p.x + u);
                    }
                    bytes += uint32_t(nfl) * 4u;
                }
                if (p.dbg & 8) {
                    ptx::mbar_arrive(&xfull[buf]);
                    continue;
                }
                ptx::mbar_arrive_expect_tx(&xfull[buf], bytes);
                for (int rho = 0; rho < tg.nrows; ++rho) {
                    const int yy = tg.y0 + rho;
                    if (yy < 0 || yy >= p.n) continue;
                    const int64_t off = (int64_t(tg.q) * p.n + yy) * nd;
                    const int64_t a0 = off & ~int64_t(3);
                    int64_t nfl = ((off - a0) + nd + 3) & ~int64_t(3);
                    if (a0 + nfl > p.x_total) nfl = (p.x_total - a0) & ~int64_t(3);
                    if (nfl > 0)
                        ptx::bulk_load(sb + int64_t(rho) * p.pitch + p.lmargin, p.x + a0, uint32_t(nfl) * 4u, &xfull[buf]);
                }
                FTR(3, lt, 2);
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ===================== epilogue =====================
        const int t = (warp & 3) * 32 + lane;
        int lt = 0;
        for (int T = blockIdx.x; T < p.tiles; T += gridDim.x, ++lt) {
            const int acc = lt & 1;
            fwait(&tfull[acc], (lt >> 1) & 1);
            if (warp == 4) FTR(2, lt, 0);
            ptx::tc_fence_after();
            if (p.dbg & 1) {
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
                continue;
            }
            const TileGeo tg = tile_geo(p, T);
            const int P = tg.P0 + t;
            const bool ok = P < tg.P1;
            float* yrow = p.y + int64_t(tg.q) * p.y_sq + int64_t(P) * p.y_sp;
            const bool plain = !p.bias && !p.relu;
#pragma unroll 1
            for (int c0 = 0; c0 < NP; c0 += 32) {
                // paced accumulator reads: the MMAs read their A operand from TMEM too, and an
                // epilogue draining 2 x 96 columns at once stalled them for ~4k cycles per tile
                // (tools/gather_probe.cu trace); spread over the next tile's MMAs: -5 % (measured)
                if (c0 && p.pace_ns) __nanosleep(uint32_t(p.pace_ns));
                uint32_t v[32];
                const uint32_t tc = tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(acc * C_::ACC_COLS + c0);
                ptx::tmem_ld_32x32b_x32(tc, v);
                if constexpr (C_::MERGE) {
                    uint32_t v2[32];
                    ptx::tmem_ld_32x32b_x32(tc + NP, v2);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + __uint_as_float(v2[j]));
                }
                ptx::tmem_ld_wait();
                if (!ok) continue;
                const int nj = min(32, p.o - c0);  // channels of this chunk that exist (uniform)
                if (!plain) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        float f = __uint_as_float(v[j]);
                        if (p.bias && j < nj) f += __ldg(p.bias + c0 + j);
                        if (p.relu) f = fmaxf(f, 0.f);
                        v[j] = __float_as_uint(f);
                    }
                }
                float* yc = yrow + int64_t(c0) * p.y_so;
                if (nj == 32 && p.y_so == 1 && (reinterpret_cast<uintptr_t>(yc) & 15) == 0) {
                    // NHWC: 32 consecutive channels of this pixel
                    float4* y4 = reinterpret_cast<float4*>(yc);
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        y4[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                            __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
                } else if (nj == 32) {
                    // NCHW: lanes = consecutive pixels of one channel plane per store (coalesced)
                    const int so = int(p.y_so);
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        *yc = __uint_as_float(v[j]);
                        yc += so;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (j < nj) yc[int64_t(j) * p.y_so] = __uint_as_float(v[j]);
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (warp == 4) FTR(2, lt, 1);
            if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
        }
    } else if (warp >= 8) {
        // ===================== gather groups =====================
        const int grp = (warp - 8) >> 2;
        const int t = (warp & 3) * 32 + lane;
        const uint32_t zero_u = ptx::smem_u32(zero_row);
        const uint32_t stage_u = ptx::smem_u32(smem + L.stage);
        const uint32_t pitch_b = uint32_t(p.pitch) * 4u;
        // this group's k-blocks are gi = grp, grp + 4, ... (over all tiles): ring slot and
        // pass over the ring walked incrementally (no division by the runtime ring depth)
        uint32_t gbase = 0;  // gi of this tile's first k-block
        int sl = grp, pass = 0;
        while (sl >= RA) { sl -= RA; ++pass; }
        int lt = 0;
        for (int T = blockIdx.x; T < p.tiles; T += gridDim.x, ++lt) {
            const int buf = lt % p.xb;
            const TileGeo tg = tile_geo(p, T);
            const int P = min(tg.P0 + t, tg.P1 - 1);
            const int r = P / p.m, c = P - (P / p.m) * p.m;
            const int yr = p.s * r - p.p;  // input row of filter row 0
            const int col0 = p.s * c - p.p;  // input column of filter column 0
            const bool border = col0 < 0 || col0 + p.k > p.n;
            // filter rows whose input row exists (others read the zero row); k <= 32
            uint32_t rok = 0;
            for (int i = 0; i < p.k; ++i)
                if (unsigned(yr + i) < unsigned(p.n)) rok |= 1u << i;
            const uint32_t slot0 = stage_u + uint32_t(buf) * uint32_t(p.xr) * pitch_b + uint32_t(p.s * (r - tg.ra)) * pitch_b;
            const int tb = col0 * p.d * 4;  // byte offset of this pixel's run within a staged row
            const int* kt = ktab + variant_of(p, tg.q) * ngroups_k;
            if (warp == 8) FTR(1, lt, 0);
            fwait(&xfull[buf], (lt / p.xb) & 1);
            if (warp == 8) FTR(1, lt, 1);
            for (int kb = int((uint32_t(grp) - gbase) & (kGatherGroups - 1)); kb < p.kb_tile; kb += kGatherGroups) {
                // gather + split first; the slot is waited for only before the TMEM store
                // the k-block's 4 group entries (uniform): filter row | zero mask | byte offset of
                // the aligned float4; all four loads issued before any use (no branches between)
                if (p.dbg & 2) {
                    if (pass > 0) fwait(&aempty[sl], (pass - 1) & 1);
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&afull[sl]);
                    sl += kGatherGroups;
                    while (sl >= RA) { sl -= RA; ++pass; }
                    continue;
                }
                const int4 e4 = *reinterpret_cast<const int4*>(kt + kb * 4);
                const int ent[4] = {e4.x, e4.y, e4.z, e4.w};
                float4 f[4];
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const int i = ent[g] & 0xFF;
                    const uint32_t slot = ((rok >> i) & 1u) ? slot0 + uint32_t(i) * pitch_b : zero_u;
                    f[g] = ptx::lds128(uint32_t(int(slot) + tb + (ent[g] >> 16)));
                }
#pragma unroll
                for (int g = 0; g < 4; ++g) {  // window columns outside the filter row's k d run
                    const int zm = ent[g] >> 8;
                    f[g].x = (zm & 1) ? 0.f : f[g].x;
                    f[g].y = (zm & 2) ? 0.f : f[g].y;
                    f[g].z = (zm & 4) ? 0.f : f[g].z;
                    f[g].w = (zm & 8) ? 0.f : f[g].w;
                }
                if (border) {  // input columns outside [0, n): zero padding (edge pixels only)
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        const int e0 = etab[variant_of(p, tg.q) * ngroups_k + kb * 4 + g];
                        float fv[4] = {f[g].x, f[g].y, f[g].z, f[g].w};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int e = e0 + u;
                            const int xc = col0 + (e >= 0 ? e / p.d : -1);
                            if (xc < 0 || xc >= p.n) fv[u] = 0.f;
                        }
                        f[g] = make_float4(fv[0], fv[1], fv[2], fv[3]);
                    }
                }
                uint32_t v[32];
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const float fa[4] = {f[g].x, f[g].y, f[g].z, f[g].w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint32_t big = __float_as_uint(fa[u]) & 0xFFFFE000u;
                        v[4 * g + u] = big;
                        v[16 + 4 * g + u] = __float_as_uint(fa[u] - __uint_as_float(big));
                    }
                }
                if (warp == 8) FTR(1, lt, 2 + kb / kGatherGroups);
                if (pass > 0) fwait(&aempty[sl], (pass - 1) & 1);
                if (warp == 8) FTR(1, lt, 10 + kb / kGatherGroups);
                ptx::tmem_st_32x32b_x32(tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(C_::A_COL) + uint32_t(sl) * 32, v);
                ptx::tmem_st_wait();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&afull[sl]);
                if (warp == 8) FTR(1, lt, 18 + kb / kGatherGroups);
                FTR(6 + warp - 8, lt, kb);  // every gather warp: its arrive for k-block kb
                sl += kGatherGroups;
                while (sl >= RA) { sl -= RA; ++pass; }
            }
            gbase += uint32_t(p.kb_tile);
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&xempty[buf]);
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512, 1>(tmem);
    }
#undef FTR
}

// kernel bank (o, k, k, d) -> per variant phi: [small rows | big rows] x Kp, filter row i's
// k d run at columns [i segw + shift, ...) of its window (run_shift), zeros elsewhere
__global__ void prep_bank_kernel(const float* __restrict__ w, float* __restrict__ w2, int o, int k, int d, int n,
                                 int pad, int segw, int kp, int nvar) {
    const int64_t total = int64_t(nvar) * 2 * o * kp;
    const int seg = k * d;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total; idx += int64_t(gridDim.x) * blockDim.x) {
        const int row = int(idx / kp), col = int(idx - int64_t(row) * kp);
        const int phi = row / (2 * o), hr = row - phi * 2 * o;
        const int oc = hr < o ? hr : hr - o;
        const int i = col / segw;
        const int e = col - i * segw - (i < k ? run_shift(nvar == 1 ? 0 : phi, i, n, d, pad) : 0);
        float v = 0.f;
        if (i < k && e >= 0 && e < seg) {
            v = w[(int64_t(oc) * k + i) * seg + e];
            if (hr < o) v -= __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);  // rows [0, o): small half
        }
        w2[idx] = v;
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

// K-major 2D map over rows x kp floats, box = 16 columns x box_rows rows, SWIZZLE_64B
bool make_kmajor_map(CUtensorMap* map, const float* base, int64_t rows, int64_t kp, int box_rows) {
    auto enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {cuuint64_t(kp), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(kp) * 4};
    cuuint32_t box[2] = {cuuint32_t(kKB), cuuint32_t(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct FwdPlan {
    int np = 0, segw = 0, kp = 0, kb = 0, nvar = 1, xr = 0, pitch = 0, lmargin = 0, stages = 0, aslots = 0;
    int tpx = 0, xb = 2;
    bool merge = true, rows_tiles = false;
    uint32_t smem = 0;
    bool ok = false;
};

FwdPlan fwd_plan(const Geo& g) {
    FwdPlan P;
    if (g.s * g.d % 4 != 0 || g.o > 192 || g.o < 1 || g.k > 32 || g.m < 1) return P;
    if (g.b * g.n * g.n * g.d >= (int64_t(1) << 40) || g.b * g.o * g.m * g.m >= (int64_t(1) << 40) ||
        g.n * g.n * g.d >= (int64_t(1) << 30) || g.b * ((g.m * g.m + kTileM - 1) / kTileM) >= (int64_t(1) << 31))
        return P;
    P.np = g.o <= 32 ? 32 : g.o <= 64 ? 64 : g.o <= 96 ? 96 : g.o <= 128 ? 128 : 192;
    P.nvar = (g.n * g.n * g.d) % 4 == 0 ? 1 : 4;
    const int seg = int(g.k * g.d);
    bool shifted = false;
    for (int phi = 0; phi < P.nvar; ++phi)
        for (int i = 0; i < g.k; ++i) shifted = shifted || run_shift(phi, i, int(g.n), int(g.d), int(g.p)) != 0;
    P.segw = (seg + (shifted ? 3 : 0) + 3) & ~3;
    P.kp = int((g.k * P.segw + kKB - 1) / kKB * kKB);
    P.kb = P.kp / kKB;
    if (P.kb * 4 > kMaxKGroups || P.kb < 2) return P;
    // CCT_TUNE_GATHER = 3 (A/B): tiles of whole output rows (m <= 128) with three row buffers
    P.rows_tiles = tuning(CCT_TUNE_GATHER) == 3 && g.m <= kTileM;
    const int64_t tr = P.rows_tiles ? kTileM / g.m : 0;
    P.tpx = int(tr ? tr * g.m : kTileM);
    const int64_t rows_span = tr ? tr : ((kTileM - 1) / g.m + 2 > g.m ? g.m : (kTileM - 1) / g.m + 2);  // output rows per tile
    P.xr = int(g.s * (rows_span - 1) + g.k);
    P.xb = P.rows_tiles ? 3 : 2;
    P.lmargin = int((g.p * g.d + 4 + 3) & ~int64_t(3));
    P.pitch = int((P.lmargin + 3 + (g.n + g.p) * g.d + P.segw + 8 + 3) & ~int64_t(3));
    if (4 * (P.lmargin + 3 + P.segw) >= 32768) return P;  // byte offsets packed as int16
    P.merge = tuning(CCT_TUNE_GATHER) != 2;  // 2: the 6-MMA form (A/B)
    P.aslots = max_aslots(P.np, P.merge);
    if (P.aslots < kGatherGroups) return P;
    for (int st = CCT_FWD_MAX_STAGES; st >= 3; --st) {
        const FwdLayout L = fwd_layout(P.np, st, P.aslots, P.xr, P.pitch, P.kb * 4, P.xb);
        if (L.total + 1024 <= uint32_t(kSmemMax)) {
            P.stages = st;
            P.smem = L.total + 1024;
            break;
        }
    }
    P.ok = P.stages > 0;
    return P;
}

template <int NP, bool MG>
cudaError_t launch_fwd(const CUtensorMap& tm, const FwdParams& fp, uint32_t smem, cudaStream_t st) {
    auto kern = conv_fwd_gather_kernel<NP, MG>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    const int grid = std::min(num_sms(), fp.tiles);
    PhaseScope ps(kPhaseGemm, st, 2.0 * double(fp.b) * fp.m * fp.m * double(fp.k) * fp.k * fp.d * fp.o, 0);
    kern<<<grid, kThreads, smem, st>>>(tm, fp);
    note_launch();
    return cudaGetLastError();
}


// ===========================================================================
// Backward-weight: dW (o x k k d) = sum over pixels of dy^T x lowered(x), computed
// transposed, dW^T (k k d x o), so the gathered operand is the tcgen05 A operand in
// TMEM: lanes = lowered columns (M-tile mt covers columns [128 mt, 128 mt + 128)),
// TMEM columns = 16 pixels of a k-block.  B = dy (NHWC: pixels x o, MN-major) streams
// through a TMA ring; 4 transform warps write its 3xTF32 small half next to it.  One
// CTA computes all M-tiles of a k-block (the staged rows and the dy tile serve every
// M-tile), accumulating M-tile mt in TMEM columns [mt NP, (mt + 1) NP).  Work = chains
// of consecutive 128-pixel tiles (<= kWgChainKB k-blocks: the fp32 accumulation-chain
// cap), each ending in a partial dW written to scratch; the partials are summed in
// chain order afterwards (deterministic).
//   warp 0        dy producer (TMA, MN-major 32-channel boxes)   [bfull / bempty]
//   warp 1        MMA issuer                                       [btdone, afull -> aempty, bempty, tfull]
//   warp 2        TMEM allocator, then the row-stage producer      [xfull / xempty]
//   warps 4-7     epilogue: TMEM -> partial dW (lanes = consecutive lowered columns)
//   warps 8-11    dy transform: small = dy - trunc(dy) in smem     [bfull -> btdone]
//   warps 12-     one gather group (4 warps) per M-tile: group mt gathers unit (k-block, mt)
// ===========================================================================
template <int MT>
constexpr int wg_threads() { return 256 + 128 + 128 * MT; }  // gather group mt owns M-tile mt
constexpr int kWgChainKB = 256;  // k-blocks per accumulation chain (= kMaxChainKB)
constexpr int kWgMaxMT = 3;      // M-tiles (k k d <= 384)

struct WgParams {
    const float* x;
    float* part;             // [chain][o][kkd]
    int64_t x_total;
    int b, n, d, k, s, p, m, o, kkd, kd;
    int mt_tiles;            // M-tiles (ceil(kkd / 128))
    int tpi, tpx, tiles, chains;  // tiles per image, pixels per tile (whole output rows when m <= 128), total tiles, chains
    int pitch, lmargin, xr;  // staged rows (as the forward)
    int xstride;             // floats per row buffer: xr rows + a guard band (the last k-block's reads
                             // past the tile's end stay in it, not in the buffer being refilled)
    int xb;                  // row-stage buffers (2 or 3)
    int bstages, aslots;
};

__device__ __forceinline__ float4 small4(float4 v) {  // x - trunc_tf32(x), exact
    v.x -= __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
    v.y -= __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
    v.z -= __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
    v.w -= __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
    return v;
}

__host__ __device__ inline uint32_t wg_bstage_bytes(int np) { return uint32_t(np) * kKB * 4u; }  // one half

struct WgLayout {
    uint32_t ring, stage, bars, total;
};
__host__ __device__ inline WgLayout wg_layout(int np, int bstages, int aslots, int xstride, int xb) {
    WgLayout L;
    L.ring = 0;
    L.stage = uint32_t(bstages) * 2u * wg_bstage_bytes(np);
    L.bars = (L.stage + uint32_t(xb) * uint32_t(xstride) * 4u + 15u) & ~15u;
    L.total = L.bars + uint32_t(3 * bstages + 2 * aslots + 2 * xb + 4) * 8u + 16u;
    return L;
}

__device__ __forceinline__ void wg_chain(const WgParams& p, int c, int& t0, int& t1) {
    t0 = int(int64_t(c) * p.tiles / p.chains);
    t1 = int(int64_t(c + 1) * p.tiles / p.chains);
}
// tile T: image q, pixels [P0, P1) (whole output rows when m <= 128: the staged rows of a tile
// are then s (rows - 1) + k, and no tile restages a partial output row)
__device__ __forceinline__ void wg_tile(const WgParams& p, int T, int& q, int& P0, int& P1) {
    q = T / p.tpi;
    P0 = (T - q * p.tpi) * p.tpx;
    P1 = min(P0 + p.tpx, p.m * p.m);
}
__device__ __forceinline__ int wg_tile_kb(const WgParams& p, int T) {
    int q, P0, P1;
    wg_tile(p, T, q, P0, P1);
    return (P1 - P0 + kKB - 1) / kKB;
}

template <int NP, bool PAD, int MT>
__global__ void __launch_bounds__(wg_threads<MT>(), 1)
    conv_wgrad_gather_kernel(const __grid_constant__ CUtensorMap tmB, const WgParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    constexpr uint32_t HB = NP * kKB * 4;  // one half (raw or small) of a dy stage
    const int RB = p.bstages, RA = p.aslots;
    const WgLayout L = wg_layout(NP, RB, RA, p.xstride, p.xb);
    uint64_t* bfull = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* btdone = bfull + RB;
    uint64_t* bempty = btdone + RB;
    uint64_t* afull = bempty + RB;
    uint64_t* aempty = afull + RA;
    uint64_t* xfull = aempty + RA;
    uint64_t* xempty = xfull + p.xb;
    uint64_t* tfull = xempty + p.xb;
    uint64_t* tempty = tfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
    constexpr uint32_t A_COL = uint32_t(MT * NP);  // A slots after the accumulators

    const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmB);
        for (int s = 0; s < RB; ++s) {
            ptx::mbar_init(&bfull[s], 1);
            ptx::mbar_init(&btdone[s], 4);
            ptx::mbar_init(&bempty[s], 1);
        }
        for (int a = 0; a < RA; ++a) {
            ptx::mbar_init(&afull[a], 4);
            ptx::mbar_init(&aempty[a], 1);
        }
        for (int a = 0; a < p.xb; ++a) {
            ptx::mbar_init(&xfull[a], 1);
            ptx::mbar_init(&xempty[a], 4 * MT);
        }
        ptx::mbar_init(tfull, 1);
        ptx::mbar_init(tempty, 4);
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<512, 1>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int nd = p.n * p.d;
    const int mm = p.m * p.m;

    if (warp == 0) {
        // ===================== dy producer (warp-uniform loop, elected issue) =====================
        int st = 0;
        uint32_t ph = 0;
        for (int c = blockIdx.x; c < p.chains; c += gridDim.x) {
            int t0, t1;
            wg_chain(p, c, t0, t1);
            for (int T = t0; T < t1; ++T) {
                int q, P0, P1;
                wg_tile(p, T, q, P0, P1);
                const int nkb = (P1 - P0 + kKB - 1) / kKB;
                for (int kb = 0; kb < nkb; ++kb) {
                    ptx::mbar_wait_sleep(&bempty[st], ph ^ 1);
                    if (ptx::elect_one()) {
                        ptx::mbar_arrive_expect_tx(&bfull[st], HB);
                        uint8_t* dst = smem + L.ring + uint32_t(st) * 2u * HB;
                        const int pix = q * mm + P0 + kb * kKB;
#pragma unroll
                        for (int cc = 0; cc < NP / 32; ++cc)
                            ptx::tma_load_2d(dst + cc * 32 * kKB * 4, &tmB, &bfull[st], 32 * cc, pix);
                    }
                    __syncwarp();
                    if (++st == RB) { st = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        constexpr uint32_t idesc = ptx::idesc_tf32(kTileM, NP, 0, 1);
        const uint32_t ring_u = ptx::smem_u32(smem + L.ring);
        int bs = 0, as = 0;
        uint32_t bph = 0, aph = 0;
        int lc = 0;
        for (int c = blockIdx.x; c < p.chains; c += gridDim.x, ++lc) {
            ptx::mbar_wait(tempty, (lc & 1) ^ 1);
            ptx::tc_fence_after();
            int t0, t1;
            wg_chain(p, c, t0, t1);
            bool first = true;
            for (int T = t0; T < t1; ++T) {
                const int nkb = wg_tile_kb(p, T);
                for (int kb = 0; kb < nkb; ++kb) {
                    // the k-block's MT units sit in consecutive A slots; one elected issue of all
                    // 6 MT MMAs and the commits (few instructions per MMA: this warp's issue rate
                    // bounded the kernel)
                    int sl[MT];
                    uint32_t sph[MT];
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        sl[mt] = as;
                        sph[mt] = aph;
                        if (++as == RA) { as = 0; aph ^= 1; }
                    }
                    ptx::mbar_wait(&btdone[bs], bph);
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) ptx::mbar_wait(&afull[sl[mt]], sph[mt]);
                    ptx::tc_fence_after();
                    const uint32_t braw = ring_u + uint32_t(bs) * 2u * HB;
                    const uint64_t dr = ptx::smem_desc(braw, 2048, 512, 1);       // K step 0; step 1: +1024 B
                    const uint64_t ds = ptx::smem_desc(braw + HB, 2048, 512, 1);
                    if (ptx::elect_one()) {
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) {
                            const uint32_t d0 = tmem + uint32_t(mt * NP);
                            const uint32_t abig = tmem + A_COL + uint32_t(sl[mt]) * 32, asml = abig + kKB;
                            // small products first, big * big last
                            ptx::mma_tf32_ts(d0, asml, dr, idesc, first ? 0u : 1u);
                            ptx::mma_tf32_ts(d0, asml + 8, dr + 64, idesc, 1u);
                            ptx::mma_tf32_ts(d0, abig, ds, idesc, 1u);
                            ptx::mma_tf32_ts(d0, abig + 8, ds + 64, idesc, 1u);
                            ptx::mma_tf32_ts(d0, abig, dr, idesc, 1u);
                            ptx::mma_tf32_ts(d0, abig + 8, dr + 64, idesc, 1u);
                            ptx::mma_commit(&aempty[sl[mt]]);
                        }
                        ptx::mma_commit(&bempty[bs]);
                    }
                    __syncwarp();
                    first = false;
                    if (++bs == RB) { bs = 0; bph ^= 1; }
                }
            }
            if (ptx::elect_one()) ptx::mma_commit(tfull);
            __syncwarp();
        }
    } else if (warp == 2) {
        // ===================== row-stage producer =====================
        if (lane == 0) {
            int lt = 0;
            for (int c = blockIdx.x; c < p.chains; c += gridDim.x) {
                int t0, t1;
                wg_chain(p, c, t0, t1);
                for (int T = t0; T < t1; ++T, ++lt) {
                    const int buf = lt % p.xb;
                    ptx::mbar_wait_sleep(&xempty[buf], ((lt / p.xb) & 1) ^ 1);
                    int q, P0, P1;
                    wg_tile(p, T, q, P0, P1);
                    const int ra = P0 / p.m, rb = (P1 - 1) / p.m;
                    const int y0 = p.s * ra - p.p, nrows = p.s * (rb - ra) + p.k;
                    float* sb = reinterpret_cast<float*>(smem + L.stage) + int64_t(buf) * p.xstride;
                    uint32_t bytes = 0;
                    for (int rho = 0; rho < nrows; ++rho) {
                        const int yy = y0 + rho;
                        if (yy < 0 || yy >= p.n) continue;
                        const int64_t off = (int64_t(q) * p.n + yy) * nd;
                        const int64_t a0 = off & ~int64_t(3);
                        int64_t nfl = ((off - a0) + nd + 3) & ~int64_t(3);
                        if (a0 + nfl > p.x_total) {
                            nfl = (p.x_total - a0) & ~int64_t(3);
                            for (int64_t u = a0 + nfl; u < p.x_total; ++u)
                                sb[int64_t(rho) * p.pitch + p.lmargin + (u - a0)] = __ldg(p.x + u);
                        }
                        bytes += uint32_t(nfl) * 4u;
                    }
                    ptx::mbar_arrive_expect_tx(&xfull[buf], bytes);
                    for (int rho = 0; rho < nrows; ++rho) {
                        const int yy = y0 + rho;
                        if (yy < 0 || yy >= p.n) continue;
                        const int64_t off = (int64_t(q) * p.n + yy) * nd;
                        const int64_t a0 = off & ~int64_t(3);
                        int64_t nfl = ((off - a0) + nd + 3) & ~int64_t(3);
                        if (a0 + nfl > p.x_total) nfl = (p.x_total - a0) & ~int64_t(3);
                        if (nfl > 0)
                            ptx::bulk_load(sb + int64_t(rho) * p.pitch + p.lmargin, p.x + a0, uint32_t(nfl) * 4u,
                                           &xfull[buf]);
                    }
                }
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ===================== epilogue: partial dW of each chain =====================
        const int qd = warp & 3;
        int lc = 0;
        for (int c = blockIdx.x; c < p.chains; c += gridDim.x, ++lc) {
            ptx::mbar_wait_sleep(tfull, lc & 1);
            ptx::tc_fence_after();
            float* part = p.part + int64_t(c) * p.o * p.kkd;
            for (int mt = 0; mt < MT; ++mt) {
                const int col = mt * kTileM + qd * 32 + lane;
#pragma unroll 1
                for (int c0 = 0; c0 < NP; c0 += 32) {
                    uint32_t v[32];
                    ptx::tmem_ld_32x32b_x32(tmem + (uint32_t(qd * 32) << 16) + uint32_t(mt * NP + c0), v);
                    ptx::tmem_ld_wait();
                    if (col < p.kkd) {
                        const int nj = min(32, p.o - c0);
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (j < nj) __stcg(part + int64_t(c0 + j) * p.kkd + col, __uint_as_float(v[j]));
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(tempty);
        }
    } else if (warp >= 8 && warp < 12) {
        // ===================== dy transform: small half =====================
        const int t = (warp - 8) * 32 + lane;
        const uint32_t ring_u = ptx::smem_u32(smem + L.ring);
        int st = 0;
        uint32_t ph = 0;
        for (int c = blockIdx.x; c < p.chains; c += gridDim.x) {
            int t0, t1;
            wg_chain(p, c, t0, t1);
            for (int T = t0; T < t1; ++T) {
                const int nkb = wg_tile_kb(p, T);
                for (int kb = 0; kb < nkb; ++kb) {
                    ptx::mbar_wait_sleep(&bfull[st], ph);
                    const uint32_t braw = ring_u + uint32_t(st) * 2u * HB;
#pragma unroll
                    for (int i = t; i < int(HB / 16); i += 128) {
                        const float4 v = ptx::lds128(braw + uint32_t(i) * 16u);
                        ptx::sts128(braw + HB + uint32_t(i) * 16u, small4(v));
                    }
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&btdone[st]);
                    if (++st == RB) { st = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp >= 12) {
        // ===================== gather groups: group mt owns M-tile mt =====================
        const int mt = (warp - 12) >> 2;
        const int qd = warp & 3;
        const uint32_t stage_u = ptx::smem_u32(smem + L.stage);
        const uint32_t pitch_b = uint32_t(p.pitch) * 4u;
        // lane constants: lowered column -> filter row i, run element e, filter column j;
        // loff = the lane's byte offset within the staged row of filter row i
        const int col = min(mt * kTileM + qd * 32 + lane, p.kkd - 1);
        const bool cok = mt * kTileM + qd * 32 + lane < p.kkd;
        const int li = col / p.kd, le = col - li * p.kd, lj = le / p.d;
        const uint32_t loff = uint32_t(li) * pitch_b + 4u * uint32_t(p.lmargin + le - p.p * p.d);
        const uint32_t lph = uint32_t((int64_t(li) * nd) & 3);
        // unit u = gk MT + mt (gk: the CTA's k-block counter) sits in A slot u % RA, pass u / RA
        int sl = mt, pass = 0;
        while (sl >= RA) { sl -= RA; ++pass; }
        int gk = 0;  // CTA k-block counter at the start of the current tile
        int lt = 0;
        for (int c = blockIdx.x; c < p.chains; c += gridDim.x) {
            int t0, t1;
            wg_chain(p, c, t0, t1);
            for (int T = t0; T < t1; ++T, ++lt) {
                const int buf = lt % p.xb;
                int q, P0, P1;
                wg_tile(p, T, q, P0, P1);
                const int ra = P0 / p.m;
                const int nkb = (P1 - P0 + kKB - 1) / kKB;
                const uint32_t sbase = stage_u + uint32_t(buf) * uint32_t(p.xstride) * 4u;
                ptx::mbar_wait_sleep(&xfull[buf], (lt / p.xb) & 1);
                int r0 = P0 / p.m, c0 = P0 - r0 * p.m;  // first pixel of k-block kb
                for (int kb = 0; kb < nkb; ++kb) {
                    // the k-block's 16 pixels lie in output row r0 (jj < split) and r0 + 1 (m >= 16);
                    // pixel jj's staged address = row base + jj s d floats (uniform stride)
                    const int split = p.m - c0;
                    const int nval = P1 - (P0 + kb * kKB);
                    const bool two = split < kKB && nval > split;  // row r0 + 1 is staged and used
                    // float offset mod 4 of input row s r - p + i of image q
                    const uint32_t ph0 = uint32_t(q * p.n + p.s * r0 - p.p) * uint32_t(nd) + lph;
                    const uint32_t ph1 = ph0 + uint32_t(p.s * nd);
                    const uint32_t sd4 = uint32_t(p.s * p.d) * 4u;
                    const uint32_t rb0 = sbase + uint32_t(p.s * (r0 - ra)) * pitch_b + loff +
                                         4u * ((ph0 & 3u) + uint32_t(p.s * c0 * p.d));
                    const uint32_t rb1 = two ? sbase + uint32_t(p.s * (r0 + 1 - ra)) * pitch_b + loff +
                                                   4u * (ph1 & 3u) - uint32_t(split) * sd4
                                             : rb0;
                    bool rv0 = true, rv1 = true;
                    if constexpr (PAD) {
                        rv0 = unsigned(p.s * r0 - p.p + li) < unsigned(p.n);
                        rv1 = unsigned(p.s * (r0 + 1) - p.p + li) < unsigned(p.n);
                    }
                    uint32_t v[32];
#pragma unroll
                    for (int jj = 0; jj < kKB; ++jj) {
                        const bool second = jj >= split;
                        // (pixels past the tile's end read the buffer's guard band; discarded below)
                        float f = ptx::lds32((second ? rb1 : rb0) + uint32_t(jj) * sd4);
                        bool ok = cok && jj < nval;
                        if constexpr (PAD) {
                            const int cc = second ? jj - split : c0 + jj;
                            ok = ok && (second ? rv1 : rv0) && unsigned(p.s * cc - p.p + lj) < unsigned(p.n);
                        }
                        f = ok ? f : 0.f;
                        const uint32_t big = __float_as_uint(f) & 0xFFFFE000u;
                        v[jj] = big;
                        v[kKB + jj] = __float_as_uint(f - __uint_as_float(big));
                    }
                    if (pass > 0) ptx::mbar_wait_sleep(&aempty[sl], (pass - 1) & 1);  // gathered before the wait
                    ptx::tmem_st_32x32b_x32(tmem + (uint32_t(qd * 32) << 16) + A_COL + uint32_t(sl) * 32, v);
                    ptx::tmem_st_wait();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&afull[sl]);
                    sl += MT;
                    while (sl >= RA) { sl -= RA; ++pass; }
                    c0 += kKB;
                    if (c0 >= p.m) { c0 -= p.m; ++r0; }
                }
                gk += nkb;
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&xempty[buf]);
            }
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512, 1>(tmem);
    }
}

// NHWC dy (pixels x o) as an MN-major operand: 32-channel x 16-pixel boxes, SWIZZLE_128B_ATOM_32B
bool make_mnmajor_map(CUtensorMap* map, const float* base, int64_t pixels, int64_t o) {
    auto enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {cuuint64_t(o), cuuint64_t(pixels)};
    cuuint64_t strides[1] = {cuuint64_t(o) * 4};
    cuuint32_t box[2] = {32, cuuint32_t(kKB)};
    cuuint32_t estr[2] = {1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct WgPlan {
    int np = 0, mt = 0, bstages = 0, aslots = 0, xr = 0, xstride = 0, xb = 0, pitch = 0, lmargin = 0, tpi = 0, tpx = 0, tiles = 0,
        chains = 0, grid = 0;
    uint32_t smem = 0;
    bool ok = false;
};

WgPlan wg_plan(const Geo& g) {
    WgPlan P;
    const int64_t kkd = g.k * g.k * g.d, mm = g.m * g.m;
    if (g.o < 1 || g.o > 128 || g.o % 4 != 0 || kkd > int64_t(kWgMaxMT) * kTileM || g.m < kKB || g.k > 32) return P;
    if (g.b * g.n * g.n * g.d >= (int64_t(1) << 40) || g.b * mm >= (int64_t(1) << 31) - kTileM ||
        g.n * g.n * g.d >= (int64_t(1) << 30) || g.o * kkd * 4096 >= (int64_t(1) << 40))
        return P;
    P.np = int((g.o + 31) / 32 * 32);
    P.mt = int((kkd + kTileM - 1) / kTileM);
    P.aslots = std::min(8, (512 - P.mt * P.np) / 32);
    if (P.aslots < 4) return P;
    // tiles of whole output rows when m <= 128 (the pixels are this GEMM's K: at most one partly
    // filled k-block per tile), else 128-pixel tiles
    const int64_t tr = g.m <= kTileM ? kTileM / g.m : 0;
    P.tpx = int(tr ? tr * g.m : kTileM);
    const int64_t rows_span = tr ? tr : ((kTileM - 1) / g.m + 2 > g.m ? g.m : (kTileM - 1) / g.m + 2);
    P.xr = int(g.s * (rows_span - 1) + g.k);
    P.lmargin = int((g.p * g.d + 4 + 3) & ~int64_t(3));
    P.pitch = int((P.lmargin + (g.n + g.p) * g.d + 8 + 3) & ~int64_t(3));
    P.xstride = int(int64_t(P.xr) * P.pitch + ((16 * g.s * g.d + 64 + 3) & ~int64_t(3)));
    if (int64_t(P.xstride) * 4 * 3 >= (int64_t(1) << 31)) return P;
    // three row-stage buffers when they fit next to >= 6 dy stages, else two
    for (int xb = 3; xb >= 2 && !P.bstages; --xb)
        for (int st = 8; st >= (xb == 3 ? 6 : 2); --st) {
            const WgLayout L = wg_layout(P.np, st, P.aslots, P.xstride, xb);
            if (L.total + 1024 <= uint32_t(kSmemMax)) {
                P.bstages = st;
                P.xb = xb;
                P.smem = L.total + 1024;
                break;
            }
        }
    if (!P.bstages) return P;
    P.tpi = int((mm + P.tpx - 1) / P.tpx);
    P.tiles = int(g.b * P.tpi);
    const int kb_tile_max = (P.tpx + kKB - 1) / kKB;
    const int cmin = (P.tiles * kb_tile_max + kWgChainKB - 1) / kWgChainKB;
    P.grid = std::min(num_sms(), P.tiles);
    P.chains = std::min(P.tiles, (cmin + P.grid - 1) / P.grid * P.grid);
    P.ok = true;
    return P;
}
int g_probe_dbg = 0;  // FwdParams::dbg of every launch (set only by tools/gather_probe.cu)
unsigned long long* g_probe_trace = nullptr;  // FwdParams::trace (likewise)
int g_probe_pace_ns = -1;                      // >= 0: FwdParams::pace_ns override (likewise)
}  // namespace gth

using namespace gth;

bool gather_fwd_ok(const Geo& g) { return fwd_plan(g).ok; }

int64_t gather_fwd_ws_floats(const Geo& g) {
    const FwdPlan P = fwd_plan(g);
    return P.ok ? int64_t(P.nvar) * 2 * g.o * P.kp : 0;
}

cudaError_t gather_fwd(const Geo& g, const float* x, const float* w, float* y, int64_t ycs, const float* bias,
                       int relu, float* ws, cudaStream_t st) {
    const FwdPlan P = fwd_plan(g);
    if (!P.ok) return cudaErrorInvalidValue;
    {
        const int64_t total = int64_t(P.nvar) * 2 * g.o * P.kp;
        prep_bank_kernel<<<grid_for(total, 256), 256, 0, st>>>(w, ws, int(g.o), int(g.k), int(g.d), int(g.n),
                                                               int(g.p), P.segw, P.kp, P.nvar);
        note_launch();
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    CUtensorMap tm;
    if (!make_kmajor_map(&tm, ws, int64_t(P.nvar) * 2 * g.o, P.kp, P.np)) return cudaErrorInvalidValue;
    FwdParams fp{};
    fp.dbg = g_probe_dbg;
    fp.trace = g_probe_trace;
    fp.pace_ns = g_probe_pace_ns >= 0 ? g_probe_pace_ns : CCT_FWD_PACE_NS;
    fp.x = x;
    fp.y = y;
    fp.bias = bias;
    fp.relu = relu;
    const int64_t mm = g.m * g.m;
    if (g.yl) {  // NHWC
        fp.y_sq = ycs ? ycs : mm * g.o;
        fp.y_so = 1;
        fp.y_sp = g.o;
    } else {
        fp.y_sq = ycs ? ycs : g.o * mm;
        fp.y_so = mm;
        fp.y_sp = 1;
    }
    fp.x_total = g.b * g.n * g.n * g.d;
    fp.b = int(g.b); fp.n = int(g.n); fp.d = int(g.d); fp.k = int(g.k); fp.s = int(g.s); fp.p = int(g.p);
    fp.m = int(g.m); fp.o = int(g.o);
    fp.seg = int(g.k * g.d);
    fp.segw = P.segw;
    fp.nvar = P.nvar;
    fp.kb_tile = P.kb;
    fp.tpx = P.tpx;
    fp.xb = P.xb;
    fp.tpi = int((mm + P.tpx - 1) / P.tpx);
    fp.tiles = int(g.b) * fp.tpi;
    fp.pitch = P.pitch;
    fp.lmargin = P.lmargin;
    fp.xr = P.xr;
    fp.stages = P.stages;
    fp.aslots = P.aslots;
    switch (P.np) {
        case 32: return P.merge ? launch_fwd<32, true>(tm, fp, P.smem, st) : launch_fwd<32, false>(tm, fp, P.smem, st);
        case 64: return P.merge ? launch_fwd<64, true>(tm, fp, P.smem, st) : launch_fwd<64, false>(tm, fp, P.smem, st);
        case 96: return P.merge ? launch_fwd<96, true>(tm, fp, P.smem, st) : launch_fwd<96, false>(tm, fp, P.smem, st);
        case 128: return launch_fwd<128, false>(tm, fp, P.smem, st);
        default: return launch_fwd<192, false>(tm, fp, P.smem, st);
    }
}


bool gather_wgrad_ok(const Geo& g) { return wg_plan(g).ok; }

int64_t gather_wgrad_ws_floats(const Geo& g) {
    const WgPlan P = wg_plan(g);
    if (!P.ok) return 0;
    const int64_t nhwc = g.yl ? 0 : (g.b * g.m * g.m * g.o + 3) / 4 * 4;  // NCHW dy -> NHWC copy
    return nhwc + int64_t(P.chains) * g.o * g.k * g.k * g.d;
}

cudaError_t gather_wgrad(const Geo& g, const float* x, const float* dy, float* dw, float* ws, cudaStream_t st) {
    const WgPlan P = wg_plan(g);
    if (!P.ok) return cudaErrorInvalidValue;
    const int64_t mm = g.m * g.m, kkd = g.k * g.k * g.d;
    const float* dyn = dy;
    float* part = ws;
    if (!g.yl) {  // NCHW dy -> NHWC (pixels x o), the MN-major B operand
        float* t = ws;
        part = ws + (g.b * mm * g.o + 3) / 4 * 4;
        cudaError_t e = transpose_batched(dy, g.o, mm, mm, g.o * mm, t, g.o, mm * g.o, g.b, kPhaseExpand, st);
        if (e != cudaSuccess) return e;
        dyn = t;
    }
    CUtensorMap tm;
    if (!make_mnmajor_map(&tm, dyn, g.b * mm, g.o)) return cudaErrorInvalidValue;
    WgParams wp{};
    wp.x = x;
    wp.part = part;
    wp.x_total = g.b * g.n * g.n * g.d;
    wp.b = int(g.b); wp.n = int(g.n); wp.d = int(g.d); wp.k = int(g.k); wp.s = int(g.s); wp.p = int(g.p);
    wp.m = int(g.m); wp.o = int(g.o);
    wp.kkd = int(kkd);
    wp.kd = int(g.k * g.d);
    wp.mt_tiles = P.mt;
    wp.tpi = P.tpi;
    wp.tpx = P.tpx;
    wp.xb = P.xb;
    wp.tiles = P.tiles;
    wp.chains = P.chains;
    wp.pitch = P.pitch;
    wp.lmargin = P.lmargin;
    wp.xr = P.xr;
    wp.xstride = P.xstride;
    wp.bstages = P.bstages;
    wp.aslots = P.aslots;
    {
        PhaseScope ps(kPhaseGemm, st, 2.0 * double(g.b) * double(mm) * double(kkd) * double(g.o), 0);
        cudaError_t e = cudaSuccess;
        auto go = [&](auto kern) {
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(P.smem));
            if (e == cudaSuccess) {
                kern<<<P.grid, 384 + 128 * P.mt, P.smem, st>>>(tm, wp);
                note_launch();
                e = cudaGetLastError();
            }
        };
        const bool pad = g.p > 0;
        switch (P.np * 10 + P.mt) {
#define CCT_WG_CASE(NP_, MT_)                                                                        \
    case NP_ * 10 + MT_:                                                                             \
        pad ? go(conv_wgrad_gather_kernel<NP_, true, MT_>) : go(conv_wgrad_gather_kernel<NP_, false, MT_>); \
        break;
            CCT_WG_CASE(32, 1) CCT_WG_CASE(32, 2) CCT_WG_CASE(32, 3)
            CCT_WG_CASE(64, 1) CCT_WG_CASE(64, 2) CCT_WG_CASE(64, 3)
            CCT_WG_CASE(96, 1) CCT_WG_CASE(96, 2) CCT_WG_CASE(96, 3)
            CCT_WG_CASE(128, 1) CCT_WG_CASE(128, 2) CCT_WG_CASE(128, 3)
#undef CCT_WG_CASE
            default: return cudaErrorInvalidValue;
        }
        if (e != cudaSuccess) return e;
    }
    const int64_t wsize = g.o * kkd;
    return splitk_reduce(part, wsize, P.chains, 1, wsize, wsize, dw, wsize, st);
}

}  // namespace cct
