// gemm_kernel.cuh -- the tcgen05 3xTF32 GEMM kernel template and its launch dispatch.
// Included by gemm.cu (host side: tensor maps, tile / split planning, run_gemm) and by the
// gemm_i<BN>_<CG>.cu instantiation units (one per tile width and CTA-group size, so the
// kernel variants compile in parallel).  See gemm.cu for the design notes.
#pragma once
#include <cudaTypedefs.h>

#include <algorithm>

#include "cct.h"
#include "common.cuh"
#include "gemm.cuh"
#include "ptx.cuh"

namespace cct {
namespace gk {


struct KParams {
    int M, N, K;
    int num_m_tiles, num_n_tiles, splits;
    int kb_total, kb_per_split;
    int units;
    int passes;
    float* C;
    int64_t mdiv, s_mq, s_mr, s_n, s_split;
    int ndiv;  // 0: column offset n * s_n; else (n / ndiv) * s_nq + (n % ndiv) * s_n
    // stream-K (sk_len > 0): CTA group g owns k-block iterations [g*sk_len, (g+1)*sk_len) of
    // the flattened (tile, k-block) space; tiles cut between two groups are summed by
    // whichever part finishes second, through sk_part / sk_cnt (see epilogue)
    int sk_len;
    float* sk_part;
    int* sk_cnt;
    int64_t s_nq;
    int64_t mlim;
    int nmlim;  // with ndiv: columns with (n % ndiv) >= nmlim are not stored
    int split_producer;  // A and B tiles issued by two producer threads
    const float* bias;  // fused epilogue: v = act(v + bias[n])
    int relu;
    // implicit (im2col) A: layer geometry (ic_d = channels per tap of the lowered index)
    int ic_d, ic_k, ic_s, ic_p, ic_m, ic_mm, ic_cpt;
};

// warps 0-3 control (TMA, MMA, TMEM alloc, spare), 4-7 epilogue, 8.. transform
#ifndef KTGROUPS
#define KTGROUPS 2
#endif
// Transform warps run as kTGroups groups of 4 that take alternate k-blocks, so the
// per-stage latency chain (ld.shared -> split -> st.shared / tcgen05.st -> proxy
// fence -> barrier arrive) of one group overlaps the next group's (measured: one
// group of 4 bounded narrow tiles at ~820 clocks per k-block).
constexpr int kTGroups = KTGROUPS;
constexpr int kTransformWarps = 4 * kTGroups;
constexpr int kThreads = 256 + 32 * kTransformWarps;

__host__ __device__ constexpr uint32_t tmem_cols_for(int bn) {
    return (2 * bn) <= 32 ? 32 : (2 * bn) <= 64 ? 64 : (2 * bn) <= 128 ? 128 : (2 * bn) <= 256 ? 256 : 512;
}

// Per-CTA tile geometry.  CG = 1: one CTA computes 128 x BN.  CG = 2 (CTA
// pair, tcgen05 cta_group::2): the pair computes 256 x BN; each CTA holds its
// 128 rows of A and BN/2 rows of B in smem and its 128 rows of D in TMEM.
template <int BN, int CG, int TRO = 0>
struct Cfg {
    static constexpr int BNL = BN / CG;  // B rows loaded by this CTA
    static constexpr uint32_t A_BYTES = kBM * kBK * 4;
    static constexpr uint32_t B_BYTES = BNL * kBK * 4;
    static constexpr uint32_t RAW_BYTES = A_BYTES + B_BYTES;
    static constexpr uint32_t STAGE_BYTES = 2 * RAW_BYTES;  // raw | small
    // transposing epilogue (TRO): one 32 x 33 fp32 staging block per epilogue warp
    static constexpr uint32_t EPI_BYTES = TRO ? 4 * 32 * 33 * 4 + 4 * 32 * 16 : 0;
    // as many ring stages as fit next to the barriers (227 KB opt-in smem per CTA)
    static constexpr int BUDGET = 225 * 1024 - int(EPI_BYTES);
    static constexpr int STAGES = (BUDGET / int(STAGE_BYTES)) > 12 ? 12 : (BUDGET / int(STAGE_BYTES));
    // full[kTGroups][STAGES] (one set per transform group, see the kernel), tdone, empty, tfull/tempty
    static constexpr uint32_t BAR_BYTES = ((2 + kTGroups) * STAGES + 4) * 8 + 16;
    static constexpr uint32_t SMEM_BYTES = STAGES * STAGE_BYTES + BAR_BYTES + EPI_BYTES + 1024;
    // Narrow tiles keep two sub-accumulators per tile (even / odd 8-wide K steps):
    // consecutive MMAs then target different TMEM regions and overlap instead of
    // serialising on one accumulator (measured: N=96 MMAs were latency-bound).
    static constexpr int NACC = (BN <= 128) ? 2 : 1;
    static constexpr uint32_t TMEM_COLS = tmem_cols_for(NACC * BN);
};

// a = big + small; big is what the tensor core reads from an fp32 operand in
// kind::tf32 (low 13 mantissa bits ignored); small is exact.
__device__ __forceinline__ float4 small_part(float4 v) {
    float4 r;
    r.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
    r.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
    r.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
    r.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
    return r;
}

// UMMA descriptor of one operand tile for K step kk (8 tf32 wide).
//   K-major tile: rows of 64 B (16 fp32), SWIZZLE_64B, 8-row atoms of 512 B.
//   MN-major tile: (rows/32) chunks of [16 K-rows x 128 B] written by TMA with
//                  SWIZZLE_128B_ATOM_32B; UMMA layout SWIZZLE_128B_BASE32B (the
//                  only MN-major smem layout for 32-bit operands), 4-K-row
//                  atoms of 512 B (SBO), chunk stride 2 KB (LBO).
template <bool MN>
__device__ __forceinline__ uint64_t tile_desc(uint32_t base, int kk) {
    if constexpr (!MN) {
        return ptx::smem_desc(base + kk * 32, 16, 512, 4);
    } else {
        return ptx::smem_desc(base + kk * 1024, 32 * kBK * 4, 512, 1);
    }
}

// first output pixel (q, r, c) of a flat pixel index
struct Pix {
    int q, r, c;
};
__device__ __forceinline__ Pix pix_of(int idx, const KParams& p) {
    Pix x;
    x.q = idx / p.ic_mm;
    const int rem = idx - x.q * p.ic_mm;
    x.r = rem / p.ic_m;
    x.c = rem - x.r * p.ic_m;
    return x;
}

// One piece of work of a CTA group: output unit u (tile, m fastest, then n, then
// split) over k-blocks [kb0, kb1).  kind 0: the whole unit; 1: leading part of a
// stream-K tile (finished by the next group); 2: trailing part (begun by the
// previous group).  Every warp role walks the same sequence.
struct Work {
    int u, kb0, kb1, kind;
};
struct WorkIter {
    int next_u, it, end;
    __device__ WorkIter(const KParams& p, int group) {
        if (p.sk_len) {
            it = group * p.sk_len;
            end = min(it + p.sk_len, p.units * p.kb_total);
            next_u = 0;
        } else {
            next_u = group;
            it = end = 0;
        }
    }
    __device__ bool next(const KParams& p, int ngroups, Work& w) {
        if (p.sk_len) {
            if (it >= end) return false;
            w.u = it / p.kb_total;
            const int lo = it - w.u * p.kb_total;
            const int stop = min(end, (w.u + 1) * p.kb_total);
            w.kb0 = lo;
            w.kb1 = lo + (stop - it);
            w.kind = (lo == 0 && w.kb1 == p.kb_total) ? 0 : (lo == 0 ? 1 : 2);
            it = stop;
            return true;
        }
        if (next_u >= p.units) return false;
        w.u = next_u;
        next_u += ngroups;
        const int sp = w.u / (p.num_m_tiles * p.num_n_tiles);
        w.kb0 = sp * p.kb_per_split;
        w.kb1 = min(w.kb0 + p.kb_per_split, p.kb_total);
        w.kind = 0;
        return true;
    }
};

// A_TM: narrow tiles keep the A operand in TMEM (tcgen05.mma A-from-TMEM): the
// transform warps read each A row once from smem and write its big / small parts
// to a 4-slot TMEM ring, so the three MMAs of a K step read only B from shared
// memory (for N <= 96 the A reads otherwise saturate the smem bus, ncu).
// TRO: transposing epilogue -- each warp stages its 32 rows x 32 columns chunk in
// smem and writes it back column by column, so an output whose ROWS are contiguous
// along the tile's N index (NCHW y of a swapped GEMM: rows = channels, columns =
// pixels) is stored as 128-byte row segments instead of 4-byte scatters.
// CH2: the tile's K range is accumulated as two chains (first / second half of the
// k-blocks) in two TMEM accumulators and summed in the epilogue (fp32 round-to-nearest),
// single-buffered: a 2-way accuracy split without partial tiles in HBM or a reduce kernel.
template <int BN, int A_MN, int B_MN, int CG, int A_IM, int A_TM = 0, int TRO = 0, int CH2 = 0>
__global__ void __launch_bounds__(kThreads, 1)
    gemm3xtf32_kernel(const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB, const KParams p) {
    using C_ = Cfg<BN, CG, TRO>;
    constexpr int STAGES = C_::STAGES;
    constexpr int BNL = C_::BNL;
    // A_TM == 2: one accumulator per tile, the freed TMEM columns deepen the A ring
    // A_TM == 3 (MG): A in TMEM, and the two products sharing A_big run as ONE N = 2 BN MMA over
    // the stage's B rows laid out [small | raw]: D[0, BN) = A_big B_small, D[BN, 2 BN) = A_big B_big
    // + A_small B_big, summed by the epilogue like two sub-accumulators (4 MMAs per k-block
    // instead of 6; an N <= 128 tf32 MMA costs ~77 cycles at any N, N = 192 ~103: tools/mma_rate.cu)
    constexpr bool MG = A_TM == 3;
    static_assert(!MG || (CG == 1 && !B_MN && !A_MN && BN <= 96 && !CH2 && !TRO), "A_TM 3 config");
    constexpr int NACC = CH2 ? 2 : (A_TM == 2) ? 1 : C_::NACC;
    // stage layout: [A raw | B raw | A small | B small]; MG: [A raw | B small | B raw | A small]
    constexpr uint32_t B_OFF = MG ? C_::A_BYTES + C_::B_BYTES : C_::A_BYTES;       // B raw
    constexpr uint32_t BS_OFF = MG ? C_::A_BYTES : C_::RAW_BYTES + C_::A_BYTES;    // B small
    static_assert(!CH2 || (!A_TM && BN > 128), "CH2 config");
    // single-buffered accumulator: CH2 (two chains), the 384-wide tile (256 + 128 columns), and
    // a 256-wide tile with A in TMEM (the A ring takes the second accumulator's columns)
    constexpr bool SB = CH2 || BN > 256 || (A_TM && BN == 256);
    constexpr uint32_t A_COL = uint32_t((SB ? 1 : 2) * NACC * BN);    // first A column
    constexpr int kASlotsFit = int((512u - A_COL) / (2 * kBK));
    constexpr int kASlots = A_TM ? (kASlotsFit < 12 ? (kASlotsFit < STAGES - 1 ? kASlotsFit : STAGES - 1)
                                                    : (12 < STAGES - 1 ? 12 : STAGES - 1))
                                 : 4;                                 // TMEM ring of A tiles
    static_assert(BN <= 256 || (BN == 384 && !CH2 && !TRO && A_IM <= 1), "BN 384 config");
    constexpr uint32_t TMEM_COLS = A_TM ? 512u : SB ? 512u : C_::TMEM_COLS;
    static_assert(!A_TM || (A_COL + kASlots * 2 * kBK <= 512 && !A_MN && STAGES > kASlots && kASlots >= 2),
                  "A_TM config");
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // align inside the shared window without leaving the shared address space
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    // full[g * STAGES + s]: stage s holding a k-block of transform group g (gi % kTGroups).
    // Each transform group waits on every phase of its own barriers in order.  (With one
    // barrier per stage and an odd ring depth, consecutive phases of a stage alternate
    // between the groups, and a parity wait for phase P + 1 passes while phase P -- the
    // other group's k-block -- is still in flight: stale operands and a tdone count skew.)
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C_::STAGE_BYTES);
    uint64_t* tdone = full + kTGroups * STAGES;
    uint64_t* empty = tdone + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    int* sk_flag = reinterpret_cast<int*>(tmem_slot + 1);
    float* epi = reinterpret_cast<float*>(smem + STAGES * C_::STAGE_BYTES + ((C_::BAR_BYTES + 15) & ~15u));

    const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0);  // warp-uniform (uniform registers)
    const int lane = threadIdx.x & 31;
    const uint32_t rank = (CG == 2) ? ptx::cluster_rank() : 0u;
    const bool leader = rank == 0;
    // work is distributed per CTA group (cluster)
    const int group = blockIdx.x / CG;
    const int ngroups = gridDim.x / CG;

    if (warp == 0 && lane == 0) {  // (warp 3 lane 0 is the B producer)
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
        // split producer: the A and B producers each arm the barrier with their own bytes
        // (two arrivals), so its transaction count never goes negative
        for (int s = 0; s < kTGroups * STAGES; ++s) ptx::mbar_init(&full[s], p.split_producer ? 2 : 1);
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(&tdone[s], 4 * CG);  // one transform group of every CTA in the group
            ptx::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], 4 * CG);  // epilogue warps of every CTA in the group
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<TMEM_COLS, CG>(tmem_slot);
    ptx::tc_fence_before();
    if constexpr (CG == 2) ptx::cluster_sync();
    else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // leader-CTA barriers seen from this CTA (remote arrive targets)
    const uint32_t tdone_leader = (CG == 2) ? ptx::mapa(ptx::smem_u32(tdone), 0) : 0u;
    const uint32_t tempty_leader = (CG == 2) ? ptx::mapa(ptx::smem_u32(tempty), 0) : 0u;

    if (warp == 0 || warp == 3) {
        // ===================== TMA producers (every CTA loads its own share) =====================
        // warp 0 issues the A tiles (and arms the stage's barrier), warp 3 the B tiles: the
        // MN-major operands take up to 4 + 8 boxes per stage and one issuing thread was the
        // limit of the backward-weight GEMMs ($CCT_SPLIT_PRODUCER=1; default 0: warp 0 issues
        // both -- the split form intermittently hangs)
        const bool role_a = warp == 0;
        const bool role_b = (warp == 3) == (p.split_producer != 0);
        // the whole warp walks the loop (coordinates stay warp-uniform, in uniform registers);
        // one elected lane arms the barrier and issues the copies
        if (role_a || role_b) {
            int stage = 0;
            uint32_t phase = 0;
            uint32_t gi = 0;  // k-blocks issued by this CTA (selects the transform group's barrier)
            WorkIter wi(p, group);
            Work w;
            while (wi.next(p, ngroups, w)) {
                const int u = w.u;
                const int mt = u % p.num_m_tiles;
                const int nt = (u / p.num_m_tiles) % p.num_n_tiles;
                const int m0 = mt * (kBM * CG) + int(rank) * kBM;
                const int n0 = nt * BN + int(rank) * BNL;
                const int kb0 = w.kb0, kb1 = w.kb1;
                // implicit lowering: each producer is one thread issuing every TMA of its
                // operand, so all im2col coordinates are per-tile constants or walked
                // incrementally (no divisions inside the k-loop)
                Pix px{};      // forward: first pixel of the tile; bwd-weight: pixel of k0
                int tap_i = 0, tap_j = 0, cc = 0;   // forward: filter tap and channel block of kb
                // bwd-weight: per 32-channel box (A rows, or B rows when B is the MN-major im2col)
                constexpr int NBW = (A_IM == 3) ? (BNL / 32 > 0 ? BNL / 32 : 1) : kBM / 32;
                int bw_ch[NBW], bw_ti[NBW], bw_tj[NBW];
                if constexpr (A_IM == 2) {  // B = im2col: the tile's pixels are its N index
                    px = pix_of(n0, p);
                    const int tap = kb0 / p.ic_cpt;
                    cc = kb0 - tap * p.ic_cpt;
                    tap_i = tap / p.ic_k;
                    tap_j = tap - tap_i * p.ic_k;
                } else if constexpr (A_IM == 3) {  // B = MN-major im2col: N = (tap, channel), K = pixels
                    px = pix_of(kb0 * kBK, p);
                    const int kkd = p.ic_k * p.ic_k * p.ic_d;
#pragma unroll
                    for (int c = 0; c < NBW; ++c) {
                        const int ncol = min(n0 + 32 * c, kkd - 32);  // columns >= N are masked later
                        const int tap = ncol / p.ic_d;
                        bw_ch[c] = ncol - tap * p.ic_d;
                        bw_ti[c] = tap / p.ic_k;
                        bw_tj[c] = tap - bw_ti[c] * p.ic_k;
                    }
                } else if constexpr (A_IM == 1 && !A_MN) {
                    px = pix_of(m0, p);
                    const int tap = kb0 / p.ic_cpt;
                    cc = kb0 - tap * p.ic_cpt;
                    tap_i = tap / p.ic_k;
                    tap_j = tap - tap_i * p.ic_k;
                } else if constexpr (A_IM == 1 && A_MN) {
                    px = pix_of(kb0 * kBK, p);
                    const int kkd = p.ic_k * p.ic_k * p.ic_d;
#pragma unroll
                    for (int c = 0; c < kBM / 32; ++c) {
                        const int mcol = min(m0 + 32 * c, kkd - 32);  // rows >= M are masked later
                        const int tap = mcol / p.ic_d;
                        bw_ch[c] = mcol - tap * p.ic_d;
                        bw_ti[c] = tap / p.ic_k;
                        bw_tj[c] = tap - bw_ti[c] * p.ic_k;
                    }
                }
                for (int kb = kb0; kb < kb1; ++kb, ++gi) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    const bool el = ptx::elect_one();
                    uint64_t* const fb = &full[int(gi % kTGroups) * STAGES + stage];
                    if (el) ptx::mbar_arrive_expect_tx(fb, (role_a && role_b) ? C_::RAW_BYTES : role_a ? C_::A_BYTES : C_::B_BYTES);
                    uint8_t* a_dst = smem + stage * C_::STAGE_BYTES;
                    uint8_t* b_dst = a_dst + B_OFF;
                    const int k0 = kb * kBK;
                    if (role_a) {
                        if constexpr (A_IM == 1 && !A_MN) {
                            // implicit lowering, forward: 128 pixels x 16 channels of filter tap (ti, tj)
                            if (el) ptx::tma_load_im2col_4d(a_dst, &tmA, fb, cc * kBK, p.ic_s * px.c - p.ic_p,
                                                    p.ic_s * px.r - p.ic_p, px.q, uint16_t(tap_j), uint16_t(tap_i));
                            if (++cc == p.ic_cpt) {
                                cc = 0;
                                if (++tap_j == p.ic_k) { tap_j = 0; ++tap_i; }
                            }
                        } else if constexpr (A_IM == 1 && A_MN) {
                            // implicit lowering, backward-weight: K rows = 16 pixels, M = (tap, ch)
#pragma unroll
                            for (int c = 0; c < kBM / 32; ++c)
                                if (el) ptx::tma_load_im2col_4d(a_dst + c * 32 * kBK * 4, &tmA, fb, bw_ch[c],
                                                        p.ic_s * px.c - p.ic_p, p.ic_s * px.r - p.ic_p, px.q,
                                                        uint16_t(bw_tj[c]), uint16_t(bw_ti[c]));
                            px.c += kBK;
                            while (px.c >= p.ic_m) {
                                px.c -= p.ic_m;
                                if (++px.r == p.ic_m) { px.r = 0; ++px.q; }
                            }
                        } else if constexpr (!A_MN) {
                            if (el) ptx::tma_load_2d(a_dst, &tmA, fb, k0, m0);
                        } else {
#pragma unroll
                            for (int c = 0; c < kBM / 32; ++c)
                                if (el) ptx::tma_load_2d(a_dst + c * 32 * kBK * 4, &tmA, fb, m0 + 32 * c, k0);
                        }
                    }
                    if (role_b) {
                        if constexpr (A_IM == 2) {
                            // B: BNL pixels x 16 channels of tap (ti, tj)
                            if (el) ptx::tma_load_im2col_4d(b_dst, &tmB, fb, cc * kBK, p.ic_s * px.c - p.ic_p,
                                                    p.ic_s * px.r - p.ic_p, px.q, uint16_t(tap_j), uint16_t(tap_i));
                            if (++cc == p.ic_cpt) {
                                cc = 0;
                                if (++tap_j == p.ic_k) { tap_j = 0; ++tap_i; }
                            }
                        } else if constexpr (A_IM == 3) {
                            // swapped backward-weight: B = 16 pixels x (BNL/32 x 32 channels of a tap)
#pragma unroll
                            for (int c = 0; c < NBW; ++c)
                                if (el) ptx::tma_load_im2col_4d(b_dst + c * 32 * kBK * 4, &tmB, fb, bw_ch[c],
                                                        p.ic_s * px.c - p.ic_p, p.ic_s * px.r - p.ic_p, px.q,
                                                        uint16_t(bw_tj[c]), uint16_t(bw_ti[c]));
                            px.c += kBK;
                            while (px.c >= p.ic_m) {
                                px.c -= p.ic_m;
                                if (++px.r == p.ic_m) { px.r = 0; ++px.q; }
                            }
                        } else if constexpr (BN == 384 && B_MN) {
                            // 32-column boxes: the CTA's columns of sub-tile 1 (256/CG), then of sub-tile 2
                            const int nb = nt * BN;
#pragma unroll
                            for (int c = 0; c < 8 / CG; ++c)
                                if (el) ptx::tma_load_2d(b_dst + c * 32 * kBK * 4, &tmB, fb,
                                                 nb + int(rank) * (256 / CG) + 32 * c, k0);
#pragma unroll
                            for (int c = 0; c < 4 / CG; ++c)
                                if (el) ptx::tma_load_2d(b_dst + (8 / CG + c) * 32 * kBK * 4, &tmB, fb,
                                                 nb + 256 + int(rank) * (128 / CG) + 32 * c, k0);
                        } else if constexpr (BN == 384) {
                            // 64-row boxes: the CTA's rows of sub-tile 1 (256/CG), then of sub-tile 2 (128/CG)
                            const int nb = nt * BN;
#pragma unroll
                            for (int c = 0; c < 4 / CG; ++c)
                                if (el) ptx::tma_load_2d(b_dst + c * 64 * kBK * 4, &tmB, fb, k0,
                                                 nb + int(rank) * (256 / CG) + 64 * c);
#pragma unroll
                            for (int c = 0; c < 2 / CG; ++c)
                                if (el) ptx::tma_load_2d(b_dst + (4 / CG + c) * 64 * kBK * 4, &tmB, fb, k0,
                                                 nb + 256 + int(rank) * (128 / CG) + 64 * c);
                        } else if constexpr (!B_MN) {
                            if (el) ptx::tma_load_2d(b_dst, &tmB, fb, k0, n0);
                        } else {
#pragma unroll
                            for (int c = 0; c < BNL / 32; ++c)
                                if (el) ptx::tma_load_2d(b_dst + c * 32 * kBK * 4, &tmB, fb, n0 + 32 * c, k0);
                        }
                    }
                    __syncwarp();
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader CTA only) =====================
        // the whole warp walks the loop (warp-uniform operands in uniform registers); one
        // elected lane issues the MMAs and commits (ptx::elect_one)
        if (leader) {
            // (BN = 384: two MMAs per step, N = 256 into columns [0, 256) and N = 128 into [256, 384))
            constexpr uint32_t idesc = ptx::idesc_tf32(kBM * CG, BN > 256 ? 256 : BN, A_MN, B_MN);
            constexpr uint32_t idesc2 = ptx::idesc_tf32(kBM * CG, BN > 256 ? BN - 256 : BN, A_MN, B_MN);
            constexpr uint32_t idesc_mg = ptx::idesc_tf32(kBM, MG ? 2 * BN : BN, 0, 0);
            int stage = 0;
            uint32_t phase = 0;
            int local = 0;
            uint32_t gi = 0;  // k-blocks issued by this CTA (A_TM slot = gi % kASlots)
            WorkIter wi(p, group);
            Work w;
            for (; wi.next(p, ngroups, w); ++local) {
                const int kb0 = w.kb0, kb1 = w.kb1;
                const int acc = SB ? 0 : (local & 1);  // single-buffered: one accumulator set
                const uint32_t use = SB ? uint32_t(local) : uint32_t(local >> 1);
                ptx::mbar_wait(&tempty[acc], (use & 1) ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + uint32_t(acc * NACC * BN);
                auto mma = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t accumulate) {
                    if constexpr (CG == 1) ptx::mma_tf32(d, a, b, idesc, accumulate);
                    else ptx::mma_tf32_cg2(d, a, b, idesc, accumulate);
                };
                auto mma2 = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t accumulate) {
                    if constexpr (CG == 1) ptx::mma_tf32(d, a, b, idesc2, accumulate);
                    else ptx::mma_tf32_cg2(d, a, b, idesc2, accumulate);
                };
                auto mma_ts = [&](uint32_t d, uint32_t a, uint64_t b, uint32_t accumulate) {
                    if constexpr (CG == 1) ptx::mma_tf32_ts(d, a, b, idesc, accumulate);
                    else ptx::mma_tf32_ts_cg2(d, a, b, idesc, accumulate);
                };
                auto mma2_ts = [&](uint32_t d, uint32_t a, uint64_t b, uint32_t accumulate) {
                    if constexpr (CG == 1) ptx::mma_tf32_ts(d, a, b, idesc2, accumulate);
                    else ptx::mma_tf32_ts_cg2(d, a, b, idesc2, accumulate);
                };
                for (int kb = kb0; kb < kb1; ++kb, ++gi) {
                    // tdone implies the raw tiles of every CTA in the group landed
                    // (each transform warp waited on its own CTA's full barrier)
                    ptx::mbar_wait(&tdone[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t a_raw = ptx::smem_u32(smem + stage * C_::STAGE_BYTES);
                    const uint32_t b_raw = a_raw + B_OFF;
                    const uint32_t a_sml = a_raw + C_::RAW_BYTES;
                    const uint32_t b_sml = a_raw + BS_OFF;
                    if (ptx::elect_one()) {
                    if constexpr (A_TM) {
                        // A big | small for this k-block in TMEM slot gi % kASlots (16 + 16 columns)
                        const uint32_t a_big = tmem_base + A_COL + (gi % kASlots) * (2 * kBK);
                        const uint32_t a_small = a_big + kBK;
                        const uint32_t first = (kb > kb0) ? 1u : 0u;
                        if constexpr (BN == 384) {
                            // composite tile: N = 256 into [0, 256), N = 128 into [256, 384), same A
                            constexpr uint32_t SUB2 = uint32_t(256 / CG) * kBK * 4;
#pragma unroll
                            for (int kk = 0; kk < 2; ++kk) {
                                const uint32_t f = kk ? 1u : first;
                                mma_ts(d_tmem, a_small + kk * 8, tile_desc<B_MN>(b_raw, kk), f);
                                mma2_ts(d_tmem + 256, a_small + kk * 8, tile_desc<B_MN>(b_raw + SUB2, kk), f);
                            }
#pragma unroll
                            for (int kk = 0; kk < 2; ++kk) {
                                mma_ts(d_tmem, a_big + kk * 8, tile_desc<B_MN>(b_sml, kk), 1u);
                                mma2_ts(d_tmem + 256, a_big + kk * 8, tile_desc<B_MN>(b_sml + SUB2, kk), 1u);
                            }
#pragma unroll
                            for (int kk = 0; kk < 2; ++kk) {
                                mma_ts(d_tmem, a_big + kk * 8, tile_desc<B_MN>(b_raw, kk), 1u);
                                mma2_ts(d_tmem + 256, a_big + kk * 8, tile_desc<B_MN>(b_raw + SUB2, kk), 1u);
                            }
                        } else if constexpr (MG) {
                            // [A_big B_small | A_big B_big] over the 2 BN rows [small | raw] (the first
                            // MMA of a tile clears both halves), then A_small B_big into the upper half
#pragma unroll
                            for (int kk = 0; kk < 2; ++kk) {
                                ptx::mma_tf32_ts(d_tmem, a_big + kk * 8, tile_desc<false>(b_sml, kk), idesc_mg,
                                                 kk ? 1u : first);
                                ptx::mma_tf32_ts(d_tmem + BN, a_small + kk * 8, tile_desc<false>(b_raw, kk), idesc, 1u);
                            }
                        } else {
#pragma unroll
                        for (int kk = 0; kk < 2; ++kk)
                            mma_ts(d_tmem + kk * (NACC - 1) * BN, a_small + kk * 8, tile_desc<B_MN>(b_raw, kk),
                                   (NACC == 1 && kk) ? 1u : first);
#pragma unroll
                        for (int kk = 0; kk < 2; ++kk)
                            mma_ts(d_tmem + kk * (NACC - 1) * BN, a_big + kk * 8, tile_desc<B_MN>(b_sml, kk), 1u);
#pragma unroll
                        for (int kk = 0; kk < 2; ++kk)
                            mma_ts(d_tmem + kk * (NACC - 1) * BN, a_big + kk * 8, tile_desc<B_MN>(b_raw, kk), 1u);
                        }
                    } else if constexpr (BN == 384) {
                        // this CTA's B rows: 256/CG of the first sub-tile, then 128/CG of the second
                        // (K-major: 256/CG rows of 64 B; MN-major: (256/CG)/32 chunks of 2 KB -- same bytes)
                        constexpr uint32_t SUB2 = uint32_t(256 / CG) * kBK * 4;
#pragma unroll
                        for (int kk = 0; kk < kBK / 8; ++kk) {
                            const uint64_t ad = tile_desc<A_MN>(a_raw, kk), as = tile_desc<A_MN>(a_sml, kk);
                            const uint64_t b1 = tile_desc<B_MN>(b_raw, kk), b2 = tile_desc<B_MN>(b_raw + SUB2, kk);
                            const uint64_t s1 = tile_desc<B_MN>(b_sml, kk), s2 = tile_desc<B_MN>(b_sml + SUB2, kk);
                            const uint32_t first = (kb > kb0 || kk > 0) ? 1u : 0u;
                            mma(d_tmem, as, b1, first);
                            mma2(d_tmem + 256, as, b2, first);
                            mma(d_tmem, ad, s1, 1u);
                            mma2(d_tmem + 256, ad, s2, 1u);
                            mma(d_tmem, ad, b1, 1u);
                            mma2(d_tmem + 256, ad, b2, 1u);
                        }
                    } else if constexpr (CH2) {
                        // chain 0: k-blocks [kb0, kbh), chain 1: [kbh, kb1), each in its accumulator
                        const int kbh = kb0 + (kb1 - kb0 + 1) / 2;
                        const uint32_t dch = d_tmem + (kb >= kbh ? uint32_t(BN) : 0u);
#pragma unroll
                        for (int kk = 0; kk < kBK / 8; ++kk) {
                            const uint64_t ad = tile_desc<A_MN>(a_raw, kk);
                            const uint64_t bd = tile_desc<B_MN>(b_raw, kk);
                            const uint32_t first = ((kb != kb0 && kb != kbh) || kk > 0) ? 1u : 0u;
                            mma(dch, tile_desc<A_MN>(a_sml, kk), bd, first);
                            mma(dch, ad, tile_desc<B_MN>(b_sml, kk), 1u);
                            mma(dch, ad, bd, 1u);
                        }
                    } else if constexpr (NACC == 1) {
#pragma unroll
                        for (int kk = 0; kk < kBK / 8; ++kk) {
                            const uint64_t ad = tile_desc<A_MN>(a_raw, kk);
                            const uint64_t bd = tile_desc<B_MN>(b_raw, kk);
                            const uint32_t first = (kb > kb0 || kk > 0) ? 1u : 0u;
                            if (p.passes == 3) {
                                // small products first, big*big last
                                mma(d_tmem, tile_desc<A_MN>(a_sml, kk), bd, first);
                                mma(d_tmem, ad, tile_desc<B_MN>(b_sml, kk), 1u);
                                mma(d_tmem, ad, bd, 1u);
                            } else {
                                mma(d_tmem, ad, bd, first);
                            }
                        }
                    } else {
                        // K step kk accumulates into sub-accumulator kk; passes interleave
                        // the two so neighbouring MMAs are independent
                        const uint32_t first = (kb > kb0) ? 1u : 0u;
                        if (p.passes == 3) {
#pragma unroll
                            for (int kk = 0; kk < 2; ++kk)
                                mma(d_tmem + kk * BN, tile_desc<A_MN>(a_sml, kk), tile_desc<B_MN>(b_raw, kk), first);
#pragma unroll
                            for (int kk = 0; kk < 2; ++kk)
                                mma(d_tmem + kk * BN, tile_desc<A_MN>(a_raw, kk), tile_desc<B_MN>(b_sml, kk), 1u);
#pragma unroll
                            for (int kk = 0; kk < 2; ++kk)
                                mma(d_tmem + kk * BN, tile_desc<A_MN>(a_raw, kk), tile_desc<B_MN>(b_raw, kk), 1u);
                        } else {
#pragma unroll
                            for (int kk = 0; kk < 2; ++kk)
                                mma(d_tmem + kk * BN, tile_desc<A_MN>(a_raw, kk), tile_desc<B_MN>(b_raw, kk), first);
                        }
                    }
                    if constexpr (CG == 1) ptx::mma_commit(&empty[stage]);
                    else ptx::mma_commit_cg2(&empty[stage], 0x3);
                    }  // elect_one
                    __syncwarp();
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                if (ptx::elect_one()) {
                    if constexpr (CG == 1) ptx::mma_commit(&tfull[acc]);
                    else ptx::mma_commit_cg2(&tfull[acc], 0x3);
                }
                __syncwarp();
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ===================== epilogue (own TMEM lanes = own 128 rows) =====================
        const int q = warp & 3;
        const int rit = q * 32 + lane;  // row within this CTA's 128-row tile
        int local = 0;
        WorkIter wi(p, group);
        Work w;
        for (; wi.next(p, ngroups, w); ++local) {
            const int u = w.u;
            const int mt = u % p.num_m_tiles;
            const int rest = u / p.num_m_tiles;
            const int nt = rest % p.num_n_tiles;
            const int sp = rest / p.num_n_tiles;
            const int acc = SB ? 0 : (local & 1);
            const uint32_t use = SB ? uint32_t(local) : uint32_t(local >> 1);
            ptx::mbar_wait(&tfull[acc], use & 1);
            ptx::tc_fence_after();
            const int64_t row = int64_t(mt) * (kBM * CG) + int64_t(rank) * kBM + rit;
            bool row_ok = row < p.M;
            int64_t off = 0;
            if (row_ok) {
                const int64_t rq = row / p.mdiv, rr = row - rq * p.mdiv;
                row_ok = rr < p.mlim;
                off = rq * p.s_mq + rr * p.s_mr + int64_t(sp) * p.s_split;
            }
            const int n0 = nt * BN;
            // final values of columns n0 + c0 .. +31 of this thread's row -> output map
            auto store32 = [&](uint32_t* v, int c0) {
                const int64_t sn = p.s_n;
                const int nlim = p.N - (n0 + c0);
                if (!row_ok) return;
                if (p.bias || p.relu) {  // fused bias + ReLU (conv layer epilogue)
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        float f = __uint_as_float(v[j]);
                        if (p.bias && j < nlim) f += __ldg(p.bias + n0 + c0 + j);
                        if (p.relu) f = fmaxf(f, 0.f);
                        v[j] = __float_as_uint(f);
                    }
                }
                if (p.ndiv) {
                    // two-level column map (slab-major dDhat): walk (n / ndiv, n % ndiv)
                    const int nq = (n0 + c0) / p.ndiv;
                    int nr = (n0 + c0) - nq * p.ndiv;
                    float* dst = p.C + off + int64_t(nq) * p.s_nq + int64_t(nr) * sn;
                    const int64_t wrap = p.s_nq - int64_t(p.ndiv) * sn;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        if (j < nlim && nr < p.nmlim) *dst = __uint_as_float(v[j]);
                        dst += sn;
                        if (++nr == p.ndiv) { nr = 0; dst += wrap; }
                    }
                    return;
                }
                float* dst = p.C + off + int64_t(n0 + c0) * sn;
                if (nlim >= 32 && sn == 1 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
                    // row-major output (lane = row): 32 consecutive floats per thread
                    float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        d4[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                            __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
                } else if (nlim >= 32) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        *dst = __uint_as_float(v[j]);
                        dst += sn;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        if (j < nlim) *dst = __uint_as_float(v[j]);
                        dst += sn;
                    }
                }
            };
            // TRO: columns n0 + c0 + lane of rows (this warp's 32) through the staging block
            // (row offsets / validity / bias: this tile's per-lane values, published once per
            // tile in a per-warp table and read back as smem broadcasts)
            if constexpr (TRO) {
                int64_t* roff = reinterpret_cast<int64_t*>(epi + 4 * 32 * 33) + q * 32;
                float* rb = reinterpret_cast<float*>(epi + 4 * 32 * 33 + 4 * 32 * 2) + q * 64;
                roff[lane] = row_ok ? off : int64_t(-1);
                rb[lane] = (p.bias && row_ok) ? __ldg(p.bias + row) : 0.f;
                __syncwarp();
            }
            auto store32_t = [&](const uint32_t* v, int c0) {
                float* buf = epi + q * 32 * 33;
                const int64_t* roff = reinterpret_cast<const int64_t*>(epi + 4 * 32 * 33) + q * 32;
                const float* rb = reinterpret_cast<const float*>(epi + 4 * 32 * 33 + 4 * 32 * 2) + q * 64;
#pragma unroll
                for (int j = 0; j < 32; ++j) buf[lane * 33 + j] = __uint_as_float(v[j]);
                __syncwarp();
                const int col = n0 + c0 + lane;
                int64_t coff = -1;
                if (col < p.N) {
                    if (p.ndiv) {
                        const int cq = col / p.ndiv;
                        coff = int64_t(cq) * p.s_nq + int64_t(col - cq * p.ndiv) * p.s_n;
                    } else {
                        coff = int64_t(col) * p.s_n;
                    }
                }
#pragma unroll 8
                for (int r = 0; r < 32; ++r) {
                    const int64_t ro = roff[r];
                    float f = buf[r * 33 + lane] + rb[r];
                    if (p.relu) f = fmaxf(f, 0.f);
                    if (ro >= 0 && coff >= 0) p.C[ro + coff] = f;
                }
                __syncwarp();
            };
            // stream-K part: this group's share of a tile cut at boundary `bnd` between
            // groups bnd and bnd + 1 (part 0 = leading k-blocks, 1 = trailing)
            const int bnd = (w.kind == 1) ? group : group - 1;
            float* part = (w.kind == 0) ? nullptr
                                        : p.sk_part + (int64_t((bnd * 2 + (w.kind - 1)) * CG + int(rank)) * BN) * kBM;
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t v[32];
                const uint32_t tcol = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * NACC * BN + c0);
                ptx::tmem_ld_32x32b_x32(tcol, v);
                if constexpr (NACC == 2) {
                    uint32_t v2[32];
                    ptx::tmem_ld_32x32b_x32(tcol + BN, v2);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + __uint_as_float(v2[j]));
                }
                ptx::tmem_ld_wait();
                if (part) {
                    // column-major partial tile: lanes (rows) coalesced
#pragma unroll
                    for (int j = 0; j < 32; ++j) __stcg(part + (c0 + j) * kBM + rit, __uint_as_float(v[j]));
                } else if constexpr (TRO) {
                    store32_t(v, c0);
                } else {
                    store32(v, c0);
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (CG == 1) ptx::mbar_arrive(&tempty[acc]);
                else ptx::mbar_arrive_remote(tempty_leader + uint32_t(acc * 8));
            }
            if (part) {
                // second finisher of the two parts sums them (part 0 + part 1: the same
                // result whichever group arrives last) and writes the tile
                __threadfence();
                ptx::named_bar_sync(1, 128);
                if (rit == 0) *sk_flag = atomicAdd(p.sk_cnt + bnd * CG + int(rank), 1);
                ptx::named_bar_sync(1, 128);
                if (*sk_flag == 1) {
                    __threadfence();
                    const float* p0 = p.sk_part + (int64_t((bnd * 2) * CG + int(rank)) * BN) * kBM;
                    const float* p1 = p0 + int64_t(CG) * BN * kBM;
#pragma unroll 1
                    for (int c0 = 0; c0 < BN; c0 += 32) {
                        uint32_t v[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            v[j] = __float_as_uint(__ldcg(p0 + (c0 + j) * kBM + rit) + __ldcg(p1 + (c0 + j) * kBM + rit));
                        if constexpr (TRO) store32_t(v, c0);
                        else store32(v, c0);
                    }
                    if (rit == 0) p.sk_cnt[bnd * CG + int(rank)] = 0;  // ready for the next launch
                }
                ptx::named_bar_sync(1, 128);  // sk_flag reuse
            }
        }
    } else if (warp >= 8) {
        // ===================== 3xTF32 transform (own tiles) =====================
        const int tg = (warp - 8) >> 2;                   // transform group: k-blocks gi % kTGroups == tg
        const int t = threadIdx.x - 256 - tg * 128;
        int stage = 0;
        uint32_t fphase = 0;  // bit s: phase parity of this group's full[tg * STAGES + s]
        uint32_t gi = 0;
        WorkIter wi(p, group);
        Work w;
        while (wi.next(p, ngroups, w)) {
            for (int kb = w.kb0; kb < w.kb1; ++kb, ++gi) {
                if (int(gi % kTGroups) != tg) {
                    if (++stage == STAGES) stage = 0;
                    continue;
                }
                ptx::mbar_wait(&full[tg * STAGES + stage], (fphase >> stage) & 1u);
                fphase ^= 1u << stage;
                const uint32_t raw = ptx::smem_u32(smem + stage * C_::STAGE_BYTES);
                if constexpr (A_TM) {
                    // the MMAs of k-block gi - kASlots (same TMEM slot) must be complete
                    if (gi >= kASlots) {
                        const uint32_t g2 = gi - kASlots;
                        ptx::mbar_wait(&empty[g2 % STAGES], (g2 / STAGES) & 1);
                    }
                    // row r of the K-major SWIZZLE_64B A tile: 16-byte chunk c at (c ^ (r/2 % 4))
                    const int r = (warp & 3) * 32 + lane;
                    uint32_t v[32];
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const float4 x = ptx::lds128(raw + r * 64 + ((c ^ ((r >> 1) & 3)) << 4));
                        const float4 sm = small_part(x);
                        v[4 * c + 0] = __float_as_uint(x.x) & 0xFFFFE000u;
                        v[4 * c + 1] = __float_as_uint(x.y) & 0xFFFFE000u;
                        v[4 * c + 2] = __float_as_uint(x.z) & 0xFFFFE000u;
                        v[4 * c + 3] = __float_as_uint(x.w) & 0xFFFFE000u;
                        v[16 + 4 * c + 0] = __float_as_uint(sm.x);
                        v[16 + 4 * c + 1] = __float_as_uint(sm.y);
                        v[16 + 4 * c + 2] = __float_as_uint(sm.z);
                        v[16 + 4 * c + 3] = __float_as_uint(sm.w);
                    }
                    ptx::tmem_st_32x32b_x32(tmem_base + (uint32_t((warp & 3) * 32) << 16) + A_COL +
                                                (gi % kASlots) * (2 * kBK),
                                            v);
                    ptx::tmem_st_wait();
                    // B small part in smem as usual
                    for (int i = t; i < int(C_::B_BYTES / 16); i += 128) {
                        const float4 x = ptx::lds128(raw + B_OFF + i * 16);
                        ptx::sts128(raw + BS_OFF + i * 16, small_part(x));
                    }
                    ptx::fence_proxy_async_smem();
                    ptx::tc_fence_before();
                } else if (p.passes == 3) {
                    constexpr int n4 = C_::RAW_BYTES / 16;
#pragma unroll 4
                    for (int i = t; i < n4; i += 128) {
                        const float4 v = ptx::lds128(raw + i * 16);
                        ptx::sts128(raw + C_::RAW_BYTES + i * 16, small_part(v));
                    }
                    ptx::fence_proxy_async_smem();
                }
                __syncwarp();
                if (lane == 0) {
                    if constexpr (CG == 1) ptx::mbar_arrive(&tdone[stage]);
                    else ptx::mbar_arrive_remote(tdone_leader + uint32_t(stage * 8));
                }
                if (++stage == STAGES) stage = 0;
            }
        }
    }

    ptx::tc_fence_before();
    if constexpr (CG == 2) ptx::cluster_sync();
    else __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<TMEM_COLS, CG>(tmem_base);
    }
}

template <int BN, int A_MN, int B_MN, int CG, int A_IM, int A_TM = 0, int TRO = 0, int CH2 = 0>
cudaError_t launch(const CUtensorMap& ta, const CUtensorMap& tb, const KParams& kp, cudaStream_t st) {
    using C_ = Cfg<BN, CG, TRO>;
    auto kern = gemm3xtf32_kernel<BN, A_MN, B_MN, CG, A_IM, A_TM, TRO, CH2>;
    // per call (idempotent, ~1 us): the attribute is per device, and callers may switch devices
    // or threads; a process-wide "done" flag would miss the second GPU
    {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C_::SMEM_BYTES);
        if (e != cudaSuccess) return e;
    }
    const int sms = num_sms() / CG * CG;
    const int grid = kp.sk_len ? sms : std::min(kp.units * CG, sms);
    PhaseScope ps(kPhaseGemm, st, 2.0 * double(kp.M) * double(kp.N) * double(kp.K), 0);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C_::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ta, tb, kp);
    note_launch();
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// CCT_TUNE_A_TMEM_WIDE (default 1): 192 / 256 / 384-wide CTA-pair tiles with a K-major A keep A
// in TMEM too (the 3xTF32 MMAs then read only B from smem): +12 % on a 192-wide microbenchmark,
// 1-4 % on the CaffeNet forward / backward-data GEMMs (the 256 / 384 tiles give up the second
// accumulator buffer for the A ring)
inline int a_tmem_wide() { return tuning(CCT_TUNE_A_TMEM_WIDE); }

// CCT_TUNE_A_TMEM: 0 keeps narrow tiles on the smem-A path, 1 A in TMEM with two
// sub-accumulators, 2 A in TMEM with one accumulator and a deeper A ring (A/B)
inline int a_in_tmem_mode() { return tuning(CCT_TUNE_A_TMEM); }

template <int BN, int CG>
cudaError_t dispatch_std(const GemmProblem& g, const CUtensorMap& ta, const CUtensorMap& tb,
                         const KParams& kp, cudaStream_t st) {
    const bool amn = g.A.major == Major::MN, bmn = g.B.major == Major::MN;
    if (g.chain2) {  // two-chain accumulation (wide tiles)
        if constexpr (BN >= 192) {
            if (g.passes != 3) return cudaErrorInvalidValue;
            if (g.im2col.x && g.im2col.operand == 1) {
                if (amn || bmn) return cudaErrorInvalidValue;
                return launch<BN, 0, 0, CG, 2, 0, 0, 1>(ta, tb, kp, st);
            }
            if (g.im2col.x && g.im2col.operand == 2) {  // swapped backward-weight of a narrow bank
                if (!bmn) return cudaErrorInvalidValue;
                return amn ? launch<BN, 1, 1, CG, 3, 0, 0, 1>(ta, tb, kp, st) : launch<BN, 0, 1, CG, 3, 0, 0, 1>(ta, tb, kp, st);
            }
            if (g.im2col.x && g.im2col.operand == 0) {  // forward (K, K) / backward-weight (MN, K | MN)
                if (!amn && !bmn) return launch<BN, 0, 0, CG, 1, 0, 0, 1>(ta, tb, kp, st);
                if (amn && bmn) return launch<BN, 1, 1, CG, 1, 0, 0, 1>(ta, tb, kp, st);
                if (amn) return launch<BN, 1, 0, CG, 1, 0, 0, 1>(ta, tb, kp, st);
                return cudaErrorInvalidValue;
            }
            if (!g.im2col.x) {
                if (!amn && !bmn) return launch<BN, 0, 0, CG, 0, 0, 0, 1>(ta, tb, kp, st);
                if (amn && !bmn) return launch<BN, 1, 0, CG, 0, 0, 0, 1>(ta, tb, kp, st);  // materialised wgrad
                if (!amn && bmn) return launch<BN, 0, 1, CG, 0, 0, 0, 1>(ta, tb, kp, st);  // swapped (narrow bank)
                if (amn && bmn) return launch<BN, 1, 1, CG, 0, 0, 0, 1>(ta, tb, kp, st);   // swapped, dy NHWC
            }
        }
        return cudaErrorInvalidValue;
    }
    if (g.C.transposed) {  // swapped forward of a narrow bank: y rows = channels
        if constexpr (CG == 1 && BN >= 192) {
            if (amn || bmn) return cudaErrorInvalidValue;
            if (g.im2col.x && g.im2col.operand == 1) return launch<BN, 0, 0, 1, 2, 0, 1>(ta, tb, kp, st);
            if (!g.im2col.x) return launch<BN, 0, 0, 1, 0, 0, 1>(ta, tb, kp, st);
        }
        return cudaErrorInvalidValue;
    }
    if constexpr (BN == 192 || BN == 256) {  // A in TMEM for wide tiles (K-major A): fewer smem reads
        if (CG == 2 && a_tmem_wide() && !amn && g.passes == 3 && !g.chain2 && !g.C.transposed) {
            if (g.im2col.x && g.im2col.operand == 1) return bmn ? cudaErrorInvalidValue : launch<BN, 0, 0, CG, 2, 1>(ta, tb, kp, st);
            if (g.im2col.x && g.im2col.operand == 0) return bmn ? cudaErrorInvalidValue : launch<BN, 0, 0, CG, 1, 1>(ta, tb, kp, st);
            if (!g.im2col.x)
                return bmn ? launch<BN, 0, 1, CG, 0, 1>(ta, tb, kp, st) : launch<BN, 0, 0, CG, 0, 1>(ta, tb, kp, st);
        }
    }
    if constexpr (BN <= 96) {
        const int atm = g.im2col.operand >= 1 ? 0 : a_in_tmem_mode();
        if constexpr (CG == 1) {
            if (!amn && !bmn && g.passes == 3 && atm == 3)
                return g.im2col.x ? launch<BN, 0, 0, 1, 1, 3>(ta, tb, kp, st) : launch<BN, 0, 0, 1, 0, 3>(ta, tb, kp, st);
        }
        if (!amn && g.passes == 3 && atm == 2) {
            if (g.im2col.x) return bmn ? cudaErrorInvalidValue : launch<BN, 0, 0, CG, 1, 2>(ta, tb, kp, st);
            return bmn ? launch<BN, 0, 1, CG, 0, 2>(ta, tb, kp, st) : launch<BN, 0, 0, CG, 0, 2>(ta, tb, kp, st);
        }
        if (!amn && g.passes == 3 && atm) {  // (atm 3 on a CTA pair or MN-major B: the two-sub-accumulator form)
            if (g.im2col.x) return bmn ? cudaErrorInvalidValue : launch<BN, 0, 0, CG, 1, 1>(ta, tb, kp, st);
            return bmn ? launch<BN, 0, 1, CG, 0, 1>(ta, tb, kp, st) : launch<BN, 0, 0, CG, 0, 1>(ta, tb, kp, st);
        }
    }
    if (g.im2col.x && g.im2col.operand == 2) {  // B = MN-major im2col (swapped backward-weight)
        if (!bmn) return cudaErrorInvalidValue;
        return amn ? launch<BN, 1, 1, CG, 3>(ta, tb, kp, st) : launch<BN, 0, 1, CG, 3>(ta, tb, kp, st);
    }
    if (g.im2col.x && g.im2col.operand == 1) {  // B = im2col (swapped implicit GEMM), K-major A and B
        if (amn || bmn) return cudaErrorInvalidValue;
        return launch<BN, 0, 0, CG, 2>(ta, tb, kp, st);
    }
    if (g.im2col.x) {  // implicit Type 1: forward / backward-data (K, K), backward-weight (MN, K|MN)
        if (!amn && !bmn) return launch<BN, 0, 0, CG, 1>(ta, tb, kp, st);
        if (amn && !bmn) return launch<BN, 1, 0, CG, 1>(ta, tb, kp, st);
        if (amn && bmn) return launch<BN, 1, 1, CG, 1>(ta, tb, kp, st);  // backward-weight, dy in NHWC
        return cudaErrorInvalidValue;
    }
    if (!amn && !bmn) return launch<BN, 0, 0, CG, 0>(ta, tb, kp, st);
    if (amn && bmn) return launch<BN, 1, 1, CG, 0>(ta, tb, kp, st);
    if (amn && !bmn) return launch<BN, 1, 0, CG, 0>(ta, tb, kp, st);
    return launch<BN, 0, 1, CG, 0>(ta, tb, kp, st);
}

template <int BN, int CG>
cudaError_t dispatch_layout(const GemmProblem& g, const CUtensorMap& ta, const CUtensorMap& tb,
                            const KParams& kp, cudaStream_t st) {
    if constexpr (BN == 384) {  // 256 + 128 composite tile; A ordinary or im2col (A side)
        const bool amn = g.A.major == Major::MN, bmn = g.B.major == Major::MN;
        if (g.chain2 || g.C.transposed || g.passes != 3 || (g.im2col.x && g.im2col.operand != 0))
            return cudaErrorInvalidValue;
        if (CG == 2 && a_tmem_wide() && !amn) {  // A in TMEM (CTA pairs: single CTAs have too few stages)
            if (g.im2col.x) return bmn ? cudaErrorInvalidValue : launch<384, 0, 0, CG, 1, 1>(ta, tb, kp, st);
            return bmn ? launch<384, 0, 1, CG, 0, 1>(ta, tb, kp, st) : launch<384, 0, 0, CG, 0, 1>(ta, tb, kp, st);
        }
        if (g.im2col.x) {
            if (!amn && !bmn) return launch<384, 0, 0, CG, 1>(ta, tb, kp, st);     // forward
            if (amn && bmn) return launch<384, 1, 1, CG, 1>(ta, tb, kp, st);       // backward-weight, dy NHWC
            if (amn) return launch<384, 1, 0, CG, 1>(ta, tb, kp, st);              // backward-weight, dRhat
            return cudaErrorInvalidValue;
        }
        if (!amn && !bmn) return launch<384, 0, 0, CG, 0>(ta, tb, kp, st);
        if (!amn && bmn) return launch<384, 0, 1, CG, 0>(ta, tb, kp, st);          // swapped materialised wgrad
        if (amn && !bmn) return launch<384, 1, 0, CG, 0>(ta, tb, kp, st);          // materialised wgrad
        return launch<384, 1, 1, CG, 0>(ta, tb, kp, st);
    } else {
        return dispatch_std<BN, CG>(g, ta, tb, kp, st);
    }
}

// explicit instantiation units (gemm_i<BN>_<CG>.cu) define these
#define CCT_GEMM_DISPATCH_DECL(BN, CG)                                                              \
    extern template cudaError_t dispatch_layout<BN, CG>(const GemmProblem&, const CUtensorMap&,     \
                                                        const CUtensorMap&, const KParams&, cudaStream_t);
CCT_GEMM_DISPATCH_DECL(384, 1) CCT_GEMM_DISPATCH_DECL(256, 1) CCT_GEMM_DISPATCH_DECL(192, 1)
CCT_GEMM_DISPATCH_DECL(128, 1) CCT_GEMM_DISPATCH_DECL(96, 1) CCT_GEMM_DISPATCH_DECL(64, 1)
CCT_GEMM_DISPATCH_DECL(384, 2) CCT_GEMM_DISPATCH_DECL(256, 2) CCT_GEMM_DISPATCH_DECL(192, 2)
CCT_GEMM_DISPATCH_DECL(128, 2) CCT_GEMM_DISPATCH_DECL(96, 2) CCT_GEMM_DISPATCH_DECL(64, 2)
#define CCT_GEMM_INSTANTIATE(BN, CG)                                                                \
    namespace cct {                                                                                 \
    namespace gk {                                                                                  \
    template cudaError_t dispatch_layout<BN, CG>(const GemmProblem&, const CUtensorMap&, const CUtensorMap&, \
                                                 const KParams&, cudaStream_t);                     \
    }                                                                                               \
    }

}  // namespace gk
}  // namespace cct
