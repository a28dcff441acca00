// lowering23.cu -- the HBM-streaming Type 2 / Type 3 kernels of the training path.
//
// Type 2 and Type 3 move k (T2) or k^2 (T3) times the output through HBM: the
// forward GEMM writes Rhat (b R m x k o, b R^2 x k^2 o) and lift sums k / k^2
// shifted taps of it; the backward expands dy into dRhat^T of the same size
// (SPEC.md:121-129 and the adjoint).  These kernels are organised so every byte
// of the big operand streams once, in long contiguous runs:
//
//   Rhat, plane-major (written by the forward GEMM's epilogue output map):
//       Rhat[((q * ncols) + col) * rpi + prow]     col = (oj, tap), prow = padded-row pixel
//     so the k^a tap planes of one output channel of one image are ONE contiguous
//     block (conv2 T3: 25 x 961 floats) -- lift_planes reads it as one stream per
//     block and writes the output plane(s) once.
//   dRhat^T (the backward GEMMs' operand, [col][ldr]): expand_planes stages the dy
//     planes of (image, 8 channels) in shared memory once and writes every tap's
//     run of rpi floats as a pure store stream.
//   Dhat2 / Dhat3 (internal row order): lower_rows writes the lowered rows of one
//     padded input row (q, Y) -- m rows of k d (T2) or R rows of d (T3), contiguous
//     -- from one coalesced read of that input row (float4, depth % 4 == 0).
//
// y / dy may be NCHW (OutputBatch) or NHWC (Geo::yl); NHWC planes go through the
// same shared-memory block so the big stream keeps its layout.
// Summation orders equal lift_kernel's (taps i then j ascending): the fast path and
// the phase-level API give bit-identical results.
#include <algorithm>

#include "common.cuh"
#include "lowering.cuh"
#include "ptx.cuh"

namespace cct {

namespace {

constexpr int kThreads = 256;
constexpr int kG = 8;  // output channels (planes) per block

// floor(v / d) for 0 <= v < 2^22 and 1 <= d < 2^10 from a float reciprocal plus one fix-up
__device__ __forceinline__ int fdiv(int v, int d, float inv) {
    int qv = __float2int_rz(float(v) * inv);
    if (qv * d > v) --qv;
    else if ((qv + 1) * d <= v) ++qv;
    return qv;
}

// One block per (image, kG output channels).  A thread owns output pixels (pix, pix + kThreads,
// ...) and, for each, walks the kG channels and their k^a taps: its (row, column) split is done
// once per pixel, and the kG x k^a loads of a pixel are independent (memory-level parallelism;
// consecutive threads read consecutive floats of a tap plane).
template <int TYPE, bool NHWC>
__global__ void __launch_bounds__(kThreads) lift_planes_kernel(const float* __restrict__ rh, float* __restrict__ y,
                                                               Geo g) {
    extern __shared__ float acc_s[];  // NHWC: kG x m^2 staged outputs
    const int m = int(g.m), mm = m * m, o = int(g.o), k = int(g.k), s = int(g.s), R = int(g.R);
    const int taps = TYPE == 2 ? k : k * k;
    const int64_t rpi = TYPE == 2 ? int64_t(R) * m : int64_t(R) * R;
    const int ngroups = (o + kG - 1) / kG;
    const float inv_m = 1.f / float(m);
    // tap strides within a channel's plane block: i (row tap), j (column tap, T3)
    const int64_t si = TYPE == 2 ? rpi + m : int64_t(k) * rpi + R, sj = rpi + 1;
    for (int64_t blk = blockIdx.x; blk < g.b * ngroups; blk += gridDim.x) {
        const int64_t q = blk / ngroups;
        const int oj0 = int(blk - q * ngroups) * kG;
        const int G = min(kG, o - oj0);
        const float* pl0 = rh + (q * o + oj0) * int64_t(taps) * rpi;
        for (int pix = threadIdx.x; pix < mm; pix += kThreads) {
            const int r = fdiv(pix, m, inv_m), c = pix - r * m;
            const int64_t off = TYPE == 2 ? int64_t(s) * r * m + c : int64_t(s) * r * R + int64_t(s) * c;
            float a[kG];
#pragma unroll
            for (int gl = 0; gl < kG; ++gl) a[gl] = 0.f;
            const float* p0 = pl0 + off;
            const int64_t sg = int64_t(taps) * rpi;  // channel stride
            // taps i then j ascending per channel (lift_kernel's order); the kG channels' loads
            // of a tap are independent
            // (measured: T2 fastest with the channels innermost, T3 with each channel's k x k
            // taps innermost -- 2.0 vs 0.4 TB/s and 2.2 vs 1.2 TB/s)
            if constexpr (TYPE == 2) {
                for (int i = 0; i < k; ++i) {
#pragma unroll
                    for (int gl = 0; gl < kG; ++gl)
                        if (gl < G) a[gl] += __ldg(p0 + gl * sg + i * si);
                }
            } else {
#pragma unroll
                for (int gl = 0; gl < kG; ++gl) {
                    if (gl < G) {
                        for (int i = 0; i < k; ++i) {
                            const float* pi = p0 + gl * sg + i * si;
#pragma unroll 3
                            for (int j = 0; j < k; ++j) a[gl] += __ldg(pi + j * sj);
                        }
                    }
                }
            }
#pragma unroll
            for (int gl = 0; gl < kG; ++gl) {
                if (gl < G) {
                    if constexpr (NHWC) acc_s[gl * mm + pix] = a[gl];
                    else y[(q * o + oj0 + gl) * mm + pix] = a[gl];
                }
            }
        }
        if constexpr (NHWC) {
            __syncthreads();
            const float inv_g = 1.f / float(G);
            for (int e = threadIdx.x; e < G * mm; e += kThreads) {
                const int pix = fdiv(e, G, inv_g), gl = e - pix * G;
                y[(q * mm + pix) * o + oj0 + gl] = acc_s[gl * mm + pix];
            }
            __syncthreads();
        }
    }
}

// Staged variant: the block's contiguous run of tap planes (G channels x k^a planes of rpi
// floats) is streamed into shared memory with coalesced loads first, so the HBM read is one
// sequential stream per block; the k^a-tap sums then read shared memory (same summation order).
template <int TYPE, bool NHWC>
__global__ void __launch_bounds__(kThreads) lift_staged_kernel(const float* __restrict__ rh, float* __restrict__ y,
                                                               Geo g, int gmax) {
    extern __shared__ float sm[];  // gmax x taps x rpi staged planes [+ NHWC: gmax x m^2 outputs]
    const int m = int(g.m), mm = m * m, o = int(g.o), k = int(g.k), s = int(g.s), R = int(g.R);
    const int taps = TYPE == 2 ? k : k * k;
    const int rpi = TYPE == 2 ? R * m : R * R;
    const int blk_floats = taps * rpi;
    const int ngroups = (o + gmax - 1) / gmax;
    const float inv_mm = 1.f / float(mm), inv_m = 1.f / float(m);
    float* acc_s = sm + gmax * blk_floats;
    for (int64_t blk = blockIdx.x; blk < g.b * ngroups; blk += gridDim.x) {
        const int64_t q = blk / ngroups;
        const int oj0 = int(blk - q * ngroups) * gmax;
        const int G = min(gmax, o - oj0);
        const float* src = rh + (q * o + oj0) * int64_t(blk_floats);
        const int total = G * blk_floats;
#pragma unroll 4
        for (int e = threadIdx.x; e < total; e += kThreads) sm[e] = __ldg(src + e);
        __syncthreads();
        for (int e = threadIdx.x; e < G * mm; e += kThreads) {
            const int gl = fdiv(e, mm, inv_mm), pix = e - gl * mm;
            const int r = fdiv(pix, m, inv_m), c = pix - r * m;
            const float* pl = sm + gl * blk_floats;
            float a = 0.f;
            if constexpr (TYPE == 2) {
                const float* p0 = pl + s * r * m + c;
                for (int i = 0; i < k; ++i) a += p0[i * (rpi + m)];
            } else {
                const float* p0 = pl + s * r * R + s * c;
                for (int i = 0; i < k; ++i) {
                    const float* pi = p0 + i * (k * rpi + R);
                    for (int j = 0; j < k; ++j) a += pi[j * (rpi + 1)];
                }
            }
            if constexpr (NHWC) acc_s[gl * mm + pix] = a;
            else y[(q * o + oj0) * mm + e] = a;
        }
        if constexpr (NHWC) {
            __syncthreads();
            const float inv_g = 1.f / float(G);
            for (int e = threadIdx.x; e < G * mm; e += kThreads) {
                const int pix = fdiv(e, G, inv_g), gl = e - pix * G;
                y[(q * mm + pix) * o + oj0 + gl] = acc_s[gl * mm + pix];
            }
        }
        __syncthreads();
    }
}

// Bulk-staged variant: the block's contiguous run of tap planes arrives by one 1D bulk copy
// (TMA engine, cp.async.bulk) into one of two shared-memory buffers while the block sums the
// previous run out of the other -- HBM streams continuously, no load instructions.  The copy
// starts at the 16-byte boundary below the run (off0 = 0..3 floats) and ends at the one above it,
// except at the end of Rhat (`total` floats), whose last <= 3 floats are plain loads.  Same
// summation order as lift_kernel (bit-identical).
template <int TYPE, bool NHWC>
__global__ void __launch_bounds__(kThreads) lift_bulk_kernel(const float* __restrict__ rh, float* __restrict__ y,
                                                             Geo g, int gmax, int64_t total) {
    extern __shared__ __align__(16) float smb[];  // 2 x (gmax x taps x rpi + 8) staged runs [+ NHWC outputs]
    __shared__ __align__(8) uint64_t bar[2];
    const int m = int(g.m), mm = m * m, o = int(g.o), k = int(g.k), s = int(g.s), R = int(g.R);
    const int taps = TYPE == 2 ? k : k * k;
    const int rpi = TYPE == 2 ? R * m : R * R;
    const int blk_floats = taps * rpi;
    const int buf_floats = (gmax * blk_floats + 8 + 3) & ~3;  // 16-byte aligned buffers
    const int ngroups = (o + gmax - 1) / gmax;
    const int64_t nblk = g.b * ngroups;
    const float inv_mm = 1.f / float(mm), inv_m = 1.f / float(m);
    float* acc_s = smb + 2 * buf_floats;
    // run [a0, a1) floats of block blk, copied to 16-byte aligned [c0, c1) (c1 <= total rounded down)
    auto span = [&](int64_t blk, int64_t& a0, int64_t& a1, int64_t& c0, int64_t& c1) {
        const int64_t q = blk / ngroups;
        const int oj0 = int(blk - q * ngroups) * gmax;
        a0 = (q * o + oj0) * int64_t(blk_floats);
        a1 = a0 + int64_t(min(gmax, o - oj0)) * blk_floats;
        c0 = a0 & ~int64_t(3);
        c1 = min((a1 + 3) & ~int64_t(3), total & ~int64_t(3));
    };
    auto issue = [&](int64_t blk, int b) {
        int64_t a0, a1, c0, c1;
        span(blk, a0, a1, c0, c1);
        const uint32_t bytes = c1 > c0 ? uint32_t(c1 - c0) * 4u : 0u;
        ptx::mbar_arrive_expect_tx(&bar[b], bytes);
        if (bytes) ptx::bulk_load(smb + b * buf_floats, rh + c0, bytes, &bar[b]);
    };
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar[0], 1);
        ptx::mbar_init(&bar[1], 1);
        ptx::fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x < nblk) issue(blockIdx.x, 0);
    int it = 0;
    for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x, ++it) {
        const int b = it & 1;
        if (threadIdx.x == 0 && blk + gridDim.x < nblk) issue(blk + gridDim.x, b ^ 1);
        int64_t a0, a1, c0, c1;
        span(blk, a0, a1, c0, c1);
        const float* sm = smb + b * buf_floats + (a0 - c0);  // the run's first float
        ptx::mbar_wait(&bar[b], uint32_t(it >> 1) & 1u);
        if (c1 < a1) {  // end of Rhat: the last floats by plain loads
            if (threadIdx.x == 0)
                for (int64_t e = max(c1, a0); e < a1; ++e) smb[b * buf_floats + (e - c0)] = __ldg(rh + e);
            __syncthreads();
        }
        const int64_t q = blk / ngroups;
        const int oj0 = int(blk - q * ngroups) * gmax;
        const int G = min(gmax, o - oj0);
        for (int e = threadIdx.x; e < G * mm; e += kThreads) {
            const int gl = fdiv(e, mm, inv_mm), pix = e - gl * mm;
            const int r = fdiv(pix, m, inv_m), c = pix - r * m;
            const float* pl = sm + gl * blk_floats;
            float a = 0.f;
            if constexpr (TYPE == 2) {
                const float* p0 = pl + s * r * m + c;
                for (int i = 0; i < k; ++i) a += p0[i * (rpi + m)];
            } else {
                const float* p0 = pl + s * r * R + s * c;
                for (int i = 0; i < k; ++i) {
                    const float* pi = p0 + i * (k * rpi + R);
                    for (int j = 0; j < k; ++j) a += pi[j * (rpi + 1)];
                }
            }
            if constexpr (NHWC) acc_s[gl * mm + pix] = a;
            else y[(q * o + oj0) * mm + e] = a;
        }
        if constexpr (NHWC) {
            __syncthreads();
            const float inv_g = 1.f / float(G);
            for (int e = threadIdx.x; e < G * mm; e += kThreads) {
                const int pix = fdiv(e, G, inv_g), gl = e - pix * G;
                y[(q * mm + pix) * o + oj0 + gl] = acc_s[gl * mm + pix];
            }
        }
        __syncthreads();  // buffer b is refilled by the issue of iteration it + 1
    }
}

// One block per (image, kG channels): the dy planes are staged in shared memory once; a thread
// owns lowered rows (idx, idx + kThreads, ...) of an image's run, splits idx once, and writes
// that row of every (channel, tap) column -- kG k^a independent stores per row, each warp a
// contiguous run.
template <int TYPE, bool NHWC>
__global__ void __launch_bounds__(kThreads) expand_planes_kernel(const float* __restrict__ dy, float* __restrict__ drt,
                                                                 Geo g, int64_t ldr) {
    extern __shared__ float sdy[];  // kG x m^2 dy values of (q, oj0 .. oj0 + G)
    const int m = int(g.m), mm = m * m, o = int(g.o), k = int(g.k), s = int(g.s), R = int(g.R);
    const int taps = TYPE == 2 ? k : k * k;
    const int rw = TYPE == 2 ? m : R;  // lowered rows per padded input row
    const int rpi = R * rw;
    const int ngroups = (o + kG - 1) / kG;
    const float inv_rw = 1.f / float(rw);
    for (int64_t blk = blockIdx.x; blk < g.b * ngroups; blk += gridDim.x) {
        const int64_t q = blk / ngroups;
        const int oj0 = int(blk - q * ngroups) * kG;
        const int G = min(kG, o - oj0);
        if constexpr (NHWC) {
            const float inv_g = 1.f / float(G);
            for (int e = threadIdx.x; e < G * mm; e += kThreads) {
                const int pix = fdiv(e, G, inv_g), gl = e - pix * G;
                sdy[gl * mm + pix] = __ldg(dy + (q * mm + pix) * o + oj0 + gl);
            }
        } else {
            const float* src = dy + (q * o + oj0) * mm;
            for (int e = threadIdx.x; e < G * mm; e += kThreads) sdy[e] = __ldg(src + e);
        }
        __syncthreads();
        float* out0 = drt + int64_t(oj0) * taps * ldr + q * rpi;
        for (int idx = threadIdx.x; idx < rpi; idx += kThreads) {
            const int Y = fdiv(idx, rw, inv_rw), X = idx - Y * rw;
            float* out = out0 + idx;
            for (int i = 0; i < k; ++i) {
                const int ty = Y - i;
                const int r = s == 1 ? ty : (ty >= 0 ? ty / s : -1);
                const bool rok = ty >= 0 && r * s == ty && r < m;
                if constexpr (TYPE == 2) {
#pragma unroll
                    for (int gl = 0; gl < kG; ++gl)
                        if (gl < G) out[(int64_t(gl) * taps + i) * ldr] = rok ? sdy[gl * mm + r * m + X] : 0.f;
                } else {
                    for (int j = 0; j < k; ++j) {
                        const int tx = X - j;
                        const int c = s == 1 ? tx : (tx >= 0 ? tx / s : -1);
                        const bool ok = rok && tx >= 0 && c * s == tx && c < m;
                        const int src = r * m + c;
#pragma unroll
                        for (int gl = 0; gl < kG; ++gl)
                            if (gl < G) out[(int64_t(gl) * taps + i * k + j) * ldr] = ok ? sdy[gl * mm + src] : 0.f;
                    }
                }
            }
        }
        __syncthreads();
    }
}

// Shift form of expand (T3 any stride, T2): column (channel gl, tap t) of an image's dRhat^T run is
// the channel's *dilated padded plane* Z (dy[r][c] at (s r, s c) of an R x rw grid, zero
// elsewhere, preceded by a zero guard of the largest tap shift) read at a constant shift:
//   T3: out[Y R + X] = Z[guard + Y R + X - (i R + j)]     T2: out[Y m + c] = Z[guard + Y m + c - i m]
// (X < j lands in the previous row's last k - 1 columns, which are zero: s (m - 1) = R - k).  A
// block builds Z of its channels in shared memory once -- in four copies offset by 0..3 floats, so
// that for every column one copy has the column's shift at the same 16-byte phase as the image's
// run in global memory -- and every column is then a copy of aligned float4s (ld.shared.v4 /
// st.global.v4, a scalar head and tail), no per-element index arithmetic.
template <int TYPE, bool NHWC>
__global__ void __launch_bounds__(kThreads) expand_shift_kernel(const float* __restrict__ dy, float* __restrict__ drt,
                                                                Geo g, int64_t ldr, int gz) {
    // [gz][4 phases][zl4]: copy f holds Z[p] at p + f; then 2 x gz x m^2: the dy planes of this
    // block and (in flight, cp.async) of the block after it
    extern __shared__ __align__(16) float zc[];
    const int m = int(g.m), mm = m * m, o = int(g.o), k = int(g.k), s = int(g.s), R = int(g.R);
    const int taps = TYPE == 2 ? k : k * k;
    const int rw = TYPE == 2 ? m : R;
    const int rpi = R * rw;
    const int guard = TYPE == 2 ? (k - 1) * rw : (k - 1) * R + (k - 1);
    const int zl4 = (guard + rpi + 3 + 3) & ~3;
    const int ngroups = (o + gz - 1) / gz;
    const int64_t nblk = g.b * ngroups;
    float* sdy = zc + gz * 4 * zl4;
    int* ctab = reinterpret_cast<int*>(sdy + 2 * gz * mm);  // gz x taps column offsets
    const float inv_mm = 1.f / float(mm), inv_m = 1.f / float(m);
    // consecutive blocks = consecutive images of one channel group
    auto fetch = [&](int64_t blk, int buf) {  // the block's dy planes -> sdy[buf] (channel-major)
        if (blk < nblk) {
            const int64_t grp = blk / g.b, q = blk - grp * g.b;
            const int oj0 = int(grp) * gz, G = min(gz, o - oj0);
            const uint32_t dst = uint32_t(__cvta_generic_to_shared(sdy + buf * gz * mm));
            if constexpr (NHWC) {
                const float inv_g = 1.f / float(G);
                for (int e = threadIdx.x; e < G * mm; e += kThreads) {
                    const int pix = fdiv(e, G, inv_g), gl = e - pix * G;
                    ptx::cp_async4(dst + uint32_t(gl * mm + pix) * 4u, dy + (q * mm + pix) * o + oj0 + gl);
                }
            } else {
                const float* src = dy + (q * o + oj0) * mm;
                for (int e = threadIdx.x; e < G * mm; e += kThreads) ptx::cp_async4(dst + uint32_t(e) * 4u, src + e);
            }
        }
        ptx::cp_async_commit();
    };
    fetch(blockIdx.x, 0);
    int it = 0;
    for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x, ++it) {
        const int64_t grp = blk / g.b, q = blk - grp * g.b;
        const int oj0 = int(grp) * gz;
        const int G = min(gz, o - oj0);
        fetch(blk + gridDim.x, (it + 1) & 1);
        {
            float4* z4 = reinterpret_cast<float4*>(zc);
            for (int e = threadIdx.x; e < G * zl4; e += kThreads) z4[e] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        ptx::cp_async_wait<1>();  // this block's planes (issued one iteration ago) landed
        __syncthreads();
        const float* sd = sdy + (it & 1) * gz * mm;
        for (int e = threadIdx.x; e < G * mm; e += kThreads) {
            const int gl = fdiv(e, mm, inv_mm), pix = e - gl * mm;
            const int r = fdiv(pix, m, inv_m), c = pix - r * m;
            const int pz = guard + (TYPE == 2 ? s * r * rw + c : s * r * R + s * c);
            float* zg = zc + gl * 4 * zl4 + pz;
            const float v = sd[e];
#pragma unroll
            for (int f = 0; f < 4; ++f) zg[f * zl4 + f] = v;
        }
        ptx::fence_proxy_async_smem();  // Z (generic-proxy writes) -> the bulk copies below read it
        __syncthreads();
        const int ga = int((q * rpi) & 3);          // 16-byte phase of the image's run (ldr % 4 == 0)
        const int h = min((4 - ga) & 3, rpi);       // scalar head up to the boundary
        const int nv = (rpi - h) >> 2, t0 = h + 4 * nv;
        float* out0 = drt + int64_t(oj0) * taps * ldr + q * rpi;
        const int ncol = G * taps;
        // per column: offset of zs (zs[idx] = Z[guard - shift + idx] in the phase-matched copy)
        for (int col = threadIdx.x; col < ncol; col += kThreads) {
            const int gl = col / taps, t = col - gl * taps;
            const int shift = TYPE == 2 ? t * rw : (t / k) * R + (t - (t / k) * k);
            const int f = (ga - guard + shift) & 3;
            ctab[col] = (gl * 4 + f) * zl4 + guard - shift + f;
        }
        __syncthreads();
        // the aligned body of every column: one 1D bulk copy (TMA engine) shared -> global per
        // column, 16-byte aligned at both ends (the phase-matched copy of Z), so the stores stream
        // without per-thread store instructions while the threads write the scalar head / tail
        if (nv > 0) {
            for (int col = threadIdx.x; col < ncol; col += kThreads)
                ptx::bulk_store(out0 + int64_t(col) * ldr + h, zc + ctab[col] + h, uint32_t(nv) * 16u);
            ptx::bulk_commit();
        }
        const int ht = h + (rpi - t0);  // scalar floats per column: head, then tail
        for (int e = threadIdx.x; e < ncol * ht; e += kThreads) {
            const int col = e / ht, u = e - col * ht;
            const int ix = u < h ? u : t0 + (u - h);
            out0[int64_t(col) * ldr + ix] = zc[ctab[col] + ix];
        }
        ptx::bulk_wait_read();  // this thread's bulk copies have read Z before it is rebuilt
        __syncthreads();
    }
    ptx::cp_async_wait<0>();
    ptx::bulk_wait_all();
}

// Type 2 / 3 lowering (internal order, depth % 4 == 0): block per padded input row
// (q, Y); its lowered rows are one contiguous span of the output.
//   T3: R rows of d floats = padded row Y, pixels [0, R) (ldc == d)
//   T2: m rows of ldc floats, row c = padded pixels [s c, s c + k) x d, zero tail to ldc
template <int TYPE>
__global__ void __launch_bounds__(kThreads) lower_rows_kernel(const float* __restrict__ x, float* __restrict__ dh,
                                                              Geo g, int64_t ldc) {
    extern __shared__ float4 srow[];  // T2: the padded input row (N x d floats)
    const int n = int(g.n), d4 = int(g.d / 4), p = int(g.p), R = int(g.R), m = int(g.m), N = int(g.N);
    const int64_t rows = g.b * R;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t qy = blockIdx.x; qy < rows; qy += gridDim.x) {
        const int64_t q = qy / R;
        const int Y = int(qy - q * R);
        const int ys = Y - p;
        const bool yok = ys >= 0 && ys < n;
        const float4* xr = x4 + ((q * n + (yok ? ys : 0)) * n) * d4;
        if constexpr (TYPE == 3) {
            float4* out = reinterpret_cast<float4*>(dh + qy * int64_t(R) * ldc);
            const float inv = 1.f / float(d4);
            for (int e = threadIdx.x; e < R * d4; e += kThreads) {
                const int X = fdiv(e, d4, inv), ch = e - X * d4;
                const int xs = X - p;
                out[e] = (yok && xs >= 0 && xs < n) ? __ldg(xr + xs * d4 + ch) : z;
            }
        } else {
            for (int e = threadIdx.x; e < N * d4; e += kThreads) {
                const int X = e / d4, ch = e - X * d4;
                const int xs = X - p;
                srow[e] = (yok && xs >= 0 && xs < n) ? __ldg(xr + xs * d4 + ch) : z;
            }
            __syncthreads();
            const int l4 = int(ldc / 4), kd4 = int(g.k) * d4, s = int(g.s);
            float4* out = reinterpret_cast<float4*>(dh + qy * int64_t(m) * ldc);
            const float inv = 1.f / float(l4);
            for (int e = threadIdx.x; e < m * l4; e += kThreads) {
                const int c = fdiv(e, l4, inv), u = e - c * l4;
                out[e] = u < kd4 ? srow[s * c * d4 + u] : z;
            }
            __syncthreads();
        }
    }
}

int blocks_for(int64_t work_blocks, int per_sm) {
    return int(std::max<int64_t>(1, std::min<int64_t>(work_blocks, int64_t(num_sms()) * per_sm)));
}

}  // namespace

bool planes_ok(const Geo& g, int type) {
    // per-block shared memory (kG planes) and 32-bit in-plane indices
    return (type == 2 || type == 3) && size_t(kG) * size_t(g.m * g.m) * 4 <= 96 * 1024 && g.R * g.R < (1 << 22) &&
           g.R * g.m < (1 << 22);
}

cudaError_t lift_planes(const Geo& g, int type, const float* rhat, float* y, cudaStream_t st) {
    if (!planes_ok(g, type)) return cudaErrorInvalidValue;
    const int taps = type == 2 ? int(g.k) : int(g.k * g.k);
    const int64_t rpi = type == 2 ? g.R * g.m : g.R * g.R;
    PhaseScope ps(kPhaseLift, st, 0, 4.0 * double(g.b * g.o) * double(taps * rpi + g.m * g.m));
    // staged form: up to kG channels' planes in 24 KB of shared memory per block (several blocks
    // per SM keep the load phase of one overlapping the sums of another)
    const int64_t blk_bytes = int64_t(taps) * rpi * 4;
    const int gmax = int(std::min<int64_t>(kG, (24 * 1024) / std::max<int64_t>(1, blk_bytes)));
    if (gmax >= 1 && (reinterpret_cast<uintptr_t>(rhat) & 15) == 0 && g.b * g.o * int64_t(taps) * rpi < (int64_t(1) << 40)) {
        // double-buffered bulk copies (buffer = the kernel's buf_floats)
        const size_t buf = ((size_t(gmax) * size_t(taps * rpi) + 8 + 3) & ~size_t(3)) * 4;
        const size_t smem = 2 * buf + (g.yl ? size_t(gmax) * size_t(g.m * g.m) * 4 : 0);
        const int grid = blocks_for(g.b * ((g.o + gmax - 1) / gmax), 4);
        const int64_t total = g.b * g.o * int64_t(taps) * rpi;
        auto go = [&](auto kern) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
            kern<<<grid, kThreads, smem, st>>>(rhat, y, g, gmax, total);
        };
        if (type == 2) g.yl ? go(lift_bulk_kernel<2, true>) : go(lift_bulk_kernel<2, false>);
        else g.yl ? go(lift_bulk_kernel<3, true>) : go(lift_bulk_kernel<3, false>);
        note_launch();
        return cudaGetLastError();
    }
    if (gmax >= 1) {
        const size_t smem = size_t(gmax) * size_t(blk_bytes) + (g.yl ? size_t(gmax) * size_t(g.m * g.m) * 4 : 0);
        if (smem <= 96 * 1024) {
            const int grid = blocks_for(g.b * ((g.o + gmax - 1) / gmax), 8);
            auto go = [&](auto kern) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
                kern<<<grid, kThreads, smem, st>>>(rhat, y, g, gmax);
            };
            if (type == 2) g.yl ? go(lift_staged_kernel<2, true>) : go(lift_staged_kernel<2, false>);
            else g.yl ? go(lift_staged_kernel<3, true>) : go(lift_staged_kernel<3, false>);
            note_launch();
            return cudaGetLastError();
        }
    }
    const size_t smem = g.yl ? size_t(kG) * size_t(g.m * g.m) * 4 : 0;
    const int grid = blocks_for(g.b * ((g.o + kG - 1) / kG), 8);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        kern<<<grid, kThreads, smem, st>>>(rhat, y, g);
    };
    if (type == 2) g.yl ? go(lift_planes_kernel<2, true>) : go(lift_planes_kernel<2, false>);
    else g.yl ? go(lift_planes_kernel<3, true>) : go(lift_planes_kernel<3, false>);
    note_launch();
    return cudaGetLastError();
}

cudaError_t expand_planes(const Geo& g, int type, const float* dy, float* drt, int64_t ldr, cudaStream_t st) {
    if (!planes_ok(g, type)) return cudaErrorInvalidValue;
    const int taps = type == 2 ? int(g.k) : int(g.k * g.k);
    const int64_t rpi = type == 2 ? g.R * g.m : g.R * g.R;
    PhaseScope ps(kPhaseExpand, st, 0, 4.0 * double(g.b * g.o) * double(taps * rpi + g.m * g.m));
    // shift form when kG (or at least 2) channels' dy + dilated planes fit in 48 KB
    const int64_t zl4 = ((type == 2 ? (g.k - 1) * g.m : (g.k - 1) * g.R + (g.k - 1)) + rpi + 6) & ~int64_t(3);
    const int64_t per_ch = (4 * zl4 + 2 * g.m * g.m + (type == 2 ? g.k : g.k * g.k)) * 4;  // 4 Z copies, 2 dy planes, column table
    const int gz = int(std::min<int64_t>(kG, (48 * 1024) / per_ch));
    if (gz >= 2 && rpi < (1 << 22) && g.m * g.m < (1 << 20) && ldr % 4 == 0 &&
        (reinterpret_cast<uintptr_t>(drt) & 15) == 0) {
        const size_t smem = size_t(gz) * size_t(per_ch);
        const int grid = blocks_for(g.b * ((g.o + gz - 1) / gz), 8);
        auto go = [&](auto kern) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
            kern<<<grid, kThreads, smem, st>>>(dy, drt, g, ldr, gz);
        };
        if (type == 2) g.yl ? go(expand_shift_kernel<2, true>) : go(expand_shift_kernel<2, false>);
        else g.yl ? go(expand_shift_kernel<3, true>) : go(expand_shift_kernel<3, false>);
    } else {
        const size_t smem = size_t(kG) * size_t(g.m * g.m) * 4;
        const int grid = blocks_for(g.b * ((g.o + kG - 1) / kG), 8);
        auto go = [&](auto kern) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
            kern<<<grid, kThreads, smem, st>>>(dy, drt, g, ldr);
        };
        if (type == 2) g.yl ? go(expand_planes_kernel<2, true>) : go(expand_planes_kernel<2, false>);
        else g.yl ? go(expand_planes_kernel<3, true>) : go(expand_planes_kernel<3, false>);
    }
    note_launch();
    // ldr padding rows (rows b*rpi .. ldr) of every column: zero (never read by a valid tile row,
    // but the GEMM's K / N tails read them)
    const int64_t rows = g.b * rpi;
    if (ldr > rows) {
        const int64_t ncols = lowered_ncols(g, type);
        cudaError_t e = cudaMemset2DAsync(drt + rows, size_t(ldr) * 4, 0, size_t(ldr - rows) * 4, size_t(ncols), st);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

bool lower_rows_ok(const Geo& g, int type, const float* x, const float* dh, int64_t ld) {
    if (!(type == 2 || type == 3) || g.d % 4 || ld % 4 || (reinterpret_cast<uintptr_t>(x) & 15) ||
        (reinterpret_cast<uintptr_t>(dh) & 15))
        return false;
    if (type == 3) return ld == g.d && g.R * (g.d / 4) < (1 << 22);
    return size_t(g.N * g.d) * 4 <= 96 * 1024 && g.m * (ld / 4) < (1 << 22);
}

cudaError_t lower_rows(const Geo& g, int type, const float* x, float* dhat, int64_t ld, cudaStream_t st) {
    if (!lower_rows_ok(g, type, x, dhat, ld)) return cudaErrorInvalidValue;
    const int64_t rpi = type == 2 ? g.R * g.m : g.R * g.R;
    PhaseScope ps(kPhaseLower, st, 0, 4.0 * double(g.b * g.n * g.n * g.d + g.b * rpi * ld));
    const int grid = blocks_for(g.b * g.R, 16);
    if (type == 3) {
        lower_rows_kernel<3><<<grid, kThreads, 0, st>>>(x, dhat, g, ld);
    } else {
        const size_t smem = size_t(g.N * g.d) * 4;
        cudaFuncSetAttribute(lower_rows_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        lower_rows_kernel<2><<<grid, kThreads, smem, st>>>(x, dhat, g, ld);
    }
    note_launch();
    return cudaGetLastError();
}

}  // namespace cct
