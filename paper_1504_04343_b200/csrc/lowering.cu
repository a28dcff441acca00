// lowering.cu -- the HBM-bound kernels of the three lowering types (see lowering.cuh).
//
// All kernels are pure gathers (no atomics): every output element is written
// exactly once by one thread, with the output index fastest-varying across a
// warp so stores are coalesced, and float4-vectorised when the channel depth is a
// multiple of 4.  Grids are grid-stride loops sized to a multiple of the SM count.
#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "lowering.cuh"
#include "ptx.cuh"

namespace cct {

RowMap rowmap_internal(const Geo& g, int type) {
    RowMap r{};
    if (type == 1) { r.ny = g.m; r.nc = g.m; }
    else if (type == 2) { r.ny = g.R; r.nc = g.m; }
    else { r.ny = g.R; r.nc = g.R; }
    r.rpi = r.ny * r.nc;
    r.sr = r.nc;
    r.sc = 1;
    return r;
}

// image block of m^2 (T1) or n^2 (T2/T3) rows, row = c*m + r / c*n + r.
RowMap rowmap_spec(const Geo& g, int type) {
    RowMap r{};
    const int64_t side = (type == 1) ? g.m : g.n;
    r.ny = side;
    r.nc = side;
    r.rpi = side * side;
    r.sr = 1;
    r.sc = side;
    return r;
}

int64_t lowered_cols(const Geo& g, int type) {
    return type == 1 ? g.k * g.k * g.d : type == 2 ? g.k * g.d : g.d;
}
int64_t lowered_ncols(const Geo& g, int type) {
    return type == 1 ? g.o : type == 2 ? g.k * g.o : g.k * g.k * g.o;
}

namespace {

constexpr int kThreads = 256;

// 4-byte asynchronous global -> shared copy (LDGSTS): the staging loops issue
// every copy before waiting, instead of one blocking load per iteration.
__device__ __forceinline__ void cp_async4(float* smem_dst, const float* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst))),
                 "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async16(float* smem_dst, const float* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst))),
                 "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }


// One warp per lowered row (q, y, c).  The row is `nruns` runs of L source
// floats that are contiguous in x (T1: k runs of k*d; T2: 1 run of k*d; T3: 1
// run of d).  The in-image part of a run is one contiguous interval, computed
// once per run, so the copy loop has no per-element index arithmetic.
template <bool VEC4>
__global__ void lower_kernel(const float* __restrict__ x, float* __restrict__ dh, Geo g, int type,
                             RowMap rm, int64_t ld, int cols, int64_t nrows_logical) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    const int n = int(g.n), d = int(g.d), k = int(g.k), s = int(g.s), p = int(g.p);
    const int nc = int(rm.nc), ny = int(rm.ny);
    const int L = (type == 3) ? d : k * d;     // run length (floats)
    const int nruns = (type == 1) ? k : 1;
    const int W = VEC4 ? 4 : 1;                 // floats per element moved
    for (int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < nrows_logical; w += warps) {
        const int c = int(w % nc);
        const int64_t t = w / nc;
        const int y = int(t % ny);
        const int64_t q = t / ny;
        float* row = dh + (q * rm.rpi + int64_t(y) * rm.sr + int64_t(c) * rm.sc) * ld;
        int ys0, xs0;
        bool zero_row = false;
        if (type == 1) { ys0 = s * y - p; xs0 = s * c - p; }
        else if (type == 2) { ys0 = y - p; xs0 = s * c - p; zero_row = (c >= g.m); }
        else { ys0 = y - p; xs0 = c - p; }
        const int taps = (type == 3) ? 1 : k;   // pixels per run
        // valid pixel interval [jlo, jhi) of the run
        const int jlo = max(0, -xs0), jhi = min(taps, n - xs0);
        const float* xq = x + q * int64_t(n) * n * d;
        if constexpr (VEC4) {
            for (int i = 0; i < nruns; ++i) {
                const int ys = ys0 + ((type == 1) ? i : 0);
                const bool row_ok = !zero_row && ys >= 0 && ys < n && jlo < jhi;
                const int lo = jlo * d / W, hi = jhi * d / W;  // in elements of W floats
                const float4* s4 = reinterpret_cast<const float4*>(xq + (int64_t(ys) * n + xs0) * d);
                float4* d4 = reinterpret_cast<float4*>(row + i * L);
#pragma unroll 4
                for (int e = lane; e < L / 4; e += 32) {
                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (row_ok && e >= lo && e < hi) v = __ldg(s4 + e);
                    d4[e] = v;
                }
            }
        } else {
            // flattened over the whole row so every lane works (run length k*d
            // is rarely a multiple of 32 when d is small, e.g. conv1 d = 3)
            const int lo = jlo * d, hi = jhi * d;
#pragma unroll 4
            for (int e = lane; e < cols; e += 32) {
                const int i = e / L, r = e - i * L;
                const int ys = ys0 + ((type == 1) ? i : 0);
                float v = 0.f;
                if (!zero_row && ys >= 0 && ys < n && r >= lo && r < hi)
                    v = __ldg(xq + (int64_t(ys) * n + xs0) * d + r);
                row[e] = v;
            }
        }
        for (int e = cols + lane; e < ld; e += 32) row[e] = 0.f;  // pad columns
    }
}

// y[q,o,r,c] = sum over taps of Rhat[row(q, s r + i, s c + j), col(o, i, j)].
// Flat over (plane, pixel) so every thread of the block works; the tap loads
// are independent and unrolled (several in flight per thread).
__global__ void lift_kernel(const float* __restrict__ rh, float* __restrict__ y, Geo g, int type,
                            RowMap rm, int64_t rs, int64_t cs) {
    const int m = int(g.m), o = int(g.o), k = int(g.k), s = int(g.s), mm = m * m;
    const int64_t total = g.b * o * int64_t(mm);
    const int64_t tap_i = rm.sr * rs, tap_j = rm.sc * rs;  // address step of one tap row / column
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t pl = e / mm;
        const int pix = int(e - pl * mm);
        const int r = pix / m, c = pix - r * m;
        const int oj = int(pl % o);
        const int64_t q = pl / o;
        const int64_t base = q * rm.rpi;
        float acc = 0.f;
        if (type == 1) {
            acc = __ldg(rh + (base + r * rm.sr + c * rm.sc) * rs + oj * cs);
        } else if (type == 2) {
            const float* p0 = rh + (base + int64_t(s) * r * rm.sr + int64_t(c) * rm.sc) * rs + int64_t(oj) * k * cs;
            const int64_t step = tap_i + cs;
#pragma unroll 4
            for (int i = 0; i < k; ++i) acc += __ldg(p0 + i * step);
        } else {
            const float* p0 = rh + (base + int64_t(s) * r * rm.sr + int64_t(s) * c * rm.sc) * rs +
                              int64_t(oj) * k * k * cs;
            for (int i = 0; i < k; ++i) {
                const float* pi = p0 + i * (tap_i + int64_t(k) * cs);
#pragma unroll 4
                for (int j = 0; j < k; ++j) acc += __ldg(pi + j * (tap_j + cs));
            }
        }
        if (g.yl) y[(q * mm + pix) * o + oj] = acc;  // NHWC y
        else y[e] = acc;
    }
}

// T1 expand: dRhat1^T[o][q*m^2 + pix] = dy[q][o][pix] -- a permutation of the
// (q, o) planes.  One block-row per group of planes; each warp copies one plane
// as a contiguous run (coalesced on both sides), 32-bit index math only.
__global__ void expand_t1_kernel(const float* __restrict__ dy, float* __restrict__ drt, int64_t b, int o,
                                 int mm, int64_t ldr) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int64_t planes = b * o;
    for (int64_t pl = int64_t(blockIdx.x) * nw + warp; pl < planes; pl += int64_t(gridDim.x) * nw) {
        const int oj = int(pl % o);
        const int64_t q = pl / o;
        const float* src = dy + pl * mm;
        float* dst = drt + int64_t(oj) * ldr + q * mm;
        int e = lane;
        for (; e + 96 < mm; e += 128) {  // four loads in flight per lane
            const float v0 = __ldg(src + e), v1 = __ldg(src + e + 32), v2 = __ldg(src + e + 64),
                        v3 = __ldg(src + e + 96);
            dst[e] = v0;
            dst[e + 32] = v1;
            dst[e + 64] = v2;
            dst[e + 96] = v3;
        }
        for (; e < mm; e += 32) dst[e] = __ldg(src + e);
    }
}

// T2/T3 expand: dRhat^T[col][row] (internal row order), zeros where lift does
// not read.  blockIdx.y = column (o, i[, j]); each thread writes 4 consecutive
// rows as one float4, walking (q, y, x) incrementally (one division per 4 rows).
__global__ void expand_kernel(const float* __restrict__ dy, float* __restrict__ drt, Geo g, int type,
                              RowMap rm, int64_t ldr) {
    const int m = int(g.m), o = int(g.o), k = int(g.k), s = int(g.s);
    const int nc = int(rm.nc), ny = int(rm.ny);
    const int col = blockIdx.y;
    int oj, i, j = 0;
    if (type == 2) { oj = col / k; i = col - oj * k; }
    else { oj = col / (k * k); const int ij = col - oj * k * k; i = ij / k; j = ij - i * k; }
    float4* out = reinterpret_cast<float4*>(drt + int64_t(col) * ldr);
    const int rows = int(g.b * rm.rpi);  // < 2^31 (checked by the launcher)
    const int rows4 = int(ldr / 4);
    for (int r4 = blockIdx.x * blockDim.x + threadIdx.x; r4 < rows4; r4 += gridDim.x * blockDim.x) {
        int row = 4 * r4;
        int t = row / nc;
        int cx = row - t * nc;
        int q = t / ny;
        int yy = t - q * ny;
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            float val = 0.f;
            if (row + u < rows) {
                const int ty = yy - i;
                int r = -1;
                if (s == 1) r = ty;
                else if (ty >= 0 && ty % s == 0) r = ty / s;
                int c = cx;
                if (type == 3) {
                    const int tx = cx - j;
                    c = -1;
                    if (s == 1) c = tx;
                    else if (tx >= 0 && tx % s == 0) c = tx / s;
                }
                if (r >= 0 && r < m && c >= 0 && c < m)
                    val = g.yl ? __ldg(dy + ((int64_t(q) * m + r) * m + c) * o + oj)
                               : __ldg(dy + ((int64_t(q) * o + oj) * m + r) * int64_t(m) + c);
            }
            v[u] = val;
            if (++cx == nc) {  // walk to the next row of the (q, y) grid
                cx = 0;
                if (++yy == ny) { yy = 0; ++q; }
            }
        }
        out[r4] = make_float4(v[0], v[1], v[2], v[3]);
    }
}

// dx[q,y,x,ch] (unpadded) = adjoint of lower: sum of the dDhat entries that
// copied Xp[q,y+p,x+p,ch].  One block-row per input row (q, y); each thread owns
// VW consecutive channels (float4 when d % 4 == 0) and walks the taps directly
// (first tap congruent mod s, then step s), several loads in flight.
template <int VW>
__global__ void col2im_kernel(const float* __restrict__ dd, int64_t ld, float* __restrict__ dx, Geo g,
                              int type) {
    using V = typename std::conditional<VW == 4, float4, float>::type;
    const int n = int(g.n), d = int(g.d), k = int(g.k), s = int(g.s), p = int(g.p), m = int(g.m),
              R = int(g.R);
    const int dv = d / VW;
    const int64_t rowsq = g.b * n;
    const int per_row = n * dv;
    for (int64_t qy = blockIdx.x; qy < rowsq; qy += gridDim.x) {
        const int yy = int(qy % n);
        const int64_t q = qy / n;
        const int py = yy + p;
        V* out = reinterpret_cast<V*>(dx + qy * int64_t(n) * d);
        // valid output-row taps i (type 1): r = (py - i)/s in [0, m)
        for (int e = threadIdx.x; e < per_row; e += blockDim.x) {
            const int xx = e / dv, cv = e - xx * dv;
            const int px = xx + p;
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
            auto add = [&](const float* ptr) {
                if constexpr (VW == 4) {
                    const float4 v = __ldg(reinterpret_cast<const float4*>(ptr) + cv);
                    a0 += v.x; a1 += v.y; a2 += v.z; a3 += v.w;
                } else {
                    a0 += __ldg(ptr + cv);
                }
            };
            // tap ranges: c = (px - j)/s in [0, m)  <=>  j in [px - s(m-1), px], j == px mod s
            const int jlo0 = px - s * (m - 1);
            int jfirst = px % s;
            if (jfirst < jlo0) jfirst += ((jlo0 - jfirst + s - 1) / s) * s;
            const int jlast = min(k - 1, px);
            if (type == 3) {
                if (py < R && px < R) add(dd + ((q * R + py) * R + px) * ld);
            } else if (type == 2) {
                if (py < R) {
                    const int64_t rowb = (q * R + py) * int64_t(m);
#pragma unroll 4
                    for (int j = jfirst; j <= jlast; j += s) add(dd + (rowb + (px - j) / s) * ld + j * d);
                }
            } else {
                const int ilo0 = py - s * (m - 1);
                int ifirst = py % s;
                if (ifirst < ilo0) ifirst += ((ilo0 - ifirst + s - 1) / s) * s;
                const int ilast = min(k - 1, py);
                for (int i = ifirst; i <= ilast; i += s) {
                    const int64_t rowb = (q * m + (py - i) / s) * int64_t(m);
#pragma unroll 4
                    for (int j = jfirst; j <= jlast; j += s)
                        add(dd + (rowb + (px - j) / s) * ld + (i * k + j) * d);
                }
            }
            if constexpr (VW == 4) out[e] = make_float4(a0, a1, a2, a3);
            else out[e] = a0;
        }
    }
}

// ---- small-channel Type 1 kernels (d % 4 != 0, e.g. conv1 d = 3) -----------
// The generic kernels move 4-byte elements with run lengths (k*d) that are not
// multiples of 4; these stage the data through shared memory so every global
// access is a float4 (or a contiguous run) and each byte moves once.

// Lowering: one CTA per output row (q, r).  The k input rows it needs
// (s*r - p + i, zero rows outside the image) are staged in smem with async
// copies, zero-padded to the padded width; each lowered row (q, r, c) is then
// written as float4s by one warp through an offset table.  All index tables
// are built once per CTA, so the per-row loops do no integer division.
// NT > 0: the lane's NT column offsets (e = lane + 32 t, ld <= 32 NT) are kept in
// registers for the whole kernel instead of re-read from smem per element (ncu: the
// per-element table read made the kernel issue-bound at 78 % issue activity).
template <int NT>
__global__ void lower_t1_smem_kernel(const float* __restrict__ x, float* __restrict__ dh, Geo g, RowMap rm,
                                     int64_t ld, int cols) {
    extern __shared__ float sm[];
    const int n = int(g.n), d = int(g.d), k = int(g.k), s = int(g.s), p = int(g.p), m = int(g.m);
    const int Wp = n + 2 * p;
    const int rowf = Wp * d;                                   // floats per staged row
    float* tile = sm;                                          // k x rowf
    int* offs = reinterpret_cast<int*>(sm + k * rowf);         // cols: lowered column -> tile index (c = 0)
    int* soff = offs + cols;                                   // rowf: staged float -> x offset in row, or -1
    for (int e = threadIdx.x; e < cols; e += blockDim.x) {
        const int i = e / (k * d), rr = e - i * (k * d), j = rr / d, ch = rr - j * d;
        offs[e] = i * rowf + j * d + ch;
    }
    for (int e = threadIdx.x; e < rowf; e += blockDim.x) {
        const int xs = e / d - p;
        soff[e] = (xs >= 0 && xs < n) ? xs * d + (e - (e / d) * d) : -1;
    }
    const int ld4 = int(ld / 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    const int64_t nqr = g.b * m;
    int oreg[NT > 0 ? NT : 1];
    if constexpr (NT > 0) {
        __syncthreads();  // offs table built
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int e = lane + 32 * t;
            oreg[t] = e < cols ? offs[e] : -1;
        }
    }
    for (int64_t qr = blockIdx.x; qr < nqr; qr += gridDim.x) {
        const int r = int(qr % m);
        const int64_t q = qr / m;
        __syncthreads();  // tables ready / previous tile consumed
        for (int e = threadIdx.x; e < rowf; e += blockDim.x) {
            const int so = soff[e];
            for (int i = 0; i < k; ++i) {
                const int ys = s * r - p + i;
                if (so >= 0 && ys >= 0 && ys < n) cp_async4(tile + i * rowf + e, x + ((q * n + ys) * int64_t(n)) * d + so);
                else tile[i * rowf + e] = 0.f;
            }
        }
        cp_async_wait_all();
        __syncthreads();
        // one warp per lowered row; lane-consecutive elements: conflict-free smem
        // gathers and 128-byte coalesced stores
        if constexpr (NT > 0) {
            for (int c = warp; c < m; c += nwarps) {
                const int base = s * c * d;
                float* row = dh + (q * rm.rpi + int64_t(r) * rm.sr + int64_t(c) * rm.sc) * ld;
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    const int e = lane + 32 * t;
                    if (e < ld4 * 4) row[e] = oreg[t] >= 0 ? tile[oreg[t] + base] : 0.f;
                }
            }
        } else {
            for (int c = warp; c < m; c += nwarps) {
                const int base = s * c * d;
                float* row = dh + (q * rm.rpi + int64_t(r) * rm.sr + int64_t(c) * rm.sc) * ld;
#pragma unroll 4
                for (int e = lane; e < ld4 * 4; e += 32) row[e] = e < cols ? tile[offs[e] + base] : 0.f;
            }
        }
    }
}

// The same lowering for unpadded layers with 16-byte aligned x and a whole number
// of float4s in x (conv1): the k input rows are staged with 16-byte cp.async from
// the float4 boundary below each row start (the row's misalignment sh_i, 0..3
// floats, is folded into the per-lane smem offsets once per tile), lowered
// columns past `cols` read a zeroed smem slot instead of taking a branch, and the
// gathers use 32-bit shared addresses.  Each thread keeps its NT = ld / 32
// (rounded up) smem offsets in registers, with i * n d mod 4 for filter row i in
// bits 28..29 (row i starts sh_0 + i n d floats past a float4 boundary).  The zero
// slot tolerates the shift (rowfS >= n d + 4 > the largest column offset + 3).
template <int NT>
__global__ void __launch_bounds__(512) lower_t1_vec_kernel(const float* __restrict__ x, float* __restrict__ dh, Geo g,
                                                             RowMap rm, int64_t ld, int cols) {
    extern __shared__ __align__(16) float sm[];
    const int n = int(g.n), d = int(g.d), k = int(g.k), s = int(g.s), m = int(g.m);
    const int rowf = n * d;                     // floats per input row
    const int rowfS = (rowf + 7) & ~3;          // slot: up to 3 leading floats + the row, float4 multiple
    const int nvmax = rowfS / 4;
    float* zero = sm + k * rowfS;               // slot k: zeros (padding columns read here)
    const uint32_t sbase = ptx::smem_u32(sm);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    for (int e = threadIdx.x; e < rowfS; e += blockDim.x) zero[e] = 0.f;
    const int kd = k * d, nd4 = rowf & 3;
    uint32_t oreg[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const int e = lane + 32 * t;
        if (e < cols) {
            const int i = e / kd, rr = e - i * kd;
            oreg[t] = uint32_t(i * rowfS + rr) | (uint32_t((i * nd4) & 3) << 28);
        } else {
            oreg[t] = uint32_t(k * rowfS);  // zero slot (no shift)
        }
    }
    const int last = int(ld) - 32 * (NT - 1);   // lanes of the final 32-column group that store
    const int64_t nqr = g.b * m;
    for (int64_t qr = blockIdx.x; qr < nqr; qr += gridDim.x) {
        const int r = int(qr % m);
        const int64_t q = qr / m;
        const int64_t g00 = ((q * n + int64_t(s) * r) * n) * d;   // float index of input row s r
        const int sh0 = int(g00 & 3);
        __syncthreads();  // previous tile consumed (and the zero slot written)
        for (int idx = threadIdx.x; idx < k * nvmax; idx += blockDim.x) {
            const int i = idx / nvmax, v = idx - i * nvmax;
            const int64_t gi = g00 + int64_t(i) * rowf;
            const int sh = int(gi & 3);
            if (4 * v < sh + rowf) cp_async16(sm + i * rowfS + 4 * v, x + (gi - sh) + 4 * v);
        }
        cp_async_wait_all();
        __syncthreads();
        uint32_t addr[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const uint32_t o = oreg[t];
            addr[t] = sbase + 4u * ((o & 0x0fffffffu) + uint32_t((sh0 + int(o >> 28)) & 3));
        }
        for (int c = warp; c < m; c += nwarps) {
            const uint32_t boff = 4u * uint32_t(s * c * d);
            float* row = dh + (q * rm.rpi + int64_t(r) * rm.sr + int64_t(c) * rm.sc) * ld + lane;
#pragma unroll
            for (int t = 0; t < NT - 1; ++t) {
                float v;
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr[t] + boff));
                row[32 * t] = v;
            }
            if (lane < last) {
                float v;
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr[NT - 1] + boff));
                row[32 * (NT - 1)] = v;
            }
        }
    }
}

// col2im (Type 1, small d): one CTA per input row (q, y).  dDhat arrives
// slab-major (col2im_slab_layout): slab (q, r, i) = the m x k*d block of rows
// (q, r, c) and filter row i, contiguous and 16-byte aligned (stride S floats),
// as the backward-data GEMM epilogue writes it.  The (r, i) slabs with
// s*r + i == y + p are staged by bulk (TMA engine) copies completing on an
// mbarrier, then every dx element of the row sums its taps from smem using
// per-element tap metadata built once (NP: compile-time bound on the slab and tap
// counts, ceil(k / s), so the sums unroll into predicated adds).  Each dDhat
// element is read once.
template <int NP>
__global__ void col2im_t1_smem_kernel(const float* __restrict__ dd, int64_t S, float* __restrict__ dx, Geo g) {
    extern __shared__ __align__(16) float sm[];
    __shared__ __align__(8) uint64_t full[2];
    const int n = int(g.n), d = int(g.d), k = int(g.k), s = int(g.s), p = int(g.p), m = int(g.m);
    const int kd = k * d;
    const int npair_max = (k + s - 1) / s;
    int* meta = reinterpret_cast<int*>(sm + 2 * npair_max * S);  // n*d: tap run per output
    // per dx column element: slab offset of its first valid tap (c < m) and the
    // number of taps (j = j0 + t s, c = c0 - t, 0 <= c < m, j < k): branch-free sums
    for (int e = threadIdx.x; e < n * d; e += blockDim.x) {
        const int xx = e / d, ch = e - xx * d, px = xx + p;
        int j = px % s, c = px / s;
        while (c >= m && j < k) { j += s; --c; }   // skip taps whose window starts past the image
        int cnt = 0;
        for (int jj = j, cc = c; jj < k && cc >= 0; jj += s, --cc) ++cnt;
        const int off = (cnt > 0) ? c * kd + j * d + ch : 0;
        meta[e] = off | (cnt << 24);                // off < 2^24 (slab <= 96 KiB)
    }
    if (threadIdx.x == 0) {
        ptx::mbar_init(&full[0], 1);
        ptx::mbar_init(&full[1], 1);
        ptx::fence_barrier_init();
    }
    __syncthreads();
    const int64_t nqy = g.b * n;
    const uint32_t slab_bytes = uint32_t(S) * 4u;
    // slabs (r, i) of dx row qy, ascending i: r from min(m-1, py/s) down while i = py - s r < k
    auto pairs = [&](int64_t row, int* rtop_out) {
        const int py = int(row % n) + p;
        const int rtop = min(m - 1, py / s);
        int np = 0;
        while (np < npair_max && rtop - np >= 0 && py - s * (rtop - np) < k) ++np;
        *rtop_out = rtop;
        return np;
    };
    // double-buffered: the slabs of the CTA's next row load while this row is summed
    auto issue = [&](int64_t row, int buf) {
        int rtop;
        const int np = pairs(row, &rtop);
        if (np == 0) return;
        const int py = int(row % n) + p;
        const int64_t q = row / n;
        ptx::mbar_arrive_expect_tx(&full[buf], uint32_t(np) * slab_bytes);
        for (int a = 0; a < np; ++a) {
            const int r = rtop - a, i = py - s * r;
            ptx::bulk_load(sm + (buf * npair_max + a) * S, dd + ((q * m + r) * int64_t(k) + i) * S, slab_bytes,
                           &full[buf]);
        }
    };
    uint32_t phase = 0;  // bit b: parity of buffer b
    if (threadIdx.x == 0 && blockIdx.x < nqy) issue(blockIdx.x, 0);
    const uint32_t sbase = ptx::smem_u32(sm);
    const uint32_t slab4 = uint32_t(S) * 4u;
    const uint32_t delta4 = uint32_t(s * d - kd) * 4u;  // slab step from tap t to t + 1 (bytes)
    int it = 0;
    for (int64_t qy = blockIdx.x; qy < nqy; qy += gridDim.x, ++it) {
        const int buf = it & 1;
        __syncthreads();  // every thread is done with the other buffer (previous row)
        if (threadIdx.x == 0 && qy + gridDim.x < nqy) issue(qy + gridDim.x, buf ^ 1);
        int rtop;
        const int np = pairs(qy, &rtop);
        if (np > 0) {
            ptx::mbar_wait(&full[buf], (phase >> buf) & 1u);
            phase ^= 1u << buf;
        }
        const uint32_t slabs = sbase + uint32_t(buf * npair_max) * slab4;
        float* out = dx + qy * int64_t(n) * d;
        for (int e = threadIdx.x; e < n * d; e += blockDim.x) {
            const int mt = meta[e];
            const int cnt = mt >> 24;
            const uint32_t a0 = slabs + 4u * uint32_t(mt & 0xFFFFFF);
            float acc = 0.f;
            if constexpr (NP > 0) {
#pragma unroll
                for (int a = 0; a < NP; ++a) {
                    if (a < np) {  // block-uniform
#pragma unroll
                        for (int t = 0; t < NP; ++t) {
                            float v = 0.f;  // +0 terms leave the sum bit-identical (it is never -0)
                            asm volatile(
                                "{\n\t.reg .pred p;\n\tsetp.lt.s32 p, %2, %3;\n\t@p ld.shared.f32 %0, [%1];\n\t}"
                                : "+f"(v)
                                : "r"(a0 + uint32_t(a) * slab4 + uint32_t(t) * delta4), "r"(t), "r"(cnt));
                            acc += v;
                        }
                    }
                }
            } else {
                for (int a = 0; a < np; ++a)
                    for (int t = 0; t < cnt; ++t) {
                        float v;
                        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a0 + uint32_t(a) * slab4 + uint32_t(t) * delta4));
                        acc += v;
                    }
            }
            out[e] = acc;
        }
    }
}

__global__ void pad_rows_kernel(const float* __restrict__ src, int64_t rows, int64_t cols, int64_t lds,
                                float* __restrict__ dst, int64_t ldd) {
    const int64_t total = rows * ldd;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / ldd, c = e - r * ldd;
        dst[e] = c < cols ? src[r * lds + c] : 0.f;
    }
}

__global__ void transpose_kernel(const float* __restrict__ src, int64_t rows, int64_t cols, int64_t lds,
                                 float* __restrict__ dst, int64_t ldd) {
    __shared__ float tile[32][33];
    const int64_t tiles_c = (cols + 31) / 32, tiles_r = (rows + 31) / 32;
    for (int64_t tix = blockIdx.x; tix < tiles_r * tiles_c; tix += gridDim.x) {
        const int64_t r0 = (tix / tiles_c) * 32, c0 = (tix % tiles_c) * 32;
        for (int i = threadIdx.y; i < 32; i += blockDim.y) {
            const int64_t r = r0 + i, c = c0 + threadIdx.x;
            tile[i][threadIdx.x] = (r < rows && c < cols) ? src[r * lds + c] : 0.f;
        }
        __syncthreads();
        for (int i = threadIdx.y; i < 32; i += blockDim.y) {
            const int64_t c = c0 + i, r = r0 + threadIdx.x;
            if (r < rows && c < cols) dst[c * ldd + r] = tile[threadIdx.x][i];
        }
        __syncthreads();
    }
}

// Batched transpose: for z < nz, dst[z*dst_z + c*ldd + r] = src[z*src_z + r*lds + c]
// (rows x cols -> cols x rows).  32 x 32 tiles through padded smem; 256 threads,
// each moving 4 elements per tile, so reads and writes are both 128-byte rows.
template <int TR>
__global__ void __launch_bounds__(256) transpose_batched_kernel(const float* __restrict__ src, int rows, int cols,
                                                                int64_t lds, int64_t src_z, float* __restrict__ dst,
                                                                int64_t ldd, int64_t dst_z, int nz) {
    // TR x 32 tiles: each thread keeps TR / 8 loads in flight (latency-bound at TR = 32)
    __shared__ float tile[TR][33];
    const int tr = (rows + TR - 1) / TR, tc = (cols + 31) >> 5;
    const int64_t per_z = int64_t(tr) * tc;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int64_t t = blockIdx.x; t < per_z * nz; t += gridDim.x) {
        const int z = int(t / per_z);
        const int rem = int(t - int64_t(z) * per_z);
        const int r0 = (rem / tc) * TR, c0 = (rem % tc) << 5;
        const float* s = src + int64_t(z) * src_z;
        float* d = dst + int64_t(z) * dst_z;
        const int c = c0 + tx;
#pragma unroll
        for (int i = 0; i < TR / 8; ++i) {
            const int r = r0 + ty + 8 * i;
            tile[ty + 8 * i][tx] = (r < rows && c < cols) ? __ldcs(s + int64_t(r) * lds + c) : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int h = 0; h < TR / 32; ++h) {
            const int r = r0 + 32 * h + tx;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int cc = c0 + ty + 8 * i;
                if (r < rows && cc < cols) d[int64_t(cc) * ldd + r] = tile[32 * h + tx][ty + 8 * i];
            }
        }
        __syncthreads();
    }
}

}  // namespace

cudaError_t lower(const Geo& g, int type, const RowMap& rm, const float* x, float* dhat, int64_t ld,
                  cudaStream_t st) {
    // Type 2 / 3 in the internal row order: whole padded input rows (lowering23.cu)
    if (type != 1 && rm.sc == 1 && rm.ny == g.R && rm.nc == (type == 2 ? g.m : g.R) && rm.sr == rm.nc &&
        lower_rows_ok(g, type, x, dhat, ld))
        return lower_rows(g, type, x, dhat, ld, st);
    const int64_t cols = lowered_cols(g, type);
    const int64_t nrows = g.b * rm.ny * rm.nc;
    PhaseScope ps(kPhaseLower, st, 0, 4.0 * double(g.b * g.n * g.n * g.d + nrows * ld));
    const bool vec = (g.d % 4 == 0) && (ld % 4 == 0) &&
                     (reinterpret_cast<uintptr_t>(x) % 16 == 0) && (reinterpret_cast<uintptr_t>(dhat) % 16 == 0);
    // small-channel Type 1 (e.g. conv1, d = 3): shared-memory staged rows
    const size_t smem1 = size_t(g.k * (g.n + 2 * g.p) * g.d) * 4 + size_t(cols) * 4 + size_t((g.n + 2 * g.p) * g.d) * 4;
    if (type == 1 && !vec && ld % 4 == 0 && reinterpret_cast<uintptr_t>(dhat) % 16 == 0 && smem1 <= 96 * 1024 &&
        rm.ny == g.m && rm.nc == g.m) {
        const int64_t nqr = g.b * g.m;
        const int grid1 = int(std::min<int64_t>(nqr, int64_t(num_sms()) * 4));
        auto go = [&](auto kern) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);  // per device
            kern<<<grid1, 512, smem1, st>>>(x, dhat, g, rm, ld, int(cols));
        };
        const int64_t nt = cdiv(ld, 32);
        const size_t smemv = size_t((g.k + 1) * ((g.n * g.d + 7) & ~int64_t(3))) * 4;
        const int64_t total = g.b * g.n * g.n * g.d;
        if (g.p == 0 && total % 4 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0 && nt >= 2 && nt <= 16 &&
            smemv <= 96 * 1024) {
            auto gov = [&](auto kern) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);  // per device
                const int threads = 512;
                int per_sm = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smemv);
                const int gridv = int(std::min<int64_t>(nqr, int64_t(num_sms()) * std::max(1, per_sm)));
                kern<<<gridv, threads, smemv, st>>>(x, dhat, g, rm, ld, int(cols));
            };
            switch (nt) {
#define CCT_LV(N) case N: gov(lower_t1_vec_kernel<N>); break;
                CCT_LV(2) CCT_LV(3) CCT_LV(4) CCT_LV(5) CCT_LV(6) CCT_LV(7) CCT_LV(8) CCT_LV(9)
                CCT_LV(10) CCT_LV(11) CCT_LV(12) CCT_LV(13) CCT_LV(14) CCT_LV(15) CCT_LV(16)
#undef CCT_LV
            }
            note_launch();
            return cudaGetLastError();
        }
        if (nt <= 4) go(lower_t1_smem_kernel<4>);
        else if (nt <= 8) go(lower_t1_smem_kernel<8>);
        else if (nt <= 12) go(lower_t1_smem_kernel<12>);
        else if (nt <= 16) go(lower_t1_smem_kernel<16>);
        else go(lower_t1_smem_kernel<0>);
        note_launch();
        return cudaGetLastError();
    }
    const int grid = grid_for(nrows * 32, kThreads);
    if (vec) lower_kernel<true><<<grid, kThreads, 0, st>>>(x, dhat, g, type, rm, ld, int(cols), nrows);
    else lower_kernel<false><<<grid, kThreads, 0, st>>>(x, dhat, g, type, rm, ld, int(cols), nrows);
    note_launch();
    return cudaGetLastError();
}

cudaError_t lift(const Geo& g, int type, const RowMap& rm, const float* rhat, int64_t rs, int64_t cs,
                 float* y, cudaStream_t st) {
    const int grid = grid_for(g.b * g.o * g.m * g.m, kThreads, 16);
    PhaseScope ps(kPhaseLift, st, 0,
                  4.0 * double(g.b * g.o * g.m * g.m) * (1.0 + (type == 1 ? 1 : type == 2 ? g.k : g.k * g.k)));
    lift_kernel<<<grid, kThreads, 0, st>>>(rhat, y, g, type, rm, rs, cs);
    note_launch();
    return cudaGetLastError();
}

cudaError_t expand(const Geo& g, int type, const float* dy, float* drt, int64_t ldr, cudaStream_t st) {
    if (type == 1 && g.yl) {
        // NHWC dy is dRhat (rows x o): dRhat^T is its transpose
        return transpose_batched(dy, g.b * g.m * g.m, g.o, g.o, 0, drt, ldr, 0, 1, kPhaseExpand, st);
    }
    if (type != 1 && planes_ok(g, type)) return expand_planes(g, type, dy, drt, ldr, st);
    const RowMap rm = rowmap_internal(g, type);
    const int64_t ncols = lowered_ncols(g, type);
    PhaseScope ps(kPhaseExpand, st, 0, 4.0 * double(g.b * g.o * g.m * g.m + ncols * g.b * rm.rpi));
    if (type == 1) {
        const int grid = grid_for(g.b * g.o * 32, kThreads, 16);  // one warp per plane
        expand_t1_kernel<<<grid, kThreads, 0, st>>>(dy, drt, g.b, int(g.o), int(g.m * g.m), ldr);
    } else {
        if (ncols > 65535 || g.b * rm.rpi >= (int64_t(1) << 31)) return cudaErrorInvalidConfiguration;
        if (ldr % 4 || reinterpret_cast<uintptr_t>(drt) % 16) return cudaErrorInvalidValue;
        const int64_t want = (int64_t(num_sms()) * 32 + ncols - 1) / ncols;
        const int gx = int(std::max<int64_t>(1, std::min<int64_t>(want, cdiv(ldr / 4, kThreads))));
        expand_kernel<<<dim3(gx, unsigned(ncols)), kThreads, 0, st>>>(dy, drt, g, type, rm, ldr);
    }
    note_launch();
    return cudaGetLastError();
}

bool col2im_slab_layout(const Geo& g, int type) {
    if (type != 1 || g.d % 4 == 0 || g.d >= 256 || g.s >= 256) return false;
    const int64_t S = slab_stride(g);
    const int64_t npair = (g.k + g.s - 1) / g.s;
    return (2 * npair * S + g.n * g.d) * 4 <= 96 * 1024;  // double-buffered slabs
}

int64_t slab_stride(const Geo& g) { return rup4(g.m * g.k * g.d); }

cudaError_t col2im(const Geo& g, int type, const float* dd, int64_t ld, float* dx, cudaStream_t st) {
    const int64_t rowsq = g.b * g.n;
    const int grid = int(std::min<int64_t>(rowsq, int64_t(num_sms()) * 16));
    const RowMap rmi = rowmap_internal(g, type);
    PhaseScope ps(kPhaseCol2im, st, 0, 4.0 * double(g.b * g.n * g.n * g.d + g.b * rmi.rpi * lowered_cols(g, type)));
    if (col2im_slab_layout(g, type)) {  // ld = slab stride
        if (ld != slab_stride(g) || reinterpret_cast<uintptr_t>(dd) % 16) return cudaErrorInvalidValue;
        cudaFuncSetAttribute(col2im_t1_smem_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        cudaFuncSetAttribute(col2im_t1_smem_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        const size_t smem1 = size_t(2 * ((g.k + g.s - 1) / g.s) * ld + g.n * g.d) * 4;
        // threads: the fewest warps that cover a dx row in the same number of passes
        // as 256 threads would (conv1: 681 floats -> 3 x 256).  Measured on conv1
        // b = 256 (ncu): 512 threads 376 us, 352 261 us, 256 219 us (5.8 TB/s), 224 225 us.
        const int64_t nd = g.n * g.d, passes = cdiv(nd, 256);
        const int threads = int(std::min<int64_t>(256, (cdiv(nd, passes) + 31) / 32 * 32));
        auto kern = (g.k + g.s - 1) / g.s <= 3 ? col2im_t1_smem_kernel<3> : col2im_t1_smem_kernel<0>;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem1);
        const int grid1 = int(std::min<int64_t>(rowsq, int64_t(num_sms()) * std::max(1, per_sm)));
        kern<<<grid1, threads, smem1, st>>>(dd, ld, dx, g);
        note_launch();
        return cudaGetLastError();
    }
    const bool vec = g.d % 4 == 0 && ld % 4 == 0 && (reinterpret_cast<uintptr_t>(dd) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(dx) % 16 == 0);
    if (vec) col2im_kernel<4><<<grid, kThreads, 0, st>>>(dd, ld, dx, g, type);
    else col2im_kernel<1><<<grid, kThreads, 0, st>>>(dd, ld, dx, g, type);
    note_launch();
    return cudaGetLastError();
}

cudaError_t pad_rows(const float* src, int64_t rows, int64_t cols, int64_t ld_src, float* dst,
                     int64_t ld_dst, cudaStream_t st) {
    PhaseScope ps(kPhaseOther, st, 0, 4.0 * double(rows * (cols + ld_dst)));
    pad_rows_kernel<<<grid_for(rows * ld_dst, kThreads), kThreads, 0, st>>>(src, rows, cols, ld_src, dst, ld_dst);
    note_launch();
    return cudaGetLastError();
}

cudaError_t transpose(const float* src, int64_t rows, int64_t cols, int64_t ld_src, float* dst,
                      int64_t ld_dst, cudaStream_t st) {
    const int64_t tiles = cdiv(rows, 32) * cdiv(cols, 32);
    const int grid = int(std::min<int64_t>(tiles, int64_t(num_sms()) * 16));
    transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(src, rows, cols, ld_src, dst, ld_dst);
    note_launch();
    return cudaGetLastError();
}

cudaError_t transpose_batched(const float* src, int64_t rows, int64_t cols, int64_t lds, int64_t src_z, float* dst,
                              int64_t ldd, int64_t dst_z, int64_t nz, int phase, cudaStream_t st) {
    if (rows <= 0 || cols <= 0 || nz <= 0) return cudaSuccess;
    if (rows >= (int64_t(1) << 31) || cols >= (int64_t(1) << 31) || nz >= (int64_t(1) << 31))
        return cudaErrorInvalidConfiguration;
    PhaseScope ps(Phase(phase), st, 0, 8.0 * double(rows * cols * nz));
    // tile height: the largest of 128 / 96 / 64 / 32 rows not above `rows` (more loads in flight)
    auto go = [&](auto tr) {
        constexpr int TR = decltype(tr)::value;
        const int64_t tiles = cdiv(rows, TR) * cdiv(cols, 32) * nz;
        const int grid = int(std::min<int64_t>(tiles, int64_t(num_sms()) * 8));
        transpose_batched_kernel<TR><<<grid, 256, 0, st>>>(src, int(rows), int(cols), lds, src_z, dst, ldd, dst_z,
                                                           int(nz));
    };
    if (rows >= 128) go(std::integral_constant<int, 128>{});
    else if (rows >= 96) go(std::integral_constant<int, 96>{});
    else if (rows >= 64) go(std::integral_constant<int, 64>{});
    else go(std::integral_constant<int, 32>{});
    note_launch();
    return cudaGetLastError();
}

}  // namespace cct
