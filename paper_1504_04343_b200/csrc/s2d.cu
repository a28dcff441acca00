// s2d.cu -- space-to-depth blocking of strided Type 1 layers (see s2d.cuh).
#include <algorithm>

#include "common.cuh"
#include "s2d.cuh"

namespace cct {

Geo s2d_geo(const Geo& g) {
    Geo v = g;
    v.k = cdiv(g.k, g.s);
    v.n = g.m + v.k - 1;
    v.d = g.s * g.s * g.d;
    v.s = 1;
    v.p = 0;
    v.m = g.m;
    v.N = v.n;
    v.R = v.n;
    return v;
}

namespace {

constexpr int kThreads = 256;

// one block per X' row (q, u); the row is n' * s^2 d contiguous floats, read from
// s input rows as runs of s d contiguous floats
__global__ void s2d_input_kernel(const float* __restrict__ x, float* __restrict__ xs, int64_t b, int n, int d,
                                 int s, int p, int ns) {
    const int sd = s * d, ds = s * sd;
    const int row_len = ns * ds;
    for (int64_t row = blockIdx.x; row < b * ns; row += gridDim.x) {
        const int64_t q = row / ns;
        const int u = int(row - q * ns);
        float* dst = xs + row * row_len;
        const float* img = x + q * int64_t(n) * n * d;
        for (int e = threadIdx.x; e < row_len; e += blockDim.x) {
            const int v = e / ds;
            const int cp = e - v * ds;
            const int a = cp / sd;
            const int t = cp - a * sd;               // b d + c
            const int r = s * u + a - p;             // input row
            const int ce = (s * v - p) * d + t;      // element offset in the input row
            float val = 0.f;
            if (r >= 0 && r < n && ce >= 0 && ce < n * d) val = __ldg(img + int64_t(r) * n * d + ce);
            dst[e] = val;
        }
    }
}

// one block per dX' row (q, u): the row (n' s^2 d contiguous floats) is staged in smem,
// then the s dx rows r = s u + a - p it covers are written coalesced:
// dx[q][r][c][ch] = dX'[q][u][v][a s d + (E - v s d)], E = (c + p) d + ch, v = E / (s d)
// (0 where v >= n').  The last block also zeroes dx rows past s n' - p (no blocked row).
__global__ void d2s_input_kernel(const float* __restrict__ dxs, float* __restrict__ dx, int64_t b, int n, int d,
                                 int s, int p, int ns) {
    extern __shared__ float row_sm[];  // n' s^2 d
    const int sd = s * d, ds = s * sd, nd = n * d;
    const int row_len = ns * ds;
    for (int64_t row = blockIdx.x; row < b * ns; row += gridDim.x) {
        const int64_t q = row / ns;
        const int u = int(row - q * ns);
        __syncthreads();
        const float* src = dxs + row * row_len;
        for (int e = threadIdx.x; e < row_len; e += blockDim.x) row_sm[e] = __ldg(src + e);
        __syncthreads();
        const int r_end = (u == ns - 1) ? n : min(n, s * u - p + s);
        for (int r = max(0, s * u - p); r < r_end; ++r) {
            const int a = r + p - s * u;  // >= s: past the blocked rows -> zero
            float* out = dx + (q * n + r) * int64_t(nd);
            for (int e = threadIdx.x; e < nd; e += blockDim.x) {
                const int E = e + p * d;
                const int v = E / sd;
                out[e] = (a < s && v < ns) ? row_sm[v * ds + a * sd + (E - v * sd)] : 0.f;
            }
        }
    }
}

__global__ void s2d_weights_kernel(const float* __restrict__ w, float* __restrict__ wsd, int o, int k, int d, int s,
                                   int ks) {
    const int sd = s * d, ds = s * sd;
    const int64_t total = int64_t(o) * ks * ks * ds;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int cp = int(idx % ds);
        const int64_t t2 = idx / ds;
        const int jp = int(t2 % ks);
        const int ip = int((t2 / ks) % ks);
        const int oo = int(t2 / (int64_t(ks) * ks));
        const int a = cp / sd, bb = (cp - a * sd) / d, c = cp - a * sd - bb * d;
        const int i = s * ip + a, j = s * jp + bb;
        wsd[idx] = (i < k && j < k) ? w[((int64_t(oo) * k + i) * k + j) * d + c] : 0.f;
    }
}

__global__ void d2s_weights_kernel(const float* __restrict__ dws, float* __restrict__ dw, int o, int k, int d, int s,
                                   int ks) {
    const int ds = s * s * d;
    const int64_t total = int64_t(o) * k * k * d;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(idx % d);
        const int64_t t2 = idx / d;
        const int j = int(t2 % k);
        const int i = int((t2 / k) % k);
        const int oo = int(t2 / (int64_t(k) * k));
        dw[idx] = dws[((int64_t(oo) * ks + i / s) * ks + j / s) * ds + ((i % s) * s + j % s) * d + c];
    }
}

int rows_grid(int64_t rows) { return int(std::min<int64_t>(rows, int64_t(num_sms()) * 8)); }

}  // namespace

cudaError_t s2d_input(const Geo& g, const float* x, float* xs, cudaStream_t st) {
    const Geo v = s2d_geo(g);
    PhaseScope ps(kPhaseLower, st, 0, 4.0 * double(g.b * g.n * g.n * g.d + g.b * v.n * v.n * v.d));
    s2d_input_kernel<<<int(std::min<int64_t>(g.b * v.n, int64_t(num_sms()) * 16)), kThreads, 0, st>>>(
        x, xs, g.b, int(g.n), int(g.d), int(g.s), int(g.p), int(v.n));
    note_launch();
    return cudaGetLastError();
}

cudaError_t d2s_input(const Geo& g, const float* dxs, float* dx, cudaStream_t st) {
    const Geo v = s2d_geo(g);
    PhaseScope ps(kPhaseCol2im, st, 0, 4.0 * double(g.b * g.n * g.n * g.d + g.b * v.n * v.n * v.d));
    const size_t sm = size_t(v.n * v.d) * 4;
    if (sm > 48 * 1024) cudaFuncSetAttribute(d2s_input_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    d2s_input_kernel<<<rows_grid(g.b * v.n), kThreads, sm, st>>>(dxs, dx, g.b, int(g.n), int(g.d), int(g.s), int(g.p),
                                                                  int(v.n));
    note_launch();
    return cudaGetLastError();
}

cudaError_t s2d_weights(const Geo& g, const float* w, float* wsd, cudaStream_t st) {
    const Geo v = s2d_geo(g);
    const int64_t total = g.o * v.k * v.k * v.d;
    PhaseScope ps(kPhaseOther, st, 0, 4.0 * double(total + g.o * g.k * g.k * g.d));
    s2d_weights_kernel<<<grid_for(total, kThreads), kThreads, 0, st>>>(w, wsd, int(g.o), int(g.k), int(g.d), int(g.s),
                                                                       int(v.k));
    note_launch();
    return cudaGetLastError();
}

cudaError_t d2s_weights(const Geo& g, const float* dws, float* dw, cudaStream_t st) {
    const Geo v = s2d_geo(g);
    const int64_t total = g.o * g.k * g.k * g.d;
    PhaseScope ps(kPhaseOther, st, 0, 4.0 * double(total + g.o * v.k * v.k * v.d));
    d2s_weights_kernel<<<grid_for(total, kThreads), kThreads, 0, st>>>(dws, dw, int(g.o), int(g.k), int(g.d), int(g.s),
                                                                       int(v.k));
    note_launch();
    return cudaGetLastError();
}

}  // namespace cct
