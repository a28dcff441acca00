// hfold_probe.cu -- where does conv_dgrad_hfold_kernel spend its time?  Times the conv1
// backward-data (b = 256) with stages dropped through Params::dbg: 1 = no epilogue fold /
// stores, 2 = no dy transform (TMEM A slots left stale), 4 = no MMAs (commits only), 8 = epilogue
// TMEM loads only, 16 = no H stores.  The
// variants compute garbage; only the times matter.  Built against the library objects:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//     -Iinclude -Ipaper_1504_04343_b200/csrc tools/hfold_probe.cu \
//     $(ls paper_1504_04343_b200/_lib/obj/*.o | grep -v -e /dgrad.o -e host_) -o tools/hfold_probe -lcuda
#include "../paper_1504_04343_b200/csrc/dgrad.cu"

#include <cstdio>
#include <vector>

int main(int argc, char** argv) {
    using namespace cct;
    const int b = argc > 1 ? atoi(argv[1]) : 256;
    Geo g{};
    g.b = b; g.n = 227; g.d = 3; g.k = 11; g.o = 96; g.s = 4; g.p = 0;
    g.m = 55; g.N = 227; g.R = 4 * 54 + 11; g.yl = 1;
    if (!hfold_dgrad_ok(g)) { printf("geometry not supported\n"); return 1; }
    const size_t ny = size_t(b) * 55 * 55 * 96, nw = 96 * 11 * 11 * 3, nx = size_t(b) * 227 * 227 * 3;
    const size_t nws = size_t(hfold_dgrad_ws_floats(g));
    float *dy, *w, *dx, *ws, *flush;
    cudaMalloc(&dy, ny * 4); cudaMalloc(&w, nw * 4); cudaMalloc(&dx, nx * 4); cudaMalloc(&ws, nws * 4);
    cudaMalloc(&flush, size_t(256) << 20);
    std::vector<float> h(ny);
    for (size_t i = 0; i < ny; ++i) h[i] = float((i * 2654435761u) % 1000) / 500.f - 1.f;
    cudaMemcpy(dy, h.data(), ny * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(w, h.data(), nw * 4, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1, k0, k1;
    cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&k0); cudaEventCreate(&k1);
    const int variants[] = {0, 3, 6, 6 | 8, 6 | 16, 2 | 16, 16, 0};
    for (int v : variants) {
        hf::g_probe_dbg = v;
        float best = 1e9f;
        for (int it = 0; it < 6; ++it) {
            cudaMemsetAsync(flush, it, size_t(256) << 20);
            cudaEventRecord(e0);
            cudaError_t err = hfold_dgrad(g, dy, w, dx, ws, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) { printf("error\n"); return 1; }
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it > 0 && ms < best) best = ms;
        }
        printf("dbg %d: hfold_dgrad (prep + hfold + vfold) %.1f us\n", v, best * 1e3f);
    }
    return 0;
}
