// gather_probe.cu -- where does conv_fwd_gather_kernel spend its time?  Times the fused conv1
// forward (b = 256, NHWC y) with stages dropped through FwdParams::dbg: 1 = no epilogue, 2 = no
// gather (TMEM A slots left stale), 4 = no MMAs (commits only), 8 = no input-row copies,
// 16 = no kernel-bank copies, 32 = plain mbarrier arrives instead of tcgen05.commit (with 4),
// 64 = spinning mbarrier waits instead of suspending ones, bits 8+: epilogue pause (x100 ns) between
// its 32-column TMEM chunks (product default 300 ns).  The
// variants compute garbage; only the times matter.  Build (as tools/hfold_probe.cu):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//     -Iinclude -Ipaper_1504_04343_b200/csrc tools/gather_probe.cu \
//     $(ls paper_1504_04343_b200/_lib/obj/*.o | grep -v -e /gather.o -e host_) -o tools/gather_probe -lcuda
#include "../paper_1504_04343_b200/csrc/gather.cu"

#include <cstdio>
#include <vector>

int main(int argc, char** argv) {
    using namespace cct;
    const int b = argc > 1 ? atoi(argv[1]) : 256;
    Geo g{};
    g.b = b; g.n = 227; g.d = 3; g.k = 11; g.o = 96; g.s = 4; g.p = 0;
    g.m = 55; g.N = 227; g.R = 4 * 54 + 11; g.yl = 1;
    if (!gather_fwd_ok(g)) { printf("geometry not supported\n"); return 1; }
    const size_t ny = size_t(b) * 55 * 55 * 96, nw = 96 * 11 * 11 * 3, nx = size_t(b) * 227 * 227 * 3;
    const size_t nws = size_t(std::max(gather_fwd_ws_floats(g), gather_wgrad_ws_floats(g)));
    float *x, *w, *y, *ws, *flush;
    cudaMalloc(&x, nx * 4); cudaMalloc(&w, nw * 4); cudaMalloc(&y, ny * 4); cudaMalloc(&ws, nws * 4);
    cudaMalloc(&flush, size_t(256) << 20);
    std::vector<float> h(nx);
    for (size_t i = 0; i < nx; ++i) h[i] = float((i * 2654435761u) % 1000) / 500.f - 1.f;
    cudaMemcpy(x, h.data(), nx * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(w, h.data(), nw * 4, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int variants[] = {0, 3 << 8, 0};
    for (int mode = 1; mode <= 1; ++mode)  // CCT_TUNE_GATHER: 1 merged products (4 MMAs / k-block), 2 six MMAs
    for (int v : variants) {
        cct_set_tuning(CCT_TUNE_GATHER, mode);
        gth::g_probe_dbg = v & 255;
        gth::g_probe_pace_ns = v ? (v >> 8) * 100 : -1;  // 0: the product default
        float best = 1e9f;
        for (int it = 0; it < 6; ++it) {
            cudaMemsetAsync(flush, it, size_t(256) << 20);
            cudaEventRecord(e0);
            cudaError_t err = gather_fwd(g, x, w, y, 0, nullptr, 0, ws, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) { printf("error\n"); return 1; }
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it > 0 && ms < best) best = ms;
        }
        printf("gather %d dbg %2d: gather_fwd (prep + kernel) %.1f us\n", mode, v, best * 1e3f);
    }
    // one traced run (dbg 0): CTA 0's event clocks, relative to its first MMA-tile start
    {
        const size_t nt = 22 * 64 * 32;
        unsigned long long* dtr;
        cudaMalloc(&dtr, nt * 8);
        cudaMemset(dtr, 0, nt * 8);
        gth::g_probe_dbg = 0;
        gth::g_probe_trace = dtr;
        cct_set_tuning(CCT_TUNE_GATHER, 1);
        gather_fwd(g, x, w, y, 0, nullptr, 0, ws, 0);
        cudaDeviceSynchronize();
        gth::g_probe_trace = nullptr;
        std::vector<unsigned long long> t(nt);
        cudaMemcpy(t.data(), dtr, nt * 8, cudaMemcpyDeviceToHost);
        auto at = [&](int role, int lt, int ev) { return t[(size_t(role) * 64 + lt) * 32 + ev]; };
        const unsigned long long t0 = at(0, 0, 0);
        auto rel = [&](unsigned long long v) { return v ? (long long)(v - t0) : -1LL; };
        printf("trace (cycles from MMA tile 0 start): per tile: MMA start / kb0 / kb12 / kb24 / end; "
               "gather grp0 start / xfull / first aempty-wait-start,-end / last arrive; epi start / end; rows xempty / issued\n");
        for (int lt = 0; lt < 44; ++lt) {
            if (!at(0, lt, 0)) break;
            printf("t%02d MMA %8lld %8lld %8lld %8lld %8lld | G %8lld %8lld %8lld %8lld %8lld | E %8lld %8lld | R %8lld %8lld\n", lt,
                   rel(at(0, lt, 0)), rel(at(0, lt, 1)), rel(at(0, lt, 13)), rel(at(0, lt, 25)), rel(at(0, lt, 30)),
                   rel(at(1, lt, 0)), rel(at(1, lt, 1)), rel(at(1, lt, 2)), rel(at(1, lt, 10)), rel(at(1, lt, 24)),
                   rel(at(2, lt, 0)), rel(at(2, lt, 1)), rel(at(3, lt, 0)), rel(at(3, lt, 2)));
        }
        // per-kb MMA issue gaps of a middle tile
        const int mt = 20;
        printf("tile %d MMA kb issue times:", mt);
        for (int kb = 0; kb < 25; ++kb) printf(" %lld", rel(at(0, mt, 1 + kb)));
        printf("\ntile %d gather grp0 (wait-start, wait-end, arrive) per its kb:", mt);
        for (int j = 0; j < 7; ++j) printf(" (%lld %lld %lld)", rel(at(1, mt, 2 + j)), rel(at(1, mt, 10 + j)), rel(at(1, mt, 18 + j)));
        printf("\n");
        for (int lt2 = 19; lt2 <= 21; ++lt2) {
            printf("tile %d per kb: MMA bfull-done / afull-done / arrive of each of the k-block's 4 gather warps\n", lt2);
            for (int kb = 0; kb < 25; ++kb) {
                const int grp = int((kb + 25 * lt2) % 4);  // gi = 25 lt + kb -> group gi % 4
                printf("  kb%02d g%d %8lld %8lld |", kb, grp, rel(at(5, lt2, 1 + kb)), rel(at(0, lt2, 1 + kb)));
                for (int w = 0; w < 4; ++w) printf(" %8lld", rel(at(6 + 4 * grp + w, lt2, kb)));
                printf("\n");
            }
        }
    }
    return 0;
}
