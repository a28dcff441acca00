// test_convlow.cpp -- the convlow C++ API (drop-in for the reference's
// include/convlow/*.hpp), exercised like the reference's declared unit tests
// (CMakeLists.txt:36-47; examples SPEC.md:57-505) and checked against the C
// restatement of the oracle (oracle/cct_oracle.h, test infrastructure only).
//
//   test_convlow cpu   -- validation, planners, RNG (no device needed)
//   test_convlow gpu   -- everything, on the B200
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "cct_oracle.h"
#include "convlow/batching.hpp"
#include "convlow/cost_model.hpp"
#include "convlow/gemm.hpp"
#include "convlow/lowering.hpp"
#include "convlow/scheduler.hpp"
#include "convlow/tensor.hpp"

using namespace convlow;

static int g_fail = 0, g_run = 0;

#define CHECK(cond)                                                                   \
    do {                                                                              \
        if (!(cond)) {                                                                \
            std::printf("    CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);   \
            throw std::runtime_error("check failed");                                 \
        }                                                                             \
    } while (0)

template <class E, class F>
static void expect_throw(F f) {
    bool thrown = false;
    try {
        f();
    } catch (const E&) {
        thrown = true;
    }
    CHECK(thrown);
}

static void run(const char* name, const std::function<void()>& f) {
    ++g_run;
    try {
        f();
        std::printf("[ok  ] %s\n", name);
    } catch (const std::exception& e) {
        ++g_fail;
        std::printf("[FAIL] %s: %s\n", name, e.what());
    }
}

static double rel_l2(const std::vector<float>& a, const std::vector<float>& b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        num += (double(a[i]) - b[i]) * (double(a[i]) - b[i]);
        den += double(b[i]) * b[i];
    }
    return std::sqrt(num / (den > 0 ? den : 1));
}

static std::vector<float> flat(const DataBatch& b) {
    std::vector<float> v;
    for (const auto& t : b.images()) v.insert(v.end(), t.values().begin(), t.values().end());
    return v;
}

// ------------------------------------------------------------------ CPU tests
static void cpu_tests() {
    run("LayerConfig::validate rejects bad shapes (tensor.cpp:23-30)", [] {
        LayerConfig L{5, 6, 1, 1, 1};
        expect_throw<config_error>([&] { L.validate(); });
        L = {5, 3, 0, 1, 1};
        expect_throw<config_error>([&] { L.validate(); });
        L = {5, 3, 1, 1, 1};
        L.validate();
        CHECK(L.m() == 3);
        L.stride = 2;
        L.pad = 1;
        CHECK(L.m() == 3);
    });
    run("DataBatch rejects empty / mixed batches", [] {
        expect_throw<config_error>([] { DataBatch b(std::vector<Tensor3>{}); });
        expect_throw<config_error>([] { DataBatch b({Tensor3(3, 1), Tensor3(4, 1)}); });
    });
    run("layer_of names both shapes (tensor.cpp:66-75)", [] {
        DataBatch b({Tensor3(4, 2)});
        try {
            layer_of(b, KernelBank(3, 3, 1));
            CHECK(false);
        } catch (const config_error& e) {
            CHECK(std::string(e.what()).find("3x3x3") != std::string::npos);
            CHECK(std::string(e.what()).find("4x4x2") != std::string::npos);
        }
    });
    run("multiply validates dims and threads before touching the device (gemm.cpp:19-34)", [] {
        expect_throw<config_error>([] { multiply(Mat(2, 3), Mat(2, 3)); });
        GemmConfig c;
        c.threads = 0;
        expect_throw<config_error>([&] { multiply(Mat(2, 2), Mat(2, 2), c); });
        c.threads = 257;
        expect_throw<config_error>([&] { multiply(Mat(2, 2), Mat(2, 2), c); });
    });
    run("RNG stream equals the oracle restatement (tensor.cpp:32-45)", [] {
        std::mt19937_64 rng(1234);
        DataBatch b = DataBatch::random(2, 5, 3, rng);
        std::vector<float> mine = flat(b), ref(mine.size());
        orc_uniform_fill(1234, 0, ref.data(), ref.size());
        CHECK(mine == ref);
    });
    run("plan_partitions (SPEC.md:310-312)", [] {
        auto p = plan_partitions(256, 16, 4);
        CHECK((p.partition_sizes == std::vector<size_t>{64, 64, 64, 64}));
        CHECK((p.threads_per_partition == std::vector<size_t>{4, 4, 4, 4}));
        CHECK((plan_partitions(7, 4, 2).partition_sizes == std::vector<size_t>{4, 3}));
        expect_throw<config_error>([] { plan_partitions(4, 4, 5); });
    });
    run("proportional_split (SPEC.md:372-374)", [] {
        auto s = proportional_split({{"cpu", 1e12, 0}, {"gpu", 2e12, 0}}, 3);
        CHECK(std::fabs(s.fractions[0] - 1.0 / 3) < 1e-12 && s.counts[0] == 1 && s.counts[1] == 2);
        auto e = proportional_split(std::vector<DeviceProfile>(8, {"b200", 1.0, 0}), 2048);
        for (size_t c : e.counts) CHECK(c == 256);
        expect_throw<config_error>([] { proportional_split({}, 4); });
    });
    run("cost model KATs (SPEC.md:246-256)", [] {
        LayerConfig L{5, 3, 2, 1, 1};
        auto e = estimate(LoweringStrategy::Type1, L);
        CHECK(e.lower_elements_written == 162 && e.gemm_flops == 324 && e.lift_adds == 0);
        LayerConfig hi{13, 3, 384, 3, 256, 1, 1}, lo{13, 3, 3, 384, 256, 1, 1};
        CostWeights fwd;
        fwd.include_backward = false;
        CHECK(select_strategy(hi, fwd).strategy == LoweringStrategy::Type3);
        CHECK(select_strategy(lo, fwd).strategy == LoweringStrategy::Type1);
        LayerConfig k1{13, 1, 64, 64, 16};
        CHECK(select_strategy(k1, fwd).strategy == LoweringStrategy::Type1);  // tie -> Type1
        CHECK(std::isinf(crossover_ratio(k1)));
        LayerConfig t{13, 3, 64, 64, 16};
        const double r = crossover_ratio(t, fwd);
        CHECK(r > 0 && std::isfinite(r));
    });
    run("footprint linear in partition size (SPEC.md:328-330)", [] {
        LayerConfig L{27, 5, 96, 256, 1, 1, 2};
        for (int t = 1; t <= 3; ++t)
            CHECK(footprint(LoweringStrategy(t), L, 256).lowered_bytes_per_partition ==
                  256 * footprint(LoweringStrategy(t), L, 1).lowered_bytes_per_partition);
        CHECK(footprint(LoweringStrategy::Type3, L, 8).lowered_bytes_per_partition <
              footprint(LoweringStrategy::Type2, L, 8).lowered_bytes_per_partition);
        CHECK(footprint(LoweringStrategy::Type2, L, 8).lowered_bytes_per_partition <
              footprint(LoweringStrategy::Type1, L, 8).lowered_bytes_per_partition);
    });
}

// ------------------------------------------------------------------ GPU tests
static void gpu_tests() {
    run("direct_convolve fixture [[6,8],[12,14]] (SPEC.md:59)", [] {
        Tensor3 d(3, 1);
        for (int i = 0; i < 9; ++i) d.values()[size_t(i)] = float(i + 1);
        KernelBank k(2, 1, 1);
        k.at(0, 0, 0, 0) = 1;
        k.at(0, 1, 1, 0) = 1;
        OutputPlane r = direct_convolve(d, k);
        CHECK((r.v == std::vector<float>{6, 8, 12, 14}));
    });
    run("direct_convolve_batch bit-identical to the oracle (tensor.cpp:77-118)", [] {
        std::mt19937_64 rng(7);
        DataBatch b = DataBatch::random(3, 9, 4, rng);
        KernelBank k = KernelBank::random(3, 4, 5, rng);
        OutputBatch y = direct_convolve_batch(b, k);
        std::vector<float> x = flat(b), ref(y.size());
        orc_direct_convolve_batch(x.data(), 3, 9, 4, k.values().data(), 3, 5, ref.data());
        CHECK(y.values() == ref);
        OutputPlane p = direct_convolve(b[1], k, 2);
        CHECK(std::memcmp(p.v.data(), y.plane(1, 2), p.v.size() * 4) == 0);
    });
    run("multiply KATs and thread invariance (SPEC.md:184-186)", [] {
        Mat a(2, 2), b(2, 2);
        a.values() = {1, 2, 3, 4};
        b.values() = {5, 6, 7, 8};
        CHECK((multiply(a, b).values() == std::vector<float>{19, 22, 43, 50}));
        std::mt19937_64 rng(3);
        Mat x = Mat::random(64, 64, rng), y = Mat::random(64, 64, rng);
        Mat c1 = multiply(x, y);
        for (size_t t : {2u, 4u, 8u}) {
            GemmConfig cfg;
            cfg.threads = t;
            CHECK(multiply(x, y, cfg).values() == c1.values());
        }
    });
    run("multiply == multiply_reference within 1e-5 up to 512^3 (SPEC.md:207)", [] {
        std::mt19937_64 rng(11);
        for (size_t n : {16u, 100u, 512u}) {
            Mat a = Mat::random(n, n + 3, rng), b = Mat::random(n + 3, n - 1, rng);
            CHECK(rel_l2(multiply(a, b).values(), multiply_reference(a, b).values()) < 1e-5);
        }
    });
    run("multiply_reference bit-identical to the oracle (gemm.cpp:124-141)", [] {
        std::mt19937_64 rng(12);
        Mat a = Mat::random(33, 65, rng), b = Mat::random(65, 17, rng);
        std::vector<float> ref(33 * 17);
        orc_multiply(a.values().data(), b.values().data(), ref.data(), 33, 65, 17);
        CHECK(multiply_reference(a, b).values() == ref);
    });
    run("lower: SPEC shapes and bit-exact matrices (SPEC.md:118-120)", [] {
        std::mt19937_64 rng(5);
        DataBatch b = DataBatch::random(2, 5, 2, rng);
        KernelBank k = KernelBank::random(3, 2, 4, rng);
        for (int t = 1; t <= 3; ++t) {
            LoweredMatrices lm = lower(b, k, LoweringStrategy(t));
            long rows, cols, kc;
            orc_lowered_shape(t, 2, 5, 2, 3, 4, &rows, &cols, &kc);
            CHECK(lm.Dhat.rows() == size_t(rows) && lm.Dhat.cols() == size_t(cols) && lm.Khat.cols() == size_t(kc));
            std::vector<float> dh(size_t(rows * cols)), kh(size_t(cols * kc)), x = flat(b);
            orc_lower(t, x.data(), k.values().data(), 2, 5, 2, 3, 4, dh.data(), kh.data());
            CHECK(lm.Dhat.values() == dh && lm.Khat.values() == kh);
        }
        DataBatch one = DataBatch::random(1, 5, 2, rng);
        KernelBank k1 = KernelBank::random(3, 2, 1, rng);
        LoweredMatrices t1 = lower(one, k1, LoweringStrategy::Type1);
        CHECK(t1.Dhat.rows() == 9 && t1.Dhat.cols() == 18 && t1.Khat.rows() == 18 && t1.Khat.cols() == 1);
    });
    run("lift(multiply(lower)) == direct for every strategy (SPEC.md:136-141)", [] {
        std::mt19937_64 rng(9);
        DataBatch b = DataBatch::random(2, 9, 4, rng);
        KernelBank k = KernelBank::random(3, 4, 5, rng);
        const std::vector<float> ref = direct_convolve_batch(b, k).values();
        for (int t = 1; t <= 3; ++t) {
            LoweredMatrices lm = lower(b, k, LoweringStrategy(t));
            OutputBatch y = lift(multiply(lm.Dhat, lm.Khat), LoweringStrategy(t), lm.layer);
            CHECK(rel_l2(y.values(), ref) < 1e-5);
        }
    });
    run("convolve_lowered n=13 k=3 d=384 o=384 b=4 (SPEC.md:138) + PhaseTimings", [] {
        std::mt19937_64 rng(1234);
        DataBatch b = DataBatch::random(4, 13, 384, rng);
        KernelBank k = KernelBank::random(3, 384, 384, rng);
        const std::vector<float> ref = direct_convolve_batch(b, k).values();
        for (int t = 1; t <= 3; ++t) {
            auto [y, pt] = convolve_lowered(b, k, LoweringStrategy(t), 8);
            CHECK(rel_l2(y.values(), ref) <= 1e-4);
            CHECK(pt.multiply_s > 0);
            if (t != 1) CHECK(pt.lift_s > 0);
        }
        expect_throw<config_error>([&] { convolve_lowered(b, k, LoweringStrategy::Type1, 0); });
    });
    run("strided / padded forward and both backward passes vs the oracle", [] {
        std::mt19937_64 rng(21);
        const size_t n = 23, kk = 11, d = 3, o = 8, bb = 2, s = 4, p = 0;
        DataBatch b = DataBatch::random(bb, n, d, rng);
        KernelBank k = KernelBank::random(kk, d, o, rng);
        const size_t m = (n + 2 * p - kk) / s + 1;
        OutputBatch dy(bb, o, m);
        std::uniform_real_distribution<float> u(-1, 1);
        for (auto& v : dy.values()) v = u(rng);
        std::vector<float> x = flat(b), ry(bb * o * m * m), rdx(x.size()), rdw(k.values().size());
        orc_conv_fwd(x.data(), k.values().data(), ry.data(), bb, n, d, kk, o, s, p);
        orc_conv_bwd_data(dy.values().data(), k.values().data(), rdx.data(), bb, n, d, kk, o, s, p);
        orc_conv_bwd_weight(x.data(), dy.values().data(), rdw.data(), bb, n, d, kk, o, s, p);
        for (int t = 1; t <= 3; ++t) {
            ConvGeometry g{s, p};
            auto [y, pt] = convolve_lowered(b, k, LoweringStrategy(t), 1, g);
            CHECK(rel_l2(y.values(), ry) <= 1e-4);
            CHECK(rel_l2(flat(convolve_backward_data(dy, k, n, LoweringStrategy(t), g)), rdx) <= 1e-4);
            CHECK(rel_l2(convolve_backward_weight(b, dy, kk, LoweringStrategy(t), g).values(), rdw) <= 1e-4);
        }
    });
    run("layer extension: groups = 2 + bias + ReLU == per-group convolutions (cct_conv_*_ex)", [] {
        std::mt19937_64 rng(31);
        const size_t n = 13, kk = 3, d = 16, o = 24, bb = 2, G = 2, s = 1, p = 1;
        DataBatch b = DataBatch::random(bb, n, d, rng);
        KernelBank k = KernelBank::random(kk, d / G, o, rng);
        LayerExtension ext;
        ext.groups = G;
        ext.relu = true;
        std::uniform_real_distribution<float> u(-1, 1);
        for (size_t j = 0; j < o; ++j) ext.bias.push_back(u(rng));
        const size_t m = (n + 2 * p - kk) / s + 1;
        OutputBatch dy(bb, o, m);
        for (auto& v : dy.values()) v = u(rng);
        // reference: each group through the oracle, then bias + ReLU; backward with the mask of y
        std::vector<float> x = flat(b), ry(bb * o * m * m), rdx(x.size()), rdw(k.values().size()), rdb(o, 0.f);
        const size_t dg = d / G, og = o / G;
        for (size_t g = 0; g < G; ++g) {
            std::vector<float> xg(bb * n * n * dg), wg(k.values().begin() + g * og * kk * kk * dg,
                                                          k.values().begin() + (g + 1) * og * kk * kk * dg);
            for (size_t i = 0; i < bb * n * n; ++i)
                for (size_t c = 0; c < dg; ++c) xg[i * dg + c] = x[i * d + g * dg + c];
            std::vector<float> yg(bb * og * m * m);
            orc_conv_fwd(xg.data(), wg.data(), yg.data(), bb, n, dg, kk, og, s, p);
            for (size_t q = 0; q < bb; ++q)
                for (size_t j = 0; j < og; ++j)
                    for (size_t e = 0; e < m * m; ++e)
                        ry[(q * o + g * og + j) * m * m + e] = std::max(0.f, yg[(q * og + j) * m * m + e] + ext.bias[g * og + j]);
        }
        auto [y, t] = convolve_lowered_ex(b, k, LoweringStrategy::Type1, ext, ConvGeometry{s, p});
        CHECK(rel_l2(y.values(), ry) <= 1e-4);
        OutputBatch dz = dy;
        for (size_t i = 0; i < dz.values().size(); ++i) dz.values()[i] = y.values()[i] > 0 ? dy.values()[i] : 0.f;
        for (size_t g = 0; g < G; ++g) {
            std::vector<float> xg(bb * n * n * dg), wg(k.values().begin() + g * og * kk * kk * dg,
                                                          k.values().begin() + (g + 1) * og * kk * kk * dg);
            for (size_t i = 0; i < bb * n * n; ++i)
                for (size_t c = 0; c < dg; ++c) xg[i * dg + c] = x[i * d + g * dg + c];
            std::vector<float> dzg(bb * og * m * m), dxg(xg.size()), dwg(wg.size());
            for (size_t q = 0; q < bb; ++q)
                for (size_t e = 0; e < og * m * m; ++e) dzg[q * og * m * m + e] = dz.values()[(q * o + g * og) * m * m + e];
            orc_conv_bwd_data(dzg.data(), wg.data(), dxg.data(), bb, n, dg, kk, og, s, p);
            orc_conv_bwd_weight(xg.data(), dzg.data(), dwg.data(), bb, n, dg, kk, og, s, p);
            for (size_t i = 0; i < bb * n * n; ++i)
                for (size_t c = 0; c < dg; ++c) rdx[i * d + g * dg + c] = dxg[i * dg + c];
            std::copy(dwg.begin(), dwg.end(), rdw.begin() + g * og * kk * kk * dg);
        }
        for (size_t q = 0; q < bb; ++q)
            for (size_t j = 0; j < o; ++j)
                for (size_t e = 0; e < m * m; ++e) rdb[j] += dz.values()[(q * o + j) * m * m + e];
        LayerGradients gr = convolve_backward_ex(b, y, dy, k, LoweringStrategy::Type1, ext, ConvGeometry{s, p});
        CHECK(rel_l2(flat(gr.dx), rdx) <= 1e-4);
        CHECK(rel_l2(gr.dw.values(), rdw) <= 1e-4);
        CHECK(rel_l2(gr.db, rdb) <= 1e-5);
        LayerExtension bad = ext;
        bad.groups = 5;
        expect_throw<config_error>([&] { convolve_lowered_ex(b, k, LoweringStrategy::Type1, bad); });
    });
    run("execute_partitioned invariant under p (SPEC.md:319, 333)", [] {
        std::mt19937_64 rng(4);
        DataBatch b = DataBatch::random(8, 11, 16, rng);
        KernelBank k = KernelBank::random(3, 16, 24, rng);
        PartitionedResult r1 = execute_partitioned(b, k, LoweringStrategy::Type1, plan_partitions(8, 8, 1));
        for (size_t p : {2u, 4u, 8u}) {
            PartitionedResult rp = execute_partitioned(b, k, LoweringStrategy::Type1, plan_partitions(8, 8, p));
            CHECK(rp.output.values() == r1.output.values());
            CHECK(rp.footprint.peak_bytes == p * rp.footprint.lowered_bytes_per_partition);
        }
    });
    run("probes: device GEMM throughput and copy bandwidth (gemm.cpp:143-200)", [] {
        ProbeResult pr = gemm_throughput_probe(1024, 1024, 1024, GemmConfig{}, 3);
        CHECK(pr.flops == 2ull * 1024 * 1024 * 1024 && pr.flops_per_s > 1e12 && pr.reps == 3);
        CHECK(memcpy_bandwidth_probe(std::size_t(256) << 20, 3) > 1e11);
        expect_throw<resource_error>([] { gemm_throughput_probe(40000, 40000, 1000, GemmConfig{}, 1); });
    });
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "gpu";
    cpu_tests();
    if (mode == "gpu") gpu_tests();
    std::printf("%d/%d passed\n", g_run - g_fail, g_run);
    return g_fail ? 1 : 0;
}
