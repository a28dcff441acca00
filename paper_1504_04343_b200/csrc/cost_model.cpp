// cost_model.cpp -- the automatic lowering optimizer (PAPER.md:76-77,
// 536-580), re-derived for this B200 implementation.
//
// Two scores are produced per (layer, type):
//   * total_score  -- the SPEC's alpha*(lower_elements + lift_adds) + beta*gemm_flops
//                     with the SPEC's exact counts;
//   * model_seconds -- a roofline model of the kernels THIS build launches
//                     (bytes each HBM-bound kernel moves / measured copy rate,
//                     executed GEMM flops / measured 3xTF32 rate with tile and
//                     wave quantisation, plus a per-launch cost), calibrated on
//                     B200 measurements.
// select_strategy takes the argmin of model_seconds; ties break T1 < T2 < T3
// (SPEC.md:236).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "cct.h"
#include "dgrad.cuh"
#include "gather.cuh"

namespace {

struct G {
    double b, n, d, k, o, s, p, m, R, N;
};

G geo(const cct_conv_desc* d) {
    G g;
    g.b = double(d->b); g.n = double(d->n); g.d = double(d->d); g.k = double(d->k);
    g.o = double(d->o); g.s = double(d->stride); g.p = double(d->pad);
    g.N = g.n + 2 * g.p;
    g.m = std::floor((g.N - g.k) / g.s) + 1;
    g.R = g.s * (g.m - 1) + g.k;
    return g;
}

double rup(double v, double q) { return std::ceil(v / q) * q; }

// Measured steady-state 3xTF32 GEMM rate (TF/s) of gemm3xtf32_kernel on B200 by
// tile width BN (rows) and reduction length K (cols): tools/gemm_bench.py
// --rate-table (M >= 16 tiles per CTA pair), re-measured on the round-2 build (warp-uniform
// MMA / TMA issue): profiles/r02/gemm_rate_table.json.  Longer K is chain-split at 4096.
const double kBN[5] = {64, 96, 128, 192, 256};
const double kK[4] = {64, 256, 1024, 4096};
const double kRate[5][4] = {
    {76.7, 147.5, 165.2, 170.4},   // BN 64
    {98.2, 185.8, 208.4, 216.2},   // BN 96
    {112.7, 193.2, 218.9, 226.6},  // BN 128
    {119.6, 240.0, 278.8, 292.4},  // BN 192
    {94.1, 193.7, 270.2, 300.1},   // BN 256
};
const double kRateRef = 300.1e12;  // table entry the calibration's gemm_flops_per_s scales

double interp_rate(double bn, double k) {
    auto pos = [](const double* xs, int n, double v, int* i0, double* f) {
        v = std::log(std::max(xs[0], std::min(xs[n - 1], v)));
        for (int i = 0; i < n - 1; ++i)
            if (v <= std::log(xs[i + 1])) {
                *i0 = i;
                *f = (v - std::log(xs[i])) / (std::log(xs[i + 1]) - std::log(xs[i]));
                return;
            }
        *i0 = n - 2;
        *f = 1.0;
    };
    int ib, ik;
    double fb, fk;
    pos(kBN, 5, bn, &ib, &fb);
    pos(kK, 4, k, &ik, &fk);
    const double r0 = kRate[ib][ik] * (1 - fk) + kRate[ib][ik + 1] * fk;
    const double r1 = kRate[ib + 1][ik] * (1 - fk) + kRate[ib + 1][ik + 1] * fk;
    return (r0 * (1 - fb) + r1 * fb) * 1e12;
}

// GEMM time: padded flops / measured rate for the tile width the kernel picks.  N a
// multiple of 384 runs the 256 + 128 composite tile (gemm.cu tile_n), measured at the
// 256-wide rate (conv4 forward: 271 TF/s algorithmic).
double gemm_seconds(double M, double N, double K, const cct_calibration* c) {
    static const double cands[] = {256, 192, 128, 96, 64};
    double bn = 256, best = 1e300;
    for (double x : cands) {
        const double pad = rup(N, x);
        if (pad < best) { best = pad; bn = x; }
    }
    const bool wide384 = cct_get_tuning(CCT_TUNE_BN384) && std::fmod(N, 384.0) == 0;
    const double rate = interp_rate(wide384 ? 256.0 : bn, std::min(K, 4096.0)) * (c->gemm_flops_per_s / kRateRef);
    return 2.0 * rup(M, 128) * rup(N, bn) * K / rate;
}

// Backward-data of Type 1 at stride 1 can run implicitly (cct_abi.cu
// run_bwd_implicit): dy -> NHWC transpose, then the forward convolution of dy
// with the rotated kernel bank straight into dx (GEMM b n^2 x d x k^2 o).
bool implicit_dgrad_possible(const G& g) {
    return cct_get_implicit_lowering() && g.s == 1 && g.p <= g.k - 1 && std::fmod(g.o, 16) == 0;
}

// seconds of the bwd-data GEMM + its data movement after dRhat is available;
// `implicit` selects the implicit form (no dDhat, no col2im)
double dgrad_seconds(const G& g, bool implicit, double rows, double cols, double ncols, double dhat, double rhat,
                     double xin, bool t3_zero_copy, const cct_calibration* c, double* by, double* launches) {
    double t = 0;
    if (implicit) {
        const double K = g.k * g.k * g.o, M = g.b * g.n * g.n;
        // pixels x d tiles (CTA pairs; the swapped d-row form is opt-in, CCT_TUNE_DGRAD_SWAP,
        // measured 8 % slower on conv2 after the warp-uniform issue fix)
        const double gt = cct_get_tuning(CCT_TUNE_DGRAD_SWAP) && g.d < 128 ? gemm_seconds(g.d, M, K, c) * 1.08
                                                                           : gemm_seconds(M, g.d, K, c);
        const double gb = rhat + xin;
        t += std::max(gt, gb / c->hbm_bytes_per_s);
        *by += gb;
        *launches += 2;  // rotate weights + GEMM
        const double chains = std::ceil(K / 4096.0);
        if (chains > 1) {  // accuracy split-K: partials written, reduced
            const double rb = (2 * chains + 1) * xin;
            t += rb / c->hbm_bytes_per_s;
            *by += rb;
            *launches += 1;
        }
        return t;
    }
    const double gt = gemm_seconds(cols, rows, ncols, c);
    const double gb = rhat + dhat;
    t += std::max(gt, gb / c->hbm_bytes_per_s);
    *by += gb;
    *launches += 1;
    if (!t3_zero_copy) {  // col2im / crop
        t += (dhat + xin) / c->hbm_bytes_per_s;
        *by += dhat + xin;
        *launches += 1;
    }
    return t;
}

// Strided Type 1 layers with s^2 d % 16 == 0 run in space-to-depth form
// (s2d.cuh, cct_abi.cu t1_s2d): the stride-1 layer of side m + k' - 1, k' = ceil(k/s)
// taps, depth s^2 d, plus the blocking / unblocking passes.
bool s2d_possible(const G& g) {
    return cct_get_tuning(CCT_TUNE_S2D) != 0 && cct_get_implicit_lowering() && g.s > 1 && std::fmod(g.s * g.s * g.d, 16) == 0;
}
G s2d_of(const G& g) {
    G v = g;
    v.k = std::ceil(g.k / g.s);
    v.n = g.m + v.k - 1;
    v.d = g.s * g.s * g.d;
    v.s = 1;
    v.p = 0;
    v.N = v.n;
    v.R = v.n;
    return v;
}

void one_pass(const G& g, int type, int pass, const cct_calibration* c, double* secs, double* bytes,
              bool allow_s2d = true, bool allow_fused = true);

// model seconds of a strided Type 1 pass with (true) / without the space-to-depth form
double t1_form_seconds(const G& g, int pass, bool s2d, const cct_calibration* c) {
    double secs = 0, bytes = 0;
    one_pass(g, 1, pass, c, &secs, &bytes, s2d, false);  // (the unfused forms)
    return secs;
}

// counts + model for one pass.  pass: 0 fwd, 1 bwd-data, 2 bwd-weight, 3 training step.
// A strided Type 1 layer takes the faster of its direct and space-to-depth forms,
// as the launcher does (cct::prefer_s2d).
// Small-channel Type 1 layers the launcher runs fused (cct_abi.cu t1_gather_fwd /
// t1_gather_wgrad / t1_hfold_dgrad: d % 16 != 0 and the fused kernels' geometry limits).
cct::Geo geo_cct(const G& g) {
    cct::Geo v;
    v.b = int64_t(g.b); v.n = int64_t(g.n); v.d = int64_t(g.d); v.k = int64_t(g.k); v.o = int64_t(g.o);
    v.s = int64_t(g.s); v.p = int64_t(g.p); v.N = int64_t(g.N); v.m = int64_t(g.m); v.R = int64_t(g.R);
    v.yl = 1;
    return v;
}
bool fused_small(const G& g) {
    return cct_get_tuning(CCT_TUNE_GATHER) != 0 && cct_get_implicit_lowering() && std::fmod(g.d, 16) != 0;
}

void one_pass(const G& g, int type, int pass, const cct_calibration* c, double* secs, double* bytes,
              bool allow_s2d, bool allow_fused) {
    const double f = 4.0;  // bytes per float
    // fused small-channel Type 1 passes (gather.cuh, dgrad.cuh): executed flops at the rates
    // measured on B200 for CaffeNet conv1 (b = 256, profiles/r02): forward 0.65, backward-weight
    // 0.59, backward-data GEMM 0.57 of the table GEMM rate; the backward-data's vertical fold
    // streams its partial rows at 1.15 x the lowering copy rate
    if (type == 1 && allow_fused && fused_small(g)) {
        const cct::Geo v = geo_cct(g);
        const bool fw = cct::gather_fwd_ok(v), wg = cct::gather_wgrad_ok(v), dg = cct::hfold_dgrad_ok(v);
        if (fw || wg || dg) {
            double t = 0, by = 0, launches = 0;
            const double flops = 2.0 * g.b * g.m * g.m * g.k * g.k * g.d * g.o;
            const double xin = g.b * g.n * g.n * g.d * f, yout = g.b * g.o * g.m * g.m * f;
            const double rate = c->gemm_flops_per_s;
            double sf = 0, bf = 0, sw = 0, bw = 0, sd = 0, bd = 0;
            if (fw) { sf = flops / (0.65 * rate); bf = xin + yout; }
            else one_pass(g, 1, 0, c, &sf, &bf, allow_s2d, false);
            if (wg) { sw = flops / (0.63 * rate); bw = xin + yout; }
            else one_pass(g, 1, 2, c, &sw, &bw, allow_s2d, false);
            if (dg) {
                const double xp = std::ceil((g.s * g.d * (g.m - 1) + g.k * g.d + 6) / 4) * 4;
                const double h = g.b * g.m * g.k * xp * f;
                sd = flops / (0.57 * rate) + (h + xin) / (1.15 * c->hbm_bytes_per_s);
                bd = 2 * yout + 2 * h + xin;
                launches += 1;
            } else {
                one_pass(g, 1, 1, c, &sd, &bd, allow_s2d, false);
            }
            launches += 2;
            if (pass == 0) { t = sf; by = bf; }
            else if (pass == 1) { t = sd; by = bd; }
            else if (pass == 2) { t = sw; by = bw; }
            else { t = sf + sd + sw; by = bf + bd + bw; }
            *secs = t + (pass == 3 ? 3 : 1) * launches / 3 * c->launch_s;
            *bytes = by;
            return;
        }
    }
    if (type == 1 && allow_s2d && s2d_possible(g)) {
        double s0 = 0, b0 = 0, s1 = 0, b1 = 0;
        one_pass(g, 1, pass, c, &s0, &b0, false, allow_fused);
        const G v = s2d_of(g);
        one_pass(v, 1, pass, c, &s1, &b1, false);
        const double xin = g.b * g.n * g.n * g.d * f, xs = v.b * v.n * v.n * v.d * f;
        // blocking of x (fwd, or wgrad without the forward's cache), unblocking of dx,
        // and the two small kernel-bank gathers; the blocking kernels run at ~0.5 of
        // the copy rate (one-thread-per-element gathers)
        const double moved = (pass == 3 ? 2.0 : 1.0) * (xin + xs);
        const double launches = pass == 0 ? 2 : pass == 3 ? 5 : 3;
        s1 += moved / (0.5 * c->hbm_bytes_per_s) + launches * c->launch_s;
        b1 += moved;
        if (s1 < s0) { *secs = s1; *bytes = b1; }
        else { *secs = s0; *bytes = b0; }
        return;
    }
    double rows, cols, ncols;
    if (type == 1) { rows = g.b * g.m * g.m; cols = g.k * g.k * g.d; ncols = g.o; }
    else if (type == 2) { rows = g.b * g.R * g.m; cols = g.k * g.d; ncols = g.k * g.o; }
    else { rows = g.b * g.R * g.R; cols = g.d; ncols = g.k * g.k * g.o; }
    const double xin = g.b * g.n * g.n * g.d * f, yout = g.b * g.o * g.m * g.m * f;
    const double dhat = rows * rup(cols, 4) * f, rhat = rows * ncols * f;
    const bool t3_zero_copy = (type == 3 && g.p == 0 && g.R == g.n && std::fmod(g.d, 4) == 0);
    // implicit Type 1 (TMA im2col operands, d % 16 == 0): no lowering, A read from x;
    // backward-weight through im2col measured ~10% slower than from a materialised Dhat,
    // and its taps are padded to dk = d rounded up to 32 channels
    const bool t1_implicit = (type == 1 && std::fmod(g.d, 16) == 0 && cct_get_implicit_lowering());
    const double wg_cols = t1_implicit ? g.k * g.k * rup(g.d, 32) : cols;
    // implicit backward-weight GEMM: MN-major im2col A; narrow banks (o <= 96) run
    // without CTA pairs (measured 0.74 of the table rate, conv1 in s2d form)
    const double wg_slow = t1_implicit ? (g.o <= 96 ? 1.35 : 1.1) : 1.0;
    // ... except that with the implicit backward (dy in NHWC) a narrow bank runs swapped
    // (cct_abi.cu wgrad_swapped): o rows of a 128-row tile, the (tap, channel) columns wide
    const bool wg_swap = t1_implicit && g.o < 128 && implicit_dgrad_possible(g) && wg_cols >= 192;
    auto wgrad_gemm = [&]() {
        // (measured on conv1 in blocked form: 1.46x the table rate -- CTA-pair-less, and the
        // producer issues 4 + 6 TMA boxes per k-block)
        return wg_swap ? gemm_seconds(g.o, wg_cols, rows, c) * 1.46 : gemm_seconds(wg_cols, ncols, rows, c) * wg_slow;
    };
    double t = 0, by = 0, launches = 0;
    // measured class rates (configs[1] sweep on the round-2 build, profiles/r02): the staged
    // relative to the lower / col2im copy rate: the bulk-copy lift streams at ~1.25 (5.3 TB/s) and
    // the shift-copy expand at ~0.98 (4.1 TB/s) -- configs[1] sweep, profiles/r02/sweep_lowering_types_b256_r2final
    const double lift_bw = c->hbm_bytes_per_s * 1.25, expand_bw = c->hbm_bytes_per_s * 0.98;
    auto hbm = [&](double b) { by += b; t += b / c->hbm_bytes_per_s; launches += 1; };
    auto hbm_at = [&](double b, double bw) { by += b; t += b / bw; launches += 1; };
    const double a_in = t1_implicit ? xin : dhat;         // bytes of the A operand stream
    // backward-data: the faster of the materialised and (Type 1, stride 1) implicit forms,
    // as the product picks it (prefer_implicit_dgrad)
    auto dgrad = [&](double* b_, double* l_) {
        double be = 0, le = 0;
        const double te = dgrad_seconds(g, false, rows, cols, ncols, dhat, rhat, xin, t3_zero_copy, c, &be, &le);
        if (type == 1 && implicit_dgrad_possible(g)) {
            double bi = 0, li = 0;
            const double ti = dgrad_seconds(g, true, rows, cols, ncols, dhat, rhat, xin, t3_zero_copy, c, &bi, &li);
            if (cct_get_implicit_lowering() == 2 || ti + li * c->launch_s < te + le * c->launch_s) {
                *b_ += bi;
                *l_ += li;
                return ti;
            }
        }
        *b_ += be;
        *l_ += le;
        return te;
    };
    if (pass == 0) {
        if (!t3_zero_copy && !t1_implicit) hbm(xin + dhat); // lower
        const double gt = gemm_seconds(rows, ncols, cols, c);
        const double gb = a_in + (type == 1 ? yout : rhat);
        t += std::max(gt, gb / c->hbm_bytes_per_s);        // GEMM (A streamed once)
        by += gb;
        launches += 1;
        if (type != 1) hbm_at(rhat + yout, lift_bw);       // lift
    } else if (pass == 1) {
        hbm_at(yout + rhat, type == 1 ? c->hbm_bytes_per_s * 0.45 : expand_bw);  // expand
        t += dgrad(&by, &launches);
    } else if (pass == 2) {
        if (!t3_zero_copy && !t1_implicit) hbm(xin + dhat); // lower
        hbm_at(yout + rhat, type == 1 ? c->hbm_bytes_per_s * 0.45 : expand_bw);  // expand
        const double gt = wgrad_gemm();
        const double gb = a_in + rhat;
        t += std::max(gt, gb / c->hbm_bytes_per_s);
        by += gb;
        launches += 2;                                     // GEMM + split-K reduce
    } else {
        // training step (cct_conv_fwd_cached + cct_conv_bwd): one lowering, one expand
        if (!t3_zero_copy && !t1_implicit) hbm(xin + dhat); // lower (fwd, cached)
        double gt = gemm_seconds(rows, ncols, cols, c);
        double gb = a_in + (type == 1 ? yout : rhat);
        t += std::max(gt, gb / c->hbm_bytes_per_s);
        by += gb;
        if (type != 1) hbm_at(rhat + yout, lift_bw);       // lift
        hbm_at(yout + rhat, type == 1 ? c->hbm_bytes_per_s * 0.45 : expand_bw);  // expand (shared)
        t += dgrad(&by, &launches);                        // bwd-data
        gt = wgrad_gemm();  // bwd-weight GEMM
        gb = a_in + rhat;
        t += std::max(gt, gb / c->hbm_bytes_per_s);
        by += gb;
        launches += 3;                                     // 2 GEMMs + split-K reduce
    }
    *secs = t + launches * c->launch_s;
    *bytes = by;
}

}  // namespace

namespace cct {
// Used by the launcher (cct_abi.cu): run a strided Type 1 layer in space-to-depth
// form when the model predicts that form faster for `pass` (0 fwd, 1 bwd-data,
// 2 bwd-weight, 3 training step).  Decided at a fixed batch (256) so that batch
// chunks and the lowered cache of a training step always agree.
bool prefer_s2d(const cct_conv_desc* desc, int pass) {
    G g = geo(desc);
    if (!s2d_possible(g)) return false;
    if (cct_get_implicit_lowering() == 2) return true;  // forced (tests)
    g.b = 256;
    cct_calibration cal;
    cct_calibration_default(&cal);
    return t1_form_seconds(g, pass, true, &cal) < t1_form_seconds(g, pass, false, &cal);
}

// Used by the launcher (cct_abi.cu): run Type 1 backward-data implicitly when
// that form is possible and the model predicts it faster.
bool prefer_implicit_dgrad(const cct_conv_desc* desc) {
    const G g = geo(desc);
    if (!implicit_dgrad_possible(g)) return false;
    if (cct_get_implicit_lowering() == 2) return true;  // forced (tests)
    cct_calibration cal;
    cct_calibration_default(&cal);
    const double f = 4.0;
    const double rows = g.b * g.m * g.m, cols = g.k * g.k * g.d, ncols = g.o;
    const double dhat = rows * rup(cols, 4) * f, rhat = rows * ncols * f, xin = g.b * g.n * g.n * g.d * f;
    double b0 = 0, l0 = 0, b1 = 0, l1 = 0;
    const double te = dgrad_seconds(g, false, rows, cols, ncols, dhat, rhat, xin, false, &cal, &b0, &l0) +
                      l0 * cal.launch_s;
    const double ti = dgrad_seconds(g, true, rows, cols, ncols, dhat, rhat, xin, false, &cal, &b1, &l1) +
                      l1 * cal.launch_s;
    return ti < te;
}
}  // namespace cct

extern "C" {

// Defaults measured on the B200 pool (profiles/):
// sustained lowering-kernel copy rate and sustained 3xTF32 algorithmic GEMM rate.
void cct_calibration_default(cct_calibration* cal) {
    if (!cal) return;
    cal->hbm_bytes_per_s = 4.15e12;  // measured lower / col2im rate (sweep, profiles/r01)
    cal->gemm_flops_per_s = 300.1e12; // measured 3xTF32 rate at BN 256, K 4096 (rate table, round 2)
    cal->launch_s = 5e-6;
    cal->alpha = 4.0 / cal->hbm_bytes_per_s * 2.0;  // one element read + written
    cal->beta = 1.0 / cal->gemm_flops_per_s;
}

cct_status cct_estimate(const cct_conv_desc* desc, cct_lowering lowering, const cct_calibration* cal,
                        int pass, cct_cost_estimate* est) {
    if (!desc || !est || lowering < CCT_LOWER_T1 || lowering > CCT_LOWER_T3) return CCT_ERR_CONFIG;
    if (desc->k < 1 || desc->d < 1 || desc->o < 1 || desc->b < 1 || desc->stride < 1 || desc->pad < 0 ||
        desc->k > desc->n + 2 * desc->pad)
        return CCT_ERR_CONFIG;
    cct_calibration def;
    if (!cal) { cct_calibration_default(&def); cal = &def; }
    const G g = geo(desc);
    const int type = int(lowering);
    const uint64_t b = uint64_t(desc->b), d = uint64_t(desc->d), k = uint64_t(desc->k), o = uint64_t(desc->o);
    const uint64_t m = uint64_t(g.m), n = uint64_t(desc->n), R = uint64_t(g.R);
    // SPEC.md:243 exact counts (stride 1, pad 0); Appendix A analogues otherwise.
    const bool spec = desc->stride == 1 && desc->pad == 0;
    uint64_t rows, cols, ncols, lower_el, lift_adds;
    if (type == 1) { rows = b * m * m; cols = k * k * d; ncols = o; lift_adds = 0; }
    else if (type == 2) { rows = spec ? b * n * n : b * R * m; cols = k * d; ncols = k * o; lift_adds = b * m * m * (k - 1) * o; }
    else { rows = spec ? b * n * n : b * R * R; cols = d; ncols = k * k * o; lift_adds = b * m * m * (k * k - 1) * o; }
    lower_el = rows * cols;
    est->lower_elements_written = lower_el;
    est->gemm_flops = 2ULL * rows * cols * ncols;
    est->lift_adds = lift_adds;
    est->lowered_bytes = lower_el * 4ULL;
    est->total_score = cal->alpha * double(lower_el + lift_adds) + cal->beta * double(est->gemm_flops);
    double secs = 0, bytes = 0;
    if (pass >= 0 && pass <= 2) {
        one_pass(g, type, pass, cal, &secs, &bytes);
    } else {  // training step: fwd (Dhat cached) + bwd-data + bwd-weight sharing one expand
        one_pass(g, type, 3, cal, &secs, &bytes);
    }
    est->model_seconds = secs;
    est->hbm_bytes = uint64_t(bytes);
    return CCT_OK;
}

cct_status cct_select_lowering(const cct_conv_desc* desc, const cct_calibration* cal, int pass,
                               cct_lowering* out, cct_cost_estimate* est) {
    if (!out) return CCT_ERR_CONFIG;
    cct_cost_estimate e[3];
    for (int t = 0; t < 3; ++t) {
        cct_status s = cct_estimate(desc, cct_lowering(t + 1), cal, pass, &e[t]);
        if (s != CCT_OK) return s;
    }
    int best = 0;
    for (int t = 1; t < 3; ++t)
        if (e[t].model_seconds < e[best].model_seconds) best = t;  // strict: ties keep the lower type
    *out = cct_lowering(best + 1);
    if (est)
        for (int t = 0; t < 3; ++t) est[t] = e[t];
    return CCT_OK;
}

}  // extern "C"
