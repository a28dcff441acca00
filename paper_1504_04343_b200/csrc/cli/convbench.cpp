// convbench -- the command-line harness of the SPEC's bench-cli module
// (the reference's src/convbench.cpp is listed in
// CMakeLists.txt:26 but absent) on the B200 path.  Every command drives the
// reference's C++ operator API (include/convlow/*.hpp) as implemented by
// libconvlow.so over the CUDA C ABI: there is no CPU compute path.
//
//   convbench verify           --layers FILE [--tolerance T] [--strategy S] [--batch B]
//   convbench sweep-ratio      --template "n k d o b [stride pad]" [--ratio-range LO:HI:STEPS]
//   convbench sweep-batch      --layers FILE --layer NAME --batch LIST [--strategy S]
//   convbench sweep-partitions --layers FILE --layer NAME --partitions LIST [--threads N]
//   convbench schedule         --devices FILE (--layers FILE --layer NAME | --template T)
//                              [--granularity G] [--audit N]
//   convbench estimate         --layers FILE          (cost model only, no GPU)
// Common flags: --out PATH  --format csv|json  --seed N  --reps N  --threads N
//
// Layer file: one record per line, `name n k d o b [stride pad]`,
// `#` starts a comment; stride / pad are this build's extension (defaults 1 / 0).
// Device profile file: `name flops overhead_seconds`.
// Records: one fixed schema for every command; CSV (header row, RFC 4180
// quoting) and JSON (array of objects with the same keys) carry identical data.
// Exit codes: 0 success, 1 verification / audit failure,
// 2 configuration error (file errors name the line), 3 resource or device error.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "cct.h"
#include "convlow/batching.hpp"
#include "convlow/cost_model.hpp"
#include "convlow/lowering.hpp"
#include "convlow/scheduler.hpp"
#include "convlow/tensor.hpp"

using namespace convlow;

namespace {

constexpr int kExitOk = 0, kExitVerify = 1, kExitConfig = 2, kExitResource = 3;
constexpr std::uint64_t kDefaultSeed = 1234;  // the reference ctest seed (CMakeLists.txt:65)

// ------------------------------------------------------------------ records
const std::vector<std::string> kFields = {
    "command", "layer", "n", "k", "d", "o", "b", "stride", "pad", "strategy", "p", "threads", "reps",
    "lower_s", "multiply_s", "lift_s", "total_s", "iqr_s", "images_per_s", "footprint_bytes", "model_seconds",
    "model_score", "model_winner", "measured_winner", "max_rel_err", "rel_l2", "adjoint_err", "passed", "kind",
    "device", "fraction", "makespan_s", "gap", "seed", "machine"};
const std::vector<std::string> kStringFields = {"command", "layer", "model_winner", "measured_winner", "passed",
                                                "kind", "device", "machine"};

struct Record {
    std::map<std::string, std::string> v;
    Record& set(const std::string& k, const std::string& s) {
        if (std::find(kFields.begin(), kFields.end(), k) == kFields.end()) throw std::logic_error("field " + k);
        v[k] = s;
        return *this;
    }
    template <class T>
    Record& num(const std::string& k, T x) {
        if constexpr (std::is_integral_v<T>) {
            return set(k, std::to_string(x));
        } else {
            std::ostringstream os;
            os.precision(10);
            os << double(x);
            return set(k, std::isfinite(double(x)) ? os.str() : std::string());
        }
    }
};

bool is_string_field(const std::string& k) {
    return std::find(kStringFields.begin(), kStringFields.end(), k) != kStringFields.end();
}

std::string csv_quote(const std::string& s) {
    if (s.find_first_of(",\"\n\r") == std::string::npos) return s;
    std::string r = "\"";
    for (char c : s) r += (c == '"') ? std::string("\"\"") : std::string(1, c);
    return r + "\"";
}

std::string json_quote(const std::string& s) {
    std::string r = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') r += '\\';
        if (c == '\n') { r += "\\n"; continue; }
        r += c;
    }
    return r + "\"";
}

void emit(const std::vector<Record>& recs, const std::string& format, std::ostream& os) {
    if (format == "csv") {
        for (size_t i = 0; i < kFields.size(); ++i) os << (i ? "," : "") << kFields[i];
        os << "\n";
        for (const Record& r : recs) {
            for (size_t i = 0; i < kFields.size(); ++i) {
                auto it = r.v.find(kFields[i]);
                os << (i ? "," : "") << (it == r.v.end() ? "" : csv_quote(it->second));
            }
            os << "\n";
        }
        return;
    }
    os << "[";
    for (size_t j = 0; j < recs.size(); ++j) {
        os << (j ? ",\n " : "\n ") << "{";
        for (size_t i = 0; i < kFields.size(); ++i) {
            auto it = recs[j].v.find(kFields[i]);
            os << (i ? ", " : "") << json_quote(kFields[i]) << ": ";
            if (it == recs[j].v.end()) os << "null";
            else if (is_string_field(kFields[i])) os << json_quote(it->second);
            else os << it->second;
        }
        os << "}";
    }
    os << "\n]\n";
}

// ------------------------------------------------------------------ flags
struct Args {
    std::string cmd;
    std::map<std::string, std::string> flags;
    std::string get(const std::string& k, const std::string& def = "") const {
        auto it = flags.find(k);
        return it == flags.end() ? def : it->second;
    }
    bool has(const std::string& k) const { return flags.count(k) != 0; }
};

const std::vector<std::string> kKnownFlags = {"layers", "strategy", "threads", "partitions", "batch", "ratio-range",
                                              "devices", "granularity", "reps", "seed", "out", "format", "tolerance",
                                              "template", "layer", "audit", "warmup"};

Args parse_args(int argc, char** argv) {
    Args a;
    if (argc < 2) throw config_error("usage: convbench <verify|sweep-ratio|sweep-batch|sweep-partitions|schedule|"
                                     "estimate> [flags]  (convbench --help)");
    a.cmd = argv[1];
    for (int i = 2; i < argc; ++i) {
        std::string f = argv[i];
        if (f.rfind("--", 0) != 0) throw config_error("unexpected argument '" + f + "'");
        f = f.substr(2);
        std::string val;
        const auto eq = f.find('=');
        if (eq != std::string::npos) {
            val = f.substr(eq + 1);
            f = f.substr(0, eq);
        } else {
            if (i + 1 >= argc) throw config_error("flag --" + f + " needs a value");
            val = argv[++i];
        }
        if (std::find(kKnownFlags.begin(), kKnownFlags.end(), f) == kKnownFlags.end())
            throw config_error("unknown flag --" + f);
        a.flags[f] = val;
    }
    return a;
}

std::size_t to_size(const std::string& s, const std::string& what) {
    char* end = nullptr;
    const long long v = std::strtoll(s.c_str(), &end, 10);
    if (s.empty() || *end != '\0' || v < 0) throw config_error(what + ": expected a non-negative integer, got '" + s + "'");
    return std::size_t(v);
}

double to_double(const std::string& s, const std::string& what) {
    char* end = nullptr;
    const double v = std::strtod(s.c_str(), &end);
    if (s.empty() || *end != '\0' || !std::isfinite(v)) throw config_error(what + ": expected a number, got '" + s + "'");
    return v;
}

std::vector<std::string> split(const std::string& s, char sep) {
    std::vector<std::string> out;
    std::string cur;
    std::istringstream is(s);
    while (std::getline(is, cur, sep))
        if (!cur.empty()) out.push_back(cur);
    return out;
}

// ------------------------------------------------------------------ files
struct NamedLayer {
    std::string name;
    LayerConfig cfg;
};

LayerConfig parse_layer_fields(const std::vector<std::string>& f, size_t first, const std::string& where) {
    if (f.size() != first + 5 && f.size() != first + 7)
        throw config_error(where + ": expected 'n k d o b [stride pad]'");
    LayerConfig c;
    c.n = to_size(f[first], where + " n");
    c.k = to_size(f[first + 1], where + " k");
    c.d = to_size(f[first + 2], where + " d");
    c.o = to_size(f[first + 3], where + " o");
    c.b = to_size(f[first + 4], where + " b");
    if (f.size() == first + 7) {
        c.stride = to_size(f[first + 5], where + " stride");
        c.pad = to_size(f[first + 6], where + " pad");
    }
    try {
        c.validate();
    } catch (const config_error& e) {
        throw config_error(where + ": " + e.what());
    }
    return c;
}

std::vector<std::string> tokens(const std::string& line) {
    std::vector<std::string> f;
    std::istringstream is(line.substr(0, line.find('#')));
    std::string t;
    while (is >> t) f.push_back(t);
    return f;
}

std::vector<NamedLayer> read_layer_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw config_error("cannot read layer file '" + path + "'");
    std::vector<NamedLayer> out;
    std::string line;
    for (int ln = 1; std::getline(in, line); ++ln) {
        const auto f = tokens(line);
        if (f.empty()) continue;
        const std::string where = path + ":" + std::to_string(ln);
        NamedLayer nl;
        nl.name = f[0];
        nl.cfg = parse_layer_fields(f, 1, where);
        for (const auto& o : out)
            if (o.name == nl.name) throw config_error(where + ": duplicate layer name '" + nl.name + "'");
        out.push_back(nl);
    }
    if (out.empty()) throw config_error("layer file '" + path + "' has no records");
    return out;
}

std::vector<DeviceProfile> read_device_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw config_error("cannot read device profile file '" + path + "'");
    std::vector<DeviceProfile> out;
    std::string line;
    for (int ln = 1; std::getline(in, line); ++ln) {
        const auto f = tokens(line);
        if (f.empty()) continue;
        const std::string where = path + ":" + std::to_string(ln);
        if (f.size() != 3) throw config_error(where + ": expected 'name flops overhead'");
        DeviceProfile d;
        d.name = f[0];
        d.flops = to_double(f[1], where + " flops");
        d.fixed_overhead = to_double(f[2], where + " overhead");
        if (!(d.flops > 0) || d.fixed_overhead < 0)
            throw config_error(where + ": need flops > 0 and overhead >= 0");
        out.push_back(d);
    }
    if (out.empty()) throw config_error("device profile file '" + path + "' has no devices");
    return out;
}

NamedLayer layer_from_args(const Args& a) {
    if (a.has("template")) {
        NamedLayer nl;
        nl.name = "template";
        nl.cfg = parse_layer_fields(tokens(a.get("template")), 0, "--template");
        return nl;
    }
    if (!a.has("layers")) throw config_error("--layers FILE (with --layer NAME) or --template is required");
    const auto layers = read_layer_file(a.get("layers"));
    const std::string want = a.get("layer", layers.front().name);
    for (const auto& l : layers)
        if (l.name == want) return l;
    throw config_error("layer '" + want + "' not in " + a.get("layers"));
}

std::vector<LoweringStrategy> strategies_of(const Args& a, const LayerConfig& L) {
    const std::string s = a.get("strategy", "all");
    if (s == "all") return {LoweringStrategy::Type1, LoweringStrategy::Type2, LoweringStrategy::Type3};
    if (s == "auto") return {select_strategy(L).strategy};
    if (s == "1" || s == "2" || s == "3") return {LoweringStrategy(std::stoi(s))};
    throw config_error("--strategy must be 1, 2, 3, auto or all, got '" + s + "'");
}

std::size_t threads_of(const Args& a) {
    const std::size_t t = to_size(a.get("threads", std::to_string(std::max(1u, std::thread::hardware_concurrency()))),
                                  "--threads");
    if (t < 1 || t > 256) throw config_error("--threads must be in [1, 256]");  // GemmConfig range (gemm.hpp:46)
    return t;
}

std::string machine() {
    char name[256];
    int sms = 0;
    const int n = cct_device_info(name, sizeof(name), &sms);
    std::ostringstream os;
    if (n > 0) os << name << " (" << sms << " SMs) x" << n;
    else os << "no CUDA device";
    os << "; host " << std::thread::hardware_concurrency() << " threads";
    return os.str();
}

Record base(const std::string& cmd, const NamedLayer& l, std::uint64_t seed) {
    Record r;
    r.set("command", cmd).set("layer", l.name);
    r.num("n", l.cfg.n).num("k", l.cfg.k).num("d", l.cfg.d).num("o", l.cfg.o).num("b", l.cfg.b);
    r.num("stride", l.cfg.stride).num("pad", l.cfg.pad).num("seed", seed);
    r.set("machine", machine());
    return r;
}

// ------------------------------------------------------------------ timing
struct Stats {
    PhaseTimings med;
    double total = 0, iqr = 0;
};

template <class F>
Stats time_phases(F&& run, int warmup, int reps) {
    for (int i = 0; i < warmup; ++i) run();
    std::vector<PhaseTimings> ts;
    std::vector<double> tot;
    for (int i = 0; i < reps; ++i) {
        ts.push_back(run());
        tot.push_back(ts.back().lower_s + ts.back().multiply_s + ts.back().lift_s);
    }
    std::vector<size_t> idx(tot.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
    std::sort(idx.begin(), idx.end(), [&](size_t x, size_t y) { return tot[x] < tot[y]; });
    Stats s;
    s.med = ts[idx[idx.size() / 2]];
    s.total = tot[idx[idx.size() / 2]];
    s.iqr = tot[idx[(3 * idx.size()) / 4]] - tot[idx[idx.size() / 4]];
    return s;
}

void put_stats(Record& r, const Stats& s, double images) {
    r.num("lower_s", s.med.lower_s).num("multiply_s", s.med.multiply_s).num("lift_s", s.med.lift_s);
    r.num("total_s", s.total).num("iqr_s", s.iqr);
    if (s.total > 0) r.num("images_per_s", images / s.total);
}

DataBatch random_batch(const LayerConfig& L, std::mt19937_64& rng) { return DataBatch::random(L.b, L.n, L.d, rng); }

// ------------------------------------------------------------------ commands
int cmd_verify(const Args& a, std::vector<Record>& out) {
    if (!a.has("layers")) throw config_error("verify needs --layers FILE");
    auto layers = read_layer_file(a.get("layers"));
    const double tol = to_double(a.get("tolerance", "1e-3"), "--tolerance");
    const std::uint64_t seed = to_size(a.get("seed", std::to_string(kDefaultSeed)), "--seed");
    const std::size_t threads = threads_of(a);
    bool all_ok = true;
    for (auto& l : layers) {
        if (a.has("batch")) l.cfg.b = to_size(a.get("batch"), "--batch");
        l.cfg.validate();
        const ConvGeometry geom{l.cfg.stride, l.cfg.pad};
        std::mt19937_64 rng(seed);
        const DataBatch x = random_batch(l.cfg, rng);
        const KernelBank w = KernelBank::random(l.cfg.k, l.cfg.d, l.cfg.o, rng);
        OutputBatch dy(l.cfg.b, l.cfg.o, l.cfg.m());
        std::uniform_real_distribution<real> u(real(-1), real(1));
        for (auto& v : dy.values()) v = u(rng);
        const OutputBatch ref = direct_convolve_batch(x, w, geom);  // exact fp64 oracle on the device
        double ref_max = 0, ref_ss = 0;
        for (real v : ref.values()) {
            ref_max = std::max(ref_max, double(std::fabs(v)));
            ref_ss += double(v) * v;
        }
        for (LoweringStrategy s : strategies_of(a, l.cfg)) {
            auto [y, t] = convolve_lowered(x, w, s, threads, geom);
            double err_max = 0, err_ss = 0, yd = 0, yd_abs = 0;
            for (size_t i = 0; i < y.size(); ++i) {
                const double e = double(y.values()[i]) - double(ref.values()[i]);
                err_max = std::max(err_max, std::fabs(e));
                err_ss += e * e;
                yd += double(y.values()[i]) * dy.values()[i];
                yd_abs += std::fabs(double(y.values()[i]) * dy.values()[i]);
            }
            // backward passes: the adjoint identity <conv(x,w),dy> = <x,dgrad(dy,w)> = <w,wgrad(x,dy)>
            const DataBatch dx = convolve_backward_data(dy, w, l.cfg.n, s, geom);
            const KernelBank dw = convolve_backward_weight(x, dy, l.cfg.k, s, geom);
            double xdx = 0, wdw = 0;
            for (size_t q = 0; q < x.b(); ++q)
                for (size_t i = 0; i < x[q].size(); ++i) xdx += double(x[q].values()[i]) * dx[q].values()[i];
            for (size_t i = 0; i < w.values().size(); ++i) wdw += double(w.values()[i]) * dw.values()[i];
            // relative to sum |y_i dy_i|: <y, dy> of random dy cancels, its own magnitude is no scale
            const double scale = std::max(yd_abs, 1e-30);
            const double adj = std::max(std::fabs(yd - xdx), std::fabs(yd - wdw)) / scale;
            const double max_rel = ref_max > 0 ? err_max / ref_max : err_max;
            const double l2 = ref_ss > 0 ? std::sqrt(err_ss / ref_ss) : std::sqrt(err_ss);
            const bool ok = max_rel <= tol && l2 <= tol && adj <= tol;
            all_ok = all_ok && ok;
            Record r = base("verify", l, seed);
            r.num("strategy", int(s)).num("threads", threads).num("reps", 1);
            r.num("lower_s", t.lower_s).num("multiply_s", t.multiply_s).num("lift_s", t.lift_s);
            r.num("total_s", t.lower_s + t.multiply_s + t.lift_s);
            r.num("max_rel_err", max_rel).num("rel_l2", l2).num("adjoint_err", adj);
            r.set("passed", ok ? "true" : "false");
            out.push_back(r);
        }
    }
    return all_ok ? kExitOk : kExitVerify;
}

int cmd_estimate(const Args& a, std::vector<Record>& out) {
    if (!a.has("layers")) throw config_error("estimate needs --layers FILE");
    for (const auto& l : read_layer_file(a.get("layers"))) {
        const StrategyChoice ch = select_strategy(l.cfg);
        for (int t = 0; t < 3; ++t) {
            const CostEstimate& e = ch.estimates[size_t(t)];
            Record r = base("estimate", l, kDefaultSeed);
            r.num("strategy", t + 1).num("model_seconds", e.model_seconds).num("model_score", e.total_score);
            r.num("footprint_bytes", e.lowered_bytes);
            r.set("model_winner", std::to_string(int(ch.strategy))).set("kind", "fwd+bwd");
            out.push_back(r);
        }
    }
    return kExitOk;
}

int cmd_sweep_ratio(const Args& a, std::vector<Record>& out) {
    NamedLayer t = layer_from_args(a);
    const auto rr = split(a.get("ratio-range", "0.0625:16:9"), ':');
    if (rr.size() != 3) throw config_error("--ratio-range must be LO:HI:STEPS");
    const double lo = to_double(rr[0], "ratio lo"), hi = to_double(rr[1], "ratio hi");
    const std::size_t steps = to_size(rr[2], "ratio steps");
    if (!(lo > 0) || !(hi >= lo) || steps < 1) throw config_error("--ratio-range needs 0 < LO <= HI, STEPS >= 1");
    const int reps = int(to_size(a.get("reps", "5"), "--reps")), warm = int(to_size(a.get("warmup", "1"), "--warmup"));
    if (reps < 1) throw config_error("--reps must be >= 1");
    const std::uint64_t seed = to_size(a.get("seed", std::to_string(kDefaultSeed)), "--seed");
    const std::size_t threads = threads_of(a);
    const double prod = double(t.cfg.d) * double(t.cfg.o);
    for (std::size_t i = 0; i < steps; ++i) {
        const double ratio = steps == 1 ? lo : lo * std::pow(hi / lo, double(i) / double(steps - 1));
        NamedLayer l = t;
        l.cfg.d = std::max<std::size_t>(1, std::size_t(std::llround(std::sqrt(prod * ratio))));
        l.cfg.o = std::max<std::size_t>(1, std::size_t(std::llround(std::sqrt(prod / ratio))));
        l.name = t.name + "@d/o=" + std::to_string(ratio);
        std::mt19937_64 rng(seed);
        const DataBatch x = random_batch(l.cfg, rng);
        const KernelBank w = KernelBank::random(l.cfg.k, l.cfg.d, l.cfg.o, rng);
        const ConvGeometry geom{l.cfg.stride, l.cfg.pad};
        std::vector<Record> recs;
        double best_meas = INFINITY, best_model = INFINITY;
        int win_meas = 0, win_model = 0;
        for (LoweringStrategy s : strategies_of(a, l.cfg)) {
            const CostEstimate e = estimate(s, l.cfg, CostWeights{0, 0, false});
            const Stats st = time_phases([&] { return convolve_lowered(x, w, s, threads, geom).second; }, warm, reps);
            Record r = base("sweep-ratio", l, seed);
            r.num("strategy", int(s)).num("threads", threads).num("reps", reps);
            put_stats(r, st, double(l.cfg.b));
            r.num("model_seconds", e.model_seconds).num("model_score", e.total_score).num("footprint_bytes", e.lowered_bytes);
            r.set("kind", "fwd");
            if (st.total < best_meas) { best_meas = st.total; win_meas = int(s); }
            if (e.model_seconds < best_model) { best_model = e.model_seconds; win_model = int(s); }
            recs.push_back(r);
        }
        for (Record& r : recs) {
            r.set("model_winner", std::to_string(win_model)).set("measured_winner", std::to_string(win_meas));
            out.push_back(r);
        }
    }
    return kExitOk;
}

int cmd_sweep_batch(const Args& a, std::vector<Record>& out) {
    const NamedLayer t = layer_from_args(a);
    if (!a.has("batch")) throw config_error("sweep-batch needs --batch LIST");
    const int reps = int(to_size(a.get("reps", "5"), "--reps")), warm = int(to_size(a.get("warmup", "1"), "--warmup"));
    if (reps < 1) throw config_error("--reps must be >= 1");
    const std::uint64_t seed = to_size(a.get("seed", std::to_string(kDefaultSeed)), "--seed");
    const std::size_t threads = threads_of(a);
    for (const auto& bs : split(a.get("batch"), ',')) {
        NamedLayer l = t;
        l.cfg.b = to_size(bs, "--batch entry");
        l.cfg.validate();
        std::mt19937_64 rng(seed);
        const DataBatch x = random_batch(l.cfg, rng);
        const KernelBank w = KernelBank::random(l.cfg.k, l.cfg.d, l.cfg.o, rng);
        const ConvGeometry geom{l.cfg.stride, l.cfg.pad};
        for (LoweringStrategy s : strategies_of(a, l.cfg)) {
            const Stats st = time_phases([&] { return convolve_lowered(x, w, s, threads, geom).second; }, warm, reps);
            Record r = base("sweep-batch", l, seed);
            r.num("strategy", int(s)).num("threads", threads).num("reps", reps).num("p", 1);
            put_stats(r, st, double(l.cfg.b));
            r.num("footprint_bytes", footprint(s, l.cfg, l.cfg.b).lowered_bytes_per_partition).set("kind", "fwd");
            out.push_back(r);
        }
    }
    return kExitOk;
}

int cmd_sweep_partitions(const Args& a, std::vector<Record>& out) {
    const NamedLayer l = layer_from_args(a);
    const int reps = int(to_size(a.get("reps", "5"), "--reps")), warm = int(to_size(a.get("warmup", "1"), "--warmup"));
    if (reps < 1) throw config_error("--reps must be >= 1");
    const std::uint64_t seed = to_size(a.get("seed", std::to_string(kDefaultSeed)), "--seed");
    const std::size_t threads = threads_of(a);
    std::mt19937_64 rng(seed);
    const DataBatch x = random_batch(l.cfg, rng);
    const KernelBank w = KernelBank::random(l.cfg.k, l.cfg.d, l.cfg.o, rng);
    const ConvGeometry geom{l.cfg.stride, l.cfg.pad};
    for (const auto& ps : split(a.get("partitions", "none,1,2,4"), ',')) {
        // "none": the Caffe-style baseline -- every image lowered and multiplied on its own
        const bool none = ps == "none";
        const std::size_t p = none ? l.cfg.b : to_size(ps, "--partitions entry");
        PartitionPlan plan;
        try {
            plan = plan_partitions(l.cfg.b, none ? l.cfg.b : threads, p);
        } catch (const config_error& e) {
            std::cerr << "convbench: skipping p=" << ps << ": " << e.what() << "\n";
            continue;
        }
        for (LoweringStrategy s : strategies_of(a, l.cfg)) {
            FootprintReport fp;
            const Stats st = time_phases(
                [&] {
                    auto res = execute_partitioned(x, w, s, plan, geom);
                    fp = res.footprint;
                    return res.timing;
                },
                warm, reps);
            Record r = base("sweep-partitions", l, seed);
            r.num("strategy", int(s)).num("threads", threads).num("reps", reps).num("p", p);
            put_stats(r, st, double(l.cfg.b));
            r.num("footprint_bytes", fp.peak_bytes).set("kind", none ? "none" : "partitioned");
            out.push_back(r);
        }
    }
    return kExitOk;
}

int cmd_schedule(const Args& a, std::vector<Record>& out) {
    if (!a.has("devices")) throw config_error("schedule needs --devices FILE");
    const auto devs = read_device_file(a.get("devices"));
    const NamedLayer l = layer_from_args(a);
    const std::size_t g = to_size(a.get("granularity", "100"), "--granularity");
    const std::uint64_t seed = to_size(a.get("seed", std::to_string(kDefaultSeed)), "--seed");
    const LoweringStrategy s = strategies_of(a, l.cfg).front();
    const SplitPlan prop = proportional_split(devs, l.cfg.b);
    const double tp = simulate_makespan(l.cfg, prop, devs, s);
    for (size_t i = 0; i < devs.size(); ++i) {
        Record r = base("schedule", l, seed);
        r.set("kind", "proportional").set("device", devs[i].name).num("strategy", int(s));
        r.num("fraction", prop.fractions[i]).num("p", prop.counts[i]).num("makespan_s", tp);
        out.push_back(r);
    }
    if (devs.size() == 2) {
        const SplitPlan opt = optimal_split_sweep(l.cfg, devs, g, s);
        const double gap = heuristic_gap(l.cfg, devs, g, s);
        Record r = base("schedule", l, seed);
        r.set("kind", "sweep-optimum").set("device", devs[1].name).num("strategy", int(s));
        r.num("fraction", opt.fractions[1]).num("p", opt.counts[1]);
        r.num("makespan_s", simulate_makespan(l.cfg, opt, devs, s)).num("gap", gap);
        out.push_back(r);
        for (std::size_t i = 0; i <= g; ++i) {  // the Fig. 9 curve: makespan vs fraction on devices[1]
            SplitPlan c;
            const double p = double(i) / double(g);
            c.fractions = {1.0 - p, p};
            Record cr = base("schedule", l, seed);
            cr.set("kind", "curve").set("device", devs[1].name).num("strategy", int(s)).num("fraction", p);
            cr.num("makespan_s", simulate_makespan(l.cfg, c, devs, s));
            out.push_back(cr);
        }
    } else {
        Record r = base("schedule", l, seed);
        r.set("kind", "gap").num("gap", 1.0).num("makespan_s", tp);  // single device / n-way: degenerate
        out.push_back(r);
    }
    if (a.has("audit")) {
        // Appendix B audit (SPEC acceptance 7): random 2-device profiles with overheads
        // <= 5% of the work time; the proportional plan must stay within 5% of the optimum
        // (bound: makespan(prop) <= W / sum(F) + max overhead, and every plan >= W / sum(F))
        const std::size_t n = to_size(a.get("audit"), "--audit");
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> lf(9.0, 13.0), fr(0.0, 0.05);
        LayerConfig one = l.cfg;
        const double work = double(estimate(s, one, CostWeights{0, 0, false}).gemm_flops);
        double worst = 1.0;
        for (std::size_t i = 0; i < n; ++i) {
            std::vector<DeviceProfile> p(2);
            for (int j = 0; j < 2; ++j) {
                p[size_t(j)].name = j ? "dev1" : "dev0";
                p[size_t(j)].flops = std::pow(10.0, lf(rng));
            }
            // overheads up to 5% of the ideal (overhead-free, proportional) work time W / sum(F)
            const double ideal = work / (p[0].flops + p[1].flops);
            for (int j = 0; j < 2; ++j) p[size_t(j)].fixed_overhead = fr(rng) * ideal;
            worst = std::max(worst, heuristic_gap(l.cfg, p, std::max<std::size_t>(g, 10), s));
        }
        Record r = base("schedule", l, seed);
        r.set("kind", "audit").num("reps", int(n)).num("gap", worst).set("passed", worst <= 1.05 ? "true" : "false");
        out.push_back(r);
        if (worst > 1.05) return kExitVerify;
    }
    return kExitOk;
}

const char* kHelp =
    "convbench -- CcT convolution-lowering harness on B200 (SPEC bench-cli)\n"
    "  verify           --layers FILE [--tolerance 1e-3] [--strategy 1|2|3|auto|all] [--batch B]\n"
    "  sweep-ratio      --template \"n k d o b [stride pad]\" [--ratio-range 0.0625:16:9] [--reps 5]\n"
    "  sweep-batch      --layers FILE --layer NAME --batch 1,16,64,256 [--strategy S]\n"
    "  sweep-partitions --layers FILE --layer NAME [--partitions none,1,2,4] [--threads N]\n"
    "  schedule         --devices FILE (--layers FILE --layer NAME | --template T) [--granularity 100] [--audit N]\n"
    "  estimate         --layers FILE\n"
    "common: --out PATH --format csv|json --seed N --reps N --warmup N --threads N\n"
    "exit: 0 ok, 1 verification/audit failure, 2 configuration error, 3 resource/device error\n";

}  // namespace

int main(int argc, char** argv) {
    if (argc >= 2 && (std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h")) {
        std::cout << kHelp;
        return kExitOk;
    }
    try {
        const Args a = parse_args(argc, argv);
        const std::string format = a.get("format", "csv");
        if (format != "csv" && format != "json") throw config_error("--format must be csv or json");
        std::vector<Record> recs;
        int rc;
        if (a.cmd == "verify") rc = cmd_verify(a, recs);
        else if (a.cmd == "estimate") rc = cmd_estimate(a, recs);
        else if (a.cmd == "sweep-ratio") rc = cmd_sweep_ratio(a, recs);
        else if (a.cmd == "sweep-batch") rc = cmd_sweep_batch(a, recs);
        else if (a.cmd == "sweep-partitions") rc = cmd_sweep_partitions(a, recs);
        else if (a.cmd == "schedule") rc = cmd_schedule(a, recs);
        else throw config_error("unknown command '" + a.cmd + "' (convbench --help)");
        if (a.has("out")) {
            std::ofstream f(a.get("out"));
            if (!f) throw config_error("cannot write '" + a.get("out") + "'");
            emit(recs, format, f);
        } else {
            emit(recs, format, std::cout);
        }
        return rc;
    } catch (const config_error& e) {
        std::cerr << "convbench: configuration error: " << e.what() << "\n";
        return kExitConfig;
    } catch (const resource_error& e) {
        std::cerr << "convbench: resource error: " << e.what() << "\n";
        return kExitResource;
    } catch (const std::exception& e) {
        std::cerr << "convbench: error: " << e.what() << "\n";
        return kExitResource;
    }
}
