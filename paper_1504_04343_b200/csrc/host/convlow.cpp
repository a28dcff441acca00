// convlow.cpp -- the reference's C++ operator API (namespace convlow) on the
// B200, implemented over the C ABI of libcct.so (include/cct.h).
//
// Value semantics are kept (inputs const&, results returned by value, as in
// tensor.hpp / gemm.hpp): each call packs the host containers into device
// buffers owned by a per-thread DeviceContext, runs the device path on that
// context's stream, copies the results back and synchronises.  Error behaviour
// mirrors the reference: the same validation messages for shapes and GemmConfig
// (tensor.cpp:23-30, 66-86; gemm.cpp:19-34), C-ABI failures rethrown as
// config_error / resource_error (common.hpp:17-24).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <sstream>
#include <string>

#include <cuda_runtime.h>

#include "cct.h"
#include "convlow/batching.hpp"
#include "convlow/cost_model.hpp"
#include "convlow/gemm.hpp"
#include "convlow/lowering.hpp"
#include "convlow/scheduler.hpp"
#include "convlow/tensor.hpp"

namespace convlow {

namespace {

[[noreturn]] void raise(cct_status s, const std::string& where) {
    const std::string msg = where + ": " + cct_last_error();
    if (s == CCT_ERR_CONFIG || s == CCT_ERR_UNSUPPORTED) throw config_error(msg);
    throw resource_error(msg);
}

void check(cct_status s, const char* where) {
    if (s != CCT_OK) raise(s, where);
}

void cuda_check(cudaError_t e, const char* where) {
    if (e != cudaSuccess) throw resource_error(std::string(where) + ": " + cudaGetErrorString(e));
}

// Per-thread device state: one stream and grow-only device buffers.
struct DeviceContext {
    cudaStream_t stream = nullptr;
    void* buf[8] = {nullptr};
    size_t cap[8] = {0};

    DeviceContext() { cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate"); }
    ~DeviceContext() {
        for (void* p : buf)
            if (p) cudaFree(p);
        if (stream) cudaStreamDestroy(stream);
    }
    void* get(int slot, size_t bytes) {
        if (bytes == 0) bytes = 16;
        if (cap[slot] < bytes) {
            if (buf[slot]) cudaFree(buf[slot]);
            buf[slot] = nullptr;
            cap[slot] = 0;
            if (cudaMalloc(&buf[slot], bytes) != cudaSuccess)
                throw resource_error("device allocation of " + std::to_string(bytes) + " bytes failed");
            cap[slot] = bytes;
        }
        return buf[slot];
    }
    void sync() { cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize"); }
};

DeviceContext& ctx() {
    static thread_local DeviceContext c;
    return c;
}

enum Slot { kX = 0, kW = 1, kY = 2, kWs = 3, kA = 4, kB = 5, kC = 6, kAux = 7 };

std::string tensor_shape_str(const Tensor3& t) {
    std::ostringstream os;
    os << t.rows() << "x" << t.cols() << "x" << t.depth();
    return os.str();
}

std::string bank_shape_str(const KernelBank& bk) {
    std::ostringstream os;
    os << bk.k() << "x" << bk.k() << "x" << bk.depth() << " (o=" << bk.o() << ")";
    return os.str();
}

cct_conv_desc make_desc(const LayerConfig& L) {
    L.validate();
    cct_conv_desc d;
    check(cct_conv_desc_init(&d, int64_t(L.n), int64_t(L.k), int64_t(L.d), int64_t(L.o), int64_t(L.b),
                             int64_t(L.stride), int64_t(L.pad)),
          "layer config");
    return d;
}

float* upload_batch(const DataBatch& batch, int slot) {
    const size_t per = batch[0].size();
    auto* d = static_cast<float*>(ctx().get(slot, per * batch.b() * sizeof(float)));
    for (size_t q = 0; q < batch.b(); ++q)
        cuda_check(cudaMemcpyAsync(d + q * per, batch[q].values().data(), per * sizeof(float), cudaMemcpyHostToDevice,
                                   ctx().stream),
                   "H2D batch");
    return d;
}

float* upload(const std::vector<real>& v, int slot) {
    auto* d = static_cast<float*>(ctx().get(slot, v.size() * sizeof(float)));
    cuda_check(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(float), cudaMemcpyHostToDevice, ctx().stream), "H2D");
    return d;
}

void download(std::vector<real>& v, const float* d) {
    cuda_check(cudaMemcpyAsync(v.data(), d, v.size() * sizeof(float), cudaMemcpyDeviceToHost, ctx().stream), "D2H");
}

// row-major host matrix -> device with a 16-byte aligned row pitch (TMA)
float* upload_padded(const Mat& m, int slot, int64_t* ld) {
    *ld = int64_t((m.cols() + 3) / 4 * 4);
    auto* d = static_cast<float*>(ctx().get(slot, size_t(*ld) * std::max<size_t>(m.rows(), 1) * sizeof(float)));
    if (m.size())
        cuda_check(cudaMemcpy2DAsync(d, size_t(*ld) * 4, m.values().data(), m.cols() * 4, m.cols() * 4, m.rows(),
                                     cudaMemcpyHostToDevice, ctx().stream),
                   "H2D matrix");
    return d;
}

void check_multiply_dims(const Mat& a, const Mat& b, const GemmConfig& cfg) {
    if (a.cols() != b.rows()) {
        std::ostringstream os;
        os << "gemm dimension mismatch: A is " << a.rows() << "x" << a.cols() << ", B is " << b.rows() << "x"
           << b.cols();
        throw config_error(os.str());
    }
    if (cfg.threads < 1 || cfg.threads > GemmConfig::kMaxThreads)
        throw config_error("gemm thread count must be in [1, " + std::to_string(GemmConfig::kMaxThreads) + "], got " +
                           std::to_string(cfg.threads));
    if (cfg.block_rows < 1 || cfg.block_cols < 1 || cfg.block_inner < 1)
        throw config_error("gemm block sizes must be >= 1");
}

cct_lowering to_c(LoweringStrategy s) { return cct_lowering(int(s)); }

LayerConfig layer_with(const LayerConfig& L, ConvGeometry g) {
    LayerConfig r = L;
    r.stride = g.stride;
    r.pad = g.pad;
    return r;
}

// PhaseTimings from the device phase profile (cct_profile_*) of one call.
struct PhaseProbe {
    PhaseProbe() {
        cct_profile_read(nullptr, nullptr, nullptr, nullptr, 1);
        cct_profile_enable(1);
    }
    PhaseTimings finish() {
        cct_profile_enable(0);
        double ms[CCT_NUM_PHASES] = {0};
        cct_profile_read(ms, nullptr, nullptr, nullptr, 1);
        PhaseTimings t;
        t.lower_s = (ms[0] + ms[3] + ms[6]) * 1e-3;   // lower (+ expand, weight padding)
        t.multiply_s = (ms[1] + ms[5]) * 1e-3;        // GEMM (+ split-K reduce)
        t.lift_s = (ms[2] + ms[4]) * 1e-3;            // lift (+ col2im)
        return t;
    }
};

}  // namespace

// ---------------------------------------------------------------- tensor.hpp
void LayerConfig::validate() const {
    if (k < 1 || k > n + 2 * pad || d < 1 || o < 1 || b < 1 || stride < 1) {
        std::ostringstream os;
        os << "invalid layer config (n=" << n << ", k=" << k << ", d=" << d << ", o=" << o << ", b=" << b;
        if (stride != 1 || pad != 0) os << ", stride=" << stride << ", pad=" << pad;
        os << "): need 1 <= k <= n, d >= 1, o >= 1, b >= 1";
        if (stride != 1 || pad != 0) os << ", stride >= 1";
        throw config_error(os.str());
    }
}

Tensor3 Tensor3::random(std::size_t n, std::size_t depth, std::mt19937_64& rng) {
    Tensor3 t(n, depth);
    std::uniform_real_distribution<real> dist(real(-1), real(1));
    for (auto& x : t.v_) x = dist(rng);
    return t;
}

KernelBank KernelBank::random(std::size_t k, std::size_t depth, std::size_t o, std::mt19937_64& rng) {
    KernelBank bk(k, depth, o);
    std::uniform_real_distribution<real> dist(real(-1), real(1));
    for (auto& x : bk.v_) x = dist(rng);
    return bk;
}

DataBatch::DataBatch(std::vector<Tensor3> images) : images_(std::move(images)) {
    if (images_.empty()) throw config_error("batch must hold at least one image");
    for (const auto& img : images_)
        if (img.rows() != images_[0].rows() || img.depth() != images_[0].depth())
            throw config_error("batch images must share one shape: found " + tensor_shape_str(img) + " and " +
                               tensor_shape_str(images_[0]));
}

DataBatch DataBatch::random(std::size_t b, std::size_t n, std::size_t depth, std::mt19937_64& rng) {
    std::vector<Tensor3> images;
    images.reserve(b);
    for (std::size_t i = 0; i < b; ++i) images.push_back(Tensor3::random(n, depth, rng));
    return DataBatch(std::move(images));
}

LayerConfig layer_of(const DataBatch& batch, const KernelBank& bank) {
    const Tensor3& first = batch[0];
    if (bank.depth() != first.depth() || bank.k() > first.rows())
        throw config_error("kernel bank " + bank_shape_str(bank) + " incompatible with data tensor " +
                           tensor_shape_str(first));
    LayerConfig layer;
    layer.n = first.rows();
    layer.k = bank.k();
    layer.d = first.depth();
    layer.o = bank.o();
    layer.b = batch.b();
    layer.validate();
    return layer;
}

OutputPlane direct_convolve(const Tensor3& data, const KernelBank& bank, std::size_t kernel_index) {
    if (bank.depth() != data.depth() || bank.k() > data.rows())
        throw config_error("kernel bank " + bank_shape_str(bank) + " incompatible with data tensor " +
                           tensor_shape_str(data));
    if (kernel_index >= bank.o())
        throw config_error("kernel index " + std::to_string(kernel_index) + " out of range for bank " +
                           bank_shape_str(bank));
    LayerConfig L;
    L.n = data.rows();
    L.k = bank.k();
    L.d = data.depth();
    L.o = 1;
    L.b = 1;
    cct_conv_desc d = make_desc(L);
    const size_t ksz = bank.k() * bank.k() * bank.depth();
    std::vector<real> wj(bank.values().begin() + long(kernel_index * ksz),
                         bank.values().begin() + long((kernel_index + 1) * ksz));
    float* dx = upload(data.values(), kX);
    float* dw = upload(wj, kW);
    OutputPlane out(L.m());
    auto* dy = static_cast<float*>(ctx().get(kY, out.v.size() * sizeof(float)));
    check(cct_direct_conv_fwd_exact(&d, dx, dw, dy, ctx().stream), "direct_convolve");
    download(out.v, dy);
    ctx().sync();
    return out;
}

OutputBatch direct_convolve_batch(const DataBatch& batch, const KernelBank& bank) {
    const LayerConfig L = layer_of(batch, bank);
    cct_conv_desc d = make_desc(L);
    float* dx = upload_batch(batch, kX);
    float* dw = upload(bank.values(), kW);
    OutputBatch out(L.b, L.o, L.m());
    auto* dy = static_cast<float*>(ctx().get(kY, out.size() * sizeof(float)));
    check(cct_direct_conv_fwd_exact(&d, dx, dw, dy, ctx().stream), "direct_convolve_batch");
    download(out.values(), dy);
    ctx().sync();
    return out;
}

// ------------------------------------------------------------------ gemm.hpp
Mat Mat::identity(std::size_t n) {
    Mat m(n, n);
    for (std::size_t i = 0; i < n; ++i) m.at(i, i) = real(1);
    return m;
}

Mat Mat::random(std::size_t rows, std::size_t cols, std::mt19937_64& rng) {
    Mat m(rows, cols);
    std::uniform_real_distribution<real> dist(real(-1), real(1));
    for (auto& x : m.v_) x = dist(rng);
    return m;
}

std::uint64_t gemm_flop_count(std::size_t rows, std::size_t inner, std::size_t cols) {
    return 2ull * rows * inner * cols;
}

namespace {
// C = A B with A, B already on the device (ld multiples of 4); C row-major ldc = N.
void device_multiply(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B, int64_t ldb,
                     float* C) {
    size_t need = 0;
    check(cct_gemm_workspace_size(M, N, K, 0, &need), "gemm workspace");
    void* ws = need ? ctx().get(kWs, need) : nullptr;
    check(cct_gemm(M, N, K, A, lda, B, ldb, C, N, 0, ws, need, ctx().stream), "multiply");
}
}  // namespace

Mat multiply(const Mat& a, const Mat& b, const GemmConfig& cfg) {
    check_multiply_dims(a, b, cfg);  // GemmConfig is validated, then ignored (one device)
    Mat c(a.rows(), b.cols());
    if (c.size() == 0) return c;
    if (a.cols() == 0) return c;
    int64_t lda, ldb;
    float* A = upload_padded(a, kA, &lda);
    float* B = upload_padded(b, kB, &ldb);
    auto* C = static_cast<float*>(ctx().get(kC, c.size() * sizeof(float)));
    device_multiply(int64_t(a.rows()), int64_t(b.cols()), int64_t(a.cols()), A, lda, B, ldb, C);
    download(c.values(), C);
    ctx().sync();
    return c;
}

Mat multiply_reference(const Mat& a, const Mat& b) {
    if (a.cols() != b.rows()) {
        std::ostringstream os;
        os << "gemm dimension mismatch: A is " << a.rows() << "x" << a.cols() << ", B is " << b.rows() << "x"
           << b.cols();
        throw config_error(os.str());
    }
    Mat c(a.rows(), b.cols());
    if (c.size() == 0) return c;
    float* A = upload(a.values(), kA);
    float* B = upload(b.values(), kB);
    auto* C = static_cast<float*>(ctx().get(kC, c.size() * sizeof(float)));
    check(cct_gemm_exact(int64_t(a.rows()), int64_t(b.cols()), int64_t(a.cols()), A, int64_t(a.cols()), B,
                         int64_t(b.cols()), C, int64_t(b.cols()), ctx().stream),
          "multiply_reference");
    download(c.values(), C);
    ctx().sync();
    return c;
}

ProbeResult gemm_throughput_probe(std::size_t rows, std::size_t inner, std::size_t cols, const GemmConfig& cfg,
                                  int reps) {
    if (reps < 1) throw config_error("probe needs reps >= 1");
    const std::uint64_t elems =
        std::uint64_t(rows) * inner + std::uint64_t(inner) * cols + std::uint64_t(rows) * cols;
    if (elems * kRealBytes > (std::uint64_t(4) << 30))
        throw resource_error("probe shape exceeds the 4 GiB working-set budget");
    Mat probe_cfg_a(1, 1), probe_cfg_b(1, 1);
    check_multiply_dims(probe_cfg_a, probe_cfg_b, cfg);
    std::mt19937_64 rng(0x9e3779b97f4a7c15ull);
    const Mat a = Mat::random(rows, inner, rng);
    const Mat b = Mat::random(inner, cols, rng);
    int64_t lda, ldb;
    float* A = upload_padded(a, kA, &lda);
    float* B = upload_padded(b, kB, &ldb);
    auto* C = static_cast<float*>(ctx().get(kC, rows * cols * sizeof(float) + 16));
    cudaEvent_t e0, e1;
    cuda_check(cudaEventCreate(&e0), "event");
    cuda_check(cudaEventCreate(&e1), "event");
    device_multiply(int64_t(rows), int64_t(cols), int64_t(inner), A, lda, B, ldb, C);  // warmup
    std::vector<double> times;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0, ctx().stream);
        device_multiply(int64_t(rows), int64_t(cols), int64_t(inner), A, lda, B, ldb, C);
        cudaEventRecord(e1, ctx().stream);
        cuda_check(cudaEventSynchronize(e1), "probe");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        times.push_back(ms * 1e-3);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    std::sort(times.begin(), times.end());
    ProbeResult res;
    res.flops = gemm_flop_count(rows, inner, cols);
    res.median_s = times[times.size() / 2];
    res.flops_per_s = res.median_s > 0 ? double(res.flops) / res.median_s : 0.0;
    res.reps = reps;
    return res;
}

double memcpy_bandwidth_probe(std::size_t buffer_bytes, int reps) {
    if (reps < 1) throw config_error("probe needs reps >= 1");
    void* src = ctx().get(kA, buffer_bytes);
    void* dst = ctx().get(kB, buffer_bytes);
    cuda_check(cudaMemsetAsync(src, 1, buffer_bytes, ctx().stream), "memset");
    cudaEvent_t e0, e1;
    cuda_check(cudaEventCreate(&e0), "event");
    cuda_check(cudaEventCreate(&e1), "event");
    cuda_check(cudaMemcpyAsync(dst, src, buffer_bytes, cudaMemcpyDeviceToDevice, ctx().stream), "copy");  // warmup
    std::vector<double> times;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0, ctx().stream);
        cudaMemcpyAsync(dst, src, buffer_bytes, cudaMemcpyDeviceToDevice, ctx().stream);
        cudaEventRecord(e1, ctx().stream);
        cuda_check(cudaEventSynchronize(e1), "probe");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        times.push_back(ms * 1e-3);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    std::sort(times.begin(), times.end());
    const double med = times[times.size() / 2];
    return med > 0 ? double(buffer_bytes) / med : 0.0;  // bytes copied per second (as the reference)
}

// -------------------------------------------------------------- lowering.hpp
LoweredMatrices lower(const DataBatch& batch, const KernelBank& bank, LoweringStrategy strategy) {
    const LayerConfig L = layer_of(batch, bank);
    cct_conv_desc d = make_desc(L);
    int64_t rows = 0, cols = 0, kcols = 0;
    check(cct_lowered_shape(&d, to_c(strategy), CCT_ROWS_SPEC, &rows, &cols, &kcols), "lower");
    float* dx = upload_batch(batch, kX);
    float* dw = upload(bank.values(), kW);
    LoweredMatrices out;
    out.strategy = strategy;
    out.layer = L;
    out.Dhat = Mat(size_t(rows), size_t(cols));
    out.Khat = Mat(size_t(cols), size_t(kcols));
    auto* dd = static_cast<float*>(ctx().get(kA, out.Dhat.size() * sizeof(float) + 16));
    auto* dk = static_cast<float*>(ctx().get(kB, out.Khat.size() * sizeof(float) + 16));
    check(cct_lower(&d, to_c(strategy), CCT_ROWS_SPEC, dx, dd, cols, ctx().stream), "lower");
    check(cct_lower_khat(&d, to_c(strategy), dw, dk, ctx().stream), "lower");
    download(out.Dhat.values(), dd);
    download(out.Khat.values(), dk);
    ctx().sync();
    return out;
}

OutputBatch lift(const Mat& Rhat, LoweringStrategy strategy, const LayerConfig& layer) {
    cct_conv_desc d = make_desc(layer);
    int64_t rows = 0, cols = 0, kcols = 0;
    check(cct_lowered_shape(&d, to_c(strategy), CCT_ROWS_SPEC, &rows, &cols, &kcols), "lift");
    if (Rhat.rows() != size_t(rows) || Rhat.cols() != size_t(kcols)) {
        std::ostringstream os;
        os << "lift: Rhat is " << Rhat.rows() << "x" << Rhat.cols() << ", strategy needs " << rows << "x" << kcols;
        throw config_error(os.str());
    }
    float* dr = upload(Rhat.values(), kA);
    OutputBatch out(layer.b, layer.o, layer.m());
    auto* dy = static_cast<float*>(ctx().get(kY, out.size() * sizeof(float)));
    check(cct_lift(&d, to_c(strategy), CCT_ROWS_SPEC, dr, kcols, dy, ctx().stream), "lift");
    download(out.values(), dy);
    ctx().sync();
    return out;
}

std::pair<OutputBatch, PhaseTimings> convolve_lowered(const DataBatch& batch, const KernelBank& bank,
                                                      LoweringStrategy strategy, std::size_t gemm_threads,
                                                      ConvGeometry geom) {
    if (gemm_threads < 1 || gemm_threads > GemmConfig::kMaxThreads)
        throw config_error("gemm thread count must be in [1, " + std::to_string(GemmConfig::kMaxThreads) + "], got " +
                           std::to_string(gemm_threads));
    const Tensor3& first = batch[0];
    if (bank.depth() != first.depth() || bank.k() > first.rows() + 2 * geom.pad)
        throw config_error("kernel bank " + bank_shape_str(bank) + " incompatible with data tensor " +
                           tensor_shape_str(first));
    LayerConfig L;
    L.n = first.rows();
    L.k = bank.k();
    L.d = first.depth();
    L.o = bank.o();
    L.b = batch.b();
    L = layer_with(L, geom);
    cct_conv_desc d = make_desc(L);
    float* dx = upload_batch(batch, kX);
    float* dw = upload(bank.values(), kW);
    OutputBatch out(L.b, L.o, L.m());
    auto* dy = static_cast<float*>(ctx().get(kY, out.size() * sizeof(float)));
    size_t need = 0;
    check(cct_workspace_size(&d, to_c(strategy), CCT_PASS_FWD, &need), "workspace");
    void* ws = ctx().get(kWs, need);
    PhaseProbe probe;
    check(cct_conv_fwd(&d, to_c(strategy), dx, dw, dy, ws, need, ctx().stream), "convolve_lowered");
    ctx().sync();
    PhaseTimings t = probe.finish();
    download(out.values(), dy);
    ctx().sync();
    return {std::move(out), t};
}

DataBatch convolve_backward_data(const OutputBatch& dy, const KernelBank& bank, std::size_t n,
                                 LoweringStrategy strategy, ConvGeometry geom) {
    LayerConfig L;
    L.n = n;
    L.k = bank.k();
    L.d = bank.depth();
    L.o = bank.o();
    L.b = dy.b();
    L = layer_with(L, geom);
    cct_conv_desc d = make_desc(L);
    if (dy.o() != L.o || dy.m() != L.m())
        throw config_error("dy is " + std::to_string(dy.b()) + "x" + std::to_string(dy.o()) + "x" +
                           std::to_string(dy.m()) + "^2, layer needs o=" + std::to_string(L.o) +
                           " m=" + std::to_string(L.m()));
    float* ddy = upload(dy.values(), kY);
    float* dw = upload(bank.values(), kW);
    const size_t per = n * n * L.d;
    auto* ddx = static_cast<float*>(ctx().get(kX, per * L.b * sizeof(float)));
    size_t need = 0;
    check(cct_workspace_size(&d, to_c(strategy), CCT_PASS_BWD_DATA, &need), "workspace");
    void* ws = ctx().get(kWs, need);
    check(cct_conv_bwd_data(&d, to_c(strategy), ddy, dw, ddx, ws, need, ctx().stream), "convolve_backward_data");
    std::vector<Tensor3> imgs(L.b, Tensor3(n, L.d));
    for (size_t q = 0; q < L.b; ++q)
        cuda_check(cudaMemcpyAsync(imgs[q].values().data(), ddx + q * per, per * sizeof(float), cudaMemcpyDeviceToHost,
                                   ctx().stream),
                   "D2H");
    ctx().sync();
    return DataBatch(std::move(imgs));
}

KernelBank convolve_backward_weight(const DataBatch& batch, const OutputBatch& dy, std::size_t k,
                                    LoweringStrategy strategy, ConvGeometry geom) {
    LayerConfig L;
    L.n = batch[0].rows();
    L.k = k;
    L.d = batch[0].depth();
    L.o = dy.o();
    L.b = batch.b();
    L = layer_with(L, geom);
    cct_conv_desc d = make_desc(L);
    if (dy.b() != L.b || dy.m() != L.m())
        throw config_error("dy batch/side does not match the layer (b=" + std::to_string(L.b) +
                           ", m=" + std::to_string(L.m()) + ")");
    float* dx = upload_batch(batch, kX);
    float* ddy = upload(dy.values(), kY);
    KernelBank dwb(k, L.d, L.o);
    auto* ddw = static_cast<float*>(ctx().get(kW, dwb.values().size() * sizeof(float)));
    size_t need = 0;
    check(cct_workspace_size(&d, to_c(strategy), CCT_PASS_BWD_WEIGHT, &need), "workspace");
    void* ws = ctx().get(kWs, need);
    check(cct_conv_bwd_weight(&d, to_c(strategy), dx, ddy, ddw, ws, need, ctx().stream), "convolve_backward_weight");
    download(dwb.values(), ddw);
    ctx().sync();
    return dwb;
}

// ----------------------------------------------------- layer extension (groups, bias, ReLU)
namespace {
LayerConfig ext_layer(const DataBatch& batch, const KernelBank& bank, const LayerExtension& ext, ConvGeometry geom) {
    const Tensor3& first = batch[0];
    if (ext.groups < 1 || first.depth() % ext.groups || bank.o() % ext.groups || bank.depth() * ext.groups != first.depth())
        throw config_error("grouped layer: kernel bank " + bank_shape_str(bank) + " with groups=" +
                           std::to_string(ext.groups) + " does not match data tensor " + tensor_shape_str(first));
    if (!ext.bias.empty() && ext.bias.size() != bank.o())
        throw config_error("bias has " + std::to_string(ext.bias.size()) + " values for o=" + std::to_string(bank.o()));
    LayerConfig L;
    L.n = first.rows();
    L.k = bank.k();
    L.d = first.depth();
    L.o = bank.o();
    L.b = batch.b();
    return layer_with(L, geom);
}
}  // namespace

std::pair<OutputBatch, PhaseTimings> convolve_lowered_ex(const DataBatch& batch, const KernelBank& bank,
                                                         LoweringStrategy strategy, const LayerExtension& ext,
                                                         ConvGeometry geom) {
    const LayerConfig L = ext_layer(batch, bank, ext, geom);
    cct_conv_desc d = make_desc(L);
    float* dx = upload_batch(batch, kX);
    float* dw = upload(bank.values(), kW);
    float* db = ext.bias.empty() ? nullptr : upload(ext.bias, kAux);
    const cct_conv_ext e{int64_t(ext.groups), db, ext.relu ? 1 : 0};
    OutputBatch out(L.b, L.o, L.m());
    auto* dy = static_cast<float*>(ctx().get(kY, out.size() * sizeof(float)));
    size_t need = 0;
    check(cct_workspace_size_ex(&d, to_c(strategy), &e, CCT_PASS_FWD, &need), "workspace");
    void* ws = ctx().get(kWs, need);
    PhaseProbe probe;
    check(cct_conv_fwd_ex(&d, to_c(strategy), &e, dx, dw, dy, ws, need, ctx().stream), "convolve_lowered_ex");
    ctx().sync();
    PhaseTimings t = probe.finish();
    download(out.values(), dy);
    ctx().sync();
    return {std::move(out), t};
}

LayerGradients convolve_backward_ex(const DataBatch& batch, const OutputBatch& y, const OutputBatch& dy,
                                    const KernelBank& bank, LoweringStrategy strategy, const LayerExtension& ext,
                                    ConvGeometry geom) {
    const LayerConfig L = ext_layer(batch, bank, ext, geom);
    if (dy.b() != L.b || dy.o() != L.o || dy.m() != L.m() || (ext.relu && (y.b() != L.b || y.o() != L.o || y.m() != L.m())))
        throw config_error("dy / y do not match the layer output (b=" + std::to_string(L.b) + ", o=" +
                           std::to_string(L.o) + ", m=" + std::to_string(L.m()) + ")");
    cct_conv_desc d = make_desc(L);
    float* dx_in = upload_batch(batch, kX);
    float* dw_in = upload(bank.values(), kW);
    float* ddy = upload(dy.values(), kY);
    float* dyo = ext.relu ? upload(y.values(), kA) : nullptr;
    const size_t per = L.n * L.n * L.d;
    auto* gdx = static_cast<float*>(ctx().get(kB, per * L.b * sizeof(float)));
    auto* gdw = static_cast<float*>(ctx().get(kC, bank.values().size() * sizeof(float)));
    auto* gdb = ext.bias.empty() ? nullptr : static_cast<float*>(ctx().get(kAux, L.o * sizeof(float)));
    const cct_conv_ext e{int64_t(ext.groups), nullptr, ext.relu ? 1 : 0};
    size_t need = 0;
    check(cct_workspace_size_ex(&d, to_c(strategy), &e, CCT_PASS_BWD, &need), "workspace");
    void* ws = ctx().get(kWs, need);
    check(cct_conv_bwd_ex(&d, to_c(strategy), &e, dx_in, dyo, ddy, dw_in, gdx, gdw, gdb, ws, need, ctx().stream),
          "convolve_backward_ex");
    LayerGradients g;
    std::vector<Tensor3> imgs(L.b, Tensor3(L.n, L.d));
    for (size_t q = 0; q < L.b; ++q)
        cuda_check(cudaMemcpyAsync(imgs[q].values().data(), gdx + q * per, per * sizeof(float), cudaMemcpyDeviceToHost,
                                   ctx().stream),
                   "D2H");
    g.dw = KernelBank(bank.k(), bank.depth(), bank.o());
    download(g.dw.values(), gdw);
    if (gdb) {
        g.db.resize(L.o);
        download(g.db, gdb);
    }
    ctx().sync();
    g.dx = DataBatch(std::move(imgs));
    return g;
}

// ------------------------------------------------------------ cost_model.hpp
namespace {
cct_calibration weights_to_cal(const CostWeights& w) {
    cct_calibration c;
    cct_calibration_default(&c);
    if (w.alpha > 0) {
        c.alpha = w.alpha;
        c.hbm_bytes_per_s = 8.0 / w.alpha;  // one element read + written
    }
    if (w.beta > 0) {
        c.beta = w.beta;
        c.gemm_flops_per_s = 1.0 / w.beta;
    }
    return c;
}
}  // namespace

CostEstimate estimate(LoweringStrategy strategy, const LayerConfig& layer, const CostWeights& w) {
    cct_conv_desc d = make_desc(layer);
    cct_calibration cal = weights_to_cal(w);
    cct_cost_estimate e;
    check(cct_estimate(&d, to_c(strategy), &cal, w.include_backward ? CCT_PASS_BWD : CCT_PASS_FWD, &e), "estimate");
    CostEstimate r;
    r.lower_elements_written = e.lower_elements_written;
    r.gemm_flops = e.gemm_flops;
    r.lift_adds = e.lift_adds;
    r.lowered_bytes = e.lowered_bytes;
    r.total_score = e.total_score;
    r.model_seconds = e.model_seconds;
    return r;
}

StrategyChoice select_strategy(const LayerConfig& layer, const CostWeights& w) {
    StrategyChoice c;
    double best = 0;
    for (int t = 0; t < 3; ++t) {
        c.estimates[size_t(t)] = estimate(LoweringStrategy(t + 1), layer, w);
        if (t == 0 || c.estimates[size_t(t)].model_seconds < best) {
            best = c.estimates[size_t(t)].model_seconds;
            c.strategy = LoweringStrategy(t + 1);
        }
    }
    c.ratio = double(layer.d) / double(layer.o);
    return c;
}

double crossover_ratio(const LayerConfig& templ, const CostWeights& w) {
    if (templ.k == 1) return INFINITY;  // identical costs, no crossover
    const double prod = double(templ.d) * double(templ.o);
    auto diff = [&](double ratio) {
        LayerConfig L = templ;
        L.d = std::max<size_t>(1, size_t(std::llround(std::sqrt(prod * ratio))));
        L.o = std::max<size_t>(1, size_t(std::llround(std::sqrt(prod / ratio))));
        return estimate(LoweringStrategy::Type1, L, w).model_seconds -
               estimate(LoweringStrategy::Type3, L, w).model_seconds;
    };
    double lo = 1.0 / 64, hi = 64.0;
    const double flo = diff(lo), fhi = diff(hi);
    if ((flo > 0) == (fhi > 0)) return fhi > 0 ? 0.0 : INFINITY;
    for (int it = 0; it < 60; ++it) {
        const double mid = std::sqrt(lo * hi);
        if ((diff(mid) > 0) == (flo > 0)) lo = mid;
        else hi = mid;
    }
    return std::sqrt(lo * hi);
}

// -------------------------------------------------------------- batching.hpp
PartitionPlan plan_partitions(std::size_t b, std::size_t total_threads, std::size_t p) {
    if (p < 1 || p > std::min(b, total_threads))
        throw config_error("partition count " + std::to_string(p) + " out of range [1, min(b=" + std::to_string(b) +
                           ", threads=" + std::to_string(total_threads) + ")]");
    PartitionPlan plan;
    plan.partitions = p;
    for (size_t i = 0; i < p; ++i) {
        plan.partition_sizes.push_back(b / p + (i < b % p ? 1 : 0));
        plan.threads_per_partition.push_back(total_threads / p + (i < total_threads % p ? 1 : 0));
    }
    return plan;
}

FootprintReport footprint(LoweringStrategy strategy, const LayerConfig& layer, std::size_t partition_size) {
    LayerConfig L = layer;
    L.b = partition_size;
    cct_conv_desc d = make_desc(L);
    int64_t rows = 0, cols = 0, kcols = 0;
    check(cct_lowered_shape(&d, to_c(strategy), CCT_ROWS_INTERNAL, &rows, &cols, &kcols), "footprint");
    FootprintReport r;
    r.strategy = strategy;
    r.lowered_bytes_per_partition = std::uint64_t(rows) * std::uint64_t(cols) * kRealBytes;
    r.peak_bytes = r.lowered_bytes_per_partition;
    return r;
}

PartitionedResult execute_partitioned(const DataBatch& batch, const KernelBank& bank, LoweringStrategy strategy,
                                      const PartitionPlan& plan, ConvGeometry geom) {
    size_t total = 0;
    for (size_t s : plan.partition_sizes) total += s;
    if (total != batch.b() || plan.partition_sizes.size() != plan.partitions)
        throw config_error("partition plan does not cover the batch");
    const Tensor3& first = batch[0];
    LayerConfig L;
    L.n = first.rows();
    L.k = bank.k();
    L.d = first.depth();
    L.o = bank.o();
    L.b = batch.b();
    L = layer_with(L, geom);
    PartitionedResult res;
    res.output = OutputBatch(L.b, L.o, L.m());
    size_t first_img = 0, max_part = 0;
    for (size_t part : plan.partition_sizes) {
        auto imgs = batch.slice(first_img, part);
        DataBatch sub(std::vector<Tensor3>(imgs.begin(), imgs.end()));
        auto [y, t] = convolve_lowered(sub, bank, strategy, 1, geom);
        std::copy(y.values().begin(), y.values().end(), res.output.plane(first_img, 0));
        res.timing.lower_s += t.lower_s;
        res.timing.multiply_s += t.multiply_s;
        res.timing.lift_s += t.lift_s;
        first_img += part;
        max_part = std::max(max_part, part);
    }
    res.footprint = footprint(strategy, L, max_part);
    res.footprint.peak_bytes = res.footprint.lowered_bytes_per_partition * plan.partitions;
    return res;
}

// ------------------------------------------------------------- scheduler.hpp
SplitPlan proportional_split(const std::vector<DeviceProfile>& devices, std::size_t b) {
    if (devices.empty()) throw config_error("proportional_split needs at least one device");
    double tot = 0;
    for (const auto& d : devices) {
        if (!(d.flops > 0)) throw config_error("device '" + d.name + "' needs flops > 0");
        tot += d.flops;
    }
    SplitPlan plan;
    std::vector<double> raw;
    size_t assigned = 0;
    for (const auto& d : devices) {
        plan.fractions.push_back(d.flops / tot);
        raw.push_back(d.flops / tot * double(b));
        plan.counts.push_back(size_t(std::floor(raw.back())));
        assigned += plan.counts.back();
    }
    std::vector<size_t> order(devices.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t c) {
        return (raw[a] - double(plan.counts[a])) > (raw[c] - double(plan.counts[c]));
    });
    for (size_t i = 0; assigned < b; ++i, ++assigned) plan.counts[order[i % order.size()]] += 1;
    return plan;
}

double simulate_makespan(const LayerConfig& layer, const SplitPlan& plan, const std::vector<DeviceProfile>& devices,
                         LoweringStrategy strategy) {
    if (plan.fractions.size() != devices.size())
        throw config_error("split plan has " + std::to_string(plan.fractions.size()) + " fractions for " +
                           std::to_string(devices.size()) + " devices");
    LayerConfig one = layer;
    one.b = 1;
    one.validate();
    const double per_image = double(estimate(strategy, one, CostWeights{0, 0, false}).gemm_flops);
    double span = 0;
    for (size_t i = 0; i < devices.size(); ++i) {
        if (!(devices[i].flops > 0)) throw config_error("device '" + devices[i].name + "' needs flops > 0");
        const double f = plan.fractions[i];
        if (f <= 0) continue;  // a device without work finishes at 0
        span = std::max(span, devices[i].fixed_overhead + f * double(layer.b) * per_image / devices[i].flops);
    }
    return span;
}

namespace {
SplitPlan two_way(double p, std::size_t b) {
    SplitPlan s;
    s.fractions = {1.0 - p, p};
    const auto c1 = std::size_t(std::llround(p * double(b)));
    s.counts = {b - std::min(b, c1), std::min(b, c1)};
    return s;
}
}  // namespace

SplitPlan optimal_split_sweep(const LayerConfig& layer, const std::vector<DeviceProfile>& devices,
                              std::size_t granularity, LoweringStrategy strategy) {
    if (devices.size() != 2)
        throw config_error("optimal_split_sweep supports exactly 2 devices (SPEC.md:393), got " +
                           std::to_string(devices.size()));
    if (granularity < 10) throw config_error("granularity must be >= 10");
    SplitPlan best = two_way(0.0, layer.b);
    double best_t = simulate_makespan(layer, best, devices, strategy);
    for (std::size_t i = 1; i <= granularity; ++i) {
        SplitPlan s = two_way(double(i) / double(granularity), layer.b);
        const double t = simulate_makespan(layer, s, devices, strategy);
        if (t < best_t) {  // strict: ties keep the smaller fraction
            best_t = t;
            best = s;
        }
    }
    return best;
}

double heuristic_gap(const LayerConfig& layer, const std::vector<DeviceProfile>& devices, std::size_t granularity,
                     LoweringStrategy strategy) {
    const SplitPlan prop = proportional_split(devices, layer.b);
    const double tp = simulate_makespan(layer, prop, devices, strategy);
    const double ts = simulate_makespan(layer, optimal_split_sweep(layer, devices, granularity, strategy), devices,
                                        strategy);
    const double opt = std::min(tp, ts);
    return opt > 0 ? tp / opt : 1.0;
}

OutputBatch direct_convolve_batch(const DataBatch& batch, const KernelBank& bank, ConvGeometry geom) {
    const Tensor3& first = batch[0];
    if (bank.depth() != first.depth() || bank.k() > first.rows() + 2 * geom.pad)
        throw config_error("kernel bank " + bank_shape_str(bank) + " incompatible with data tensor " +
                           tensor_shape_str(first));
    LayerConfig L;
    L.n = first.rows();
    L.k = bank.k();
    L.d = first.depth();
    L.o = bank.o();
    L.b = batch.b();
    L = layer_with(L, geom);
    cct_conv_desc d = make_desc(L);
    float* dx = upload_batch(batch, kX);
    float* dw = upload(bank.values(), kW);
    OutputBatch out(L.b, L.o, L.m());
    auto* dy = static_cast<float*>(ctx().get(kY, out.size() * sizeof(float)));
    check(cct_direct_conv_fwd_exact(&d, dx, dw, dy, ctx().stream), "direct_convolve_batch");
    download(out.values(), dy);
    ctx().sync();
    return out;
}

}  // namespace convlow
