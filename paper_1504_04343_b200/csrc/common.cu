// common.cu -- device property cache, launch counter, thread-local error text.
#include "common.cuh"

#include "cct.h"

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

namespace cct {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
int g_sms[64] = {0};
}  // namespace

int num_sms() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (!g_sms[dev]) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
            v = 148;
        g_sms[dev] = v;
    }
    return g_sms[dev];
}

// Tuning switches (cct_set_tuning): explicit, process-wide; the library reads no
// environment variables, so results and tile choices depend only on the caller's calls.
namespace {
constexpr int kTuneDefaults[CCT_TUNE_COUNT] = {
    /* SPLIT_PRODUCER */ 0, /* A_TMEM */ 1,     /* A_TMEM_WIDE */ 1, /* CTA_PAIRS */ 0,
    /* BN384 */ 0,          /* STREAMK */ 1,    /* CHAIN2 */ 1,      /* S2D */ 1,
    /* IMPLICIT_BWD */ 1,   /* WGRAD_SWAP */ 1, /* DGRAD_SWAP */ 0,  /* FWD_SWAP */ 0,
    /* TRACE_PHASES */ 0,   /* GATHER */ 1,     /* FUSED_T23 */ 0,   /* OVERLAP */ 1};
constexpr int kTuneMax[CCT_TUNE_COUNT] = {1, 3, 1, 2, 1, 1, 1, 2, 2, 1, 2, 1, 1, 3, 1, 1};
std::atomic<int> g_tune[CCT_TUNE_COUNT] = {
    {kTuneDefaults[0]}, {kTuneDefaults[1]}, {kTuneDefaults[2]},  {kTuneDefaults[3]},  {kTuneDefaults[4]},
    {kTuneDefaults[5]}, {kTuneDefaults[6]}, {kTuneDefaults[7]},  {kTuneDefaults[8]},  {kTuneDefaults[9]},
    {kTuneDefaults[10]}, {kTuneDefaults[11]}, {kTuneDefaults[12]}, {kTuneDefaults[13]}, {kTuneDefaults[14]},
    {kTuneDefaults[15]}};
}  // namespace

int tuning(int key) { return (key >= 0 && key < CCT_TUNE_COUNT) ? g_tune[key].load(std::memory_order_relaxed) : 0; }

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }
void reset_launch_count() { g_launches.store(0, std::memory_order_relaxed); }

namespace {
struct Rec {
    cudaEvent_t a, b;
    int phase;
    double flops, bytes;
};
std::mutex g_pm;
std::atomic<bool> g_prof{false};
std::vector<Rec> g_recs;
double g_acc_ms[kNumPhases], g_acc_fl[kNumPhases], g_acc_by[kNumPhases];
uint64_t g_acc_n[kNumPhases];
}  // namespace

void profile_enable(bool on) { g_prof.store(on); }

namespace {
struct ForkSet {
    Fork f[16] = {};
    bool made[16] = {};
    ~ForkSet() {
        for (int i = 0; i < 16; ++i)
            if (made[i]) {
                cudaStreamDestroy(f[i].side);
                cudaEventDestroy(f[i].fork);
                cudaEventDestroy(f[i].join);
            }
    }
};
thread_local ForkSet t_fork;
}  // namespace

const Fork* fork_resources() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return nullptr;
    if (!t_fork.made[dev]) {
        int lo = 0, hi = 0;
        Fork& f = t_fork.f[dev];
        if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess ||
            cudaStreamCreateWithPriority(&f.side, cudaStreamNonBlocking, hi) != cudaSuccess)
            return nullptr;
        if (cudaEventCreateWithFlags(&f.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&f.join, cudaEventDisableTiming) != cudaSuccess) {
            cudaStreamDestroy(f.side);
            return nullptr;
        }
        t_fork.made[dev] = true;
    }
    return &t_fork.f[dev];
}

PhaseScope::PhaseScope(Phase ph, cudaStream_t s, double flops, double bytes) : slot(-1), st(s) {
    if (tuning(CCT_TUNE_TRACE_PHASES)) fprintf(stderr, "cct-phase %d bytes %.0f flops %.0f\n", int(ph), bytes, flops);
    if (!g_prof.load(std::memory_order_relaxed)) return;
    Rec r{};
    if (cudaEventCreate(&r.a) != cudaSuccess || cudaEventCreate(&r.b) != cudaSuccess) return;
    r.phase = ph;
    r.flops = flops;
    r.bytes = bytes;
    cudaEventRecord(r.a, st);
    std::lock_guard<std::mutex> lk(g_pm);
    slot = int(g_recs.size());
    g_recs.push_back(r);
}

PhaseScope::~PhaseScope() {
    if (slot < 0) return;
    std::lock_guard<std::mutex> lk(g_pm);
    cudaEventRecord(g_recs[size_t(slot)].b, st);
}

void profile_read(double* ms, double* flops, double* bytes, uint64_t* launches, bool reset) {
    std::lock_guard<std::mutex> lk(g_pm);
    for (Rec& r : g_recs) {
        cudaEventSynchronize(r.b);
        float t = 0.f;
        cudaEventElapsedTime(&t, r.a, r.b);
        g_acc_ms[r.phase] += t;
        g_acc_fl[r.phase] += r.flops;
        g_acc_by[r.phase] += r.bytes;
        g_acc_n[r.phase] += 1;
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    g_recs.clear();
    for (int i = 0; i < kNumPhases; ++i) {
        if (ms) ms[i] = g_acc_ms[i];
        if (flops) flops[i] = g_acc_fl[i];
        if (bytes) bytes[i] = g_acc_by[i];
        if (launches) launches[i] = g_acc_n[i];
        if (reset) g_acc_ms[i] = g_acc_fl[i] = g_acc_by[i] = 0, g_acc_n[i] = 0;
    }
}

void set_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }

}  // namespace cct

extern "C" {
cct_status cct_set_tuning(cct_tuning key, int value) {
    const int k = int(key);
    if (k < 0 || k >= CCT_TUNE_COUNT) {
        cct::set_error("unknown tuning key " + std::to_string(k));
        return CCT_ERR_CONFIG;
    }
    if (value < 0 || value > cct::kTuneMax[k]) {
        cct::set_error("tuning key " + std::to_string(k) + ": value " + std::to_string(value) + " out of range [0, " +
                       std::to_string(cct::kTuneMax[k]) + "]");
        return CCT_ERR_CONFIG;
    }
    cct::g_tune[k].store(value);
    return CCT_OK;
}
int cct_get_tuning(cct_tuning key) { return (int(key) >= 0 && int(key) < CCT_TUNE_COUNT) ? cct::tuning(int(key)) : -1; }
void cct_reset_tuning(void) {
    for (int k = 0; k < CCT_TUNE_COUNT; ++k) cct::g_tune[k].store(cct::kTuneDefaults[k]);
}
}  // extern "C"
