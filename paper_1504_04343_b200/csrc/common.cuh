// common.cuh -- shared host helpers: device properties, launch accounting,
// thread-local error message (cct_last_error).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace cct {

int num_sms();              // SM count of the current device (cached per device)
void note_launch();
int tuning(int key);        // cct_set_tuning value of a cct_tuning key         // count one kernel launch (cct_launch_count)
void set_error(const std::string& msg);
const char* last_error();

// PhaseTimings on the device: when enabled, every launch is
// bracketed by CUDA events on its stream and attributed to a phase.
enum Phase : int { kPhaseLower = 0, kPhaseGemm = 1, kPhaseLift = 2, kPhaseExpand = 3, kPhaseCol2im = 4,
                   kPhaseReduce = 5, kPhaseOther = 6, kNumPhases = 7 };
struct PhaseScope {
    PhaseScope(Phase ph, cudaStream_t st, double flops = 0, double bytes = 0);
    ~PhaseScope();
    int slot;
    cudaStream_t st;
};
void profile_enable(bool on);

// In-call fork / join (CCT_TUNE_OVERLAP): per host thread and device, a high-priority side stream
// and two events, so independent work inside one ABI call (the backward-weight beside the
// backward-data's fold) runs concurrently.  Null when they cannot be created.
struct Fork {
    cudaStream_t side;
    cudaEvent_t fork, join;
};
const Fork* fork_resources();
// sync + accumulate: ms, flops, bytes, launches per phase (arrays of kNumPhases)
void profile_read(double* ms, double* flops, double* bytes, uint64_t* launches, bool reset);

inline int64_t rup4(int64_t v) { return (v + 3) & ~int64_t(3); }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// grid size for a grid-stride elementwise kernel: a multiple of the SM count
inline int grid_for(int64_t work_items, int threads, int per_sm = 8) {
    const int64_t want = cdiv(work_items, threads);
    const int64_t cap = int64_t(num_sms()) * per_sm;
    return int(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace cct
