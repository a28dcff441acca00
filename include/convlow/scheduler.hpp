// convlow/scheduler.hpp -- device-split planning and simulation (
// the reference's src/scheduler.cpp is absent, CMakeLists.txt:25).  The planner
// (proportional_split) is on the B200 path: the batch split over GPUs.  The
// makespan simulator, the sweep optimum and the heuristic gap (SPEC.md:375-401,
// PAPER Appendix B) are pure arithmetic, used by `convbench schedule`.
#pragma once

#include <string>
#include <vector>

#include "convlow/common.hpp"
#include "convlow/lowering.hpp"

namespace convlow {

struct DeviceProfile {
    std::string name;
    double flops = 0.0;
    double fixed_overhead = 0.0;
};

struct SplitPlan {
    std::vector<double> fractions;
    std::vector<std::size_t> counts;
};

// fraction_i = flops_i / sum(flops); counts by largest remainder (sum == b).
SplitPlan proportional_split(const std::vector<DeviceProfile>& devices, std::size_t b);

// max over devices with work of fixed_overhead_i + work(fraction_i b) / flops_i, where
// work = the GEMM FLOPs of the layer's lowering per image.
// config_error when the plan and the device list differ in length.
double simulate_makespan(const LayerConfig& layer, const SplitPlan& plan, const std::vector<DeviceProfile>& devices,
                         LoweringStrategy strategy = LoweringStrategy::Type1);

// Two devices only: scan the fraction p of devices[1] over
// {0, 1/g, ..., 1} (g >= 10) for the smallest makespan; ties keep the smaller p.
SplitPlan optimal_split_sweep(const LayerConfig& layer, const std::vector<DeviceProfile>& devices,
                              std::size_t granularity, LoweringStrategy strategy = LoweringStrategy::Type1);

// makespan(proportional) / makespan(best of the sweep and the proportional plan) >= 1
// (Appendix B: "within 5% of the optimal").
double heuristic_gap(const LayerConfig& layer, const std::vector<DeviceProfile>& devices, std::size_t granularity,
                     LoweringStrategy strategy = LoweringStrategy::Type1);

}  // namespace convlow
