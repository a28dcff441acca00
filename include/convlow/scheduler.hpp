// convlow/scheduler.hpp -- the proportional device split (the
// reference's src/scheduler.cpp is absent, CMakeLists.txt:25).  Only the
// planner is on the B200 path (the batch split over GPUs); the makespan
// simulator of SPEC.md:375-401 is out of scope.
#pragma once

#include <string>
#include <vector>

#include "convlow/common.hpp"

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

}  // namespace convlow
