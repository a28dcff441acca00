// convlow/cost_model.hpp -- the automatic lowering optimizer (
// the reference's src/cost_model.cpp is absent, CMakeLists.txt:23).
//
// estimate() returns the SPEC's exact counts plus the B200 model
// time of the kernels this build launches; select_strategy() takes the argmin
// of the model time (ties: Type1 < Type2 < Type3).
#pragma once

#include <array>
#include <cstdint>

#include "convlow/lowering.hpp"

namespace convlow {

struct CostEstimate {
    std::uint64_t lower_elements_written = 0;
    std::uint64_t gemm_flops = 0;
    std::uint64_t lift_adds = 0;
    std::uint64_t lowered_bytes = 0;
    double total_score = 0.0;    // alpha (lower + lift) + beta flops
    double model_seconds = 0.0;  // calibrated B200 time of fwd (or fwd + bwd)
};

struct StrategyChoice {
    LoweringStrategy strategy = LoweringStrategy::Type1;
    std::array<CostEstimate, 3> estimates{};
    double ratio = 0.0;  // d / o
};

// Calibration weights; defaults are the measured B200 values.
struct CostWeights {
    double alpha = 0.0;  // s per element moved (0 = default)
    double beta = 0.0;   // s per flop (0 = default)
    bool include_backward = true;
};

CostEstimate estimate(LoweringStrategy strategy, const LayerConfig& layer, const CostWeights& w = {});
StrategyChoice select_strategy(const LayerConfig& layer, const CostWeights& w = {});
// d/o at which Type 1 and Type 3 model times cross, bisection over [1/64, 64]
// with d*o fixed; +inf / 0 when no crossing (k = 1: +inf).
double crossover_ratio(const LayerConfig& templ, const CostWeights& w = {});

}  // namespace convlow
