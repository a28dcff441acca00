// convlow/lowering.hpp -- the three lowering strategies (the
// reference's src/lowering.cpp is absent, CMakeLists.txt:22).
//
// lower / lift / convolve_lowered keep the SPEC contracts (shapes SPEC.md:101-104,
// row order c*m + r, zero-filled Type 2 rows).  On B200 the phases are device
// kernels (include/cct.h) and PhaseTimings are CUDA-event device times.
// Extensions required by the north star: stride / pad (ConvGeometry) and the
// backward-data / backward-weight passes.
#pragma once

#include <utility>
#include <vector>

#include "convlow/gemm.hpp"
#include "convlow/tensor.hpp"

namespace convlow {

enum class LoweringStrategy { Type1 = 1, Type2 = 2, Type3 = 3 };

struct LoweredMatrices {
    LoweringStrategy strategy = LoweringStrategy::Type1;
    Mat Dhat;  // Type1 (b m^2) x (k^2 d); Type2 (b n^2) x (k d); Type3 (b n^2) x d
    Mat Khat;  // Type1 (k^2 d) x o;       Type2 (k d) x (k o);    Type3 d x (k^2 o)
    LayerConfig layer;
};

struct PhaseTimings {
    double lower_s = 0.0;
    double multiply_s = 0.0;
    double lift_s = 0.0;
};

// Extension: stride / zero padding of the convolution (defaults = Eq. 1).
struct ConvGeometry {
    std::size_t stride = 1;
    std::size_t pad = 0;
};

LoweredMatrices lower(const DataBatch& batch, const KernelBank& bank, LoweringStrategy strategy);
OutputBatch lift(const Mat& Rhat, LoweringStrategy strategy, const LayerConfig& layer);

// lift(multiply(lower(...))): the hot path, on the device.  gemm_threads is
// validated like GemmConfig::threads and otherwise ignored.
std::pair<OutputBatch, PhaseTimings> convolve_lowered(const DataBatch& batch, const KernelBank& bank,
                                                      LoweringStrategy strategy, std::size_t gemm_threads,
                                                      ConvGeometry geom = {});

// Extension of direct_convolve_batch (tensor.hpp) to stride / pad: the exact
// fp64 device oracle of the generalised layer (checker for convbench verify).
OutputBatch direct_convolve_batch(const DataBatch& batch, const KernelBank& bank, ConvGeometry geom);

// Backward passes (north_star).  dy has the OutputBatch layout of the forward
// output; the results have the layouts of the forward inputs.
DataBatch convolve_backward_data(const OutputBatch& dy, const KernelBank& bank, std::size_t n,
                                 LoweringStrategy strategy, ConvGeometry geom = {});
KernelBank convolve_backward_weight(const DataBatch& batch, const OutputBatch& dy, std::size_t k,
                                    LoweringStrategy strategy, ConvGeometry geom = {});

// Layer extension (beyond the reference, whose SPEC puts groups out of
// scope): grouped convolution as in bvlc_reference_caffenet and the bias + ReLU
// epilogue around the layer.  The KernelBank holds (o, k, k, d / groups); output channel j
// reads input-channel group j / (o / groups).  y = relu ? max(conv + bias, 0) : conv + bias
// (empty bias = none).  Over cct_conv_fwd_ex / cct_conv_bwd_ex (include/cct.h).
struct LayerExtension {
    std::size_t groups = 1;
    std::vector<real> bias;  // o values, or empty
    bool relu = false;
};

std::pair<OutputBatch, PhaseTimings> convolve_lowered_ex(const DataBatch& batch, const KernelBank& bank,
                                                         LoweringStrategy strategy, const LayerExtension& ext,
                                                         ConvGeometry geom = {});

struct LayerGradients {
    DataBatch dx;          // gradient of the input
    KernelBank dw;         // (o, k, k, d / groups)
    std::vector<real> db;  // o values (empty when the layer has no bias)
};

// dy: gradient of the layer output y (after the ReLU; y is the forward's output).
LayerGradients convolve_backward_ex(const DataBatch& batch, const OutputBatch& y, const OutputBatch& dy,
                                    const KernelBank& bank, LoweringStrategy strategy, const LayerExtension& ext,
                                    ConvGeometry geom = {});

}  // namespace convlow
