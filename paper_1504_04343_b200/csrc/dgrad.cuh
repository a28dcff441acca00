// dgrad.cuh -- fused backward-data of small-channel strided Type 1 layers (CaffeNet conv1
// class) without the materialised dDhat.
//
// The materialised path writes dDhat = dRhat Khat (b m^2 x k^2 d, 1.13 GB for conv1 at
// b = 256) and col2im sums it into dx (SPEC.md:139-143 adjoint of the Type 1 lowering,
// tensor.cpp:77-106).  Here the GEMM tile keeps one output-row pair's dDhat in TMEM (lanes =
// pixels, columns = (filter row i, run element e)) and its epilogue folds the horizontal
// overlap of neighbouring pixels (pixel c's run for filter row i covers padded input floats
// [s d c, s d c + k d) of input row s r + i, so at most ceil(k d / s d) pixels meet in a
// float) with warp shuffles: each pixel writes only the s d floats it owns (the last pixel
// of a row also the tail) of a per-(output row, filter row) partial row H.  A streaming pass
// then sums the <= ceil(k / s) partial rows of every input row (the vertical overlap) into dx.
// HBM traffic: H is 0.42 GB instead of dDhat's 1.13 GB written and read back.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

#include "lowering.cuh"

namespace cct {

bool hfold_dgrad_ok(const Geo& g);
int64_t hfold_dgrad_ws_floats(const Geo& g);
// dx (NHWC) = backward-data of dy (layout g.yl) through the kernel bank w (o, k, k, d), on st:
// the GEMM + horizontal fold, then the vertical fold (vfold_kernel, reading H from ws).  When
// gemm_done is not null it is recorded on st between the two (the caller may fork there).
cudaError_t hfold_dgrad(const Geo& g, const float* dy, const float* w, float* dx, float* ws, cudaStream_t st,
                        cudaEvent_t gemm_done = nullptr);

}  // namespace cct
