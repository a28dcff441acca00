// gather.cuh -- fused small-channel Type 1 convolution (the lowered matrix is never
// materialised): CaffeNet conv1 class layers, d * s % 4 == 0 (d = 3, stride 4).
//
// The Type 1 lowering of such a layer reads, for output pixel (r, c)
// and filter row i, one contiguous run of k d floats of input row s r - p + i starting
// at column s c - p.  The fused kernels stage whole input rows in shared memory (1D
// bulk copies, TMA engine) and gather warps assemble each 16-column k-block of Dhat
// (forward: 128 pixels x 16 lowered columns; backward-weight: 128 lowered columns x
// 16 pixels) in registers, split it into its 3xTF32 big / small halves and write those
// straight into TMEM, where tcgen05.mma reads its A operand.  The other operand (the
// kernel bank, or dy) streams through a TMA ring.  No Dhat reaches HBM
// (the fused lowering).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

#include "lowering.cuh"

namespace cct {

// Whether the fused forward / backward-weight kernels take this layer (geometry,
// shared-memory budget, 32-bit index ranges).
bool gather_fwd_ok(const Geo& g);
bool gather_wgrad_ok(const Geo& g);
// scratch floats of the fused passes (prepared kernel bank / partial dW tiles)
int64_t gather_fwd_ws_floats(const Geo& g);
int64_t gather_wgrad_ws_floats(const Geo& g);

// y (layout g.yl; image stride ycs floats when > 0) = conv(x, w) (+ bias, ReLU)
cudaError_t gather_fwd(const Geo& g, const float* x, const float* w, float* y, int64_t ycs, const float* bias,
                       int relu, float* ws, cudaStream_t st);
// dw (o, k, k, d) = sum over pixels of dy x lowered(x); dy in layout g.yl
cudaError_t gather_wgrad(const Geo& g, const float* x, const float* dy, float* dw, float* ws, cudaStream_t st);

}  // namespace cct
