// epilogue.cuh -- the layer epilogue around a convolution: bias + ReLU forward
// and its backward (the adjacent steps either side of a conv
// layer in CaffeNet).  The forward is fused into the GEMM epilogue (OutMap::bias /
// relu) whenever the GEMM writes y directly (Type 1, unsplit); these kernels cover
// the remaining paths and the backward.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace cct {

// y (b, o, mm) NCHW in place: y = act(y + bias[j]) for channels j < o of each image,
// images `ostride` planes apart (ostride > o: one channel group of a wider y);
// bias may be null
cudaError_t bias_act(float* y, const float* bias, int relu, int64_t b, int64_t o, int64_t mm, int64_t ostride,
                     cudaStream_t st);

// dz = relu ? (y > 0 ? dy : 0) : dy  (y = the layer's post-activation output), and
// the bias gradient db[j] = sum over (q, pixels) of dz, deterministic (per-plane
// block sums, then a fixed-order sum over images).  dz may alias dy only when
// relu == 0 (then nothing is written); db may be null.  partial: b * o floats.
cudaError_t relu_bias_bwd(const float* dy, const float* y, float* dz, float* db, float* partial, int relu, int64_t b,
                          int64_t o, int64_t mm, cudaStream_t st);

// strided copies for channel groups (cudaMemcpy2DAsync on the stream)
cudaError_t copy2d(float* dst, int64_t dpitch, const float* src, int64_t spitch, int64_t width, int64_t rows,
                   cudaStream_t st);

}  // namespace cct
