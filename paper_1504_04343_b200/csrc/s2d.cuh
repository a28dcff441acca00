// s2d.cuh -- space-to-depth form of a strided Type 1 layer.
//
// A stride-s convolution (k x k taps, pad p, depth d) equals a stride-1, unpadded
// convolution of the blocked input
//     X'[q][u][v][(a s + b) d + c] = Xp[q][s u + a][s v + b][c]      (a, b < s)
// with the blocked kernel bank
//     W'[o][i'][j'][(a s + b) d + c] = W[o][s i' + a][s j' + b][c]   (0 outside k)
// of k' = ceil(k / s) taps and depth s^2 d, on an input of side n' = m + k' - 1
// (Xp = x zero-padded by p; rows / columns past the padded input read as 0).
// The output y is unchanged.  CaffeNet conv1 (k 11, s 4, d 3) becomes a 3 x 3
// convolution of depth 48: an implicit (TMA im2col) Type 1 GEMM with K = 432
// instead of a materialised 1.1 GB Dhat, and a stride-1 backward.
// The adjoints gather dx from dX' and dW from dW' (rows / taps no output touches
// get 0).  All four kernels are HBM-bound gathers (one thread per output element,
// output-coalesced).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

#include "lowering.cuh"

namespace cct {

// the stride-1 layer on X' (n', k', s^2 d, o, s = 1, p = 0; same m)
Geo s2d_geo(const Geo& g);

// X' from x (NHWC, b x n x n x d); X' is b x n' x n' x s^2 d
cudaError_t s2d_input(const Geo& g, const float* x, float* xs, cudaStream_t st);
// W' (o x k' x k' x s^2 d) from W (o x k x k x d)
cudaError_t s2d_weights(const Geo& g, const float* w, float* ws, cudaStream_t st);
// dx (b x n x n x d) from dX' (b x n' x n' x s^2 d)
cudaError_t d2s_input(const Geo& g, const float* dxs, float* dx, cudaStream_t st);
// dW (o x k x k x d) from dW' (o x k' x k' x s^2 d)
cudaError_t d2s_weights(const Geo& g, const float* dws, float* dw, cudaStream_t st);

}  // namespace cct
