// reduce.cuh -- deterministic split-K reduction (fixed ascending split order).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace cct {

// out[r*ld_out + c] = sum_{s<splits} part[s*split_stride + r*ld_in + c]   (r<rows, c<cols)
cudaError_t splitk_reduce(const float* part, int64_t split_stride, int splits, int64_t rows,
                          int64_t cols, int64_t ld_in, float* out, int64_t ld_out, cudaStream_t st);

}  // namespace cct
