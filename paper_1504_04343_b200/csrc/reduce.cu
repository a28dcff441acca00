// reduce.cu -- deterministic split-K reduction for the backward-weight GEMMs.
// Each output element sums its split partials in ascending split order, so the
// result is run-to-run bit-identical (no atomics).
#include "common.cuh"
#include "reduce.cuh"

namespace cct {

namespace {
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int64_t sstride, int splits,
                                     int64_t rows, int64_t cols, int64_t ldi, float* __restrict__ out,
                                     int64_t ldo) {
    const int64_t total = rows * cols;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / cols, c = e - r * cols;
        const float* p = part + r * ldi + c;
        float acc = 0.f;
        for (int s = 0; s < splits; ++s) acc += p[int64_t(s) * sstride];
        out[r * ldo + c] = acc;
    }
}
}  // namespace

cudaError_t splitk_reduce(const float* part, int64_t split_stride, int splits, int64_t rows,
                          int64_t cols, int64_t ld_in, float* out, int64_t ld_out, cudaStream_t st) {
    const int threads = 256;
    PhaseScope ps(kPhaseReduce, st, 0, 4.0 * double(rows * cols) * double(splits + 1));
    splitk_reduce_kernel<<<grid_for(rows * cols, threads), threads, 0, st>>>(
        part, split_stride, splits, rows, cols, ld_in, out, ld_out);
    note_launch();
    return cudaGetLastError();
}

}  // namespace cct
