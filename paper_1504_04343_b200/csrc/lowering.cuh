// lowering.cuh -- HBM-bound data-side kernels of the three lowering types.
//
// Replace the reference's lower / lift (spec-only)
// and add their adjoints for the backward passes:
//   lower_t{1,2,3}   : x (NHWC)      -> Dhat   (row-major, rows x ld)
//   lift_t{1,2,3}    : Rhat          -> y (NCHW)         Type 2/3 sum k / k^2 taps
//   expand_t{1,2,3}  : dy (NCHW)     -> dRhat^T (column-major: [col][ldr]) adjoint of lift
//   col2im_t{1,2}    : dDhat         -> dx (NHWC)        adjoint of lower (gather form)
//   crop_t3          : dXp (padded)  -> dx
// Row order of a lowered matrix is described by RowMap: row(q, y, c) =
// q*rpi + y*sr + c*sc, which covers both the SPEC order (c*m + r) and the
// internal row-major order.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace cct {

struct Geo {
    int64_t b, n, d, k, o, s, p;
    int64_t m, R, N;  // output side, touched padded extent, padded side
    int64_t yl = 0;   // layout of y / dy: 0 NCHW (OutputBatch), 1 NHWC
};

struct RowMap {
    int64_t rpi, sr, sc;  // rows per image, stride of y (row) and c (col) index
    int64_t ny, nc;       // extents of y and c covered (rows outside are zero / absent)
};

// which lowered matrix a RowMap describes
RowMap rowmap_internal(const Geo& g, int type);
RowMap rowmap_spec(const Geo& g, int type);  // s = 1, p = 0 only

int64_t lowered_cols(const Geo& g, int type);   // k^2 d, k d, d
int64_t lowered_ncols(const Geo& g, int type);  // Khat columns: o, k o, k^2 o

cudaError_t lower(const Geo& g, int type, const RowMap& rm, const float* x, float* dhat, int64_t ld,
                  cudaStream_t st);
// Rhat element (row, col) at rhat[row*rs + col*cs]
cudaError_t lift(const Geo& g, int type, const RowMap& rm, const float* rhat, int64_t rs, int64_t cs,
                 float* y, cudaStream_t st);
// dRhat^T[col*ldr + row], internal row order, zero where lift does not read
cudaError_t expand(const Geo& g, int type, const float* dy, float* drt, int64_t ldr, cudaStream_t st);
// Small-channel Type 1 (d % 4 != 0, e.g. conv1): dDhat is produced slab-major --
// slab (q, r, i) = rows (q, r, 0..m-1) x columns [i k d, (i+1) k d), contiguous,
// slab stride slab_stride(g) floats -- so col2im stages whole slabs.
bool col2im_slab_layout(const Geo& g, int type);
int64_t slab_stride(const Geo& g);
// dx from dDhat (internal order, row-major with ld -- or slab-major with ld = slab
// stride when col2im_slab_layout); type 3 = crop of dXp
cudaError_t col2im(const Geo& g, int type, const float* dd, int64_t ld, float* dx, cudaStream_t st);
// dst[r*ld_dst + c] = src[r*ld_src + c] for c < cols, 0 for cols <= c < ld_dst
cudaError_t pad_rows(const float* src, int64_t rows, int64_t cols, int64_t ld_src, float* dst,
                     int64_t ld_dst, cudaStream_t st);
// dst[c*ld_dst + r] = src[r*ld_src + c]  (rows x cols -> cols x rows)
cudaError_t transpose(const float* src, int64_t rows, int64_t cols, int64_t ld_src, float* dst,
                      int64_t ld_dst, cudaStream_t st);

// batched: dst[z*dst_z + c*ldd + r] = src[z*src_z + r*lds + c] for z < nz (strides may be
// negative); `phase` = the profiling phase the copy is accounted to
cudaError_t transpose_batched(const float* src, int64_t rows, int64_t cols, int64_t lds, int64_t src_z, float* dst,
                              int64_t ldd, int64_t dst_z, int64_t nz, int phase, cudaStream_t st);

// ---- Type 2 / 3 streaming kernels (lowering23.cu) ----------------------------------
// Rhat plane-major: Rhat[((q * ncols) + col) * rpi + prow] (the forward GEMM's output map)
bool planes_ok(const Geo& g, int type);
cudaError_t lift_planes(const Geo& g, int type, const float* rhat, float* y, cudaStream_t st);
// dy -> dRhat^T[col * ldr + row] (internal row order), zero rows ldr tail included
cudaError_t expand_planes(const Geo& g, int type, const float* dy, float* drt, int64_t ldr, cudaStream_t st);
// Dhat2 / Dhat3 in internal row order from whole padded input rows (d % 4 == 0)
bool lower_rows_ok(const Geo& g, int type, const float* x, const float* dh, int64_t ld);
cudaError_t lower_rows(const Geo& g, int type, const float* x, float* dhat, int64_t ld, cudaStream_t st);

}  // namespace cct
