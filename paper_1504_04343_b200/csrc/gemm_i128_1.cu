// gemm_i128_1.cu -- kernel variants of tile width 128, CTA group 1 (see gemm_kernel.cuh)
#include "gemm_kernel.cuh"

CCT_GEMM_INSTANTIATE(128, 1)
