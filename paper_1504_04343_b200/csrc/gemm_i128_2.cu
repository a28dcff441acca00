// gemm_i128_2.cu -- kernel variants of tile width 128, CTA group 2 (see gemm_kernel.cuh)
#include "gemm_kernel.cuh"

CCT_GEMM_INSTANTIATE(128, 2)
