// gemm_i192_1.cu -- kernel variants of tile width 192, CTA group 1 (see gemm_kernel.cuh)
#include "gemm_kernel.cuh"

CCT_GEMM_INSTANTIATE(192, 1)
