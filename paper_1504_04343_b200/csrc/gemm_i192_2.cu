// gemm_i192_2.cu -- kernel variants of tile width 192, CTA group 2 (see gemm_kernel.cuh)
#include "gemm_kernel.cuh"

CCT_GEMM_INSTANTIATE(192, 2)
