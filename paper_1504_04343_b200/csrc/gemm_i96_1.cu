// gemm_i96_1.cu -- kernel variants of tile width 96, CTA group 1 (see gemm_kernel.cuh)
#include "gemm_kernel.cuh"

CCT_GEMM_INSTANTIATE(96, 1)
