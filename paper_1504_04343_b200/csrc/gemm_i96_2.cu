// gemm_i96_2.cu -- kernel variants of tile width 96, CTA group 2 (see gemm_kernel.cuh)
#include "gemm_kernel.cuh"

CCT_GEMM_INSTANTIATE(96, 2)
