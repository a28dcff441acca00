// gemm_i256_2.cu -- kernel variants of tile width 256, CTA group 2 (see gemm_kernel.cuh)
#include "gemm_kernel.cuh"

CCT_GEMM_INSTANTIATE(256, 2)
