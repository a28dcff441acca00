// gemm_i256_1.cu -- kernel variants of tile width 256, CTA group 1 (see gemm_kernel.cuh)
#include "gemm_kernel.cuh"

CCT_GEMM_INSTANTIATE(256, 1)
