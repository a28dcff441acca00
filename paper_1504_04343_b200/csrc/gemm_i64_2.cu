// gemm_i64_2.cu -- kernel variants of tile width 64, CTA group 2 (see gemm_kernel.cuh)
#include "gemm_kernel.cuh"

CCT_GEMM_INSTANTIATE(64, 2)
