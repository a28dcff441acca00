// gemm_i384_1.cu -- kernel variants of tile width 384, CTA group 1 (see gemm_kernel.cuh)
#include "gemm_kernel.cuh"

CCT_GEMM_INSTANTIATE(384, 1)
