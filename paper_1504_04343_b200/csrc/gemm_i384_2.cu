// gemm_i384_2.cu -- kernel variants of tile width 384, CTA group 2 (see gemm_kernel.cuh)
#include "gemm_kernel.cuh"

CCT_GEMM_INSTANTIATE(384, 2)
