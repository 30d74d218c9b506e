// gemm_wide.cu -- the kernels of gemm.cu for the wide formats (L = 64, 128, 256, 288
// limbs: up to 9216 bits), compiled with limb loops instead of full unrolling
// (mp_arith.cuh MPG_UNROLL); mantissas live in local memory.
#define MPG_WIDE 1
#include "gemm.cu"
