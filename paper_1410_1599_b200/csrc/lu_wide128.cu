// lu_wide128.cu -- the kernels of lu.cu for L = 128 limbs (wide format, limb loops
// instead of full unrolling: mp_arith.cuh MPG_UNROLL); one limb count per translation unit.
#define MPG_WIDE 1
#define MPG_WIDE_L 128
#include "lu.cu"
