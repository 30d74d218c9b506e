// lu_wide64.cu -- the kernels of lu.cu for L = 64 limbs (wide format, limb loops
// instead of full unrolling: mp_arith.cuh MPG_UNROLL); one limb count per translation unit.
#define MPG_WIDE 1
#define MPG_WIDE_L 64
#include "lu.cu"
