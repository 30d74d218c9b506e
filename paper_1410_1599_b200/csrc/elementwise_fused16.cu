// elementwise_fused16.cu -- the fused two-level pre-/post-addition kernels (elementwise.cu
// preadd2_kernel / postadd2_kernel) for one group of limb counts, as their own translation unit
// so that they compile beside elementwise.cu.
#define MPG_EW_PART 2
#include "elementwise.cu"
