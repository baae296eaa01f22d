// rkc_step_o128.cu -- the step kernels (rkc_step_impl.cuh) for pools with up
// to 128 object slots (the ABI maximum): 6.5 KB of warp state, 30 CTAs per SM.
#define RKC_OMAX 128
#define RKC_STEP_NS o128
#include "rkc_step_impl.cuh"
