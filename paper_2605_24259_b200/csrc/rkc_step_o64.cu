// rkc_step_o64.cu -- the step kernels (rkc_step_impl.cuh) for pools with at
// most 64 object slots: 6 KB of warp state, 32 resident CTAs per SM.
#define RKC_OMAX 64
#define RKC_STEP_NS o64
#include "rkc_step_impl.cuh"
