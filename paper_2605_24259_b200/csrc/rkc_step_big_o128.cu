// rkc_step_big_o128.cu -- the step kernels (rkc_step_impl.cuh) for pools of more than 1024 blocks (block words streamed)
// with at most 128 object slots.
#define RKC_OMAX 128
#define RKC_BIG 1
#define RKC_STEP_NS big_o128
#include "rkc_step_impl.cuh"
