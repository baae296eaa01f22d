// rkc_step_small_o128.cu -- the step kernels (rkc_step_impl.cuh) for pools of at most 1024 blocks (keys staged in shared memory)
// with at most 128 object slots.
#define RKC_OMAX 128
#define RKC_BIG 0
#define RKC_STEP_NS small_o128
#include "rkc_step_impl.cuh"
