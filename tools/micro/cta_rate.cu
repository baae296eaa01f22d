// CTA launch-rate microbenchmark (B200): how many CTAs per microsecond the
// hardware dispatches for trivially short CTAs of 1..8 warps.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void empty_kernel(int* sink) {
  if (threadIdx.x == 0 && blockIdx.x == 0x7FFFFFFF) sink[0] = 1;
}
// a CTA that does ~1 us of dependent work (a trace-step-like latency chain)
__global__ void short_kernel(int* sink, int iters) {
  unsigned v = threadIdx.x;
  for (int i = 0; i < iters; ++i) v = v * 1664525u + 1013904223u;
  if (v == 0x12345678u) sink[0] = v;
}

int main() {
  int* sink;
  cudaMalloc(&sink, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int threads : {32, 64, 128, 256}) {
    for (int grid : {100000, 625000, 1000000}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        empty_kernel<<<grid, threads>>>(sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("empty  threads=%3d grid=%8d  %8.1f us  %.3f CTAs/ns\n", threads, grid, ms * 1e3, grid / (ms * 1e6));
      }
    }
  }
  for (int iters : {0, 100, 1000}) {
    for (int threads : {32, 64}) {
      int grid = 625000 * 32 / threads;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        short_kernel<<<grid, threads>>>(sink, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("short iters=%4d threads=%3d grid=%8d  %8.1f us  %.3f CTAs/ns\n", iters, threads, grid, ms * 1e3, grid / (ms * 1e6));
      }
    }
  }
  return 0;
}
