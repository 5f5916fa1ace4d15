// Measures the cost of a grid-wide barrier on B200: cooperative-groups
// grid.sync() vs a sense-reversing atomic barrier (one arrival per CTA).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, int* sink) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) *sink = iters;
}

__device__ __forceinline__ void my_barrier(unsigned* count, volatile unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g0 = *gen;
    __threadfence();
    const unsigned arrived = atomicAdd(count, 1u);
    if (arrived == nblocks - 1) {
      *count = 0;
      __threadfence();
      atomicAdd((unsigned*)gen, 1u);
    } else {
      while (*gen == g0) { __nanosleep(20); }
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void k_my(int iters, unsigned* count, unsigned* gen) {
  for (int i = 0; i < iters; ++i) my_barrier(count, gen, gridDim.x);
}

int main() {
  int* sink; unsigned* cnt; unsigned* gen;
  cudaMalloc(&sink, 4); cudaMalloc(&cnt, 4); cudaMalloc(&gen, 4);
  cudaMemset(cnt, 0, 4); cudaMemset(gen, 0, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int grid : {4, 16, 32, 64, 128, 148}) {
    for (int nth : {128, 256}) {
      int iters = 2000;
      void* args[] = {&iters, &sink};
      cudaLaunchCooperativeKernel((void*)k_cg, grid, nth, args, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_cg, grid, nth, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      void* args2[] = {&iters, &cnt, &gen};
      cudaLaunchCooperativeKernel((void*)k_my, grid, nth, args2, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_my, grid, nth, args2, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms2; cudaEventElapsedTime(&ms2, a, b);
      printf("grid %3d nth %3d  cg.sync %.3f us   atomic barrier %.3f us  (%s)\n", grid, nth, ms * 1e3 / iters,
             ms2 * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
