// cluster barrier + DSMEM fetch latency for cluster sizes 2..16 (B200)
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void k(long long* out, int n, int mode) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double v[32];
  __shared__ double got[16];
  const int C = cl.num_blocks(), tid = threadIdx.x;
  if (tid < 32) v[tid] = tid;
  cl.sync();
  long long t0 = clock64();
  double acc = 0;
  for (int i = 0; i < n; ++i) {
    if (mode >= 1) {
      if (tid < 32) v[tid] = acc + i;
      __syncthreads();
    }
    cl.sync();
    if (mode >= 2) {
      if (tid < C) got[tid] = *cl.map_shared_rank(&v[i & 31], tid);
      __syncthreads();
      acc += got[(i + 1) % C];
    }
  }
  long long t1 = clock64();
  if (tid == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = (long long)acc; }
}
int main() {
  long long* o; cudaMalloc(&o, 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int C : {2, 4, 8, 16})
    for (int mode = 0; mode < 3; ++mode) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      cfg.gridDim = dim3(C); cfg.blockDim = dim3(256);
      at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      const int n = 2000;
      cudaLaunchKernelEx(&cfg, k, o, n, mode);
      cudaLaunchKernelEx(&cfg, k, o, n, mode);
      long long h[2]; cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
      printf("C=%2d mode=%d (%s): %.0f cycles/iter  %s\n", C, mode, mode == 0 ? "cluster.sync" : mode == 1 ? "+smem write+syncthreads" : "+DSMEM fetch of C values+syncthreads", (double)h[0] / n, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
