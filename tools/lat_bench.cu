// FP64 / shuffle latency microbenchmark (one warp, dependent chains, clock64).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double a, double b) {
  double x = a;
  long long t0, t1;
  const int N = 1024;
  // DFMA chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = fma(x, b, a);
  t1 = clock64();
  cyc[0] = t1 - t0;
  // DADD chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x + b;
  t1 = clock64();
  cyc[1] = t1 - t0;
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < 64; ++i) x = sqrt(x + 1.0);
  t1 = clock64();
  cyc[2] = t1 - t0;
  // div chain
  t0 = clock64();
  for (int i = 0; i < 64; ++i) x = b / (x + 1.0);
  t1 = clock64();
  cyc[3] = t1 - t0;
  // rsqrt chain
  t0 = clock64();
  for (int i = 0; i < 64; ++i) x = rsqrt(x + 1.0);
  t1 = clock64();
  cyc[4] = t1 - t0;
  // shfl (double) chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < 256; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 0.0;
  t1 = clock64();
  cyc[5] = t1 - t0;
  // FFMA chain (float)
  float y = (float)a, fb = (float)b;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) y = fmaf(y, fb, (float)a);
  t1 = clock64();
  cyc[6] = t1 - t0;
  out[threadIdx.x] = x + y;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 64 * sizeof(double));
  cudaMallocManaged(&c, 16 * sizeof(long long));
  lat<<<1, 32>>>(o, c, 0.5, 0.999);
  cudaDeviceSynchronize();
  lat<<<1, 32>>>(o, c, 0.5, 0.999);
  cudaDeviceSynchronize();
  printf("DFMA %.1f  DADD %.1f  sqrt %.1f  div %.1f  rsqrt %.1f  shfl+dadd %.1f  FFMA %.1f cycles\n", c[0] / 1024.0,
         c[1] / 1024.0, c[2] / 64.0, c[3] / 64.0, c[4] / 64.0, c[5] / 256.0, c[6] / 1024.0);
  return 0;
}
