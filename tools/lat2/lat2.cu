// latency microbenchmark: dependent chains of the primitives the Jacobi
// rotation parameters use (one thread; cycles per link)
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rsq_approx(double x) {
  double y;
  asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ double rcp_approx(double x) {
  double y;
  asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ double rj_rsqrt(double x) {
  double y = rsq_approx(x);
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y * fma(-h * y, y, 1.5);
}
__global__ void k(double* out, long long* cyc, double x0, int n) {
  double x = x0;
  float f = (float)x0;
  long long t0, t1;
#define BENCH(slot, body)            \
  x = x0; f = (float)x0;             \
  t0 = clock64();                    \
  for (int i = 0; i < n; ++i) { body; } \
  t1 = clock64();                    \
  cyc[slot] = t1 - t0; out[slot] = x + f;
  BENCH(0, x = fma(x, 1.0000001, 1e-9))
  BENCH(1, x = rsq_approx(x) + 0.5)
  BENCH(2, x = rj_rsqrt(x) + 0.5)
  BENCH(3, x = sqrt(x) + 0.5)
  BENCH(4, x = 1.0 / (x + 1.0) + 0.5)
  BENCH(5, f = sqrtf(f) + 0.5f)
  BENCH(6, f = 1.0f / (f + 1.0f) + 0.5f)
  BENCH(7, f = __fdividef(1.0f, f + 1.0f) + 0.5f)
  BENCH(8, f = __frsqrt_rn(f) + 0.5f)
  BENCH(9, x = (double)(float)x + 0.5)
  BENCH(10, x = rcp_approx(x) + 0.5)
  BENCH(11, f = rsqrtf(f) + 0.5f)
  BENCH(12, x = __shfl_xor_sync(0xffffffffu, x, 1) + 0.5)
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 64 * 8); cudaMalloc(&c, 64 * 8);
  const int n = 1000;
  k<<<1, 32>>>(o, c, 1.7, n);
  k<<<1, 32>>>(o, c, 1.7, n);
  long long h[16];
  cudaMemcpy(h, c, 13 * 8, cudaMemcpyDeviceToHost);
  const char* nm[] = {"dfma", "rsqrt.approx.f64", "rj_rsqrt (3 Newton)", "sqrt f64", "div f64", "sqrtf", "divf",
                      "__fdividef", "__frsqrt_rn", "cvt f64->f32->f64", "rcp.approx.f64", "rsqrtf", "shfl f64"};
  for (int i = 0; i < 13; ++i) printf("%-22s %.1f cycles/link\n", nm[i], (double)h[i] / n);
  return 0;
}
