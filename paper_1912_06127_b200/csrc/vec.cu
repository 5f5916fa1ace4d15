// Elementwise helpers: diag(V) scalings (inverse-singular-value merge,
// PAPER.md:361-365), copies, deterministic reductions.
#include "common.cuh"
#include "kernels.h"

#include <map>
#include <mutex>
#include <utility>

namespace {

inline int grid_for(long long n, int tpb = 256) {
  long long b = (n + tpb - 1) / tpb;
  return (int)std::max<long long>(1, std::min<long long>(b, 8LL * g_num_sms));
}

__global__ void scale_rows_kernel(cplx* out, const cplx* __restrict__ in, const double* __restrict__ v, int rows,
                                  long long cols) {
  const long long n = rows * cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / cols;
    out[e] = cscale(in[e], v[r]);
  }
}

__global__ void scale_cols_kernel(cplx* out, const cplx* __restrict__ in, const double* __restrict__ v,
                                  long long rows, int cols) {
  const long long n = rows * cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e % cols);
    out[e] = cscale(in[e], v[c]);
  }
}

__global__ void copy_kernel(cplx* dst, const cplx* __restrict__ src, long long n) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    dst[e] = src[e];
}

__global__ void fill_kernel(cplx* dst, cplx v, long long n) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    dst[e] = v;
}

// block partial sums of x*y, last block reduces partials in block order
__global__ void sum_products_kernel(const cplx* __restrict__ x, const cplx* __restrict__ y, long long n, cplx* result,
                                    double* partials, unsigned* counter) {
  __shared__ double sr[32], si[32];
  __shared__ bool last;
  double ar = 0, ai = 0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const cplx p = cmul(x[e], y[e]);
    ar += p.x;
    ai += p.y;
  }
  ar = warp_sum(ar);
  ai = warp_sum(ai);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { sr[wid] = ar; si[wid] = ai; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tr = 0, tq = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { tr += sr[w]; tq += si[w]; }
    partials[2 * blockIdx.x] = tr;
    partials[2 * blockIdx.x + 1] = tq;
    __threadfence();
    const unsigned t = atomicAdd(counter, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double tr = 0, tq = 0;
    for (int b = 0; b < (int)gridDim.x; ++b) {
      tr += ((volatile double*)partials)[2 * b];
      tq += ((volatile double*)partials)[2 * b + 1];
    }
    *result = cmk(tr, tq);
    *counter = 0u;
  }
}

__global__ void nonfinite_kernel(const cplx* __restrict__ x, long long n, int* flag) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const cplx v = x[e];
    if (!isfinite(v.x) || !isfinite(v.y)) { *flag = 1; }
  }
}

}  // namespace

cudaError_t scale_rows(cudaStream_t st, cplx* out, const cplx* in, const double* v, int rows, long long cols) {
  const long long n = rows * cols;
  if (n <= 0) return cudaSuccess;
  scale_rows_kernel<<<grid_for(n), 256, 0, st>>>(out, in, v, rows, cols);
  return cudaGetLastError();
}
cudaError_t scale_cols(cudaStream_t st, cplx* out, const cplx* in, const double* v, long long rows, int cols) {
  const long long n = rows * cols;
  if (n <= 0) return cudaSuccess;
  scale_cols_kernel<<<grid_for(n), 256, 0, st>>>(out, in, v, rows, cols);
  return cudaGetLastError();
}
cudaError_t copy_cplx(cudaStream_t st, cplx* dst, const cplx* src, long long n) {
  if (n <= 0) return cudaSuccess;
  copy_kernel<<<grid_for(n), 256, 0, st>>>(dst, src, n);
  return cudaGetLastError();
}
cudaError_t fill_cplx(cudaStream_t st, cplx* dst, cplx v, long long n) {
  if (n <= 0) return cudaSuccess;
  fill_kernel<<<grid_for(n), 256, 0, st>>>(dst, v, n);
  return cudaGetLastError();
}
cudaError_t sum_products(cudaStream_t st, const cplx* x, const cplx* y, long long n, cplx* result, double* partials,
                         unsigned* counter) {
  const int nb = (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, 2LL * g_num_sms));
  sum_products_kernel<<<nb, 256, 0, st>>>(x, y, n, result, partials, counter);
  return cudaGetLastError();
}
cudaError_t any_nonfinite(cudaStream_t st, const cplx* x, long long n, int* flag) {
  if (n <= 0) return cudaSuccess;
  nonfinite_kernel<<<grid_for(n), 256, 0, st>>>(x, n, flag);
  return cudaGetLastError();
}

cudaError_t set_smem_attr(const void* fn, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  // lock-free fast path: a small per-thread cache of (device, kernel) -> bytes already opted in
  struct Ent { int dev; const void* fn; int bytes; };
  static thread_local Ent cache[32];
  static thread_local int ncache = 0;
  for (int i = 0; i < ncache; ++i)
    if (cache[i].fn == fn && cache[i].dev == dev && cache[i].bytes >= bytes) return cudaSuccess;
  std::lock_guard<std::mutex> lk(mu);
  auto remember = [&](int b) {
    if (ncache < 32) cache[ncache++] = Ent{dev, fn, b};
  };
  auto key = std::make_pair(dev, fn);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) {
    remember(it->second);
    return cudaSuccess;
  }
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) {
    done[key] = bytes;
    remember(bytes);
  }
  return e;
}

cudaError_t set_cluster_nonportable(const void* fn) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(dev, fn);
  if (done.count(key)) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e == cudaSuccess) done[key] = 1;
  return e;
}
