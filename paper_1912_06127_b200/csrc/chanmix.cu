// Sparse MPO-channel contraction (the W_j / W_{j+1} stages of H_eff and the
// environment updates).  The MPO tensors are sparse finite-state machines
// (nnz(W) = 12 of 100 entries for nearest-neighbour XXZ), so this stage is an
// HBM-bound gather/FMA over the (chi x chi) plane, not a GEMM: one thread per
// (outer, inner) point loops over all output channels; consecutive threads
// walk the contiguous inner index so every load/store is coalesced.
#include <mutex>
#include "common.cuh"
#include "kernels.h"

namespace {

constexpr int TPB = 128;

__global__ void __launch_bounds__(TPB) chanmix_kernel(ChanMix cm, int n_inner, const cplx* __restrict__ in,
                                                      long long so_in, long long si_in, Strides3 ich,
                                                      cplx* __restrict__ out, long long so_out, long long si_out,
                                                      Strides3 och, const double* skip) {
  if (skip != nullptr && *skip != 0.0) return;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  // stage the (small) sparse tables in shared memory
  cplx* s_coef = reinterpret_cast<cplx*>(sm_raw);
  long long* s_ioff = reinterpret_cast<long long*>(s_coef + cm.nnz);
  long long* s_ooff = s_ioff + cm.nnz;
  int* s_row = reinterpret_cast<int*>(s_ooff + cm.n_oc);
  for (int e = threadIdx.x; e < cm.nnz; e += TPB) {
    s_coef[e] = cm.coef[e];
    const int4 c = cm.ic_idx[e];
    s_ioff[e] = c.x * ich.s0 + c.y * ich.s1 + c.z * ich.s2;
  }
  for (int q = threadIdx.x; q < cm.n_oc; q += TPB) {
    const int4 c = cm.oc_idx[q];
    s_ooff[q] = c.x * och.s0 + c.y * och.s1 + c.z * och.s2;
  }
  for (int q = threadIdx.x; q <= cm.n_oc; q += TPB) s_row[q] = cm.rowptr[q];
  __syncthreads();

  const int i = blockIdx.x * TPB + threadIdx.x;
  if (i >= n_inner) return;
  const long long o = blockIdx.y;
  const cplx* src = in + o * so_in + i * si_in;
  cplx* dst = out + o * so_out + i * si_out;
  for (int q = 0; q < cm.n_oc; ++q) {
    cplx acc = cmk(0.0, 0.0);
    const int e1 = s_row[q + 1];
    for (int e = s_row[q]; e < e1; ++e) cfma(acc, s_coef[e], __ldg(src + s_ioff[e]));
    dst[s_ooff[q]] = acc;
  }
}

// Gather variant (n_ic <= GMAX distinct input channels): every thread first
// issues the loads of all its distinct input channels (independent, in flight
// together: one memory latency instead of one per sparse entry), parks them in
// shared memory, then forms the output channels from the CSR rows.
constexpr int GMAX = 32, GCH = 16;
__global__ void __launch_bounds__(TPB) chanmix_gather_kernel(ChanMix cm, int n_inner, const cplx* __restrict__ in,
                                                             long long so_in, long long si_in, Strides3 ich,
                                                             cplx* __restrict__ out, long long so_out, long long si_out,
                                                             Strides3 och, const double* skip) {
  if (skip != nullptr && *skip != 0.0) return;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  cplx* s_val = reinterpret_cast<cplx*>(sm_raw);          // [n_ic][TPB]
  cplx* s_coef = s_val + (size_t)cm.n_ic * TPB;           // [nnz]
  long long* s_icoff = reinterpret_cast<long long*>(s_coef + cm.nnz);  // [n_ic]
  long long* s_ooff = s_icoff + cm.n_ic;                  // [n_oc]
  int* s_slot = reinterpret_cast<int*>(s_ooff + cm.n_oc);  // [nnz]
  int* s_row = s_slot + cm.nnz;                            // [n_oc + 1]
  for (int e = threadIdx.x; e < cm.nnz; e += TPB) {
    s_coef[e] = cm.coef[e];
    s_slot[e] = cm.slot[e];
  }
  for (int k = threadIdx.x; k < cm.n_ic; k += TPB) {
    const int4 c = cm.icu_idx[k];
    s_icoff[k] = c.x * ich.s0 + c.y * ich.s1 + c.z * ich.s2;
  }
  for (int q = threadIdx.x; q < cm.n_oc; q += TPB) {
    const int4 c = cm.oc_idx[q];
    s_ooff[q] = c.x * och.s0 + c.y * och.s1 + c.z * och.s2;
  }
  for (int q = threadIdx.x; q <= cm.n_oc; q += TPB) s_row[q] = cm.rowptr[q];
  __syncthreads();
  const int i = blockIdx.x * TPB + threadIdx.x;
  const bool valid = i < n_inner;
  const long long o = blockIdx.y;
  const cplx* src = in + o * so_in + (long long)(valid ? i : 0) * si_in;
  for (int k0 = 0; k0 < cm.n_ic; k0 += GCH) {
    cplx v[GCH];
#pragma unroll
    for (int k = 0; k < GCH; ++k)
      if (valid && k0 + k < cm.n_ic) v[k] = __ldg(src + s_icoff[k0 + k]);
#pragma unroll
    for (int k = 0; k < GCH; ++k)
      if (k0 + k < cm.n_ic) s_val[(size_t)(k0 + k) * TPB + threadIdx.x] = v[k];
  }
  if (!valid) return;  // each thread reads only its own s_val column: no barrier needed
  cplx* dst = out + o * so_out + (long long)i * si_out;
  for (int q = 0; q < cm.n_oc; ++q) {
    cplx acc = cmk(0.0, 0.0);
    const int e1 = s_row[q + 1];
    for (int e = s_row[q]; e < e1; ++e) cfma(acc, s_coef[e], s_val[(size_t)s_slot[e] * TPB + threadIdx.x]);
    dst[s_ooff[q]] = acc;
  }
}

std::mutex& gmu() {
  static std::mutex m;
  return m;
}

}  // namespace

cudaError_t chanmix(cudaStream_t st, const ChanMix& cm, int n_outer, int n_inner, const cplx* in, long long so_in,
                    long long si_in, Strides3 in_ch, cplx* out, long long so_out, long long si_out,
                    Strides3 out_ch, const double* skip) {
  if (n_outer <= 0 || n_inner <= 0) return cudaSuccess;
  if (cm.n_ic > 0 && cm.n_ic <= GMAX && cm.slot != nullptr) {
    const size_t smg = (size_t)cm.n_ic * TPB * sizeof(cplx) + (size_t)cm.nnz * (sizeof(cplx) + sizeof(int)) +
                       (size_t)(cm.n_ic + cm.n_oc) * sizeof(long long) + (size_t)(cm.n_oc + 1) * sizeof(int);
    cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(chanmix_gather_kernel), 100 * 1024);
    if (e != cudaSuccess) return e;
    if (smg <= 100 * 1024) {
      dim3 grid((n_inner + TPB - 1) / TPB, n_outer);
      chanmix_gather_kernel<<<grid, TPB, smg, st>>>(cm, n_inner, in, so_in, si_in, in_ch, out, so_out, si_out,
                                                    out_ch, skip);
      return cudaGetLastError();
    }
  }
  const size_t sm = (size_t)cm.nnz * (sizeof(cplx) + sizeof(long long)) + (size_t)cm.n_oc * sizeof(long long) +
                    (size_t)(cm.n_oc + 1) * sizeof(int);
  if (sm > 48 * 1024) {
    cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(chanmix_kernel), (int)sm);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((n_inner + TPB - 1) / TPB, n_outer);
  chanmix_kernel<<<grid, TPB, sm, st>>>(cm, n_inner, in, so_in, si_in, in_ch, out, so_out, si_out, out_ch, skip);
  return cudaGetLastError();
}
