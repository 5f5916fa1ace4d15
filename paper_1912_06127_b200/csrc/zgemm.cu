// Complex-FP64 GEMM on the sm_100a FP64 tensor pipe (DMMA.8x8x4).
//
// tcgen05.mma has no f64 kind, so the FP64 tensor path on B200 is the
// warp-level mma.sync.m8n8k4.f64 (SASS DMMA).  One complex product is THREE
// real DMMAs (3M / Gauss: P1 = ar br, P2 = ai bi, P3 = (ar + ai)(br + bi);
// re = P1 - P2, im = P3 - P1 - P2; normwise stable, |error| <= ~3 eps |a||b|
// per product), 25% fewer tensor-pipe operations than the four-product form.
// Operands are staged through a 4-stage cp.async (LDGSTS) shared-memory
// pipeline; tiles are 64x64 complex per CTA of 8 warps (32x16 per warp), or
// 32x32 per CTA when 64x64 tiles would give
// fewer than two waves on the 148 SMs; deterministic split-K on top.  op(A), op(B) in {N, T, C, R(conj only)};
// everything is row-major.  Used for every dense contraction on the hot path
// (H_eff stages 1 and 4, H1, environment updates, Theta merge, measurement).
#include "common.cuh"
#include "kernels.h"

#include <atomic>

namespace {

constexpr int BK = 8, STAGES = 4, NT = 256;
constexpr int PA = BK + 4;   // [BM][PA]  k contiguous   (conflict-free fragment reads)
constexpr int PBT = BK + 4;  // [BN][PBT] k contiguous
// [BK][BM + 2] (m contiguous) and [BK][BN + 2] (n contiguous) for the other layouts

struct GemmArgs {
  int M, N, K;
  cplx alpha, beta;
  const cplx* A;
  long long lda, sA;
  const cplx* B;
  long long ldb, sB;
  cplx* C;
  long long ldc, sC;
  int ksplit, kchunk;
  cplx* work;  // split-K partials [batch*ksplit][M][N]
  const double* skip;  // != 0 on device: return at once (Lanczos converged, krylov_tol > 0)
  GemmMask mask;       // block-sparse operands: visit only the k-chunks both masks allow
};
constexpr int MAXKL = 1024;  // k-chunk list capacity (K <= 8192 with masks)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int OPA, int OPB, int BM, int BN>
__global__ void __launch_bounds__(NT, 2) zgemm_dmma_kernel(GemmArgs g) {
  if (g.skip != nullptr && *g.skip != 0.0) return;
  constexpr bool TA = (OPA == 1 || OPA == 2), CA = (OPA == 2 || OPA == 3);
  constexpr bool TB = (OPB == 1 || OPB == 2), CB = (OPB == 2 || OPB == 3);
  constexpr int PAT = BM + 2, PB = BN + 2;
  constexpr int MT = BM / 16, NTL = BN / 32;  // 8x8 sub-tiles per warp (2 x 4 warps)
  constexpr int A_ST = TA ? BK * PAT : BM * PA;
  constexpr int B_ST = TB ? BN * PBT : BK * PB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* sA = reinterpret_cast<cplx*>(smem_raw);
  cplx* sB = sA + STAGES * A_ST;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int z = blockIdx.z;
  const int batch = z / g.ksplit, split = z - batch * g.ksplit;
  const int kbeg = split * g.kchunk;
  const int kend = min(g.K, kbeg + g.kchunk);
  const cplx* A = g.A + batch * g.sA;
  const cplx* B = g.B + batch * g.sB;
  const int M = g.M, N = g.N;
  const long long lda = g.lda, ldb = g.ldb;

  auto load_tile = [&](int stage, int kt) {
    const int k0 = kbeg + kt * BK;
    cplx* a_dst = sA + stage * A_ST;
    cplx* b_dst = sB + stage * B_ST;
#pragma unroll
    for (int i = 0; i < (BM * BK) / NT; ++i) {
      const int c = tid + i * NT;
      if (!TA) {
        const int r = c >> 3, kk = c & 7;
        const int gm = m0 + r, gk = k0 + kk;
        const bool v = (gm < M) && (gk < kend);
        cp_async16(a_dst + r * PA + kk, v ? (const void*)(A + gm * lda + gk) : (const void*)A, v);
      } else {
        const int kr = c / BM, mm = c % BM;
        const int gm = m0 + mm, gk = k0 + kr;
        const bool v = (gm < M) && (gk < kend);
        cp_async16(a_dst + kr * PAT + mm, v ? (const void*)(A + gk * lda + gm) : (const void*)A, v);
      }
    }
#pragma unroll
    for (int i = 0; i < (BN * BK) / NT; ++i) {
      const int c = tid + i * NT;
      if (!TB) {
        const int kr = c / BN, nn = c % BN;
        const int gn = n0 + nn, gk = k0 + kr;
        const bool v = (gn < N) && (gk < kend);
        cp_async16(b_dst + kr * PB + nn, v ? (const void*)(B + gk * ldb + gn) : (const void*)B, v);
      } else {
        const int r = c >> 3, kk = c & 7;
        const int gn = n0 + r, gk = k0 + kk;
        const bool v = (gn < N) && (gk < kend);
        cp_async16(b_dst + r * PBT + kk, v ? (const void*)(B + gn * ldb + gk) : (const void*)B, v);
      }
    }
  };

  double acc1[MT][NTL][2], acc2[MT][NTL][2], acc3[MT][NTL][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NTL; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) acc1[i][j][h] = acc2[i][j][h] = acc3[i][j][h] = 0.0;

  // k-chunks to visit: all, or (block-sparse operands) those where this CTA's
  // rows of op(A) and columns of op(B) may both be nonzero, compacted in order
  __shared__ int s_kl[MAXKL];
  __shared__ int s_wcnt[NT / 32];
  const bool masked = g.mask.a != nullptr;
  int nk = (kend > kbeg) ? (kend - kbeg + BK - 1) / BK : 0;
  if (masked) {
    const int kc0 = kbeg / BK, nkc = nk;
    const int r0 = m0 / 32, r1 = min((M - 1) / 32, (m0 + BM - 1) / 32);
    const int c0 = n0 / 32, c1 = min((N - 1) / 32, (n0 + BN - 1) / 32);
    int cnt = 0;
    for (int base = 0; base < nkc; base += NT) {
      const int kc = kc0 + base + tid;
      bool on = false;
      if (base + tid < nkc) {
        bool a = false, b = false;
        for (int r = r0; r <= r1; ++r) a |= g.mask.a[(long long)r * g.mask.ldA + kc] != 0;
        for (int c = c0; c <= c1; ++c) b |= g.mask.b[(long long)kc * g.mask.ldB + c] != 0;
        on = a && b;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, on);
      if (lane == 0) s_wcnt[warp] = __popc(bal);
      __syncthreads();
      int off = cnt;
      for (int w = 0; w < warp; ++w) off += s_wcnt[w];
      if (on) s_kl[off + __popc(bal & ((1u << lane) - 1u))] = kc - kc0;
      int tot = 0;
      for (int w = 0; w < NT / 32; ++w) tot += s_wcnt[w];
      cnt += tot;
      __syncthreads();
    }
    nk = cnt;
  }
  auto kt_of = [&](int kt) { return masked ? s_kl[kt] : kt; };
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_tile(s, kt_of(s));
    cp_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nt = kt + STAGES - 1;
      if (nt < nk) load_tile(nt % STAGES, kt_of(nt));
      cp_commit();
    }
    const cplx* a_s = sA + (kt % STAGES) * A_ST;
    const cplx* b_s = sB + (kt % STAGES) * B_ST;
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      const int kq = ks + (lane & 3);
      cplx af[MT], bf[NTL];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int row = wm * (BM / 2) + mt * 8 + (lane >> 2);
        af[mt] = TA ? a_s[kq * PAT + row] : a_s[row * PA + kq];
        if (CA) af[mt].y = -af[mt].y;
      }
#pragma unroll
      for (int nt = 0; nt < NTL; ++nt) {
        const int col = wn * (BN / 4) + nt * 8 + (lane >> 2);
        bf[nt] = TB ? b_s[col * PBT + kq] : b_s[kq * PB + col];
        if (CB) bf[nt].y = -bf[nt].y;
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const double as = af[mt].x + af[mt].y;
#pragma unroll
        for (int nt = 0; nt < NTL; ++nt) {
          dmma(acc1[mt][nt][0], acc1[mt][nt][1], af[mt].x, bf[nt].x);
          dmma(acc2[mt][nt][0], acc2[mt][nt][1], af[mt].y, bf[nt].y);
          dmma(acc3[mt][nt][0], acc3[mt][nt][1], as, bf[nt].x + bf[nt].y);
        }
      }
    }
  }
  cp_wait<0>();

  // epilogue
  const bool partial = g.ksplit > 1;
  cplx* C = partial ? g.work + (long long)z * M * N : g.C + batch * g.sC;
  const long long ldc = partial ? (long long)N : g.ldc;
  const cplx alpha = g.alpha, beta = g.beta;
  const bool use_beta = (beta.x != 0.0 || beta.y != 0.0);
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int r = m0 + wm * (BM / 2) + mt * 8 + (lane >> 2);
    if (r >= M) continue;
#pragma unroll
    for (int nt = 0; nt < NTL; ++nt) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = n0 + wn * (BN / 4) + nt * 8 + 2 * (lane & 3) + h;
        if (c >= N) continue;
        const double p1 = acc1[mt][nt][h], p2 = acc2[mt][nt][h];
        cplx v = cmk(p1 - p2, acc3[mt][nt][h] - p1 - p2);
        cplx* p = C + r * ldc + c;
        if (partial) {
          *p = v;
        } else {
          cplx out = cmul(alpha, v);
          if (use_beta) out = cadd(out, cmul(beta, *p));
          *p = out;
        }
      }
    }
  }
}

__global__ void splitk_reduce_kernel(int M, int N, int ksplit, int batch, const cplx* __restrict__ work, cplx alpha,
                                     cplx beta, cplx* C, long long ldc, long long sC, const double* skip) {
  if (skip != nullptr && *skip != 0.0) return;
  const long long MN = (long long)M * N;
  const long long total = MN * batch;
  const bool use_beta = (beta.x != 0.0 || beta.y != 0.0);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / MN, rc = e - b * MN;
    const int r = (int)(rc / N), c = (int)(rc - (long long)r * N);
    cplx s = cmk(0, 0);
    for (int k = 0; k < ksplit; ++k) s = cadd(s, work[(b * ksplit + k) * MN + rc]);
    cplx* p = C + b * sC + (long long)r * ldc + c;
    cplx out = cmul(alpha, s);
    if (use_beta) out = cadd(out, cmul(beta, *p));
    *p = out;
  }
}

__global__ void scale_matrix_kernel(int M, int N, cplx beta, cplx* C, long long ldc) {
  const long long total = (long long)M * N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e / N), c = (int)(e - (long long)r * N);
    cplx* p = C + (long long)r * ldc + c;
    *p = (beta.x == 0.0 && beta.y == 0.0) ? cmk(0, 0) : cmul(beta, *p);
  }
}

template <int OPA, int OPB, int BM, int BN>
constexpr size_t smem_bytes() {
  constexpr bool TA = (OPA == 1 || OPA == 2);
  constexpr bool TB = (OPB == 1 || OPB == 2);
  return (size_t)STAGES * ((TA ? BK * (BM + 2) : BM * PA) + (TB ? BN * PBT : BK * (BN + 2))) * sizeof(cplx);
}

template <int OPA, int OPB, int BM, int BN>
cudaError_t launch_t(const GemmArgs& g, dim3 grid, cudaStream_t st) {
  // opt-in once per device (lock-free fast path: one bit per device)
  static std::atomic<unsigned long long> dev_mask{0};
  constexpr size_t sm = smem_bytes<OPA, OPB, BM, BN>();
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(dev_mask.load(std::memory_order_acquire) & bit)) {
    cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(zgemm_dmma_kernel<OPA, OPB, BM, BN>), (int)sm);
    if (e != cudaSuccess) return e;
    dev_mask.fetch_or(bit, std::memory_order_acq_rel);
  }
  zgemm_dmma_kernel<OPA, OPB, BM, BN><<<grid, NT, sm, st>>>(g);
  return cudaGetLastError();
}

template <int BM, int BN, int OPA>
cudaError_t launch_b(int opB, const GemmArgs& g, dim3 grid, cudaStream_t st) {
  switch (opB) {
    case 0: return launch_t<OPA, 0, BM, BN>(g, grid, st);
    case 1: return launch_t<OPA, 1, BM, BN>(g, grid, st);
    case 2: return launch_t<OPA, 2, BM, BN>(g, grid, st);
    default: return launch_t<OPA, 3, BM, BN>(g, grid, st);
  }
}

template <int BM, int BN>
cudaError_t launch_ab(int opA, int opB, const GemmArgs& g, dim3 grid, cudaStream_t st) {
  switch (opA) {
    case 0: return launch_b<BM, BN, 0>(opB, g, grid, st);
    case 1: return launch_b<BM, BN, 1>(opB, g, grid, st);
    case 2: return launch_b<BM, BN, 2>(opB, g, grid, st);
    default: return launch_b<BM, BN, 3>(opB, g, grid, st);
  }
}

}  // namespace

int g_num_sms = 148;

cudaError_t zgemm(cudaStream_t st, int opA, int opB, int M, int N, int K, cplx alpha, const cplx* A, long long lda,
                  const cplx* B, long long ldb, cplx beta, cplx* C, long long ldc, int batch, long long sA,
                  long long sB, long long sC, cplx* work, size_t work_elems, const double* skip,
                  const GemmMask* mask) {
  if (M <= 0 || N <= 0 || batch <= 0) return cudaSuccess;
  if (K <= 0) {
    for (int b = 0; b < batch; ++b) {
      scale_matrix_kernel<<<std::max(1, std::min(4096, (M * N + 255) / 256)), 256, 0, st>>>(M, N, beta, C + b * sC, ldc);
    }
    return cudaGetLastError();
  }
  GemmArgs g;
  g.M = M; g.N = N; g.K = K;
  g.alpha = alpha; g.beta = beta;
  g.A = A; g.lda = lda; g.sA = sA;
  g.B = B; g.ldb = ldb; g.sB = sB;
  g.C = C; g.ldc = ldc; g.sC = sC;
  g.work = work;
  g.skip = skip;
  if (mask != nullptr && mask->a != nullptr && mask->b != nullptr && (K + BK - 1) / BK <= MAXKL) g.mask = *mask;
  // tile choice: 64x64 when that gives >= 2 waves of CTAs, else 32x32 (4x more CTAs)
  const long long tiles64 = (long long)((M + 63) / 64) * ((N + 63) / 64) * batch;
  const bool small = tiles64 < 2LL * g_num_sms;
  const int bm = small ? 32 : 64, bn = bm;
  const long long tiles = (long long)((M + bm - 1) / bm) * ((N + bn - 1) / bn) * batch;
  int ksplit = 1;
  const long long target = 2LL * g_num_sms;
  if (work != nullptr && tiles < target && K >= 256) {
    ksplit = (int)std::min<long long>((target + tiles - 1) / tiles, K / 128);
    ksplit = std::min(ksplit, 16);
    while (ksplit > 1 && (size_t)ksplit * batch * (size_t)M * N > work_elems) --ksplit;
  }
  int kchunk = K;
  if (ksplit > 1) {
    kchunk = ((K + ksplit - 1) / ksplit + BK - 1) / BK * BK;
    ksplit = (K + kchunk - 1) / kchunk;
  }
  g.ksplit = ksplit;
  g.kchunk = kchunk;
  dim3 grid((N + bn - 1) / bn, (M + bm - 1) / bm, batch * ksplit);
  cudaError_t e = small ? launch_ab<32, 32>(opA, opB, g, grid, st) : launch_ab<64, 64>(opA, opB, g, grid, st);
  if (e != cudaSuccess || ksplit == 1) return e;
  const long long total = (long long)M * N * batch;
  const int blocks = (int)std::min<long long>(4LL * g_num_sms, (total + 255) / 256);
  splitk_reduce_kernel<<<blocks, 256, 0, st>>>(M, N, ksplit, batch, work, alpha, beta, C, ldc, sC, skip);
  return cudaGetLastError();
}
