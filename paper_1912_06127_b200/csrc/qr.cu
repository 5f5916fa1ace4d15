// Blocked Householder QR (compact WY) for the QR-preconditioned Jacobi SVD
// (svd.cu).  Not a step of the paper's method by itself: it changes only how
// fast the one-sided Jacobi of PAPER.md:455 (Fig 6 "SVD") converges
// (Drmac-Veselic preconditioning: Jacobi on R^H of A = QR, twice).
//
// A is column-major (m x n, ld = lda, m >= n).  Panel p covers columns
// [k0, k0 + kb), kb = qr_kb_for(m) (the panel fits 128 KB of shared memory).
// One CTA factors a panel, producing
//   - R in the upper triangle of A, the reflector tails below the diagonal,
//   - Vc: the reflectors as explicit rows (n x m row-major: row k = v_k, with
//     v_k[k] = 1 and zeros above),
//   - T_p: the kb x kb upper-triangular factor, H_k0 ... H_{k0+kb-1} = I - V T V^H.
// The trailing columns are updated with three DMMA GEMMs (zgemm.cu), and Q is
// applied to a matrix the same way (panels in reverse order).
// Conventions follow LAPACK zgeqr2/zlarfg/zlarft: H = I - tau v v^H,
// R = H_n^H ... H_1^H A, beta = -sign(Re alpha) ||x||.
#include <cmath>
#include <cooperative_groups.h>
#include "common.cuh"
#include "kernels.h"

namespace {

// Factor panel [k0, k0+kb) of column-major A (rows k0..m-1), kb <= KB.  The
// panel is staged in shared memory (column j at P + j*ldp, row r - k0); each
// reflector: warp 0 forms it (zlarfg), all threads scale its tail, then warp w
// owns columns j = w, w + NW, ...: j > i get w_j = v^H a_j and the update
// a_j -= conj(tau) v w_j, j < i get z_j = v_j^H v_i (for T).
template <int KB, int NT>
__global__ void __launch_bounds__(NT, 1) qr_panel_kernel(cplx* A, long long lda, int m, int k0, int kb, cplx* tau,
                                                         cplx* Vc, long long ldv, cplx* T) {
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) unsigned char qr_sm[];
  cplx* P = reinterpret_cast<cplx*>(qr_sm);
  const int rows = m - k0;
  const int ldp = rows;
  __shared__ cplx s_z[KB][KB + 1];  // s_z[j][i] = v_j^H v_i (j < i)
  __shared__ cplx s_tau[KB];
  __shared__ cplx s_T[KB][KB + 1];
  __shared__ cplx s_scale;
  __shared__ int s_refl;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int e = tid; e < rows * kb; e += NT) {
    const int j = e / rows, r = e - j * rows;
    P[j * ldp + r] = A[(long long)(k0 + j) * lda + k0 + r];
  }
  __syncthreads();
  for (int i = 0; i < kb; ++i) {
    const int pr = i;  // pivot row within the panel
    cplx* vi = P + i * ldp;
    if (wid == 0) {
      double xn2 = 0.0;
      for (int r = pr + 1 + lane; r < rows; r += 32) xn2 += cabs2(vi[r]);
      xn2 = warp_sum(xn2);
      if (lane == 0) {
        const double ar = vi[pr].x, ai = vi[pr].y;
        cplx t_i = cmk(0.0, 0.0), scale = cmk(1.0, 0.0);
        double beta = ar;
        const bool refl = !(xn2 == 0.0 && ai == 0.0);
        if (refl) {
          beta = -copysign(sqrt(ar * ar + ai * ai + xn2), ar);
          t_i = cmk((beta - ar) / beta, -ai / beta);
          const double dr = ar - beta, di = ai;
          const double den = dr * dr + di * di;
          scale = cmk(dr / den, -di / den);  // 1 / (alpha - beta)
        }
        s_tau[i] = t_i;
        s_scale = scale;
        s_refl = refl;
        vi[pr] = cmk(beta, 0.0);  // R_pp; the reflector uses v_p = 1 implicitly
      }
    }
    __syncthreads();
    if (s_refl) {
      const cplx sc = s_scale;
      for (int r = pr + 1 + tid; r < rows; r += NT) vi[r] = cmul(vi[r], sc);
    }
    __syncthreads();
    const cplx ct = cconj(s_tau[i]);
    for (int j = wid; j < kb; j += NW) {
      if (j == i) continue;
      cplx* aj = P + j * ldp;
      double dr = 0.0, di = 0.0;
      if (j > i) {
        // w_j = v^H a_j over rows >= pr (v_pr = 1)
        for (int r = pr + lane; r < rows; r += 32) {
          const cplx v = (r == pr) ? cmk(1.0, 0.0) : vi[r];
          const cplx x = cdotc(v, aj[r]);
          dr += x.x;
          di += x.y;
        }
        dr = warp_sum(dr);
        di = warp_sum(di);
        const cplx f = cmul(ct, cmk(dr, di));
        for (int r = pr + lane; r < rows; r += 32) {
          const cplx v = (r == pr) ? cmk(1.0, 0.0) : vi[r];
          aj[r] = csub(aj[r], cmul(v, f));
        }
      } else {
        // z_j = v_j^H v_i over rows >= pr (v_j has unit entry at row j < pr)
        for (int r = pr + lane; r < rows; r += 32) {
          const cplx v = (r == pr) ? cmk(1.0, 0.0) : vi[r];
          const cplx x = cdotc(aj[r], v);
          dr += x.x;
          di += x.y;
        }
        dr = warp_sum(dr);
        di = warp_sum(di);
        if (lane == 0) s_z[j][i] = cmk(dr, di);
      }
    }
    __syncthreads();
  }
  // ---- T (zlarft forward/columnwise): T_ii = tau_i, T[0:i, i] = -tau_i T[0:i,0:i] z[0:i, i]
  if (tid == 0) {
    for (int i = 0; i < kb; ++i) {
      s_T[i][i] = s_tau[i];
      for (int r = 0; r < i; ++r) {
        cplx acc = cmk(0.0, 0.0);
        for (int c = r; c < i; ++c) acc = cadd(acc, cmul(s_T[r][c], s_z[c][i]));
        s_T[r][i] = cmul(cmk(-s_tau[i].x, -s_tau[i].y), acc);
      }
      for (int r = i + 1; r < kb; ++r) s_T[r][i] = cmk(0.0, 0.0);
    }
  }
  __syncthreads();
  for (int e = tid; e < KB * KB; e += NT) T[e] = (e / KB < kb && e % KB < kb) ? s_T[e / KB][e % KB] : cmk(0.0, 0.0);
  for (int e = tid; e < kb; e += NT) tau[k0 + e] = s_tau[e];
  // ---- write back the panel and the explicit reflector rows Vc[k0 + j][k0 + r]
  for (int e = tid; e < rows * kb; e += NT) {
    const int j = e / rows, r = e - j * rows;
    const cplx a = P[j * ldp + r];
    A[(long long)(k0 + j) * lda + k0 + r] = a;
    const cplx v = (r < j) ? cmk(0.0, 0.0) : (r == j) ? cmk(1.0, 0.0) : a;
    Vc[(long long)(k0 + j) * ldv + k0 + r] = v;
  }
}

// R^H (n x n, lower) from the upper triangle of column-major QR output A (ld lda)
// into column-major X (ld ldx); rows [n, rows_total) of X zeroed.
__global__ void qr_rh_kernel(const cplx* __restrict__ A, long long lda, int n, cplx* X, long long ldx, int rows_total) {
  const long long total = (long long)rows_total * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e / rows_total), r = (int)(e - (long long)c * rows_total);
    // X[r][c] = conj(R[c][r]) for r >= c (R upper: R[c][r] with c <= r)
    cplx v = cmk(0.0, 0.0);
    if (r < n && r >= c) v = cconj(A[(long long)r * lda + c]);
    X[(long long)c * ldx + r] = v;
  }
}

}  // namespace

// panel width by the row count (the panel lives in registers)
int qr_kb_for(int m) { return m <= 256 ? 32 : m <= 512 ? 16 : m <= 1024 ? 8 : 0; }

cudaError_t qr_factor(cudaStream_t st, const QrWork& w, cplx* A, long long lda, int m, int n) {
  const int KBm = qr_kb_for(m);
  if (m < n || n < 1 || KBm == 0 || KBm != w.kb) return cudaErrorInvalidValue;
  const cplx one = cmk(1.0, 0.0), zero = cmk(0.0, 0.0), mone = cmk(-1.0, 0.0);
  for (int k0 = 0, p = 0; k0 < n; k0 += KBm, ++p) {
    const int kb = std::min(KBm, n - k0);
    const int rows = m - k0;
    cplx* T = w.T + (long long)p * KBm * KBm;
    const size_t smem = (size_t)rows * kb * sizeof(cplx);
    static bool attr = false;
    if (!attr) {  // panels need <= 128 KB (rows * kb * 16 B)
      cudaError_t ea;
      if ((ea = cudaFuncSetAttribute(qr_panel_kernel<32, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     128 * 1024)) != cudaSuccess ||
          (ea = cudaFuncSetAttribute(qr_panel_kernel<16, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     128 * 1024)) != cudaSuccess ||
          (ea = cudaFuncSetAttribute(qr_panel_kernel<8, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     128 * 1024)) != cudaSuccess)
        return ea;
      attr = true;
    }
    if (KBm == 32) qr_panel_kernel<32, 256><<<1, 256, smem, st>>>(A, lda, m, k0, kb, w.tau, w.Vc, w.ldv, T);
    else if (KBm == 16) qr_panel_kernel<16, 256><<<1, 256, smem, st>>>(A, lda, m, k0, kb, w.tau, w.Vc, w.ldv, T);
    else qr_panel_kernel<8, 256><<<1, 256, smem, st>>>(A, lda, m, k0, kb, w.tau, w.Vc, w.ldv, T);
    const int nt = n - k0 - kb;
    if (nt <= 0) continue;
    // trailing A_t = A[k0:m, k0+kb:n]; row-major view Ar_t (nt x rows, ld lda)
    cplx* Art = A + (long long)(k0 + kb) * lda + k0;
    const cplx* Vp = w.Vc + (long long)k0 * w.ldv + k0;  // kb x rows, ld ldv
    cudaError_t e;
    // Wt = Ar_t Vc^H                     (nt x kb)
    if ((e = zgemm(st, OP_N, OP_C, nt, kb, rows, one, Art, lda, Vp, w.ldv, zero, w.W1, kb)) != cudaSuccess) return e;
    // Wt2 = Wt conj(T)                   (= (T^H W)^T)
    if ((e = zgemm(st, OP_N, OP_R, nt, kb, kb, one, w.W1, kb, T, KBm, zero, w.W2, kb)) != cudaSuccess) return e;
    // Ar_t -= Wt2 Vc
    if ((e = zgemm(st, OP_N, OP_N, nt, rows, kb, mone, w.W2, kb, Vp, w.ldv, one, Art, lda)) != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t qr_apply_q(cudaStream_t st, const QrWork& w, int m, int n, cplx* C, long long ldc, int nc) {
  const cplx one = cmk(1.0, 0.0), zero = cmk(0.0, 0.0), mone = cmk(-1.0, 0.0);
  const int KBm = w.kb;
  const int np = (n + KBm - 1) / KBm;
  for (int p = np - 1; p >= 0; --p) {
    const int k0 = p * KBm, kb = std::min(KBm, n - k0), rows = m - k0;
    const cplx* T = w.T + (long long)p * KBm * KBm;
    const cplx* Vp = w.Vc + (long long)k0 * w.ldv + k0;
    cplx* Crt = C + k0;  // row-major view of column-major C: nc x rows, ld ldc
    cudaError_t e;
    // Wt = Cr_t Vc^H ; Wt2 = Wt T^T (= (T W)^T) ; Cr_t -= Wt2 Vc
    if ((e = zgemm(st, OP_N, OP_C, nc, kb, rows, one, Crt, ldc, Vp, w.ldv, zero, w.W1, kb)) != cudaSuccess) return e;
    if ((e = zgemm(st, OP_N, OP_T, nc, kb, kb, one, w.W1, kb, T, KBm, zero, w.W2, kb)) != cudaSuccess) return e;
    if ((e = zgemm(st, OP_N, OP_N, nc, rows, kb, mone, w.W2, kb, Vp, w.ldv, one, Crt, ldc)) != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t qr_r_conjtrans(cudaStream_t st, const cplx* A, long long lda, int n, cplx* X, long long ldx,
                           int rows_total) {
  const long long total = (long long)rows_total * n;
  const int blocks = (int)std::max<long long>(1, std::min<long long>((total + 255) / 256, 4LL * g_num_sms));
  qr_rh_kernel<<<blocks, 256, 0, st>>>(A, lda, n, X, ldx, rows_total);
  return cudaGetLastError();
}

// ===========================================================================
// Cluster-resident Householder QR for n <= 16 * cw columns (one thread-block
// cluster; CTA c owns columns [c*cw, (c+1)*cw) in shared memory).  Per
// reflector k: the owner CTA forms v_k (zlarfg) in its shared memory, one
// cluster barrier, every CTA copies v_k through DSMEM and applies
// H_k^H = I - conj(tau_k) v_k v_k^H to its columns > k (warp per column).
// No GEMM launches and no T factors: the reflectors are applied to a matrix
// later by qr_apply_refl_kernel.
namespace {

template <int NT>
__global__ void __launch_bounds__(NT, 1)
    qrc_factor_kernel(cplx* A, long long lda, int m, int n, int cw, cplx* tau, cplx* RH, long long ldrh, int rh_rows) {
  namespace cgq = cooperative_groups;
  cgq::cluster_group cluster = cgq::this_cluster();
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) unsigned char qc_sm[];
  cplx* Aloc = reinterpret_cast<cplx*>(qc_sm);  // cw columns x m rows
  cplx* vbuf = Aloc + (long long)cw * m;        // m
  __shared__ cplx s_tau[2];  // double-buffered: the owner of k+1 may write before readers of k finish
  __shared__ cplx s_scale;
  __shared__ int s_refl;
  __shared__ double s_red[NW];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int crank = (int)cluster.block_rank();
  const int c0 = crank * cw, c1 = min(n, c0 + cw), ncl = max(0, c1 - c0);
  for (int e = tid; e < ncl * m; e += NT) {
    const int j = e / m, r = e - j * m;
    Aloc[e] = A[(long long)(c0 + j) * lda + r];
  }
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    const int owner = k / cw;
    if (crank == owner) {
      __syncthreads();  // column k was updated by another warp in the previous phase B
      cplx* col = Aloc + (long long)(k - c0) * m;
      double xn2 = 0.0;
      for (int r = k + 1 + tid; r < m; r += NT) xn2 += cabs2(col[r]);
      xn2 = warp_sum(xn2);
      if (lane == 0) s_red[wid] = xn2;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < NW; ++w) t += s_red[w];
        const double ar = col[k].x, ai = col[k].y;
        cplx t_i = cmk(0.0, 0.0), scale = cmk(1.0, 0.0);
        double beta = ar;
        const bool refl = !(t == 0.0 && ai == 0.0);
        if (refl) {
          beta = -copysign(sqrt(ar * ar + ai * ai + t), ar);
          t_i = cmk((beta - ar) / beta, -ai / beta);
          const double dr = ar - beta, di = ai;
          const double den = dr * dr + di * di;
          scale = cmk(dr / den, -di / den);
        }
        s_tau[k & 1] = t_i;
        s_scale = scale;
        s_refl = refl;
        col[k] = cmk(beta, 0.0);
      }
      __syncthreads();
      if (s_refl) {
        const cplx sc = s_scale;
        for (int r = k + 1 + tid; r < m; r += NT) col[r] = cmul(col[r], sc);
      }
    }
    cluster.sync();
    // every CTA: v_k and tau_k from the owner (DSMEM), then update columns > k
    const cplx* rcol = cluster.map_shared_rank(Aloc + (long long)(k - owner * cw) * m, owner);
    for (int r = k + 1 + tid; r < m; r += NT) vbuf[r] = rcol[r];
    if (tid == 0) vbuf[k] = cmk(1.0, 0.0);
    const cplx tk = *cluster.map_shared_rank(&s_tau[k & 1], owner);
    __syncthreads();
    const cplx ct = cconj(tk);
    if (tk.x != 0.0 || tk.y != 0.0) {
      for (int jl = wid; jl < ncl; jl += NW) {
        if (c0 + jl <= k) continue;
        cplx* aj = Aloc + (long long)jl * m;
        double dr = 0.0, di = 0.0;
        for (int r = k + lane; r < m; r += 32) {
          const cplx x = cdotc(vbuf[r], aj[r]);
          dr += x.x;
          di += x.y;
        }
        dr = warp_sum(dr);
        di = warp_sum(di);
        const cplx f = cmul(ct, cmk(dr, di));
        for (int r = k + lane; r < m; r += 32) aj[r] = csub(aj[r], cmul(vbuf[r], f));
      }
    }
    if (crank == owner && tid == 0) tau[k] = tk;
  }
  __syncthreads();
  for (int e = tid; e < ncl * m; e += NT) {
    const int j = e / m, r = e - j * m;
    A[(long long)(c0 + j) * lda + r] = Aloc[e];
  }
  // [R^H ; 0] (rh_rows x n): RH[r][c] = conj(R[c][r]) for c <= r < n, column c of RH from row c of R
  if (RH != nullptr) {
    for (int e = tid; e < ncl * rh_rows; e += NT) {
      const int j = e / rh_rows, r = e - j * rh_rows;  // our column c = c0 + j of R = row c of RH^T
      const int c = c0 + j;
      // R[i][c] (i <= c) lands at RH[c][i] (row c, column i)
      if (r <= c && r < n) RH[(long long)r * ldrh + c] = cconj(Aloc[(long long)j * m + r]);
    }
  }
  cluster.sync();  // keep shared memory alive until every CTA finished its DSMEM reads
}

// C (m x nc, column-major, ld ldc) <- H_0 H_1 ... H_{n-1} C with the
// reflectors of qrc_factor_kernel / zgeqr2 (v_k = [0..0, 1, A[k+1:, k]]).
// One CTA per 8 columns of C held in registers (RPT rows per thread); per
// reflector one reduction of 16 doubles (warp reduce-scatter + one
// __syncthreads), v_k read from L2.
template <int RPT, int NT>
__global__ void __launch_bounds__(NT)
    qr_apply_refl_kernel(const cplx* __restrict__ A, long long lda, const cplx* __restrict__ tau, int m, int n, cplx* C,
                         long long ldc, int nc) {
  constexpr int CB = 8, NV = 2 * CB, NW = NT / 32;
  __shared__ double red[2][NW][NV];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int cb0 = blockIdx.x * CB;
  cplx c[RPT][CB];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int r = tid + q * NT;
#pragma unroll
    for (int j = 0; j < CB; ++j)
      c[q][j] = (r < m && cb0 + j < nc) ? C[(long long)(cb0 + j) * ldc + r] : cmk(0.0, 0.0);
  }
  int buf = 0;
  for (int k = n - 1; k >= 0; --k) {
    const cplx tk = tau[k];
    if (tk.x == 0.0 && tk.y == 0.0) continue;  // uniform across the CTA
    cplx v[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int r = tid + q * NT;
      v[q] = (r == k) ? cmk(1.0, 0.0) : (r > k && r < m) ? __ldg(A + (long long)k * lda + r) : cmk(0.0, 0.0);
    }
    double val[NV];
#pragma unroll
    for (int j = 0; j < CB; ++j) {
      double sr = 0.0, si = 0.0;
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const cplx p = cdotc(v[q], c[q][j]);
        sr += p.x;
        si += p.y;
      }
      val[2 * j] = sr;
      val[2 * j + 1] = si;
    }
    // reduce-scatter over the warp: lane l holds value l >> 1
#pragma unroll
    for (int lev = 0; lev < 4; ++lev) {
      const int msk = 16 >> lev, h = NV >> (lev + 1);
      const bool up = (lane & msk) != 0;
#pragma unroll
      for (int j = 0; j < h; ++j) {
        const double send = up ? val[j] : val[j + h];
        const double keep = up ? val[j + h] : val[j];
        val[j] = keep + __shfl_xor_sync(0xffffffffu, send, msk);
      }
    }
    double t = val[0] + __shfl_xor_sync(0xffffffffu, val[0], 1);
    if ((lane & 1) == 0) red[buf][wid][lane >> 1] = t;
    __syncthreads();
    double tot = 0.0;
    if (lane < NV)
#pragma unroll
      for (int w = 0; w < NW; ++w) tot += red[buf][w][lane];
    buf ^= 1;
#pragma unroll
    for (int j = 0; j < CB; ++j) {
      const cplx wj = cmk(__shfl_sync(0xffffffffu, tot, 2 * j), __shfl_sync(0xffffffffu, tot, 2 * j + 1));
      const cplx f = cmul(tk, wj);
#pragma unroll
      for (int q = 0; q < RPT; ++q) c[q][j] = csub(c[q][j], cmul(v[q], f));
    }
  }
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int r = tid + q * NT;
#pragma unroll
    for (int j = 0; j < CB; ++j)
      if (r < m && cb0 + j < nc) C[(long long)(cb0 + j) * ldc + r] = c[q][j];
  }
}

}  // namespace

// Cluster QR (n <= 16 * cw with the panel fitting shared memory); returns
// cudaErrorNotSupported otherwise.  Optionally writes [R^H ; 0] (rh_rows x n)
// to RH (the strictly upper part of RH must be zero on entry or is ignored).
cudaError_t qr_factor_cluster(cudaStream_t st, cplx* A, long long lda, int m, int n, cplx* tau, cplx* RH,
                              long long ldrh, int rh_rows) {
  if (m < n || n < 1) return cudaErrorInvalidValue;
  const int C = std::min(16, n);
  const int cw = (n + C - 1) / C;
  const int Cu = (n + cw - 1) / cw;
  const size_t smem = ((size_t)cw * m + m) * sizeof(cplx);
  if (smem > 200 * 1024) return cudaErrorNotSupported;
  cudaError_t e;
  static bool attr = false;
  if (!attr) {
    if ((e = cudaFuncSetAttribute(qrc_factor_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)) !=
        cudaSuccess)
      return e;
    if ((e = cudaFuncSetAttribute(qrc_factor_kernel<256>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) !=
        cudaSuccess)
      return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3(Cu);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = Cu;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (RH != nullptr) {
    // zero RH first (the kernel writes the lower triangle only)
    if ((e = cudaMemset2DAsync(RH, (size_t)ldrh * sizeof(cplx), 0, (size_t)rh_rows * sizeof(cplx), n, st)) !=
        cudaSuccess)
      return e;
  }
  return cudaLaunchKernelEx(&cfg, qrc_factor_kernel<256>, A, lda, m, n, cw, tau, RH, ldrh, rh_rows);
}

cudaError_t qr_apply_refl(cudaStream_t st, const cplx* A, long long lda, const cplx* tau, int m, int n, cplx* C,
                          long long ldc, int nc) {
  const int blocks = (nc + 7) / 8;
  if (m <= 256) qr_apply_refl_kernel<1, 256><<<blocks, 256, 0, st>>>(A, lda, tau, m, n, C, ldc, nc);
  else if (m <= 512) qr_apply_refl_kernel<2, 256><<<blocks, 256, 0, st>>>(A, lda, tau, m, n, C, ldc, nc);
  else if (m <= 1024) qr_apply_refl_kernel<4, 256><<<blocks, 256, 0, st>>>(A, lda, tau, m, n, C, ldc, nc);
  else return cudaErrorNotSupported;
  return cudaGetLastError();
}
