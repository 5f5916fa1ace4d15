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
#include <cstdio>
#include <cstdlib>
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
  if (wid == 0) {  // column i depends on the earlier columns; its rows r < i are independent (lane r)
    for (int i = 0; i < kb; ++i) {
      const int r = lane;
      if (r < i) {
        cplx acc = cmk(0.0, 0.0);
        for (int c = r; c < i; ++c) acc = cadd(acc, cmul(s_T[r][c], s_z[c][i]));
        s_T[r][i] = cmul(cmk(-s_tau[i].x, -s_tau[i].y), acc);
      } else if (r == i) {
        s_T[i][i] = s_tau[i];
      } else if (r < kb) {
        s_T[r][i] = cmk(0.0, 0.0);
      }
      __syncwarp();
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

// Panel [k0, k0+kb) of column-major A (rows k0..m-1, kb <= 32) factored by ONE
// thread-block cluster of C CTAs: CTA c holds rows [c*rc, (c+1)*rc) of the
// panel in its shared memory.  ONE cluster barrier per reflector i: every CTA
// forms, over its rows g >= i, the partial sums
//   s_j = x^H a_j (j > i),  s_j = v_j^H x (j < i),  s_i = |x below the pivot|^2
// with x = column i BEFORE the reflector is known, and the owner of pivot row
// i publishes that row (alpha = x_i, a_j[i], v_j[i]); after the barrier every
// CTA sums the C partials in rank order (identical everywhere) and forms
// zlarfg (beta, tau, scale = 1/(alpha - beta)) and, since v = (x - beta e_i) scale,
//   w_j = v^H a_j = conj(scale) (s_j - beta a_j[i])          (j > i)
//   z_j = v_j^H v = scale (s_j - beta conj(v_j[i]))           (j < i, for T)
// (algebraically the LAPACK dots with the explicit v; |scale| <= 1/||x|| keeps
// the rounding at eps ||a_j||), then updates its rows of a_j -= conj(tau) v w_j.
// The DSMEM slots are double-buffered by reflector parity, so the next
// reflector's partials never overwrite ones a slower CTA is still reading.
// Output as qr_panel_kernel (R / reflector tails in A, explicit rows Vc, tau, T).
constexpr int QPW = 32;   // max panel width
constexpr int QPNT = 256;
__global__ void __launch_bounds__(QPNT, 1) qr_panel_cl_kernel(cplx* A, long long lda, int m, int k0, int kb, int rc,
                                                               cplx* tau, cplx* Vc, long long ldv, cplx* T) {
  namespace cgx = cooperative_groups;
  cgx::cluster_group cluster = cgx::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int crank = (int)cluster.block_rank();
  extern __shared__ __align__(16) unsigned char qr_sm[];
  cplx* P = reinterpret_cast<cplx*>(qr_sm);  // [kb][rc] column j at P + j*rc
  __shared__ cplx s_w[2][QPW];                // partial sums of this CTA (by reflector parity)
  __shared__ cplx s_row[2][QPW];              // pivot row (owner CTA, by parity)
  __shared__ cplx s_pw[QPW][16];              // partial sums of all CTAs
  __shared__ cplx s_rowt[QPW];                // pivot row fetched from its owner
  __shared__ cplx s_wt[QPW];                  // w_j (j > i)
  __shared__ cplx s_z[QPW][QPW + 1];          // (CTA 0) z[j][i] = v_j^H v_i
  __shared__ cplx s_tau[QPW];
  __shared__ cplx s_T[QPW][QPW + 1];
  __shared__ cplx s_scale;
  __shared__ double s_beta;
  __shared__ int s_refl;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int rows = m - k0;
  const int r0 = crank * rc;                       // first panel row of this CTA
  const int nr = max(0, min(rc, rows - r0));       // rows held
  for (int e = tid; e < kb * rc; e += QPNT) {
    const int j = e / rc, r = e - j * rc;
    P[j * rc + r] = (r < nr) ? A[(long long)(k0 + j) * lda + k0 + r0 + r] : cmk(0.0, 0.0);
  }
  __syncthreads();
  // thread (h, rr): rows rr and rr + 128 of this CTA, panel columns [16 h, 16 h + 16)
  const int h = tid >> 7, rr = tid & 127;
  __shared__ double s_red[QPNT / 32][32];
  for (int i = 0; i < kb; ++i) {
    const int pr = i, par = i & 1;  // pivot row within the panel
    cplx* vi = P + i * rc;
    // ---- (1) partial sums over this CTA's rows g >= pr: 16 columns per thread,
    // then a warp reduce-scatter (lane l: value l) and the 4 warps of a half
    {
      double val[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) val[u] = 0.0;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int r = rr + 128 * q, g = r0 + r;
        if (r >= nr || g < pr) continue;
        const cplx x = vi[r];
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const int j = 16 * h + jj;
          if (j >= kb) continue;
          const cplx a = P[j * rc + r];
          cplx t;
          if (j > i) t = cdotc(x, a);
          else if (j < i) t = cdotc(a, x);
          else t = cmk(g > pr ? cabs2(x) : 0.0, 0.0);
          val[2 * jj] += t.x;
          val[2 * jj + 1] += t.y;
        }
      }
#pragma unroll
      for (int lev = 0; lev < 5; ++lev) {
        const int msk = 16 >> lev, hh = 16 >> lev;
        const bool up = (lane & msk) != 0;
#pragma unroll
        for (int u = 0; u < hh; ++u) {
          const double send = up ? val[u] : val[u + hh];
          const double keep = up ? val[u + hh] : val[u];
          val[u] = keep + __shfl_xor_sync(0xffffffffu, send, msk);
        }
      }
      s_red[wid][lane] = val[0];
    }
    __syncthreads();
    if (tid < 64) {
      const int hh = tid >> 5, l = tid & 31, j = 16 * hh + (l >> 1);
      const double t = ((s_red[4 * hh][l] + s_red[4 * hh + 1][l]) + s_red[4 * hh + 2][l]) + s_red[4 * hh + 3][l];
      if (j < kb) reinterpret_cast<double*>(&s_w[par][j])[l & 1] = t;
    } else if (tid < 64 + kb) {
      if (pr >= r0 && pr < r0 + nr) s_row[par][tid - 64] = P[(tid - 64) * rc + pr - r0];
    }
    __syncthreads();
    cluster.sync();
    // kb x C partials and the pivot row fetched in parallel (one DSMEM round trip)
    for (int e = tid; e < kb * C; e += QPNT) {
      const int j = e / C, c = e - j * C;
      s_pw[j][c] = *cluster.map_shared_rank(&s_w[par][j], c);
    }
    if (tid >= QPNT - QPW && tid - (QPNT - QPW) < kb)
      s_rowt[tid - (QPNT - QPW)] = *cluster.map_shared_rank(&s_row[par][tid - (QPNT - QPW)], pr / rc);
    // every thread keeps its rows of x (column i) for step (3)
    cplx xq[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int r = rr + 128 * q;
      xq[q] = r < nr ? vi[r] : cmk(0.0, 0.0);
    }
    __syncthreads();
    // ---- (2) zlarfg and the dots, every CTA (identical sums in a fixed
    // pairwise order over the C = 8 or 16 ranks, identical results)
    if (tid < kb) {
      cplx t[16];
      double xn[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        t[c] = c < C ? s_pw[tid][c] : cmk(0.0, 0.0);
        xn[c] = c < C ? s_pw[i][c].x : 0.0;
      }
#pragma unroll
      for (int w = 1; w < 16; w *= 2)
#pragma unroll
        for (int c = 0; c + w < 16; c += 2 * w) {
          t[c] = cadd(t[c], t[c + w]);
          xn[c] += xn[c + w];
        }
      const cplx sj = t[0];
      const double xn2 = xn[0];
      const cplx al = s_rowt[i];
      const double ar = al.x, ai = al.y;
      cplx t_i = cmk(0.0, 0.0), scale = cmk(1.0, 0.0);
      double beta = ar;
      const bool refl = !(xn2 == 0.0 && ai == 0.0);
      if (refl) {
        beta = -copysign(sqrt(ar * ar + ai * ai + xn2), ar);
        const double ib = 1.0 / beta;
        t_i = cmk((beta - ar) * ib, -ai * ib);
        const double dr = ar - beta, di = ai;
        const double iden = 1.0 / (dr * dr + di * di);
        scale = cmk(dr * iden, -di * iden);  // 1 / (alpha - beta)
      }
      if (tid > i) {
        s_wt[tid] = cmul(cconj(t_i), cmul(cconj(scale), csub(sj, cscale(s_rowt[tid], beta))));  // conj(tau) w_j
      } else if (tid < i) {
        if (crank == 0) s_z[tid][i] = cmul(scale, csub(sj, cscale(cconj(s_rowt[tid]), beta)));
      } else {
        s_tau[i] = t_i;
        s_scale = scale;
        s_beta = beta;
        s_refl = refl;
      }
    }
    __syncthreads();
    // ---- (3) v_i = (x - beta e_pr) scale; a_j -= v_i conj(tau) w_j (j > i);
    // the half holding column i writes v_i (R_pp = beta at the pivot)
    {
      const cplx sc = s_scale;
      const bool refl = s_refl != 0;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int r = rr + 128 * q, g = r0 + r;
        if (r >= nr || g < pr) continue;
        const cplx v = (g == pr) ? cmk(1.0, 0.0) : (refl ? cmul(xq[q], sc) : xq[q]);
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const int j = 16 * h + jj;
          if (j <= i || j >= kb) continue;
          P[j * rc + r] = csub(P[j * rc + r], cmul(v, s_wt[j]));
        }
        if (h == (i >> 4)) vi[r] = (g == pr) ? cmk(s_beta, 0.0) : v;
      }
    }
    __syncthreads();
  }
  // ---- T (zlarft forward/columnwise) on CTA 0, one warp: column i of T
  // depends on the earlier columns; its rows r < i are independent (lane r)
  if (crank == 0 && wid == 0) {
    for (int i = 0; i < kb; ++i) {
      const int r = lane;
      if (r < i) {
        cplx acc = cmk(0.0, 0.0);
        for (int c = r; c < i; ++c) acc = cadd(acc, cmul(s_T[r][c], s_z[c][i]));
        s_T[r][i] = cmul(cmk(-s_tau[i].x, -s_tau[i].y), acc);
      } else if (r == i) {
        s_T[i][i] = s_tau[i];
      } else if (r < kb) {
        s_T[r][i] = cmk(0.0, 0.0);
      }
      __syncwarp();
    }
  }
  __syncthreads();
  if (crank == 0) {
    for (int e = tid; e < QPW * QPW; e += QPNT)
      T[e] = (e / QPW < kb && e % QPW < kb) ? s_T[e / QPW][e % QPW] : cmk(0.0, 0.0);
    for (int e = tid; e < kb; e += QPNT) tau[k0 + e] = s_tau[e];
  }
  for (int e = tid; e < kb * rc; e += QPNT) {
    const int j = e / rc, r = e - j * rc;
    if (r >= nr) continue;
    const int g = r0 + r;
    const cplx a = P[j * rc + r];
    A[(long long)(k0 + j) * lda + k0 + g] = a;
    const cplx v = (g < j) ? cmk(0.0, 0.0) : (g == j) ? cmk(1.0, 0.0) : a;
    Vc[(long long)(k0 + j) * ldv + k0 + g] = v;
  }
  cluster.sync();  // shared memory stays alive until every CTA finished its DSMEM reads
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
int qr_kb_for(int m) { return m <= 4096 ? 32 : 0; }

cudaError_t qr_factor(cudaStream_t st, const QrWork& w, cplx* A, long long lda, int m, int n) {
  const int KBm = qr_kb_for(m);
  if (m < n || n < 1 || KBm == 0 || KBm != w.kb) return cudaErrorInvalidValue;
  const cplx one = cmk(1.0, 0.0), zero = cmk(0.0, 0.0), mone = cmk(-1.0, 0.0);
  for (int k0 = 0, p = 0; k0 < n; k0 += KBm, ++p) {
    const int kb = std::min(KBm, n - k0);
    const int rows = m - k0;
    cplx* T = w.T + (long long)p * KBm * KBm;
    cudaError_t e;
    if (rows <= 64) {
      const size_t smem = (size_t)rows * kb * sizeof(cplx);
      if ((e = set_smem_attr(reinterpret_cast<const void*>(qr_panel_kernel<32, 256>), 128 * 1024)) != cudaSuccess)
        return e;
      qr_panel_kernel<32, 256><<<1, 256, smem, st>>>(A, lda, m, k0, kb, w.tau, w.Vc, w.ldv, T);
    } else {
      // cluster panel: C CTAs of rc rows each (rc * kb * 16 B of shared memory)
      const int C = rows <= 512 ? 4 : rows <= 1024 ? 8 : 16;
      const int rc = (rows + C - 1) / C;
      const size_t smem = (size_t)rc * kb * sizeof(cplx);
      if ((e = set_smem_attr(reinterpret_cast<const void*>(qr_panel_cl_kernel), (int)std::max<size_t>(smem, 48 * 1024))) !=
          cudaSuccess)
        return e;
      if ((e = set_cluster_nonportable(reinterpret_cast<const void*>(qr_panel_cl_kernel))) != cudaSuccess) return e;
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      cfg.gridDim = dim3(C);
      cfg.blockDim = dim3(QPNT);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      if ((e = cudaLaunchKernelEx(&cfg, qr_panel_cl_kernel, A, lda, m, k0, kb, rc, w.tau, w.Vc, w.ldv, T)) !=
          cudaSuccess)
        return e;
    }
    const int nt = n - k0 - kb;
    if (nt <= 0) continue;
    // trailing A_t = A[k0:m, k0+kb:n]; row-major view Ar_t (nt x rows, ld lda)
    cplx* Art = A + (long long)(k0 + kb) * lda + k0;
    const cplx* Vp = w.Vc + (long long)k0 * w.ldv + k0;  // kb x rows, ld ldv
    // Wt = Ar_t Vc^H                     (nt x kb; K = rows: split-K into w.gw)
    if ((e = zgemm(st, OP_N, OP_C, nt, kb, rows, one, Art, lda, Vp, w.ldv, zero, w.W1, kb, 1, 0, 0, 0, w.gw,
                   w.gw_elems)) != cudaSuccess)
      return e;
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
    if ((e = zgemm(st, OP_N, OP_C, nc, kb, rows, one, Crt, ldc, Vp, w.ldv, zero, w.W1, kb, 1, 0, 0, 0, w.gw,
                   w.gw_elems)) != cudaSuccess)
      return e;
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

// Look-ahead variant (default).  CTA c owns columns [c*cw, (c+1)*cw).  No
// cluster-wide barrier per reflector: reflectors are published point to point.
//  phase 1: CTA c applies the reflectors 0 .. c*cw-1 of the earlier CTAs to its
//           columns as they appear: it spins on a counter in its own shared
//           memory that the producer raises with a cluster-scope release store,
//           then copies v_k and tau_k through DSMEM (batches of up to NB).
//  phase 2: CTA c factors its band: warp 0 (the panel warp) forms v_k from
//           column k, publishes it, and applies it to column k+1 (look-ahead)
//           while warps 1.. apply it to the band's remaining columns; one named
//           barrier per reflector.
// flag in CTA `rank`'s shared memory (shared::cluster window), release/acquire at cluster scope
__device__ __forceinline__ void st_release_cluster_rank(const unsigned* local, unsigned rank, unsigned v) {
  const unsigned la = (unsigned)__cvta_generic_to_shared(local);
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
  asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"(ra), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_cluster_local(const unsigned* local) {
  const unsigned la = (unsigned)__cvta_generic_to_shared(local);
  unsigned v;
  asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(la) : "memory");
  return v;
}

__device__ unsigned long long g_qr_prof[16][4];
// 1/x for normal nonzero x: MUFU seed + two Newton steps (full double precision)
__device__ __forceinline__ double qr_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
__device__ unsigned long long g_qr_ph[8];
__constant__ int qr_ph_cta = 15;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#ifndef QR_PUB
#define QR_PUB 1
#endif
// GRID = false: one thread-block cluster, counters in each CTA's shared memory
// raised by cluster-scope release stores.  GRID = true: a cooperative grid (up
// to one CTA per SM, for bands that do not fit one cluster), one counter in
// global memory (`gcnt`, zero on entry) raised with a GPU-scope release.
template <int NT, int NB, bool GRID, int RPL = 0>
__global__ void __launch_bounds__(NT, 1)
    qrc3_factor_kernel(cplx* A, long long lda, int m, int n, int cw, cplx* tau, cplx* RH, long long ldrh, int rh_rows,
                       unsigned* gcnt) {
  namespace cgq = cooperative_groups;
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) unsigned char qc_sm[];
  cplx* Aloc = reinterpret_cast<cplx*>(qc_sm);  // cw columns x m rows (own band)
  cplx* vb = Aloc + (long long)cw * m;          // NB received reflectors x m rows
  cplx* s_tau = vb + (long long)NB * m;         // [cw] published taus of the own band
  __shared__ cplx s_vt[NB];
  __shared__ unsigned s_npub;  // reflectors published to this CTA (written remotely)
  __shared__ int s_nav;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int crank = GRID ? (int)blockIdx.x : (int)cgq::this_cluster().block_rank();
  const int ncta = GRID ? (int)gridDim.x : (int)cgq::this_cluster().num_blocks();
  auto all_sync = [&]() {
    if (GRID) cgq::this_grid().sync();
    else cgq::this_cluster().sync();
  };
  const int c0 = crank * cw, c1 = min(n, c0 + cw), ncl = max(0, c1 - c0);
  for (int e = tid; e < ncl * m; e += NT) {
    const int j = e / m, r = e - j * m;
    Aloc[e] = A[(long long)(c0 + j) * lda + r];
  }
  if (tid == 0) s_npub = 0u;
  all_sync();  // every counter initialised before any remote release
  if (tid == 0 && crank < 16) g_qr_prof[crank][0] = gtime();
  int nbatches = 0;
  // ---------------- phase 1: apply the earlier CTAs' reflectors 0 .. c0-1
  for (int k = 0; k < c0;) {
    if (tid == 0) {
      unsigned a;
      if (GRID) {
        while ((a = *(volatile unsigned*)gcnt) <= (unsigned)k) __nanosleep(64);
        __threadfence();
      } else {
        while ((a = ld_acquire_cluster_local(&s_npub)) <= (unsigned)k) __nanosleep(64);
      }
      s_nav = min((int)a, min(c0, k + NB)) - k;  // batch of available reflectors
    }
    __syncthreads();
    const int nb = s_nav;
    // copy v_{k..k+nb-1} (rows >= k) and their taus from the owners
    for (int e = tid; e < nb * (m - k); e += NT) {
      const int b = e / (m - k), r = k + (e - b * (m - k));
      const int kk = k + b;
      vb[(long long)b * m + r] =
          (r < kk) ? cmk(0.0, 0.0) : (r == kk) ? cmk(1.0, 0.0) : __ldcg(A + (long long)kk * lda + r);
    }
    if (tid < nb) s_vt[tid] = __ldcg(tau + k + tid);
    __syncthreads();
    for (int jl = wid; jl < ncl; jl += NW) {
      cplx* aj = Aloc + (long long)jl * m;
      for (int b = 0; b < nb; ++b) {
        const cplx ct = cconj(s_vt[b]);
        if (ct.x == 0.0 && ct.y == 0.0) continue;
        const int kk = k + b;
        const cplx* v = vb + (long long)b * m;
        double dr = 0.0, di = 0.0;
        for (int r = kk + lane; r < m; r += 32) {
          const cplx x = cdotc(v[r], aj[r]);
          dr += x.x;
          di += x.y;
        }
        dr = warp_sum(dr);
        di = warp_sum(di);
        const cplx f = cmul(ct, cmk(dr, di));
        for (int r = kk + lane; r < m; r += 32) aj[r] = csub(aj[r], cmul(v[r], f));
      }
    }
    __syncthreads();  // vb reused by the next batch
    k += nb;
    ++nbatches;
  }
  if (tid == 0 && crank < 16) g_qr_prof[crank][1] = gtime();
  // ---------------- phase 2: factor the own band with look-ahead
  // warp 0 carries ||A[k+1:, k]||^2 of the next pivot column from its
  // look-ahead update, so a reflector costs one pass over its column
  double xn2_next = 0.0;
  if (wid == 0 && ncl > 0) {
    for (int r = c0 + 1 + lane; r < m; r += 32) xn2_next += cabs2(Aloc[r]);
    xn2_next = warp_sum(xn2_next);
  }
  if constexpr (RPL > 0) {
    // m <= 32 RPL: warp 0 keeps the pivot column in registers (row r = lane +
    // 32 t in slot t), so the reflector, the scaling and the look-ahead update
    // of the next column run on registers with one shared-memory load of that
    // column per reflector; the workers still read v from shared memory
    cplx pc[RPL];
    if (wid == 0) {
#pragma unroll
      for (int t = 0; t < RPL; ++t) {
        const int r = lane + 32 * t;
        pc[t] = (ncl > 0 && r < m) ? Aloc[r] : cmk(0.0, 0.0);
      }
    }
    for (int i = 0; i < ncl; ++i) {
      const int k = c0 + i;
      cplx* col = Aloc + (long long)i * m;
      cplx vr[RPL];
      if (wid == 0) {
        const double xn2 = xn2_next;
        cplx akk = cmk(0.0, 0.0);
#pragma unroll
        for (int t = 0; t < RPL; ++t)
          if (t == (k >> 5)) akk = pc[t];
        const double ar = __shfl_sync(0xffffffffu, akk.x, k & 31), ai = __shfl_sync(0xffffffffu, akk.y, k & 31);
        cplx t_i = cmk(0.0, 0.0), scale = cmk(1.0, 0.0);
        double beta = ar;
        const bool refl = !(xn2 == 0.0 && ai == 0.0);
        if (refl) {
          beta = -copysign(sqrt(ar * ar + ai * ai + xn2), ar);
          const double ib = qr_rcp(beta);
          t_i = cmk((beta - ar) * ib, -ai * ib);
          const double dr = ar - beta, di = ai;
          const double iden = qr_rcp(dr * dr + di * di);
          scale = cmk(dr * iden, -di * iden);
        }
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
          const int r = lane + 32 * t;
          if (r > k && r < m) {
            const cplx v = refl ? cmul(pc[t], scale) : pc[t];
            vr[t] = v;
            col[r] = v;  // the publisher warp copies it to global (off this warp's chain)
          } else {
            vr[t] = (r == k) ? cmk(1.0, 0.0) : cmk(0.0, 0.0);
          }
        }
        if (lane == (k & 31)) col[k] = cmk(beta, 0.0);
        if (lane == 0) s_tau[i] = t_i;
      }
      asm volatile("bar.sync 2, %0;" ::"n"(NT) : "memory");
      if (wid == NW - 1) {
        // publisher warp: v_k and tau_k to global, then release them to the
        // later CTAs (every QR_PUB-th reflector and the band's last)
        for (int r = k + 1 + lane; r < m; r += 32) __stcg(A + (long long)k * lda + r, col[r]);
        if (lane == 0) __stcg(tau + k, s_tau[i]);
        __syncwarp();
        if (((i + 1) % QR_PUB) == 0 || i + 1 == ncl) {
          if (GRID) {
            if (lane == 0) {
              __threadfence();
              *(volatile unsigned*)gcnt = (unsigned)(k + 1);
            }
          } else {
            for (int c = crank + 1 + lane; c < ncta; c += 32)
              st_release_cluster_rank(&s_npub, (unsigned)c, (unsigned)(k + 1));
          }
        }
      }
      const cplx ct = cconj(s_tau[i]);
      const bool upd = ct.x != 0.0 || ct.y != 0.0;
      if (wid == 0) {
        if (i + 1 < ncl) {
          // look-ahead: column i+1 (rows >= k) <- H_k column i+1, kept in registers
          const cplx* aj = Aloc + (long long)(i + 1) * m;
          double dr = 0.0, di = 0.0;
#pragma unroll
          for (int t = 0; t < RPL; ++t) {
            const int r = lane + 32 * t;
            pc[t] = (r >= k && r < m) ? aj[r] : cmk(0.0, 0.0);
            const cplx x = cdotc(vr[t], pc[t]);
            dr += x.x;
            di += x.y;
          }
          cplx f = cmk(0.0, 0.0);
          if (upd) {
            dr = warp_sum(dr);
            di = warp_sum(di);
            f = cmul(ct, cmk(dr, di));
          }
          double nx = 0.0;
#pragma unroll
          for (int t = 0; t < RPL; ++t) {
            const int r = lane + 32 * t;
            if (upd) pc[t] = csub(pc[t], cmul(vr[t], f));
            if (r > k + 1 && r < m) nx += cabs2(pc[t]);
          }
          xn2_next = warp_sum(nx);
#pragma unroll
          for (int t = 0; t < RPL; ++t)
            if (lane + 32 * t == k) Aloc[(long long)(i + 1) * m + k] = pc[t];  // R[k][i+1] is final
        }
      } else if (wid < NW - 1) {
        // workers (warps 1 .. NW-2): columns i+2, ... with reflector i (v from shared memory)
        for (int jl = i + 1 + wid; jl < ncl; jl += NW - 2) {
          cplx* aj = Aloc + (long long)jl * m;
          if (!upd) continue;
          double dr = 0.0, di = 0.0;
          for (int r = k + lane; r < m; r += 32) {
            const cplx v = (r == k) ? cmk(1.0, 0.0) : col[r];
            const cplx x = cdotc(v, aj[r]);
            dr += x.x;
            di += x.y;
          }
          dr = warp_sum(dr);
          di = warp_sum(di);
          const cplx f = cmul(ct, cmk(dr, di));
          for (int r = k + lane; r < m; r += 32) {
            const cplx v = (r == k) ? cmk(1.0, 0.0) : col[r];
            aj[r] = csub(aj[r], cmul(v, f));
          }
        }
      }
    }
  } else {
  for (int i = 0; i < ncl; ++i) {
    const int k = c0 + i;
    cplx* col = Aloc + (long long)i * m;
    if (wid == 0) {
      const double xn2 = xn2_next;
      const double ar = col[k].x, ai = col[k].y;
      cplx t_i = cmk(0.0, 0.0), scale = cmk(1.0, 0.0);
      double beta = ar;
      const bool refl = !(xn2 == 0.0 && ai == 0.0);
      if (refl) {
        beta = -copysign(sqrt(ar * ar + ai * ai + xn2), ar);
        const double ib = qr_rcp(beta);
        t_i = cmk((beta - ar) * ib, -ai * ib);
        const double dr = ar - beta, di = ai;
        const double iden = qr_rcp(dr * dr + di * di);
        scale = cmk(dr * iden, -di * iden);
      }
      // scale the tail into v_k and hand it to the consumers through L2 (not
      // DSMEM: a producer's shared-memory port would serve every later CTA)
      for (int r = k + 1 + lane; r < m; r += 32) {
        const cplx v = refl ? cmul(col[r], scale) : col[r];
        col[r] = v;
      }
      if (lane == 0) {
        col[k] = cmk(beta, 0.0);
        s_tau[i] = t_i;
      }
      __syncwarp();
    }
    asm volatile("bar.sync 2, %0;" ::"n"(NT) : "memory");
    const cplx ct = cconj(s_tau[i]);
    if (wid == NW - 1) {
      // publisher warp: v_k and tau_k to global, then release them (off warp 0's chain)
      for (int r = k + 1 + lane; r < m; r += 32) __stcg(A + (long long)k * lda + r, col[r]);
      if (lane == 0) __stcg(tau + k, s_tau[i]);
      __syncwarp();
      if (((i + 1) % QR_PUB) == 0 || i + 1 == ncl) {
        if (GRID) {
          if (lane == 0) {
            __threadfence();
            *(volatile unsigned*)gcnt = (unsigned)(k + 1);
          }
        } else {
          for (int c = crank + 1 + lane; c < ncta; c += 32)
            st_release_cluster_rank(&s_npub, (unsigned)c, (unsigned)(k + 1));
        }
      }
      continue;
    }
    if (wid == 0) xn2_next = 0.0;
    // warp 0: column i+1 (the next pivot, also its norm below row k+1);
    // warps 1 .. NW-2: columns i+2, ...
    const int jstart = (wid == 0) ? i + 1 : i + 1 + wid;
    const int jstep = (wid == 0) ? ncl : NW - 2;
    for (int jl = jstart; jl < ncl; jl += jstep) {
      cplx* aj = Aloc + (long long)jl * m;
      const bool upd = ct.x != 0.0 || ct.y != 0.0;
      cplx f = cmk(0.0, 0.0);
      if (upd) {
        double dr = 0.0, di = 0.0;
        for (int r = k + lane; r < m; r += 32) {
          const cplx v = (r == k) ? cmk(1.0, 0.0) : col[r];
          const cplx x = cdotc(v, aj[r]);
          dr += x.x;
          di += x.y;
        }
        dr = warp_sum(dr);
        di = warp_sum(di);
        f = cmul(ct, cmk(dr, di));
      }
      double nx = 0.0;
      for (int r = k + lane; r < m; r += 32) {
        const cplx v = (r == k) ? cmk(1.0, 0.0) : col[r];
        const cplx a = upd ? csub(aj[r], cmul(v, f)) : aj[r];
        aj[r] = a;
        if (r > k + 1) nx += cabs2(a);
      }
      if (wid == 0) {
        xn2_next = warp_sum(nx);
        break;
      }
    }
    // next iteration: warp 0 reads column i+1 (updated by itself); the workers'
    // updates of column i+2 are ordered before warp 0 touches it by the next
    // bar.sync 2
  }
  }  // RPL == 0
  __syncthreads();
  if (tid == 0 && crank < 16) {
    g_qr_prof[crank][2] = gtime();
    g_qr_prof[crank][3] = nbatches;
  }
  for (int e = tid; e < ncl * m; e += NT) {
    const int j = e / m, r = e - j * m;
    A[(long long)(c0 + j) * lda + r] = Aloc[e];
  }
  if (RH != nullptr) {
    for (int e = tid; e < ncl * rh_rows; e += NT) {
      const int j = e / rh_rows, r = e - j * rh_rows;
      const int c = c0 + j;
      if (r <= c && r < n) RH[(long long)r * ldrh + c] = cconj(Aloc[(long long)j * m + r]);
    }
  }
  all_sync();  // keep shared memory alive until every CTA finished its reads
}

// C (m x nc, column-major, ld ldc) <- H_0 H_1 ... H_{n-1} C with the
// reflectors of qrc_factor_kernel / zgeqr2 (v_k = [0..0, 1, A[k+1:, k]]).
// One CTA per 8 columns of C held in registers (RPT rows per thread); per
// reflector one reduction of 16 doubles (warp reduce-scatter + one
// __syncthreads), v_k read from L2.
struct QrApplyJob {
  const cplx* A;
  long long lda;
  const cplx* tau;
  int m, n;
  cplx* C;
  long long ldc;
  int nc;
};

// blocks [0, nb0) run job j0, blocks [nb0, ...) job j1 (two independent applications in one launch)
template <int RPT, int NT>
__global__ void __launch_bounds__(NT) qr_apply_refl_kernel(QrApplyJob j0, QrApplyJob j1, int nb0) {
  constexpr int CB = 8, NV = 2 * CB, NW = NT / 32;
  __shared__ double red[2][NW][NV];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool second = (int)blockIdx.x >= nb0;
  const QrApplyJob& J = second ? j1 : j0;
  const cplx* __restrict__ A = J.A;
  const long long lda = J.lda;
  const cplx* __restrict__ tau = J.tau;
  const int m = J.m, n = J.n, nc = J.nc;
  cplx* C = J.C;
  const long long ldc = J.ldc;
  const int cb0 = (second ? (int)blockIdx.x - nb0 : (int)blockIdx.x) * CB;
  cplx c[RPT][CB];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int r = tid + q * NT;
#pragma unroll
    for (int j = 0; j < CB; ++j)
      c[q][j] = (r < m && cb0 + j < nc) ? C[(long long)(cb0 + j) * ldc + r] : cmk(0.0, 0.0);
  }
  int buf = 0;
  // software prefetch of the next reflector (L2 latency off the chain)
  cplx vn[RPT];
  cplx tn = (n > 0) ? tau[n - 1] : cmk(0.0, 0.0);
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int r = tid + q * NT, k = n - 1;
    vn[q] = (k >= 0 && r > k && r < m) ? __ldg(A + (long long)k * lda + r) : cmk(0.0, 0.0);
  }
  for (int k = n - 1; k >= 0; --k) {
    const cplx tk = tn;
    cplx v[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int r = tid + q * NT;
      v[q] = (r == k) ? cmk(1.0, 0.0) : vn[q];
    }
    if (k > 0) {
      tn = tau[k - 1];
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int r = tid + q * NT;
        vn[q] = (r > k - 1 && r < m) ? __ldg(A + (long long)(k - 1) * lda + r) : cmk(0.0, 0.0);
      }
    }
    if (tk.x == 0.0 && tk.y == 0.0) continue;  // uniform across the CTA
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
  if (cw > 32) return cudaErrorNotSupported;
  constexpr int NB = 8;
  // >= 116 KB so that the 16 CTAs land on 16 different SMs (2 per SM halves the producer's pace)
  const size_t smem = std::max<size_t>(((size_t)cw * m + (size_t)NB * m + cw) * sizeof(cplx), 116 * 1024);
  if (smem > 200 * 1024) return cudaErrorNotSupported;
  cudaError_t e;
  // 512 threads: one warp per trailing column of a band (the per-reflector
  // critical path); m <= 256: the pivot column in registers (measured fastest)
  const bool reg = m <= 256;
  auto fn = reg ? qrc3_factor_kernel<512, NB, false, 8> : qrc3_factor_kernel<512, NB, false>;
  const int nthreads = 512;
  if ((e = set_smem_attr(reinterpret_cast<const void*>(fn), 200 * 1024)) != cudaSuccess) return e;
  if ((e = set_cluster_nonportable(reinterpret_cast<const void*>(fn))) != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3(Cu);
  cfg.blockDim = dim3(nthreads);
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
  unsigned* nog = nullptr;
  e = cudaLaunchKernelEx(&cfg, fn, A, lda, m, n, cw, tau, RH, ldrh, rh_rows, nog);
  static const int prof = std::getenv("TDVP_QR_PROF") ? 1 : 0;  // thread-safe once (lanes call this concurrently)
  if (prof && e == cudaSuccess) {
    unsigned long long z[16][4];
    cudaMemcpyFromSymbolAsync(z, g_qr_prof, sizeof(z), 0, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    unsigned long long ph[8];
    cudaMemcpyFromSymbolAsync(ph, g_qr_ph, sizeof(ph), 0, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    std::fprintf(stderr, "qrc3 cta1 phase-2 cycles: norm %llu params %llu scale+publish %llu bar %llu lookahead %llu\n",
                 ph[0], ph[1], ph[2], ph[3], ph[4]);
    unsigned long long zz[8] = {0};
    cudaMemcpyToSymbolAsync(g_qr_ph, zz, sizeof(zz), 0, cudaMemcpyHostToDevice, st);
    std::fprintf(stderr, "qrc3 m=%d n=%d cw=%d ctas=%d (us from start: phase1 end / phase2 end / batches)\n", m, n, cw, Cu);
    for (int c = 0; c < Cu && c < 16; ++c)
      std::fprintf(stderr, "  cta %2d: %8.1f %8.1f %4llu\n", c, (z[c][1] - z[0][0]) * 1e-3, (z[c][2] - z[0][0]) * 1e-3,
                   z[c][3]);
  }
  return e;
}

// Grid variant: bands of cw columns on up to one CTA per SM (cooperative launch)
cudaError_t qr_factor_grid(cudaStream_t st, cplx* A, long long lda, int m, int n, cplx* tau, cplx* RH, long long ldrh,
                           int rh_rows, unsigned* gcnt) {
  if (m < n || n < 1 || gcnt == nullptr) return cudaErrorInvalidValue;
  constexpr int NB = 4;
  auto fn = qrc3_factor_kernel<256, NB, true>;
  cudaError_t e;
  if ((e = set_smem_attr(reinterpret_cast<const void*>(fn), 200 * 1024)) != cudaSuccess) return e;
  // smallest band width whose shared memory fits and whose CTAs are co-resident
  int cw = std::max(1, (n + g_num_sms - 1) / g_num_sms);
  const size_t per_col = (size_t)m * sizeof(cplx);
  if (((size_t)cw * m + (size_t)NB * m + cw) * sizeof(cplx) > 200 * 1024) return cudaErrorNotSupported;
  (void)per_col;
  // prefer bands of 8+ columns (fewer, busier CTAs) while they fit
  while (cw < 8 && ((size_t)(2 * cw) * m + (size_t)NB * m + 2 * cw) * sizeof(cplx) <= 200 * 1024) cw *= 2;
  const int nct = (n + cw - 1) / cw;
  const size_t smem = ((size_t)cw * m + (size_t)NB * m + cw) * sizeof(cplx);
  int occ = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, smem)) != cudaSuccess) return e;
  if (occ * g_num_sms < nct) return cudaErrorNotSupported;
  if (RH != nullptr) {
    if ((e = cudaMemset2DAsync(RH, (size_t)ldrh * sizeof(cplx), 0, (size_t)rh_rows * sizeof(cplx), n, st)) !=
        cudaSuccess)
      return e;
  }
  if ((e = cudaMemsetAsync(gcnt, 0, sizeof(unsigned), st)) != cudaSuccess) return e;
  void* args[] = {(void*)&A, (void*)&lda, (void*)&m, (void*)&n, (void*)&cw, (void*)&tau, (void*)&RH, (void*)&ldrh,
                  (void*)&rh_rows, (void*)&gcnt};
  return cudaLaunchCooperativeKernel((void*)fn, dim3(nct), dim3(256), args, smem, st);
}

cudaError_t qr_apply_refl(cudaStream_t st, const cplx* A, long long lda, const cplx* tau, int m, int n, cplx* C,
                          long long ldc, int nc) {
  return qr_apply_refl2(st, A, lda, tau, m, n, C, ldc, nc, nullptr, 0, nullptr, 0, 0, nullptr, 0, 0);
}

cudaError_t qr_apply_refl2(cudaStream_t st, const cplx* A0, long long lda0, const cplx* tau0, int m0, int n0, cplx* C0,
                           long long ldc0, int nc0, const cplx* A1, long long lda1, const cplx* tau1, int m1, int n1,
                           cplx* C1, long long ldc1, int nc1) {
  const QrApplyJob j0{A0, lda0, tau0, m0, n0, C0, ldc0, nc0};
  const QrApplyJob j1{A1, lda1, tau1, m1, n1, C1, ldc1, nc1};
  const int nb0 = (nc0 + 7) / 8, nb1 = A1 ? (nc1 + 7) / 8 : 0;
  const int m = std::max(m0, A1 ? m1 : 0);
  const int blocks = nb0 + nb1;
  // measured: 128 threads (1-2 rows each) fastest up to 256 rows
  if (m <= 128) qr_apply_refl_kernel<1, 128><<<blocks, 128, 0, st>>>(j0, j1, nb0);
  else if (m <= 256) qr_apply_refl_kernel<2, 128><<<blocks, 128, 0, st>>>(j0, j1, nb0);
  else if (m <= 512) qr_apply_refl_kernel<2, 256><<<blocks, 256, 0, st>>>(j0, j1, nb0);
  else if (m <= 1024) qr_apply_refl_kernel<4, 256><<<blocks, 256, 0, st>>>(j0, j1, nb0);
  else return cudaErrorNotSupported;
  return cudaGetLastError();
}
