// Truncated SVD of the two-site matrix Theta' (PAPER.md:455 Fig 6, :493-499
// eq:discweight, :510 epsilon) by blocked one-sided (Hestenes) Jacobi.
//
// The matrix (or its conjugate transpose, so that rows >= cols) is held
// column-major together with the accumulated right rotations:
//   Y = [X ; V]  (mr + nc rows, nc columns),  X = M V  ->  columns U_c sigma_c.
// A sweep is a round-robin tournament over column blocks of b = 16; in each
// round one CTA per block pair
//   1. forms the 32 x 32 Gram matrix of its columns (X rows only),
//   2. measures max |g_ij| / sqrt(g_ii g_jj) (convergence, relative),
//   3. diagonalises the Gram matrix by parallel-ordered complex Jacobi
//      rotations in shared memory, accumulating the unitary Q,
//   4. applies Y_pair <- Y_pair Q over all mr + nc rows.
// Singular values are the column norms of X (recomputed from the columns, so
// they carry the one-sided method's accuracy).  Then on device: descending
// order, the truncation rule (O-7 incl. the AMB-9 multiplet guard), discarded
// weight, and the split Psi_L = U S, Lambda = S, V = 1/S, Psi_R = S W^dagger.
#include <cfloat>
#include <cmath>
#include "common.cuh"
#include "kernels.h"

namespace {

constexpr int TB = 16;     // columns per block
constexpr int PC = 2 * TB; // columns per block pair
constexpr int NTH = 256;
constexpr int TR = 16;     // row tile
constexpr int OPT = TR * PC / NTH;  // apply outputs per thread

__device__ __forceinline__ void rr_pair(int n, int round, int i, int& a, int& b) {
  // circle method on n (even) players: player n-1 fixed
  const int m = n - 1;
  if (i == 0) {
    a = n - 1;
    b = round % m;
  } else {
    a = (round + i) % m;
    b = (round - i + m) % m;
  }
  if (a > b) { const int t = a; a = b; b = t; }
}

__global__ void svd_init_kernel(cplx* Y, long long ldy, const cplx* __restrict__ th, int m, int n, int mr, int nc,
                                bool transposed) {
  const long long rows = (long long)mr + nc;
  const long long total = rows * nc;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e / rows);
    const int r = (int)(e - (long long)c * rows);
    cplx v;
    if (r < mr) {
      v = transposed ? cconj(th[(long long)c * n + r]) : th[(long long)r * n + c];
    } else {
      v = cmk((r - mr) == c ? 1.0 : 0.0, 0.0);
    }
    Y[(long long)c * ldy + r] = v;
  }
}

__global__ void __launch_bounds__(NTH) svd_round_kernel(cplx* Y, long long ldy, int mr, int nc, int nb, int nbe,
                                                        int round, double tol, double* offmax) {
  __shared__ cplx G[PC][PC + 1];
  __shared__ cplx Qm[PC][PC + 1];
  __shared__ cplx tile[TR][PC + 1];
  __shared__ int cols[PC];
  __shared__ int s_ncols;
  __shared__ int rp[PC / 2], rq[PC / 2];
  __shared__ double rc[PC / 2];
  __shared__ cplx rs[PC / 2];
  __shared__ double s_off[NTH / 32];
  __shared__ double s_offall;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  if (tid == 0) {
    int a, b;
    rr_pair(nbe, round, blockIdx.x, a, b);
    int k = 0;
    for (int blk : {a, b}) {
      if (blk >= nb) continue;
      for (int c = blk * TB; c < min(nc, blk * TB + TB); ++c) cols[k++] = c;
    }
    s_ncols = k;
  }
  __syncthreads();
  const int ncols = s_ncols;
  if (ncols < 2) return;

  // ---- 1. Gram matrix of the X rows
  cplx acc[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) acc[s] = cmk(0, 0);
  for (int r0 = 0; r0 < mr; r0 += TR) {
    for (int e = tid; e < TR * PC; e += NTH) {
      const int c = e / TR, rr = e - c * TR;
      cplx v = cmk(0, 0);
      if (c < ncols && r0 + rr < mr) v = Y[(long long)cols[c] * ldy + r0 + rr];
      tile[rr][c] = v;
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int i = wid + 8 * s, j = lane;
#pragma unroll 8
      for (int rr = 0; rr < TR; ++rr) {
        const cplx a = tile[rr][i], b = tile[rr][j];
        acc[s].x = fma(a.x, b.x, acc[s].x);
        acc[s].x = fma(a.y, b.y, acc[s].x);
        acc[s].y = fma(a.x, b.y, acc[s].y);
        acc[s].y = fma(-a.y, b.x, acc[s].y);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int s = 0; s < 4; ++s) G[wid + 8 * s][lane] = acc[s];
  for (int e = tid; e < PC * PC; e += NTH) {
    const int i = e / PC, j = e - i * PC;
    Qm[i][j] = cmk(i == j ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();

  // ---- 2. relative off-diagonal measure
  auto measure_off = [&]() -> double {
    double off = 0.0;
    for (int e = tid; e < PC * PC; e += NTH) {
      const int i = e / PC, j = e - i * PC;
      if (i < j && j < ncols) {
        const double di = G[i][i].x, dj = G[j][j].x;
        if (di > 0.0 && dj > 0.0) off = fmax(off, sqrt(cabs2(G[i][j])) / sqrt(di * dj));
      }
    }
    off = warp_max(off);
    if (lane == 0) s_off[wid] = off;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < NTH / 32; ++w) t = fmax(t, s_off[w]);
      s_offall = t;
    }
    __syncthreads();
    return s_offall;
  };
  const double off0 = measure_off();
  if (tid == 0) atomic_max_nonneg(offmax, off0);
  if (off0 <= tol) return;

  // ---- 3. parallel-ordered Jacobi diagonalisation of G, Q accumulates
  const int n2 = ncols + (ncols & 1);
  for (int sweep = 0; sweep < 10; ++sweep) {
    for (int r = 0; r < n2 - 1; ++r) {
      if (tid < n2 / 2) {
        int p, q;
        rr_pair(n2, r, tid, p, q);
        double cs = 1.0;
        cplx sn = cmk(0, 0);  // sn * e^{i phi}
        if (q < ncols) {
          const double a = G[p][p].x, c = G[q][q].x;
          const cplx g = G[p][q];
          const double ag = sqrt(cabs2(g));
          if (ag > 0.0 && ag > 1e-300 && !(ag <= 0.25 * tol * sqrt(fmax(a, 0.0) * fmax(c, 0.0)))) {
            const double zeta = (c - a) / (2.0 * ag);
            const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            cs = 1.0 / sqrt(1.0 + t * t);
            const double s = cs * t;
            sn = cmk(s * g.x / ag, s * g.y / ag);
          }
        }
        rp[tid] = p;
        rq[tid] = q;
        rc[tid] = cs;
        rs[tid] = sn;
      }
      __syncthreads();
      // column updates of G and Q:  X_p' = cs X_p - conj(sn) X_q ; X_q' = sn X_p + cs X_q
      for (int e = tid; e < (n2 / 2) * PC; e += NTH) {
        const int pi = e / PC, row = e - pi * PC;
        const int p = rp[pi], q = rq[pi];
        if (q >= ncols || row >= ncols) continue;
        const double cs = rc[pi];
        const cplx sn = rs[pi];
        if (cs == 1.0 && sn.x == 0.0 && sn.y == 0.0) continue;
        {
          const cplx gp = G[row][p], gq = G[row][q];
          G[row][p] = csub(cscale(gp, cs), cmul(cconj(sn), gq));
          G[row][q] = cadd(cmul(sn, gp), cscale(gq, cs));
        }
        {
          const cplx qp = Qm[row][p], qq = Qm[row][q];
          Qm[row][p] = csub(cscale(qp, cs), cmul(cconj(sn), qq));
          Qm[row][q] = cadd(cmul(sn, qp), cscale(qq, cs));
        }
      }
      __syncthreads();
      // row updates of G:  G_p' = cs G_p - sn G_q ; G_q' = conj(sn) G_p + cs G_q
      for (int e = tid; e < (n2 / 2) * PC; e += NTH) {
        const int pi = e / PC, col = e - pi * PC;
        const int p = rp[pi], q = rq[pi];
        if (q >= ncols || col >= ncols) continue;
        const double cs = rc[pi];
        const cplx sn = rs[pi];
        if (cs == 1.0 && sn.x == 0.0 && sn.y == 0.0) continue;
        const cplx gp = G[p][col], gq = G[q][col];
        G[p][col] = csub(cscale(gp, cs), cmul(sn, gq));
        G[q][col] = cadd(cmul(cconj(sn), gp), cscale(gq, cs));
      }
      __syncthreads();
      if (tid < n2 / 2) {
        const int p = rp[tid], q = rq[tid];
        if (q < ncols && !(rc[tid] == 1.0 && rs[tid].x == 0.0 && rs[tid].y == 0.0)) {
          G[p][q] = cmk(0, 0);
          G[q][p] = cmk(0, 0);
          G[p][p].y = 0.0;
          G[q][q].y = 0.0;
        }
      }
      __syncthreads();
    }
    if (measure_off() <= 0.25 * tol) break;
  }

  // ---- 4. Y_pair <- Y_pair Q over all rows (X and accumulated V)
  const int rows = mr + nc;
  for (int r0 = 0; r0 < rows; r0 += TR) {
    for (int e = tid; e < TR * PC; e += NTH) {
      const int c = e / TR, rr = e - c * TR;
      cplx v = cmk(0, 0);
      if (c < ncols && r0 + rr < rows) v = Y[(long long)cols[c] * ldy + r0 + rr];
      tile[rr][c] = v;
    }
    __syncthreads();
    cplx outv[OPT];
#pragma unroll
    for (int s = 0; s < OPT; ++s) {
      const int e = tid + s * NTH;
      const int c = e / TR, rr = e - c * TR;
      cplx a = cmk(0, 0);
      if (c < ncols) {
        for (int k = 0; k < ncols; ++k) cfma(a, tile[rr][k], Qm[k][c]);
      }
      outv[s] = a;
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < OPT; ++s) {
      const int e = tid + s * NTH;
      const int c = e / TR, rr = e - c * TR;
      if (c < ncols && r0 + rr < rows) Y[(long long)cols[c] * ldy + r0 + rr] = outv[s];
    }
  }
}

__global__ void svd_colnorm_kernel(const cplx* __restrict__ Y, long long ldy, int mr, int nc, double* sigma,
                                   int* nonfinite) {
  const int warps = blockDim.x >> 5;
  const int c = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= nc) return;
  double s = 0.0;
  for (int r = lane; r < mr; r += 32) s += cabs2(Y[(long long)c * ldy + r]);
  s = warp_sum(s);
  if (lane == 0) {
    const double v = sqrt(s);
    sigma[c] = v;
    if (!isfinite(v)) *nonfinite = 1;
  }
}

// single CTA: order columns by descending sigma, apply the truncation rule
__global__ void svd_truncate_kernel(const double* __restrict__ sigma, int nc, int* order, TruncParams tp, int* ires,
                                    double* dres) {
  extern __shared__ double s_sorted[];  // [nc] sorted sigma, then [nc+1] suffix sums
  double* s_tail = s_sorted + nc;
  for (int c = threadIdx.x; c < nc; c += blockDim.x) {
    const double v = sigma[c];
    int rank = 0;
    for (int o = 0; o < nc; ++o) {
      const double u = sigma[o];
      rank += (u > v) || (u == v && o < c);
    }
    order[rank] = c;
    s_sorted[rank] = v;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int r = nc;
  const double s1 = s_sorted[0];
  const double eps = tp.eps > 0.0 ? tp.eps : 1e-14;
  int chi_eps = 0, nz = 0;
  for (int k = 0; k < r; ++k) {
    chi_eps += (s_sorted[k] >= eps * s1);
    nz += (s_sorted[k] > 0.0);
  }
  int chi_w = nz;
  if (tp.w_max > 0.0) {
    s_tail[r] = 0.0;
    for (int k = r - 1; k >= 0; --k) s_tail[k] = s_tail[k + 1] + s_sorted[k] * s_sorted[k];
    chi_w = nz;
    for (int c = 0; c <= r; ++c)
      if (s_tail[c] <= tp.w_max) { chi_w = c; break; }
    chi_w = max(chi_w, 1);
  }
  int chi = max(1, min(min(chi_eps, chi_w), tp.chi_max));
  // multiplet guard (AMB-9 + reading R-9b: absolute floor 1e-13 sigma_1)
  while (chi > 1 && chi < r && s_sorted[chi - 1] - s_sorted[chi] <= tp.delta * s_sorted[chi - 1] + 1e-13 * s1) --chi;
  double w = 0.0;
  for (int k = chi; k < r; ++k) w += s_sorted[k] * s_sorted[k];
  ires[0] = chi;
  ires[1] = chi_eps;
  ires[3] = r;
  dres[0] = w;
  dres[1] = s1;
}

__global__ void svd_write_kernel(const cplx* __restrict__ Y, long long ldy, const int* __restrict__ order,
                                 const double* __restrict__ sigma, const int* __restrict__ ires, int m, int n, int mr,
                                 bool transposed, cplx* psiL, cplx* psiR, double* lam, double* vinv) {
  const int chi = ires[0];
  // Psi_L: m x chi ; Psi_R: chi x n
  const long long nL = (long long)m * chi, nR = (long long)chi * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nL + nR + chi;
       e += (long long)gridDim.x * blockDim.x) {
    if (e < nL) {
      const int r = (int)(e / chi), k = (int)(e - (long long)r * chi);
      const int c = order[k];
      psiL[e] = transposed ? cscale(Y[(long long)c * ldy + mr + r], sigma[c]) : Y[(long long)c * ldy + r];
    } else if (e < nL + nR) {
      const long long f = e - nL;
      const int k = (int)(f / n), col = (int)(f - (long long)k * n);
      const int c = order[k];
      psiR[f] = transposed ? cconj(Y[(long long)c * ldy + col])
                           : cscale(cconj(Y[(long long)c * ldy + mr + col]), sigma[c]);
    } else {
      const int k = (int)(e - nL - nR);
      const double s = sigma[order[k]];
      lam[k] = s;
      vinv[k] = 1.0 / s;
    }
  }
}

}  // namespace

size_t svd_work_elems(int m, int n) {
  const long long mr = std::max(m, n), nc = std::min(m, n);
  return (size_t)(mr + nc) * nc;
}

cudaError_t svd_truncate_split(cudaStream_t st, const SvdDev& d, const cplx* theta, int m, int n,
                               const TruncParams& tp, cplx* psiL, cplx* psiR, double* lam, double* vinv,
                               int* chi_out, double* w_out, int* r_out, int* chi_eps_out, int* sweeps_out) {
  const bool transposed = m < n;
  const int mr = std::max(m, n), nc = std::min(m, n);
  const long long ldy = (long long)mr + nc;
  cudaError_t e;
  {
    const long long total = ldy * nc;
    const int blocks = (int)std::max<long long>(1, std::min<long long>((total + 255) / 256, 8LL * g_num_sms));
    svd_init_kernel<<<blocks, 256, 0, st>>>(d.Y, ldy, theta, m, n, mr, nc, transposed);
  }
  const int nb = (nc + TB - 1) / TB;
  const int nbe = std::max(2, nb + (nb & 1));
  const double tol = std::max(4.0 * DBL_EPSILON * std::sqrt((double)mr), 1e-15);
  int sweeps = 0;
  if (nc >= 2) {
    for (sweeps = 1; sweeps <= 40; ++sweeps) {
      if ((e = cudaMemsetAsync(d.offmax, 0, sizeof(double), st)) != cudaSuccess) return e;
      for (int r = 0; r < nbe - 1; ++r) svd_round_kernel<<<nbe / 2, NTH, 0, st>>>(d.Y, ldy, mr, nc, nb, nbe, r, tol, d.offmax);
      if ((e = cudaMemcpyAsync(d.h_buf, d.offmax, sizeof(double), cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
      if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
      if (!(d.h_buf[0] > tol)) break;
    }
  }
  if ((e = cudaMemsetAsync(d.ires, 0, 4 * sizeof(int), st)) != cudaSuccess) return e;
  svd_colnorm_kernel<<<(nc + 7) / 8, 256, 0, st>>>(d.Y, ldy, mr, nc, d.sigma, d.ires + 2);
  svd_truncate_kernel<<<1, 1024, (2 * nc + 1) * sizeof(double), st>>>(d.sigma, nc, d.order, tp, d.ires, d.dres);
  if ((e = cudaMemcpyAsync(d.h_ibuf, d.ires, 4 * sizeof(int), cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(d.h_buf + 1, d.dres, 2 * sizeof(double), cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  if (d.h_ibuf[2] != 0 || !std::isfinite(d.h_buf[1]) || !(d.h_buf[2] > 0.0)) return cudaErrorUnknown;
  const int chi = d.h_ibuf[0];
  {
    const long long total = (long long)m * chi + (long long)chi * n + chi;
    const int blocks = (int)std::max<long long>(1, std::min<long long>((total + 255) / 256, 8LL * g_num_sms));
    svd_write_kernel<<<blocks, 256, 0, st>>>(d.Y, ldy, d.order, d.sigma, d.ires, m, n, mr, transposed, psiL, psiR,
                                             lam, vinv);
  }
  *chi_out = chi;
  *w_out = d.h_buf[1];
  *r_out = d.h_ibuf[3];
  *chi_eps_out = d.h_ibuf[1];
  *sweeps_out = sweeps;
  return cudaGetLastError();
}
