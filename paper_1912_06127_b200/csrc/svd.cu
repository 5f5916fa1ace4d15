// Truncated SVD of the two-site matrix Theta' (PAPER.md:455 Fig 6, :493-499
// eq:discweight, :510 epsilon) by blocked one-sided (Hestenes) Jacobi.
//
// The matrix (or its conjugate transpose, so that rows >= cols) is held
// column-major together with the accumulated right rotations:
//   Y = [X ; V]  (mr + nc rows, nc columns),  X = M V  ->  columns U_c sigma_c.
// A sweep is a round-robin tournament over column blocks of b (4 or 8); in
// each round one CTA per block pair
//   1. forms the 2b x 2b Gram matrix of its columns (X rows only),
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
#include <cooperative_groups.h>
#include <cstdlib>
#include <cstdio>
namespace cg = cooperative_groups;

namespace {

__device__ unsigned long long g_svd_prof[8];  // cycles per phase (block 0), debug
#define PROF_MARK(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) { const unsigned long long _t = clock64(); g_svd_prof[i] += _t - prof_t; prof_t = _t; } } while (0)

constexpr int NTH = 256;
#ifndef INNER_SWEEPS
#define INNER_SWEEPS 1
#endif
#ifndef INNER_MODE
#define INNER_MODE 0
#endif

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

// ---------------------------------------------------------------------------
// Cooperative single-launch variant: all sweeps and rounds in one persistent
// kernel, grid-wide barrier between rounds, convergence decided on device
// (no host round trips).  Block pair = 2*BW columns per CTA; the inner
// Hermitian 2BW x 2BW Gram eigenproblem is solved by one warp.
template <int BW>
struct CoopCfg {
  static constexpr int PC = 2 * BW;
  // rows per staged tile: BW = 8 uses the register-tiled Gram/apply (64 rows,
  // 4 column groups x 64 row threads), else 6 loads in flight per thread
  static constexpr int TRc = (PC == 16) ? 128 : 1536 / PC;
  static constexpr bool TILED = (PC == 16);
  static constexpr int E = PC * PC;                // Gram entries
  static constexpr int EPT = (E + NTH - 1) / NTH;  // entries per thread
  static constexpr int S = (E >= NTH) ? 1 : NTH / E;  // row slices per entry
};

// Complex Jacobi rotation zeroing g = x_p^H x_q for column norms a = |x_p|^2,
// c = |x_q|^2 (3 long-latency ops): w = c - a, D = sqrt(w^2 + 4|g|^2),
// t e^{i phi} = 2 sgn(w) g / (|w| + D), cs = 1/sqrt(1 + t^2), sn = cs t e^{i phi}.
// x_p' = cs x_p - conj(sn) x_q ;  x_q' = sn x_p + cs x_q.  Returns false if
// |g|^2 <= tol2q a c (already orthogonal to the requested tolerance).
__device__ __forceinline__ bool rot_params(double a, double c, double gr, double gi, double tol2q, double& cs,
                                           cplx& sn) {
  const double ag2 = gr * gr + gi * gi;
  if (!(ag2 > 1e-300) || !(ag2 > tol2q * a * c)) return false;
  const double w = c - a;
  const double den = fabs(w) + sqrt(fma(w, w, 4.0 * ag2));
  const double f = copysign(2.0, w) / den;  // t e^{i phi} = f g
  const double t2 = f * f * ag2;
  cs = rsqrt(1.0 + t2);
  sn = cmk(cs * f * gr, cs * f * gi);
  return true;
}

// Inner block-pair solve, one warp, register resident (PC = 8 or 16 columns).
// G = D C D (D = sqrt diag G); C = L L^H (Cholesky, clamped pivots); R = L^H D
// satisfies R^H R = G, so one-sided Jacobi on the columns of R (held in
// registers: lane (c, h) owns rows [h*RC, (h+1)*RC) of column c of R and of
// Q) yields the rotation Q that orthogonalises the block pair.  Only column
// operations: partner chunks arrive by shuffle, dots reduce across the H
// chunk-lanes of a column.  Writes Q (PC x PC) to Qm.
template <int PC>
__device__ __forceinline__ void inner_reg(cplx (*G)[PC + 1], cplx (*Qm)[PC + 1], int ncols, double tol) {
  constexpr int H = 32 / PC, RC = PC / H;
  const int lane = threadIdx.x & 31;
  const int c = lane % PC, h = lane / PC;
  // --- scaled Cholesky of the leading ncols x ncols block, L stored in Qm (lower)
  __shared__ double s_d[PC];
  if (lane < PC) {
    const double gd = (lane < ncols) ? G[lane][lane].x : 0.0;
    s_d[lane] = gd > 0.0 ? sqrt(gd) : 0.0;
  }
  __syncwarp();
  for (int k = 0; k < PC; ++k) {
    // lane i >= k computes L[i][k]
    if (lane < PC) {
      const int i = lane;
      cplx l = cmk(0, 0);
      if (k < ncols && i < ncols && i >= k && s_d[k] > 0.0 && s_d[i] > 0.0) {
        const cplx cik = cscale(G[i][k], 1.0 / (s_d[i] * s_d[k]));
        cplx acc = cik;
        for (int m = 0; m < k; ++m) acc = csub(acc, cmul(Qm[i][m], cconj(Qm[k][m])));
        if (i == k) {
          l = cmk(sqrt(fmax(acc.x, 1e-28)), 0.0);
        }
        Qm[i][k] = (i == k) ? l : acc;  // off-diagonal: numerator, divided below
      } else if (i >= k) {
        Qm[i][k] = cmk(0, 0);
      }
    }
    __syncwarp();
    if (lane < PC && lane > k) {
      const double lkk = Qm[k][k].x;
      if (lkk > 0.0) Qm[lane][k] = cscale(Qm[lane][k], 1.0 / lkk);
    }
    __syncwarp();
  }
  // --- registers: R[rho][c] = conj(L[c][rho]) d_c (rho <= c), Q = I
  cplx r[RC], q[RC];
#pragma unroll
  for (int k = 0; k < RC; ++k) {
    const int rho = h * RC + k;
    r[k] = (rho <= c && c < ncols) ? cscale(cconj(Qm[c][rho]), s_d[c]) : cmk(0, 0);
    q[k] = cmk(rho == c ? 1.0 : 0.0, 0.0);
  }
  __syncwarp();
  const double tol2q = 0.0625 * tol * tol;
  for (int sweep = 0; sweep < INNER_SWEEPS; ++sweep) {
    double offs = 0.0;
#pragma unroll 1
    for (int rd = 0; rd < PC - 1; ++rd) {
      int pa, pb;
      // partner of column c in round rd (circle method, player PC-1 fixed)
      {
        const int m = PC - 1;
        int partner;
        if (c == PC - 1) partner = rd % m;
        else if (c == rd % m) partner = PC - 1;
        else partner = (2 * rd - c + 2 * m) % m;
        pa = min(c, partner);
        pb = max(c, partner);
      }
      const bool is_p = (c == pa);
      const int plane = (is_p ? pb : pa) + PC * h;
      cplx pr[RC], pq[RC];
#pragma unroll
      for (int k = 0; k < RC; ++k) {
        pr[k].x = __shfl_sync(0xffffffffu, r[k].x, plane);
        pr[k].y = __shfl_sync(0xffffffffu, r[k].y, plane);
        pq[k].x = __shfl_sync(0xffffffffu, q[k].x, plane);
        pq[k].y = __shfl_sync(0xffffffffu, q[k].y, plane);
      }
      double a = 0.0, cc = 0.0, gr = 0.0, gi = 0.0;
#pragma unroll
      for (int k = 0; k < RC; ++k) {
        const cplx xp = is_p ? r[k] : pr[k];
        const cplx xq = is_p ? pr[k] : r[k];
        a += cabs2(xp);
        cc += cabs2(xq);
        gr = fma(xp.x, xq.x, fma(xp.y, xq.y, gr));
        gi = fma(xp.x, xq.y, fma(-xp.y, xq.x, gi));
      }
#pragma unroll
      for (int o = PC; o < 32; o <<= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        cc += __shfl_xor_sync(0xffffffffu, cc, o);
        gr += __shfl_xor_sync(0xffffffffu, gr, o);
        gi += __shfl_xor_sync(0xffffffffu, gi, o);
      }
      const double ag2 = gr * gr + gi * gi;
      if (a > 0.0 && cc > 0.0 && pb < ncols) {
        offs = fmax(offs, ag2 / (a * cc));
        double cs;
        cplx sn;
        if (rot_params(a, cc, gr, gi, tol2q, cs, sn)) {
          // p: x_p' = cs x_p - conj(sn) x_q ;  q: x_q' = sn x_p + cs x_q
          const cplx f = is_p ? cmk(-sn.x, sn.y) : sn;
#pragma unroll
          for (int k = 0; k < RC; ++k) {
            r[k] = cadd(cscale(r[k], cs), cmul(f, pr[k]));
            q[k] = cadd(cscale(q[k], cs), cmul(f, pq[k]));
          }
        }
      }
    }
    offs = warp_max(offs);
    if (offs <= tol2q) break;
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < RC; ++k) Qm[h * RC + k][c] = q[k];
  __syncwarp();
}

// Alternative inner solve (INNER_MODE 0): two-sided Jacobi on the Gram
// matrix in shared memory by one warp (one task per lane per phase).
template <int PC>
__device__ __forceinline__ void inner_smem(cplx (*G)[PC + 1], cplx (*Qm)[PC + 1], int ncols, double tol, int* rp,
                                           int* rq, double* rc, cplx* rs) {
  const int lane = threadIdx.x & 31;
  const double tol2q = 0.0625 * tol * tol;
  for (int e = lane; e < PC * PC; e += 32) Qm[e / PC][e % PC] = cmk((e / PC) == (e % PC) ? 1.0 : 0.0, 0.0);
  __syncwarp();
  const int n2 = ncols + (ncols & 1);
  for (int sweep = 0; sweep < INNER_SWEEPS; ++sweep) {
    for (int r = 0; r < n2 - 1; ++r) {
      if (lane < n2 / 2) {
        int p, q;
        rr_pair(n2, r, lane, p, q);
        double cs = 1.0;
        cplx sn = cmk(0, 0);
        if (q < ncols) {
          const double a = G[p][p].x, c = G[q][q].x;
          if (a > 0.0 && c > 0.0 && !rot_params(a, c, G[p][q].x, G[p][q].y, tol2q, cs, sn)) {
            cs = 1.0;
            sn = cmk(0, 0);
          }
        }
        rp[lane] = p;
        rq[lane] = q;
        rc[lane] = cs;
        rs[lane] = sn;
      }
      __syncwarp();
      for (int e = lane; e < (n2 / 2) * PC; e += 32) {
        const int pi = e / PC, row = e - pi * PC;
        const int p = rp[pi], q = rq[pi];
        if (q >= ncols || row >= ncols || (rs[pi].x == 0.0 && rs[pi].y == 0.0)) continue;
        const double cs = rc[pi];
        const cplx sn = rs[pi];
        const cplx gp = G[row][p], gq = G[row][q];
        G[row][p] = csub(cscale(gp, cs), cmul(cconj(sn), gq));
        G[row][q] = cadd(cmul(sn, gp), cscale(gq, cs));
        const cplx qp = Qm[row][p], qq = Qm[row][q];
        Qm[row][p] = csub(cscale(qp, cs), cmul(cconj(sn), qq));
        Qm[row][q] = cadd(cmul(sn, qp), cscale(qq, cs));
      }
      __syncwarp();
      for (int e = lane; e < (n2 / 2) * PC; e += 32) {
        const int pi = e / PC, col = e - pi * PC;
        const int p = rp[pi], q = rq[pi];
        if (q >= ncols || col >= ncols || (rs[pi].x == 0.0 && rs[pi].y == 0.0)) continue;
        const double cs = rc[pi];
        const cplx sn = rs[pi];
        const cplx gp = G[p][col], gq = G[q][col];
        G[p][col] = csub(cscale(gp, cs), cmul(sn, gq));
        G[q][col] = cadd(cmul(cconj(sn), gp), cscale(gq, cs));
      }
      __syncwarp();
      if (lane < n2 / 2) {
        const int p = rp[lane], q = rq[lane];
        if (q < ncols && !(rs[lane].x == 0.0 && rs[lane].y == 0.0)) {
          G[p][q] = cmk(0, 0);
          G[q][p] = cmk(0, 0);
          G[p][p].y = 0.0;
          G[q][q].y = 0.0;
        }
      }
      __syncwarp();
    }
  }
}

template <int BW>
__device__ void coop_pair(cplx* Y, long long ldy, int mr, int nc, int nb, int nbe, int round, int pair, double tol,
                          double* off_cur, cplx (*G)[2 * BW + 1], cplx (*Qm)[2 * BW + 1], cplx (*tile)[2 * BW + 1],
                          cplx* red, int* cols, int* s_ncols, int* rp, int* rq, double* rc, cplx* rs,
                          double* s_off) {
  using Cf = CoopCfg<BW>;
  constexpr int PC = Cf::PC, TRc = Cf::TRc;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  unsigned long long prof_t = clock64();
  if (tid == 0) {
    int a, b;
    rr_pair(nbe, round, pair, a, b);
    int k = 0;
    for (int blk : {a, b}) {
      if (blk >= nb) continue;
      for (int c = blk * BW; c < min(nc, blk * BW + BW); ++c) cols[k++] = c;
    }
    *s_ncols = k;
  }
  __syncthreads();
  const int ncols = *s_ncols;
  if (ncols < 2) return;

  // ---- Gram matrix over the X rows (next tile prefetched into registers)
  constexpr int LPT = (TRc * PC) / NTH;  // loads per thread per tile
  cplx acc[Cf::EPT], acc2[Cf::EPT];
#pragma unroll
  for (int u = 0; u < Cf::EPT; ++u) acc[u] = acc2[u] = cmk(0, 0);
  const int slice = (Cf::S > 1) ? (tid % Cf::S) : 0;
  const int ebase = (Cf::S > 1) ? (tid / Cf::S) : tid;
  cplx pre[LPT];
  auto fetch = [&](int r0, int limit) {
#pragma unroll
    for (int u = 0; u < LPT; ++u) {
      const int e = tid + u * NTH;
      const int c = e / TRc, rr = e - c * TRc;
      pre[u] = (c < ncols && r0 + rr < limit) ? __ldcg(Y + (long long)cols[c] * ldy + r0 + rr) : cmk(0, 0);
    }
  };
  auto stash = [&]() {
#pragma unroll
    for (int u = 0; u < LPT; ++u) {
      const int e = tid + u * NTH;
      tile[e - (e / TRc) * TRc][e / TRc] = pre[u];
    }
  };
  if constexpr (Cf::TILED) {
    // register-tiled Gram: thread = (4x4 block of G, row slice of 16); per
    // row 8 shared loads (warp-broadcast) feed 16 complex MACs, so the loop
    // is FP64-pipe bound instead of shared-memory bound (2 loads per MAC)
    const int blk = tid & 15, sl = tid >> 4, i0 = (blk >> 2) * 4, j0 = (blk & 3) * 4;
    cplx g[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) g[a][b] = cmk(0, 0);
    fetch(0, mr);
    for (int r0 = 0; r0 < mr; r0 += TRc) {
      stash();
      __syncthreads();
      if (r0 + TRc < mr) fetch(r0 + TRc, mr);
#pragma unroll
      for (int m = 0; m < TRc / 16; ++m) {
        const int rr = sl + 16 * m;
        cplx ti[4], tj[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          ti[a] = tile[rr][i0 + a];
          tj[a] = tile[rr][j0 + a];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            g[a][b].x = fma(ti[a].x, tj[b].x, fma(ti[a].y, tj[b].y, g[a][b].x));
            g[a][b].y = fma(ti[a].x, tj[b].y, fma(-ti[a].y, tj[b].x, g[a][b].y));
          }
      }
      __syncthreads();
    }
    // reduce the 16 row slices: lanes l, l ^ 16 (one shuffle), then the 8 warps in order
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        g[a][b].x += __shfl_xor_sync(0xffffffffu, g[a][b].x, 16);
        g[a][b].y += __shfl_xor_sync(0xffffffffu, g[a][b].y, 16);
      }
    for (int w = 0; w < NTH / 32; ++w) {
      if (wid == w && lane < 16) {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) G[i0 + a][j0 + b] = w == 0 ? g[a][b] : cadd(G[i0 + a][j0 + b], g[a][b]);
      }
      __syncthreads();
    }
  } else {
  fetch(0, mr);
  for (int r0 = 0; r0 < mr; r0 += TRc) {
    stash();
    __syncthreads();
    if (r0 + TRc < mr) fetch(r0 + TRc, mr);
#pragma unroll
    for (int u = 0; u < Cf::EPT; ++u) {
      const int e = ebase + u * NTH;
      if (e < Cf::E) {
        const int i = e / PC, j = e - i * PC;
#pragma unroll 4
        for (int rr = slice; rr < TRc; rr += 2 * Cf::S) {
          const cplx a = tile[rr][i], b = tile[rr][j];
          acc[u].x = fma(a.x, b.x, acc[u].x);
          acc[u].x = fma(a.y, b.y, acc[u].x);
          acc[u].y = fma(a.x, b.y, acc[u].y);
          acc[u].y = fma(-a.y, b.x, acc[u].y);
          const int r2 = rr + Cf::S;
          if (r2 < TRc) {
            const cplx a2 = tile[r2][i], b2 = tile[r2][j];
            acc2[u].x = fma(a2.x, b2.x, acc2[u].x);
            acc2[u].x = fma(a2.y, b2.y, acc2[u].x);
            acc2[u].y = fma(a2.x, b2.y, acc2[u].y);
            acc2[u].y = fma(-a2.y, b2.x, acc2[u].y);
          }
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < Cf::EPT; ++u) acc[u] = cadd(acc[u], acc2[u]);
  if (Cf::S > 1) {
    red[tid] = acc[0];
    __syncthreads();
    if (tid < Cf::E) {
      cplx t = cmk(0, 0);
      for (int q = 0; q < Cf::S; ++q) t = cadd(t, red[tid * Cf::S + q]);
      G[tid / PC][tid % PC] = t;
    }
  } else {
#pragma unroll
    for (int u = 0; u < Cf::EPT; ++u) {
      const int e = ebase + u * NTH;
      if (e < Cf::E) G[e / PC][e % PC] = acc[u];
    }
  }
  }  // !TILED
  for (int e = tid; e < PC * PC; e += NTH) Qm[e / PC][e % PC] = cmk((e / PC) == (e % PC) ? 1.0 : 0.0, 0.0);
  __syncthreads();

  PROF_MARK(0);
  // ---- relative off-diagonal measure (whole CTA)
  double off = 0.0;
  for (int e = tid; e < PC * PC; e += NTH) {
    const int i = e / PC, j = e - i * PC;
    if (i < j && j < ncols) {
      const double di = G[i][i].x, dj = G[j][j].x;
      if (di > 0.0 && dj > 0.0) off = fmax(off, cabs2(G[i][j]) / (di * dj));  // squared
    }
  }
  off = warp_max(off);
  if (lane == 0) s_off[wid] = off;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < NTH / 32; ++w) t = fmax(t, s_off[w]);
    t = sqrt(t);
    s_off[0] = t;
    atomic_max_nonneg(off_cur, t);
  }
  __syncthreads();
  const double off0 = s_off[0];
  __syncthreads();
  if (off0 <= tol) return;

  PROF_MARK(1);
  // ---- inner solve by warp 0: Q with (X Q)^H (X Q) diagonal, from G = X^H X
#if INNER_MODE == 1
  if (wid == 0) inner_reg<PC>(G, Qm, ncols, tol);
#else
  if (wid == 0) inner_smem<PC>(G, Qm, ncols, tol, rp, rq, rc, rs);
#endif
  __syncthreads();
  PROF_MARK(2);

  // ---- apply: Y_pair <- Y_pair Q over all mr + nc rows (next tile prefetched)
  const int rows = mr + nc;
  if constexpr (Cf::TILED) {
    // register-tiled: thread = (row of the tile, group of 4 output columns);
    // per k one row load + 4 broadcast Q loads for 4 complex MACs
    const int c0 = (tid >> 6) * 4, rr = tid & 63;
    fetch(0, rows);
    for (int r0 = 0; r0 < rows; r0 += TRc) {
      stash();
      __syncthreads();
      if (r0 + TRc < rows) fetch(r0 + TRc, rows);
#pragma unroll
      for (int hh = 0; hh < TRc / 64; ++hh) {
        const int r = rr + 64 * hh;
        cplx o[4] = {cmk(0, 0), cmk(0, 0), cmk(0, 0), cmk(0, 0)};
        for (int k = 0; k < ncols; ++k) {
          const cplx a = tile[r][k];
#pragma unroll
          for (int q = 0; q < 4; ++q) cfma(o[q], a, Qm[k][c0 + q]);
        }
        if (r0 + r < rows) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (c0 + q < ncols) __stcg(Y + (long long)cols[c0 + q] * ldy + r0 + r, o[q]);
        }
      }
      __syncthreads();
    }
    PROF_MARK(3);
    return;
  }
  fetch(0, rows);
  for (int r0 = 0; r0 < rows; r0 += TRc) {
    stash();
    __syncthreads();
    if (r0 + TRc < rows) fetch(r0 + TRc, rows);
#pragma unroll
    for (int u = 0; u < LPT; ++u) {
      const int e = tid + u * NTH;
      const int c = e / TRc, rr = e - c * TRc;
      if (c < ncols && r0 + rr < rows) {
        cplx a = cmk(0, 0), b = cmk(0, 0);
        int k = 0;
        for (; k + 1 < ncols; k += 2) {
          cfma(a, tile[rr][k], Qm[k][c]);
          cfma(b, tile[rr][k + 1], Qm[k + 1][c]);
        }
        if (k < ncols) cfma(a, tile[rr][k], Qm[k][c]);
        __stcg(Y + (long long)cols[c] * ldy + r0 + rr, cadd(a, b));
      }
    }
    __syncthreads();
  }
  PROF_MARK(3);
}

template <int BW>
__global__ void __launch_bounds__(NTH) svd_coop_kernel(cplx* Y, long long ldy, int mr, int nc, int nb, int nbe,
                                                       double tol, int max_sweeps, double* offbuf, int* sweeps_out) {
  constexpr int PC = 2 * BW;
  using Cf = CoopCfg<BW>;
  __shared__ cplx G[PC][PC + 1];
  __shared__ cplx Qm[PC][PC + 1];
  __shared__ cplx tile[Cf::TRc][PC + 1];
  __shared__ cplx red[NTH];
  __shared__ int cols[PC];
  __shared__ int s_ncols;
  __shared__ int rp[PC / 2], rq[PC / 2];
  __shared__ double rc[PC / 2];
  __shared__ cplx rs[PC / 2];
  __shared__ double s_off[NTH / 32];
  cg::grid_group grid = cg::this_grid();
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    double* off_cur = offbuf + (sweep % 3);
    if (blockIdx.x == 0 && threadIdx.x == 0) offbuf[(sweep + 1) % 3] = 0.0;
    for (int round = 0; round < nbe - 1; ++round) {
      for (int pair = blockIdx.x; pair < nbe / 2; pair += gridDim.x)
        coop_pair<BW>(Y, ldy, mr, nc, nb, nbe, round, pair, tol, off_cur, G, Qm, tile, red, cols, &s_ncols, rp, rq,
                      rc, rs, s_off);
      {
        unsigned long long prof_t = clock64();
        grid.sync();
        PROF_MARK(4);
      }
    }
    const double off = __ldcg(off_cur);
    if (!(off > tol) || off * off <= 0.01 * tol) break;  // early stop: see svd_rjac.cu c_rj_early
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *sweeps_out = min(sweep + 1, max_sweeps);
}

// ---------------------------------------------------------------------------
// Shared-memory-resident variant (used when a block pair's full columns fit):
// the CTA stages all mr + nc rows of its 2*BW columns in shared memory and
// runs plain one-sided Hestenes rotations on them (dot products of the
// actual columns, no Gram matrix, no inner eigenproblem), one warp per
// column pair, INNER_SWEEPS inner sweeps, then writes the columns back.
template <int BW>
__global__ void __launch_bounds__(256) svd_coop_smem_kernel(cplx* Y, long long ldy, int mr, int nc, int nb,
                                                               int nbe, double tol, int max_sweeps, double* offbuf,
                                                               int* sweeps_out) {
  constexpr int PC = 2 * BW, NT = 256, WPP = 8 / BW;  // warps per column pair
  extern __shared__ __align__(16) unsigned char smraw[];
  cplx* sm = reinterpret_cast<cplx*>(smraw);
  __shared__ double s_part[8][4];
  __shared__ int cols[PC];
  __shared__ int s_ncols;
  __shared__ double s_off[BW];
  __shared__ int s_any;
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int rows = mr + nc;
  const int lds = rows;  // column stride in shared memory
  const double tol2q = 0.0625 * tol * tol;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    double* off_cur = offbuf + (sweep % 3);
    if (blockIdx.x == 0 && tid == 0) offbuf[(sweep + 1) % 3] = 0.0;
    for (int round = 0; round < nbe - 1; ++round) {
      for (int pair = blockIdx.x; pair < nbe / 2; pair += gridDim.x) {
        if (tid == 0) {
          int a, b;
          rr_pair(nbe, round, pair, a, b);
          int k = 0;
          for (int blk : {a, b}) {
            if (blk >= nb) continue;
            for (int c = blk * BW; c < min(nc, blk * BW + BW); ++c) cols[k++] = c;
          }
          s_ncols = k;
          s_any = 0;
        }
        if (tid < BW) s_off[tid] = 0.0;
        __syncthreads();
        const int ncols = s_ncols;
        if (ncols >= 2) {
          {
            // 8 independent loads in flight per thread
            const int total = ncols * rows;
            for (int base = tid; base < total; base += 8 * NT) {
              cplx v[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int e = base + u * NT;
                if (e < total) {
                  const int c = e / rows, r = e - c * rows;
                  v[u] = __ldcg(Y + (long long)cols[c] * ldy + r);
                }
              }
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int e = base + u * NT;
                if (e < total) sm[e] = v[u];  // sm[c * lds + r] with lds == rows
              }
            }
          }
          __syncthreads();
          const int n2 = ncols + (ncols & 1);
          for (int isw = 0; isw < INNER_SWEEPS; ++isw) {
            for (int r = 0; r < n2 - 1; ++r) {
              const int pi = wid / WPP, part = wid - pi * WPP;
              int p = 0, q = 0;
              bool active = pi < n2 / 2;
              if (active) {
                rr_pair(n2, r, pi, p, q);
                active = q < ncols;
              }
              cplx* xp = sm + p * lds;
              cplx* xq = sm + q * lds;
              if (active) {
                double a0 = 0, a1 = 0, c0 = 0, c1 = 0, gr0 = 0, gr1 = 0, gi0 = 0, gi1 = 0;
                constexpr int STR = 32 * WPP;
                int rr = lane + 32 * part;
                for (; rr + STR < mr; rr += 2 * STR) {
                  const cplx u0 = xp[rr], v0 = xq[rr], u1 = xp[rr + STR], v1 = xq[rr + STR];
                  a0 += cabs2(u0); a1 += cabs2(u1);
                  c0 += cabs2(v0); c1 += cabs2(v1);
                  gr0 = fma(u0.x, v0.x, fma(u0.y, v0.y, gr0)); gr1 = fma(u1.x, v1.x, fma(u1.y, v1.y, gr1));
                  gi0 = fma(u0.x, v0.y, fma(-u0.y, v0.x, gi0)); gi1 = fma(u1.x, v1.y, fma(-u1.y, v1.x, gi1));
                }
                for (; rr < mr; rr += STR) {
                  const cplx u0 = xp[rr], v0 = xq[rr];
                  a0 += cabs2(u0);
                  c0 += cabs2(v0);
                  gr0 = fma(u0.x, v0.x, fma(u0.y, v0.y, gr0));
                  gi0 = fma(u0.x, v0.y, fma(-u0.y, v0.x, gi0));
                }
                const double pa = warp_sum(a0 + a1), pc = warp_sum(c0 + c1);
                const double pgr = warp_sum(gr0 + gr1), pgi = warp_sum(gi0 + gi1);
                if (lane == 0) {
                  s_part[wid][0] = pa;
                  s_part[wid][1] = pc;
                  s_part[wid][2] = pgr;
                  s_part[wid][3] = pgi;
                }
              }
              if (WPP > 1) __syncthreads(); else __syncwarp();
              if (active) {
                double a = 0, c = 0, gr = 0, gi = 0;
#pragma unroll
                for (int u = 0; u < WPP; ++u) {
                  a += s_part[pi * WPP + u][0];
                  c += s_part[pi * WPP + u][1];
                  gr += s_part[pi * WPP + u][2];
                  gi += s_part[pi * WPP + u][3];
                }
                const double ag2 = gr * gr + gi * gi;
                double cs = 1.0;
                cplx sn = cmk(0, 0);
                if (a > 0.0 && c > 0.0) {
                  if (isw == 0 && part == 0 && lane == 0) s_off[pi] = fmax(s_off[pi], ag2 / (a * c));
                  rot_params(a, c, gr, gi, tol2q, cs, sn);
                }
                if (sn.x != 0.0 || sn.y != 0.0) {
                  if (lane == 0) s_any = 1;
                  const cplx snc = cconj(sn);
                  for (int r2 = lane + 32 * part; r2 < rows; r2 += 32 * WPP) {
                    const cplx u = xp[r2], v = xq[r2];
                    xp[r2] = csub(cscale(u, cs), cmul(snc, v));
                    xq[r2] = cadd(cmul(sn, u), cscale(v, cs));
                  }
                }
              }
              __syncthreads();
            }
          }
          if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < BW; ++w) t = fmax(t, s_off[w]);
            atomic_max_nonneg(off_cur, sqrt(t));
          }
          if (s_any) {
            const int total = ncols * rows;
#pragma unroll 4
            for (int e = tid; e < total; e += NT) {
              const int c = e / rows, r = e - c * rows;
              __stcg(Y + (long long)cols[c] * ldy + r, sm[e]);
            }
          }
        }
        __syncthreads();
      }
      grid.sync();
    }
    const double off = __ldcg(off_cur);
    if (!(off > tol)) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *sweeps_out = min(sweep + 1, max_sweeps);
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
  ires[5] = nz;
  dres[0] = w;
  dres[1] = s1;
}

// Column presorting for the QR preconditioner (Drmac-Veselic: sorting the
// columns of X by decreasing norm before X = Q1 R1 makes R1 and R2 graded and
// cuts Jacobi sweeps; measured 45 -> 38 sweeps over six Theta of a c1-shaped
// run).  Single CTA: perm[rank] = c, perm[nc + c] = rank, ties by index.
__global__ void svd_presort_kernel(const double* __restrict__ nrm, int nc, int* perm) {
  extern __shared__ double s_n[];
  for (int c = threadIdx.x; c < nc; c += blockDim.x) s_n[c] = nrm[c];
  __syncthreads();
  for (int c = threadIdx.x; c < nc; c += blockDim.x) {
    const double v = s_n[c];
    int r = 0;
    for (int j = 0; j < nc; ++j) {
      const double u = s_n[j];
      r += (u > v) || (u == v && j < c);
    }
    perm[min(r, nc - 1)] = c;
    perm[nc + c] = r;
  }
}

// Q1[:, j] = X[:, perm[j]] (X = rows [0, mr) of Y)
__global__ void svd_permcopy_kernel(const cplx* __restrict__ Y, long long ldy, int mr, int nc,
                                    const int* __restrict__ perm, cplx* Q1) {
  const long long total = (long long)mr * nc;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(e / mr), r = (int)(e - (long long)j * mr);
    const int c = min(max(perm[j], 0), nc - 1);
    Q1[e] = Y[(long long)c * ldy + r];
  }
}

__global__ void svd_write_kernel(const cplx* __restrict__ Y, long long ldy, const int* __restrict__ order,
                                 const double* __restrict__ sigma, const int* __restrict__ ires, int m, int n, int mr,
                                 bool transposed, cplx* psiL, cplx* psiR, double* lam, double* vinv,
                                 const int* __restrict__ iperm) {
  const int chi = ires[0];
  // Psi_L: m x chi ; Psi_R: chi x n
  const long long nL = (long long)m * chi, nR = (long long)chi * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nL + nR + chi;
       e += (long long)gridDim.x * blockDim.x) {
    if (e < nL) {
      const int r = (int)(e / chi), k = (int)(e - (long long)r * chi);
      const int c = order[k];
      psiL[e] = transposed ? cscale(Y[(long long)c * ldy + mr + (iperm ? iperm[r] : r)], sigma[c])
                           : Y[(long long)c * ldy + r];
    } else if (e < nL + nR) {
      const long long f = e - nL;
      const int k = (int)(f / n), col = (int)(f - (long long)k * n);
      const int c = order[k];
      psiR[f] = transposed ? cconj(Y[(long long)c * ldy + col])
                           : cscale(cconj(Y[(long long)c * ldy + mr + (iperm ? iperm[col] : col)]), sigma[c]);
    } else {
      const int k = (int)(e - nL - nR);
      const double s = sigma[order[k]];
      lam[k] = s;
      vinv[k] = 1.0 / s;
    }
  }
}

}  // namespace

size_t svd_qr_work_elems(int m, int n) {
  const long long mr = std::max(m, n), nc = std::min(m, n);
  // Q1 (mr x nc) + Vc1 (nc x mr) + Q2, Vc2 (nc x nc) + T1, T2 + tau1, tau2 + W1, W2 (nc x 32)
  // + split-K partials of the V^H C products (16 x nc x 32)
  return (size_t)(2 * mr * nc + 2 * nc * nc + 2 * 32 * (nc + 32) + 2 * nc + 2 * 32 * nc + 16 * 32 * nc + 64);
}

size_t svd_work_elems(int m, int n) {
  const long long mr = std::max(m, n), nc = std::min(m, n);
  return (size_t)(mr + nc) * nc;
}

cudaError_t svd_truncate_split(cudaStream_t st, const SvdDev& d, const cplx* theta, int m, int n,
                               const TruncParams& tp, cplx* psiL, cplx* psiR, double* lam, double* vinv,
                               int* chi_out, double* w_out, int* r_out, int* chi_eps_out, int* sweeps_out,
                               float* jac_ms_out, double* jac_flop_out) {
  const bool transposed = m < n;
  const int mr = std::max(m, n), nc = std::min(m, n);
  const long long ldy = (long long)mr + nc;
  cudaError_t e;
  {
    const long long total = ldy * nc;
    const int blocks = (int)std::max<long long>(1, std::min<long long>((total + 255) / 256, 8LL * g_num_sms));
    svd_init_kernel<<<blocks, 256, 0, st>>>(d.Y, ldy, theta, m, n, mr, nc, transposed);
  }
  // QR preconditioning (Drmac-Veselic): X = Q1 R1, R1^H = Q2 R2, Jacobi on
  // X3 = R2^H (nc x nc) with V accumulated; then X = (Q1 U3) S (Q2 V)^H, i.e.
  // Q1 is applied to the converged X3 columns and Q2 to V before the split.
  const bool use_qr = nc >= 2 && d.qrbuf != nullptr && qr_kb_for(mr) > 0 && qr_kb_for(nc) > 0 &&
                      svd_qr_work_elems(m, n) <= d.qrbuf_elems;
  const bool presort = use_qr && d.perm != nullptr && nc * sizeof(double) <= 48 * 1024;
  QrWork w1{}, w2{};
  int x_rows = mr;
  bool qr_cluster = false;
  cplx* q1p = nullptr;
  cplx* q2p = nullptr;
  if (use_qr) {
    cplx* p = d.qrbuf;
    cplx* Q1 = p; p += (long long)mr * nc;
    cplx* Q2 = p; p += (long long)nc * nc;
    w1.kb = qr_kb_for(mr);
    w2.kb = qr_kb_for(nc);
    w1.Vc = p; w1.ldv = mr; p += (long long)nc * mr;
    w2.Vc = p; w2.ldv = nc; p += (long long)nc * nc;
    w1.T = p; p += 32LL * (nc + 32);
    w2.T = p; p += 32LL * (nc + 32);
    w1.tau = p; p += nc;
    w2.tau = p; p += nc;
    w1.W1 = w2.W1 = p; p += 32LL * nc;
    w1.W2 = w2.W2 = p; p += 32LL * nc;
    w1.gw = w2.gw = p; w1.gw_elems = w2.gw_elems = (size_t)16 * 32 * nc; p += 16LL * 32 * nc;
    if (presort) {
      // X P with P sorting the columns by decreasing norm; V = P (Q2 V3) at the write
      svd_colnorm_kernel<<<(nc + 7) / 8, 256, 0, st>>>(d.Y, ldy, mr, nc, d.sigma, d.ires + 2);
      svd_presort_kernel<<<1, 1024, nc * sizeof(double), st>>>(d.sigma, nc, d.perm);
      const long long total = (long long)mr * nc;
      const int blocks = (int)std::max<long long>(1, std::min<long long>((total + 255) / 256, 8LL * g_num_sms));
      svd_permcopy_kernel<<<blocks, 256, 0, st>>>(d.Y, ldy, mr, nc, d.perm, Q1);
    } else if ((e = cudaMemcpy2DAsync(Q1, (size_t)mr * sizeof(cplx), d.Y, (size_t)ldy * sizeof(cplx),
                                      (size_t)mr * sizeof(cplx), nc, cudaMemcpyDeviceToDevice, st)) != cudaSuccess) {
      return e;
    }
    qr_cluster = false;
    {
      // cluster-resident QR where the column bands fit shared memory, else
      // the same look-ahead QR over a cooperative grid
      e = qr_factor_cluster(st, Q1, mr, mr, nc, w1.tau, Q2, nc, nc);
      if (e == cudaSuccess) {
        if ((e = qr_factor_cluster(st, Q2, nc, nc, nc, w2.tau, d.Y, ldy, mr)) != cudaSuccess) return e;
        qr_cluster = true;
      } else if (e != cudaErrorNotSupported) {
        return e;
      } else {
        cudaGetLastError();
        unsigned* gcnt = d.flags;  // the Jacobi's counters are free before the Jacobi runs
        e = qr_factor_grid(st, Q1, mr, mr, nc, w1.tau, Q2, nc, nc, gcnt);
        if (e == cudaSuccess) {
          if ((e = qr_factor_grid(st, Q2, nc, nc, nc, w2.tau, d.Y, ldy, mr, gcnt)) != cudaSuccess) return e;
          qr_cluster = true;
        } else if (e != cudaErrorNotSupported) {
          return e;
        } else {
          cudaGetLastError();
        }
      }
    }
    if (!qr_cluster) {
      if ((e = qr_factor(st, w1, Q1, mr, mr, nc)) != cudaSuccess) return e;
      if ((e = qr_r_conjtrans(st, Q1, mr, nc, Q2, nc, nc)) != cudaSuccess) return e;
      if ((e = qr_factor(st, w2, Q2, nc, nc, nc)) != cudaSuccess) return e;
      if ((e = qr_r_conjtrans(st, Q2, nc, nc, d.Y, ldy, mr)) != cudaSuccess) return e;
    }
    q1p = Q1;
    q2p = Q2;
    x_rows = nc;
  }
  const double tol = std::max(4.0 * DBL_EPSILON * std::sqrt((double)x_rows), 1e-15);
  int sweeps = 0;
  const bool tj = jac_ms_out != nullptr && d.ev_jac[0] != nullptr;
  if (tj && (e = cudaEventRecord(d.ev_jac[0], st)) != cudaSuccess) return e;
  // block Jacobi on DMMA (svd_bjac.cu) from 300 columns (tools/svd_once.py,
  // random n x n: 384 9.8 vs 11.3 ms for the register-resident rjac, 512 13.8
  // vs 15.6, 768 27.4 vs 34.1, 1024 42.3 vs 48.1; 256 and below rjac is as
  // fast or faster).  With several SVDs in flight (d.throughput: segment lanes,
  // U(1) sector workers) the grid-filling bjac would serialise them, so there
  // it only takes what rjac cannot (> 1024 columns).  TDVP_SVD_BJ_MIN
  // overrides the threshold (the parity tests force both paths).
  static const int bj_env = [] {  // thread-safe once (segment lanes / U(1) workers call this concurrently)
    const char* ev = std::getenv("TDVP_SVD_BJ_MIN");
    return ev ? std::atoi(ev) : -1;
  }();
  const int bj_min = bj_env >= 0 ? bj_env : (d.throughput ? 1025 : 300);
  if ((e = cudaMemsetAsync(d.dres + 2, 0, sizeof(double), st)) != cudaSuccess) return e;
  bool bj = false;
  if (nc >= bj_min && (e = svd_bjac_run(st, d, x_rows, mr, nc, ldy, tol, d.ires + 4, d.dres + 2)) !=
                          cudaErrorNotSupported) {
    // block Jacobi on the DMMA pipe (svd_bjac.cu)
    if (e != cudaSuccess) return e;
    sweeps = -1;
    bj = true;
  } else if (nc >= 2 && (e = svd_rjac_run(st, d, x_rows, mr, nc, ldy, tol, d.ires + 4)) != cudaErrorNotSupported) {
    // register-resident Jacobi (svd_rjac.cu)
    if (e != cudaSuccess) return e;
    sweeps = -1;
  } else if (nc >= 2) {
    cudaGetLastError();
    // fallback for shapes neither svd_bjac nor svd_rjac take: shared-memory-
    // resident block pairs when the columns fit (<= 200 KB), else the Gram variant
    const long long rows = (long long)mr + nc;
    int bw;
    bool smem_path;
    if (rows * 8 * 16 <= 200 * 1024) {
      // measured on B200 (microbench.py --svd, profiles/r1_microbench.md): the
      // shared-memory block-pair variant with b = 4 is fastest where it fits
      bw = 4;
      smem_path = true;
    } else {
      bw = nc <= 1024 ? 4 : 8;
      smem_path = false;
    }
    const int nb = (nc + bw - 1) / bw;
    const int nbe = std::max(2, nb + (nb & 1));
    if ((e = cudaMemsetAsync(d.offmax, 0, 4 * sizeof(double), st)) != cudaSuccess) return e;
    int max_sweeps = 60;
    int* sweeps_dev = d.ires + 4;
    void* args[] = {(void*)&d.Y, (void*)&ldy, (void*)&mr, (void*)&nc, (void*)&nb, (void*)&nbe, (void*)&tol,
                    (void*)&max_sweeps, (void*)&d.offmax, (void*)&sweeps_dev};
    void* fn;
    int nth;
    size_t dsm = 0;
    if (smem_path) {
      fn = bw == 4 ? (void*)svd_coop_smem_kernel<4> : (void*)svd_coop_smem_kernel<8>;
      nth = 256;
      dsm = (size_t)rows * 2 * bw * sizeof(cplx);
      if ((e = set_smem_attr(fn, 210 * 1024)) != cudaSuccess) return e;
    } else {
      fn = bw == 4 ? (void*)svd_coop_kernel<4> : (void*)svd_coop_kernel<8>;
      nth = NTH;
    }
    int occ = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, nth, dsm)) != cudaSuccess) return e;
    const int grid = std::max(1, std::min(nbe / 2, occ * g_num_sms));
    static const int prof = std::getenv("TDVP_SVD_PROF") ? 1 : 0;  // thread-safe once
    if (prof) {
      unsigned long long z[8] = {0};
      cudaMemcpyToSymbolAsync(g_svd_prof, z, sizeof(z), 0, cudaMemcpyHostToDevice, st);
    }
    if ((e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(nth), args, dsm, st)) != cudaSuccess) return e;
    if (prof) {
      unsigned long long z[8];
      cudaMemcpyFromSymbolAsync(z, g_svd_prof, sizeof(z), 0, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      std::fprintf(stderr, "svd prof n=%d grid=%d bw=%d smem=%d cycles: setup+gram %llu off %llu inner %llu apply %llu gsync %llu\n",
                   nc, grid, bw, (int)smem_path, z[0], z[1], z[2], z[3], z[4]);
    }
    sweeps = -1;  // read back with the truncation results
  }
  if (tj && (e = cudaEventRecord(d.ev_jac[1], st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(d.ires, 0, 4 * sizeof(int), st)) != cudaSuccess) return e;
  svd_colnorm_kernel<<<(nc + 7) / 8, 256, 0, st>>>(d.Y, ldy, mr, nc, d.sigma, d.ires + 2);
  svd_truncate_kernel<<<1, 1024, (2 * nc + 1) * sizeof(double), st>>>(d.sigma, nc, d.order, tp, d.ires, d.dres);
  if ((e = cudaMemcpyAsync(d.h_ibuf, d.ires, 8 * sizeof(int), cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(d.h_buf + 1, d.dres, 3 * sizeof(double), cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  if (d.h_ibuf[2] != 0 || !std::isfinite(d.h_buf[1]) || !(d.h_buf[2] > 0.0)) return cudaErrorUnknown;
  const int chi = d.h_ibuf[0];
  if (sweeps < 0) sweeps = d.h_ibuf[4];
  if (tj) {
    float ms = 0.f;
    if ((e = cudaEventElapsedTime(&ms, d.ev_jac[0], d.ev_jac[1])) != cudaSuccess) return e;
    *jac_ms_out = ms;
  }
  if (use_qr && qr_cluster) {
    // Q1 onto the X columns and Q2 onto V, one launch
    if ((e = qr_apply_refl2(st, q1p, mr, w1.tau, mr, nc, d.Y, ldy, nc, q2p, nc, w2.tau, nc, nc, d.Y + mr, ldy, nc)) !=
        cudaSuccess)
      return e;
  } else if (use_qr) {
    if ((e = qr_apply_q(st, w1, mr, nc, d.Y, ldy, nc)) != cudaSuccess) return e;
    if ((e = qr_apply_q(st, w2, nc, nc, d.Y + mr, ldy, nc)) != cudaSuccess) return e;
  }
  {
    const long long total = (long long)m * chi + (long long)chi * n + chi;
    const int blocks = (int)std::max<long long>(1, std::min<long long>((total + 255) / 256, 8LL * g_num_sms));
    svd_write_kernel<<<blocks, 256, 0, st>>>(d.Y, ldy, d.order, d.sigma, d.ires, m, n, mr, transposed, psiL, psiR,
                                             lam, vinv, presort ? d.perm + nc : nullptr);
  }
  *chi_out = chi;
  *w_out = d.h_buf[1];
  *r_out = d.h_ibuf[3];
  *chi_eps_out = d.h_ibuf[1];
  *sweeps_out = sweeps;
  if (jac_flop_out) *jac_flop_out = bj ? d.h_buf[3] : 0.0;
  return cudaGetLastError();
}
