// Register-resident blocked one-sided (Hestenes) Jacobi for the truncated SVD
// of the two-site matrix Theta' (Fig 6 "SVD"; truncation
// PAPER.md:493-499, :510).  Replaces the Jacobi stage of svd.cu for the
// shapes listed in kTab; init (Y = [X ; I]), column norms, truncation and the
// split are svd.cu's.
//
// Y (column-major, ld = ldy) holds the work matrix X (mr x nc, mr >= nc) in
// rows [0, mr) and the accumulated right rotations V (nc x nc) in rows
// [vofs, vofs + nc) (vofs >= mr; the QR-preconditioned path runs on an
// nc x nc X while V stays at the full problem's offset).  The right factor is accumulated (not recovered afterwards
// by a GEMM with Theta) because the inverse-canonical form multiplies both
// factors by V_j = 1/Lambda_j: each factor must be accurate
// RELATIVE to sigma_k, which only the rotated columns/rows give.
//
// One CTA per block pair (2*BW columns); each thread holds RX rows of X and
// RV rows of V of all 2*BW columns in REGISTERS.  All sweeps of the
// round-robin tournament over column blocks run in ONE persistent launch;
// between rounds the blocks go through L2 and the CTAs meet at a cluster
// barrier (all CTAs in one thread-block cluster, <= 16) or a grid barrier
// (cooperative launch).  An inner step applies BW disjoint rotations: the
// 4*BW dot products (|x_p|^2, |x_q|^2, x_p^H x_q) are reduced by a warp
// reduce-scatter butterfly and one shared-memory exchange (one
// __syncthreads per step); every warp derives the same rotation parameters.
// Round 0 of a sweep runs the full 2BW-column round robin (intra- and
// cross-block pairs), the other rounds the BW cross-block steps, so a sweep
// visits every column pair exactly once.
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cooperative_groups.h>
#include "common.cuh"
#include "kernels.h"
namespace cg = cooperative_groups;

namespace {

constexpr unsigned FULL = 0xffffffffu;

// Early stop (quadratic convergence of cyclic Jacobi): a sweep whose largest
// pair cosine c satisfies c^2 <= c_rj_early * tol leaves cosines ~ c^2 << tol,
// so the confirming sweep that would measure them is skipped (TDVP_RJ_EARLY=0:
// always confirm).  Measured off sequences: 7.6e-4, 6.1e-7, 1.0e-12, 2.5e-15.
__constant__ double c_rj_early = 0.01;

__device__ unsigned long long g_rj_prof[12];

__device__ __forceinline__ void rj_rr_pair(int n, int round, int i, int& a, int& b) {
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

// step s, slot i of the inner schedule (compile-time after unrolling)
template <int BW, bool CROSS>
__device__ __forceinline__ void rj_pq(int s, int i, int& p, int& q) {
  if (CROSS) {
    p = i;
    q = BW + (i + s) % BW;
  } else {
    constexpr int N = 2 * BW, M = N - 1;
    int a, b;
    if (i == 0) {
      a = N - 1;
      b = s % M;
    } else {
      a = (s + i) % M;
      b = (s - i + M) % M;
    }
    p = a < b ? a : b;
    q = a < b ? b : a;
  }
}

// 1/x and 1/sqrt(x) for normal positive x: MUFU seed + Newton steps (full
// double precision; the arguments below are always normal numbers).
__device__ __forceinline__ double rj_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ double rj_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y * fma(-h * y, y, 1.5);
}

// Complex Jacobi rotation zeroing g = x_p^H x_q (a = |x_p|^2, c = |x_q|^2):
// t e^{i phi} = 2 sgn(c-a) g / (|c-a| + sqrt((c-a)^2 + 4|g|^2)), cs = 1/sqrt(1+t^2),
// sn = cs t e^{i phi};  x_p' = cs x_p - conj(sn) x_q,  x_q' = sn x_p + cs x_q.
// Skipped (identity) when |g|^2 <= tol2q a c.
__device__ __forceinline__ bool rj_params(double a, double c, double gr, double gi, double tol2q, double& cs,
                                          double& sr, double& si, bool fastp) {
  const double ag2 = gr * gr + gi * gi;
  if (!(ag2 > 1e-300) || !(ag2 > tol2q * a * c)) return false;
  const double w = c - a;
  if (!fastp) {
    const double den = fabs(w) + sqrt(fma(w, w, 4.0 * ag2));
    const double f = copysign(2.0, w) / den;
    cs = rsqrt(fma(f * f, ag2, 1.0));
    sr = cs * f * gr;
    si = cs * f * gi;
    return true;
  }
  const double s = fma(w, w, 4.0 * ag2);
  const double den = fabs(w) + s * rj_rsqrt(s);
  const double f = copysign(2.0, w) * rj_rcp(den);
  cs = rj_rsqrt(fma(f * f, ag2, 1.0));
  sr = cs * f * gr;
  si = cs * f * gi;
  return true;
}

// per-step phase profile (block 0, thread 0): [4] dots [5] reduce+store [6] barrier [7] params+apply
#define RJ_T(i)                              \
  if (sprof) {                               \
    const unsigned long long _t = clock64(); \
    g_rj_prof[i] += _t - spt;                \
    spt = _t;                                \
  }

// CTA barrier over the NT threads doing the steps: __syncthreads when they
// are the whole CTA (NAMED = false), else named barrier 1 over NT threads.
template <int NT, bool NAMED>
__device__ __forceinline__ void rj_bar(int barid = 1) {
  if (NAMED) asm volatile("bar.sync %0, %1;" ::"r"(barid), "n"(NT) : "memory");
  else __syncthreads();
}

template <int BW, int RX, int RV, int NT, bool CROSS, bool NAMED = false>
__device__ __forceinline__ void rj_step(cplx (&x)[RX][2 * BW], cplx (&v)[(RV > 0 ? RV : 1)][2 * BW], int s,
                                        double (*red)[BW * 4],
                                        int lane, int wid, double tol2q, double& offacc, bool& rot, bool sprof,
                                        bool fastp, double (*pout)[3] = nullptr, int barid = 1) {
  constexpr int NV = 4 * BW;
  constexpr int H = (NV == 32) ? 5 : (NV == 16) ? 4 : 3;
  constexpr int SH = 5 - H;
  constexpr int NW = NT / 32;
  unsigned long long spt = sprof ? clock64() : 0ull;
  double val[NV];
#pragma unroll
  for (int i = 0; i < BW; ++i) {
    int p, q;
    rj_pq<BW, CROSS>(s, i, p, q);
    double a = 0.0, c = 0.0, gr = 0.0, gi = 0.0;
#pragma unroll
    for (int k = 0; k < RX; ++k) {
      const cplx u = x[k][p], w = x[k][q];
      a = fma(u.x, u.x, fma(u.y, u.y, a));
      c = fma(w.x, w.x, fma(w.y, w.y, c));
      gr = fma(u.x, w.x, fma(u.y, w.y, gr));
      gi = fma(u.x, w.y, fma(-u.y, w.x, gi));
    }
    val[4 * i] = a;
    val[4 * i + 1] = c;
    val[4 * i + 2] = gr;
    val[4 * i + 3] = gi;
  }
  if (sprof && val[0] + val[NV - 1] == -1.2345e300) g_rj_prof[11]++;
  RJ_T(4)
  // warp reduce-scatter: afterwards lane l holds the warp sum of value l >> SH
#pragma unroll
  for (int lev = 0; lev < H; ++lev) {
    const int msk = 16 >> lev;
    const int h = NV >> (lev + 1);
    const bool up = (lane & msk) != 0;
#pragma unroll
    for (int j = 0; j < h; ++j) {
      const double send = up ? val[j] : val[j + h];
      const double keep = up ? val[j + h] : val[j];
      val[j] = keep + __shfl_xor_sync(FULL, send, msk);
    }
  }
  double t = val[0];
#pragma unroll
  for (int msk = (16 >> H); msk >= 1; msk >>= 1) t += __shfl_xor_sync(FULL, t, msk);
  if ((lane & ((1 << SH) - 1)) == 0) red[wid][lane >> SH] = t;
  RJ_T(5)
  rj_bar<NT, NAMED>(barid);
  RJ_T(6)
  // every warp: CTA totals (tree over warps), rotation parameters of pair (lane % BW)
  double tot = 0.0;
  if (lane < NV) {
    double part[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) part[w] = red[w][lane];
#pragma unroll
    for (int st = 1; st < NW; st <<= 1)
#pragma unroll
      for (int w = 0; w + st < NW; w += 2 * st) part[w] += part[w + st];
    tot = part[0];
  }
  const int pi = lane % BW;
  const double a = __shfl_sync(FULL, tot, 4 * pi);
  const double c = __shfl_sync(FULL, tot, 4 * pi + 1);
  const double gr = __shfl_sync(FULL, tot, 4 * pi + 2);
  const double gi = __shfl_sync(FULL, tot, 4 * pi + 3);
  if (sprof && a + c + gr + gi == -1.2345e300) g_rj_prof[11]++;  // timer waits for the totals
  RJ_T(8)
  double cs = 1.0, sr = 0.0, si = 0.0;
  if (a > 0.0 && c > 0.0) {
    offacc = fmax(offacc, (gr * gr + gi * gi) / (a * c));
    rj_params(a, c, gr, gi, tol2q, cs, sr, si, fastp);
  }
  if (pout != nullptr && wid == 0 && lane < BW) {
    pout[lane][0] = cs;
    pout[lane][1] = sr;
    pout[lane][2] = si;
  }
  if (sprof && cs + sr + si == -1.2345e300) g_rj_prof[11]++;  // timer waits for the parameters
  RJ_T(9)
#pragma unroll
  for (int i = 0; i < BW; ++i) {
    int p, q;
    rj_pq<BW, CROSS>(s, i, p, q);
    const double csi = __shfl_sync(FULL, cs, i);
    const double sri = __shfl_sync(FULL, sr, i);
    const double sii = __shfl_sync(FULL, si, i);
    if (sri != 0.0 || sii != 0.0) {  // warp-uniform (identical in every warp)
      rot = true;
#pragma unroll
      for (int k = 0; k < RX; ++k) {
        const cplx u = x[k][p], w = x[k][q];
        x[k][p] = cmk(fma(csi, u.x, -fma(sri, w.x, sii * w.y)), fma(csi, u.y, -fma(sri, w.y, -sii * w.x)));
        x[k][q] = cmk(fma(csi, w.x, fma(sri, u.x, -sii * u.y)), fma(csi, w.y, fma(sri, u.y, sii * u.x)));
      }
#pragma unroll
      for (int k = 0; k < RV; ++k) {
        const cplx u = v[k][p], w = v[k][q];
        v[k][p] = cmk(fma(csi, u.x, -fma(sri, w.x, sii * w.y)), fma(csi, u.y, -fma(sri, w.y, -sii * w.x)));
        v[k][q] = cmk(fma(csi, w.x, fma(sri, u.x, -sii * u.y)), fma(csi, w.y, fma(sri, u.y, sii * u.x)));
      }
    }
  }
  if (sprof && x[RX - 1][0].x + v[0][2 * BW - 1].y == -1.2345e300) g_rj_prof[11]++;
  RJ_T(7)
}

template <int BW, int RX, int RV, int NT, bool CLUSTER>
__global__ void __launch_bounds__(NT, 1)
    rjac_kernel(cplx* Y, long long ldy, int mr, int vofs, int nc, int nb, int nbe, double tol, int max_sweeps, int full_rounds,
                double* offbuf, int* sweeps_out, int prof, int fastp) {
  constexpr int PC = 2 * BW, NV = 4 * BW, NW = NT / 32;
  __shared__ double red[2][NW][NV];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double tol2q = 0.0625 * tol * tol;
  cplx x[RX][PC], v[RV][PC];
  int sweep = 0, buf = 0;
  unsigned long long pt = 0;
  const bool pr = prof && blockIdx.x == 0 && tid == 0;
  auto mark = [&](int i) {
    if (pr) {
      const unsigned long long t = clock64();
      if (pt) g_rj_prof[i] += t - pt;
      pt = t;
    }
  };
  mark(0);
  for (; sweep < max_sweeps; ++sweep) {
    double* off_cur = offbuf + (sweep % 3);
    if (blockIdx.x == 0 && tid == 0) offbuf[(sweep + 1) % 3] = 0.0;
    for (int round = 0; round < nbe - 1; ++round) {
      int a, b;
      rj_rr_pair(nbe, round, blockIdx.x, a, b);
#pragma unroll
      for (int j = 0; j < PC; ++j) {
        const int blk = j < BW ? a : b;
        const int col = blk * BW + (j % BW);
        const bool valid = blk < nb && col < nc;
        const cplx* src = Y + (long long)col * ldy;
#pragma unroll
        for (int k = 0; k < RX; ++k) {
          const int r = tid + k * NT;
          x[k][j] = (valid && r < mr) ? __ldcg(src + r) : cmk(0.0, 0.0);
        }
#pragma unroll
        for (int k = 0; k < RV; ++k) {
          const int r = tid + k * NT;
          v[k][j] = (valid && r < nc) ? __ldcg(src + vofs + r) : cmk(0.0, 0.0);
        }
      }
      mark(0);
      double offacc = 0.0;
      bool rot = false;
      if (round == 0 || full_rounds) {
#pragma unroll
        for (int s = 0; s < PC - 1; ++s) {
          rj_step<BW, RX, RV, NT, false>(x, v, s, red[buf], lane, wid, tol2q, offacc, rot, pr && prof > 1, fastp);
          buf ^= 1;
        }
      } else {
#pragma unroll
        for (int s = 0; s < BW; ++s) {
          rj_step<BW, RX, RV, NT, true>(x, v, s, red[buf], lane, wid, tol2q, offacc, rot, pr && prof > 1, fastp);
          buf ^= 1;
        }
      }
      mark(1);
      if (rot) {
#pragma unroll
        for (int j = 0; j < PC; ++j) {
          const int blk = j < BW ? a : b;
          const int col = blk * BW + (j % BW);
          if (blk < nb && col < nc) {
            cplx* dst = Y + (long long)col * ldy;
#pragma unroll
            for (int k = 0; k < RX; ++k) {
              const int r = tid + k * NT;
              if (r < mr) __stcg(dst + r, x[k][j]);
            }
#pragma unroll
            for (int k = 0; k < RV; ++k) {
              const int r = tid + k * NT;
              if (r < nc) __stcg(dst + vofs + r, v[k][j]);
            }
          }
        }
      }
      if (wid == 0) {
        offacc = warp_max(offacc);
        if (lane == 0 && offacc > 0.0) atomic_max_nonneg(off_cur, sqrt(offacc));
      }
      mark(2);
      if (CLUSTER) {
        cg::this_cluster().sync();
      } else {
        cg::this_grid().sync();
      }
      mark(3);
    }
    const double off = __ldcg(off_cur);
    if (!(off > tol) || off * off <= c_rj_early * tol) break;
  }
  if (blockIdx.x == 0 && tid == 0) *sweeps_out = min(sweep + 1, max_sweeps);
}

// ---------------------------------------------------------------------------
// Norm-tracked step (rjac2 MODE 1).  The column norms a_j = |x_j|^2 are
// reduced once per round and then updated by every rotation (a_p' = a_p - d,
// a_q' = a_q + d with d = t |g|, exact for the zeroing rotation), so a step
// reduces only the BW inner products g = x_p^H x_q.  A norm that loses more
// than 99% in one rotation is marked stale: its pairs are skipped for the rest
// of the round and the sweep is not allowed to converge (the next round
// recomputes the norms from the data).  The rotation angle is formed in FP32
// from zeta = (c - a) / (2|g|); cs = 1/sqrt(1 + t^2) and sn = cs t g/|g| are
// FP64, so the rotation is unitary to FP64 rounding whatever t is (an angle
// off by ~1e-7 only leaves a ~1e-7 residual for the next sweep).
__device__ __forceinline__ void rj2_params(double a, double c, double gr, double gi, double& cs, double& sr,
                                           double& si, double& dnorm) {
  const double ag2 = gr * gr + gi * gi;
  const double rg = rj_rsqrt(ag2);  // 1/|g|
  const double zeta = 0.5 * (c - a) * rg;
  double t;
  if (fabs(zeta) < 1e15) {
    const float z = (float)zeta;
    const float az = fabsf(z);
    const float tf = copysignf(1.0f, z) / (az + sqrtf(fmaf(z, z, 1.0f)));
    t = (double)tf;
  } else {
    t = 0.5 / zeta;
  }
  cs = rj_rsqrt(fma(t, t, 1.0));
  const double f = cs * t * rg;
  sr = f * gr;
  si = f * gi;
  dnorm = t * ag2 * rg;  // t |g|
}

template <int BW, int RX, int NT, bool CROSS>
__device__ __forceinline__ void rj2_step(cplx (&x)[RX][2 * BW], double (&nrm)[2 * BW], unsigned& stale, int s,
                                         double (*red)[BW * 4], int lane, int wid, double tol2q, double tolc2,
                                         double& cmax, bool& rot, double (*pout)[3], int barid = 1) {
  constexpr int NV = 2 * BW;
  constexpr int H = (NV == 16) ? 4 : (NV == 8) ? 3 : 2;
  constexpr int SH = 5 - H;
  constexpr int NW = NT / 32;
  double val[NV];
#pragma unroll
  for (int i = 0; i < BW; ++i) {
    int p, q;
    rj_pq<BW, CROSS>(s, i, p, q);
    double gr = 0.0, gi = 0.0;
#pragma unroll
    for (int k = 0; k < RX; ++k) {
      const cplx u = x[k][p], w = x[k][q];
      gr = fma(u.x, w.x, fma(u.y, w.y, gr));
      gi = fma(u.x, w.y, fma(-u.y, w.x, gi));
    }
    val[2 * i] = gr;
    val[2 * i + 1] = gi;
  }
#pragma unroll
  for (int lev = 0; lev < H; ++lev) {
    const int msk = 16 >> lev;
    const int h = NV >> (lev + 1);
    const bool up = (lane & msk) != 0;
#pragma unroll
    for (int j = 0; j < h; ++j) {
      const double send = up ? val[j] : val[j + h];
      const double keep = up ? val[j + h] : val[j];
      val[j] = keep + __shfl_xor_sync(FULL, send, msk);
    }
  }
  double tt = val[0];
#pragma unroll
  for (int msk = (16 >> H); msk >= 1; msk >>= 1) tt += __shfl_xor_sync(FULL, tt, msk);
  if ((lane & ((1 << SH) - 1)) == 0) red[wid][lane >> SH] = tt;
  rj_bar<NT, true>(barid);
  double tot = 0.0;
  if (lane < NV) {
#pragma unroll
    for (int w = 0; w < NW; ++w) tot += red[w][lane];
  }
  // lane pi (mod BW) forms the rotation of pair pi
  const int pi = lane % BW;
  const double gr = __shfl_sync(FULL, tot, 2 * pi);
  const double gi = __shfl_sync(FULL, tot, 2 * pi + 1);
  double a = 0.0, c = 0.0;
  int pidx = 0, qidx = 0;
#pragma unroll
  for (int i = 0; i < BW; ++i) {
    int p, q;
    rj_pq<BW, CROSS>(s, i, p, q);
    if (pi == i) {
      a = nrm[p];
      c = nrm[q];
      pidx = p;
      qidx = q;
    }
  }
  double cs = 1.0, sr = 0.0, si = 0.0, dn = 0.0;
  int flag = 0;  // 1: not converged, 2: a norm went stale
  const bool st = ((stale >> pidx) | (stale >> qidx)) & 1u;
  if (a > 0.0 && c > 0.0) {
    const double ag2 = gr * gr + gi * gi;
    if (st) {
      flag = 1;
    } else if (ag2 > 1e-300 && ag2 > tol2q * a * c) {
      rj2_params(a, c, gr, gi, cs, sr, si, dn);
      if (ag2 > tolc2 * a * c) flag = 1;
      if (a - dn < 0.01 * a || c + dn < 0.01 * c) flag |= 2;
    } else if (ag2 > tolc2 * a * c) {
      flag = 1;
    }
    cmax = fmax(cmax, st ? 1.0 : ag2 / (a * c));  // squared cosine of the pair (a stale norm: unknown)
  }
  if (pout != nullptr && wid == 0 && lane < BW) {
    pout[lane][0] = cs;
    pout[lane][1] = sr;
    pout[lane][2] = si;
  }
#pragma unroll
  for (int i = 0; i < BW; ++i) {
    int p, q;
    rj_pq<BW, CROSS>(s, i, p, q);
    const double csi = __shfl_sync(FULL, cs, i);
    const double sri = __shfl_sync(FULL, sr, i);
    const double sii = __shfl_sync(FULL, si, i);
    const double dni = __shfl_sync(FULL, dn, i);
    const int fl = __shfl_sync(FULL, flag, i);
    if (sri != 0.0 || sii != 0.0) {  // warp-uniform
      rot = true;
#pragma unroll
      for (int k = 0; k < RX; ++k) {
        const cplx u = x[k][p], w = x[k][q];
        x[k][p] = cmk(fma(csi, u.x, -fma(sri, w.x, sii * w.y)), fma(csi, u.y, -fma(sri, w.y, -sii * w.x)));
        x[k][q] = cmk(fma(csi, w.x, fma(sri, u.x, -sii * u.y)), fma(csi, w.y, fma(sri, u.y, sii * u.x)));
      }
      nrm[p] -= dni;
      nrm[q] += dni;
      if (fl & 2) stale |= (1u << p) | (1u << q);
    }
  }
}

// column norms of the 2BW register columns, reduced over the NT X threads
template <int BW, int RX, int NT>
__device__ __forceinline__ void rj2_norms(const cplx (&x)[RX][2 * BW], double (&nrm)[2 * BW], double (*red)[BW * 4],
                                          int lane, int wid, int barid = 1) {
  constexpr int NV = 2 * BW;
  constexpr int H = (NV == 16) ? 4 : (NV == 8) ? 3 : 2;
  constexpr int SH = 5 - H;
  constexpr int NW = NT / 32;
  double val[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < RX; ++k) t = fma(x[k][j].x, x[k][j].x, fma(x[k][j].y, x[k][j].y, t));
    val[j] = t;
  }
#pragma unroll
  for (int lev = 0; lev < H; ++lev) {
    const int msk = 16 >> lev;
    const int h = NV >> (lev + 1);
    const bool up = (lane & msk) != 0;
#pragma unroll
    for (int j = 0; j < h; ++j) {
      const double send = up ? val[j] : val[j + h];
      const double keep = up ? val[j + h] : val[j];
      val[j] = keep + __shfl_xor_sync(FULL, send, msk);
    }
  }
  double tt = val[0];
#pragma unroll
  for (int msk = (16 >> H); msk >= 1; msk >>= 1) tt += __shfl_xor_sync(FULL, tt, msk);
  if ((lane & ((1 << SH) - 1)) == 0) red[wid][lane >> SH] = tt;
  rj_bar<NT, true>(barid);
  double tot = 0.0;
  if (lane < NV) {
#pragma unroll
    for (int w = 0; w < NW; ++w) tot += red[w][lane];
  }
#pragma unroll
  for (int j = 0; j < NV; ++j) nrm[j] = __shfl_sync(FULL, tot, j);
}

// ---------------------------------------------------------------------------
// rjac2: the right factor V is NOT on the critical path.  Warps [0, NTX/32)
// ("X warps") run the rounds on X only and publish every step's rotation
// parameters in shared memory; warps [NTX/32, ...) ("V warps") replay the
// PREVIOUS round's rotations on that round's V blocks (streamed from L2 in
// chunks of rows) while the X warps work on the next round.  The V update of
// round R completes before barrier R+1 and the blocks it touched are next
// used by V warps after that barrier, so V sees every round in order.
template <int BW, bool CROSS>
__device__ __forceinline__ void rj_v_round(cplx (&v)[2 * BW], const double (*P)[BW][3]) {
  constexpr int NS = CROSS ? BW : 2 * BW - 1;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
#pragma unroll
    for (int i = 0; i < BW; ++i) {
      int p, q;
      rj_pq<BW, CROSS>(s, i, p, q);
      const double csi = P[s][i][0], sri = P[s][i][1], sii = P[s][i][2];
      if (sri != 0.0 || sii != 0.0) {
        const cplx u = v[p], w = v[q];
        v[p] = cmk(fma(csi, u.x, -fma(sri, w.x, sii * w.y)), fma(csi, u.y, -fma(sri, w.y, -sii * w.x)));
        v[q] = cmk(fma(csi, w.x, fma(sri, u.x, -sii * u.y)), fma(csi, w.y, fma(sri, u.y, sii * u.x)));
      }
    }
  }
}

template <int BW, int RX, int NTX, int NTV, bool CLUSTER, int MODE, int G>
__global__ void __launch_bounds__(G * NTX + NTV, 1)
    rjac2_kernel(cplx* Y, long long ldy, int mr, int vofs, int nc, int nb, int nbe, double tol, int max_sweeps,
                 double* offbuf, int* sweeps_out, int prof, unsigned* flags) {
  // flags != nullptr: between rounds, point-to-point per-block counters in
  // global memory (xflag[b] = rounds whose X update of block b is stored,
  // vflag[b] = rounds whose V update is stored) instead of a grid barrier;
  // one grid barrier per sweep (the convergence decision).
  // G block pairs per CTA ("pair groups" of NTX X threads each, named barrier
  // 1 + g), one set of NTV V threads serving all groups
  constexpr int PC = 2 * BW, NV = 4 * BW, NWX = NTX / 32;
  __shared__ double red_all[G][2][NWX][NV];
  __shared__ double Ps_all[G][2][2 * BW - 1][BW][3];
  __shared__ int s_blk_all[G][2][4];  // a, b, rotated, full round
  const int tid0 = threadIdx.x, lane = tid0 & 31;
  const bool xthr = tid0 < G * NTX;
  const int grp = xthr ? tid0 / NTX : 0;
  const int tid = xthr ? tid0 - grp * NTX : tid0 - (G - 1) * NTX;  // V threads: tid - NTX >= 0
  const int wid = tid >> 5;
  const int barid = 1 + grp;
  const int pair = blockIdx.x * G + grp;
  const int npairs = nbe / 2;
  auto& red = red_all[grp];
  auto& Ps = Ps_all[grp];
  auto& s_blk = s_blk_all[grp];
  const double tol2q = 0.0625 * tol * tol;
  cplx x[RX][PC], dummy[1][PC];
  int sweep = 0, buf = 0, R = 0;
  unsigned long long pt = 0;
  const bool pr = prof && blockIdx.x == 0 && tid0 == 0;
  auto mark = [&](int i) {
    if (pr) {
      const unsigned long long t = clock64();
      if (pt) g_rj_prof[i] += t - pt;
      pt = t;
    }
  };
  // V warps: replay round slot sb's rotations on its V blocks
  unsigned* xflag = flags;
  unsigned* vflag = flags ? flags + nbe : nullptr;
  const int tv = tid0 - G * NTX;  // V thread index
  auto wait_flag = [&](const unsigned* f, unsigned need) {
    while (*(volatile const unsigned*)f < need) __nanosleep(32);
    __threadfence();
  };
  auto apply_v = [&](int sb, int Rdone) {  // Rdone = the round whose rotations are replayed
   for (int g = 0; g < G; ++g) {
    const int a = s_blk_all[g][sb][0], b = s_blk_all[g][sb][1];
    if (a < 0) continue;  // idle group
    if (flags) {
      // V blocks a, b were last updated by round Rdone-1's replay
      if (tv == 0) {
        if (a < nb) wait_flag(vflag + a, (unsigned)Rdone);
        if (b < nb) wait_flag(vflag + b, (unsigned)Rdone);
      }
      asm volatile("bar.sync 15, %0;" ::"n"(NTV) : "memory");
    }
    if (s_blk_all[g][sb][2]) {
    const bool full = s_blk_all[g][sb][3] != 0;
    long long off[PC];
    bool ok[PC];
#pragma unroll
    for (int j = 0; j < PC; ++j) {
      const int blk = j < BW ? a : b;
      const int col = blk * BW + (j % BW);
      ok[j] = blk < nb && col < nc;
      off[j] = (long long)col * ldy + vofs;
    }
    // rows streamed from L2 with the next row's load in flight (latency off the chain)
    cplx v[PC], vn[PC];
    int r = tid - NTX;
#pragma unroll
    for (int j = 0; j < PC; ++j) v[j] = (ok[j] && r < nc) ? __ldcg(Y + off[j] + r) : cmk(0.0, 0.0);
    for (; r < nc; r += NTV) {
      const int rn = r + NTV;
#pragma unroll
      for (int j = 0; j < PC; ++j) vn[j] = (ok[j] && rn < nc) ? __ldcg(Y + off[j] + rn) : cmk(0.0, 0.0);
      if (full) rj_v_round<BW, false>(v, Ps_all[g][sb]);
      else rj_v_round<BW, true>(v, Ps_all[g][sb]);
#pragma unroll
      for (int j = 0; j < PC; ++j) {
        if (ok[j]) __stcg(Y + off[j] + r, v[j]);
        v[j] = vn[j];
      }
    }
    }
    if (flags) {
      asm volatile("bar.sync 15, %0;" ::"n"(NTV) : "memory");
      if (tv == 0) {
        __threadfence();
        if (a < nb) *(volatile unsigned*)(vflag + a) = (unsigned)(Rdone + 1);
        if (b < nb) *(volatile unsigned*)(vflag + b) = (unsigned)(Rdone + 1);
      }
    }
   }
  };
  mark(0);
  for (; sweep < max_sweeps; ++sweep) {
    double* off_cur = offbuf + (sweep % 3);
    if (blockIdx.x == 0 && tid0 == 0) offbuf[(sweep + 1) % 3] = 0.0;
    for (int round = 0; round < nbe - 1; ++round, ++R) {
      if (xthr && pair >= npairs) {
        if (tid == 0) {
          s_blk[R & 1][0] = -1;  // idle group (odd pair count)
          s_blk[R & 1][2] = 0;
        }
      } else if (xthr) {
        int a, b;
        rj_rr_pair(nbe, round, pair, a, b);
        const int sb = R & 1;
        if (flags) {
          // blocks a, b were stored by round R-1
          if (tid == 0) {
            if (a < nb) wait_flag(xflag + a, (unsigned)R);
            if (b < nb) wait_flag(xflag + b, (unsigned)R);
          }
          rj_bar<NTX, true>(barid);
        }
#pragma unroll
        for (int j = 0; j < PC; ++j) {
          const int blk = j < BW ? a : b;
          const int col = blk * BW + (j % BW);
          const bool valid = blk < nb && col < nc;
          const cplx* src = Y + (long long)col * ldy;
#pragma unroll
          for (int k = 0; k < RX; ++k) {
            const int r = tid + k * NTX;
            x[k][j] = (valid && r < mr) ? __ldcg(src + r) : cmk(0.0, 0.0);
          }
        }
        mark(0);
        double offacc = 0.0;
        bool rot = false;
        if (MODE == 1) {
          double nrm[PC];
          unsigned stale = 0u;
          double cmax = 0.0;
          rj2_norms<BW, RX, NTX>(x, nrm, red[buf], lane, wid, barid);
          buf ^= 1;
          if (round == 0) {
#pragma unroll
            for (int s = 0; s < PC - 1; ++s) {
              rj2_step<BW, RX, NTX, false>(x, nrm, stale, s, red[buf], lane, wid, tol2q, tol * tol, cmax, rot,
                                           Ps[sb][s], barid);
              buf ^= 1;
            }
          } else {
#pragma unroll
            for (int s = 0; s < BW; ++s) {
              rj2_step<BW, RX, NTX, true>(x, nrm, stale, s, red[buf], lane, wid, tol2q, tol * tol, cmax, rot,
                                          Ps[sb][s], barid);
              buf ^= 1;
            }
          }
          offacc = cmax;
        } else if (round == 0) {
#pragma unroll
          for (int s = 0; s < PC - 1; ++s) {
            rj_step<BW, RX, 0, NTX, false, true>(x, dummy, s, red[buf], lane, wid, tol2q, offacc, rot, false, false,
                                                 Ps[sb][s], barid);
            buf ^= 1;
          }
        } else {
#pragma unroll
          for (int s = 0; s < BW; ++s) {
            rj_step<BW, RX, 0, NTX, true, true>(x, dummy, s, red[buf], lane, wid, tol2q, offacc, rot, false, false,
                                                Ps[sb][s], barid);
            buf ^= 1;
          }
        }
        mark(1);
        if (rot) {
#pragma unroll
          for (int j = 0; j < PC; ++j) {
            const int blk = j < BW ? a : b;
            const int col = blk * BW + (j % BW);
            if (blk < nb && col < nc) {
              cplx* dst = Y + (long long)col * ldy;
#pragma unroll
              for (int k = 0; k < RX; ++k) {
                const int r = tid + k * NTX;
                if (r < mr) __stcg(dst + r, x[k][j]);
              }
            }
          }
        }
        if (tid == 0) {
          s_blk[sb][0] = a;
          s_blk[sb][1] = b;
          s_blk[sb][2] = rot ? 1 : 0;
          s_blk[sb][3] = round == 0 ? 1 : 0;
        }
        if (flags) {
          rj_bar<NTX, true>(barid);  // every X store of this group issued
          if (tid == 0) {
            __threadfence();
            if (a < nb) *(volatile unsigned*)(xflag + a) = (unsigned)(R + 1);
            if (b < nb) *(volatile unsigned*)(xflag + b) = (unsigned)(R + 1);
          }
        }
        if (wid == 0) {
          offacc = warp_max(offacc);
          if (lane == 0 && offacc > 0.0) atomic_max_nonneg(off_cur, sqrt(offacc));
        }
        mark(2);
      } else if (R > 0) {
        apply_v((R - 1) & 1, R - 1);
      }
      if (flags) {
        __syncthreads();  // X and V warps of this CTA: the shared parameter buffers rotate
      } else if (CLUSTER) {
        cg::this_cluster().sync();
      } else {
        cg::this_grid().sync();
      }
      mark(3);
    }
    if (flags) {
      if (CLUSTER) cg::this_cluster().sync();
      else cg::this_grid().sync();
    }
    const double off = __ldcg(off_cur);
    if (!(off > tol) || off * off <= c_rj_early * tol) break;
  }
  // the last round's V update
  if (!xthr && R > 0) apply_v((R - 1) & 1, R - 1);
  if (blockIdx.x == 0 && tid0 == 0) *sweeps_out = min(sweep + 1, max_sweeps);
}

struct RjVariant {
  void* fn;
  bool cluster;
};

template <int BW, int RX, int RV, int NT>
RjVariant rj_pick(bool cluster) {
  return RjVariant{cluster ? (void*)rjac_kernel<BW, RX, RV, NT, true> : (void*)rjac_kernel<BW, RX, RV, NT, false>,
                   cluster};
}
template <int BW, int RX, int NTX, int NTV, int MODE = 1, int G = 1>
RjVariant rj2_pick(bool cluster) {
  return RjVariant{cluster ? (void*)rjac2_kernel<BW, RX, NTX, NTV, true, MODE, G>
                           : (void*)rjac2_kernel<BW, RX, NTX, NTV, false, MODE, G>,
                   cluster};
}

// variant table.  kind 1 (rjac): X and V rows in registers, rx/rv rows per
// thread, nt threads.  kind 2 (rjac2): X rows in registers (rx per X thread,
// nt X threads), V streamed by ntv V threads.
struct Row {
  int kind, bw, rx, rv, nt, ntv, groups = 1;
};
constexpr Row kTab[] = {
    {1, 8, 1, 1, 256, 0},    // 0
    {1, 4, 1, 1, 256, 0},    // 1
    {1, 4, 2, 1, 256, 0},    // 2
    {1, 8, 2, 1, 256, 0},    // 3
    {1, 4, 2, 2, 256, 0},    // 4
    {1, 4, 2, 2, 128, 0},    // 5
    {2, 4, 2, 0, 128, 128},  // 6: X <= 256 rows
    {2, 4, 4, 0, 128, 128},  // 7: X <= 512
    {2, 4, 4, 0, 256, 64},   // 8: X <= 1024
    {2, 8, 1, 0, 256, 128},  // 9: X <= 256, BW 8 (one cluster up to nc = 256)
    {2, 4, 2, 0, 256, 128},  // 10: X <= 512
    {2, 4, 2, 0, 128, 128},  // 11: as 6 with exact (non-tracked) norms and FP64 angles
    {2, 8, 2, 0, 128, 128},  // 12: X <= 256, BW 8: one cluster up to nc = 256
    {2, 8, 2, 0, 128, 128},  // 13: as 12, exact norms
    {2, 4, 2, 0, 128, 128, 2},  // 14: as 6 with 2 block pairs per CTA (one cluster up to nc = 256)
    {2, 4, 1, 0, 256, 128},     // 15: X <= 256 rows, 8 X warps (1 row each)
    {2, 4, 1, 0, 256, 256},     // 16: as 15 with 8 V warps
    {2, 4, 4, 0, 64, 128},      // 17: X <= 256 rows, 2 X warps (4 rows each)
    {2, 4, 8, 0, 32, 128},      // 18: X <= 256 rows, 1 X warp (8 rows each)
    {2, 4, 4, 0, 256, 128},     // 19: X <= 1024, 4 V warps
    {2, 4, 2, 0, 256, 64},      // 20: X <= 512, 2 V warps
};
constexpr int kNTab = sizeof(kTab) / sizeof(kTab[0]);

RjVariant rj_variant(int row, bool cl) {
  switch (row) {
    case 0: return rj_pick<8, 1, 1, 256>(cl);
    case 1: return rj_pick<4, 1, 1, 256>(cl);
    case 2: return rj_pick<4, 2, 1, 256>(cl);
    case 3: return rj_pick<8, 2, 1, 256>(cl);
    case 4: return rj_pick<4, 2, 2, 256>(cl);
    case 5: return rj_pick<4, 2, 2, 128>(cl);
    case 6: return rj2_pick<4, 2, 128, 128>(cl);
    case 7: return rj2_pick<4, 4, 128, 128>(cl);
    case 8: return rj2_pick<4, 4, 256, 64>(cl);
    case 9: return rj2_pick<8, 1, 256, 128>(cl);
    case 10: return rj2_pick<4, 2, 256, 128>(cl);
    case 11: return rj2_pick<4, 2, 128, 128, 0>(cl);
    case 12: return rj2_pick<8, 2, 128, 128>(cl);
    case 13: return rj2_pick<8, 2, 128, 128, 0>(cl);
    case 14: return rj2_pick<4, 2, 128, 128, 1, 2>(cl);
    case 15: return rj2_pick<4, 1, 256, 128>(cl);
    case 16: return rj2_pick<4, 1, 256, 256>(cl);
    case 17: return rj2_pick<4, 4, 64, 128>(cl);
    case 18: return rj2_pick<4, 8, 32, 128>(cl);
    case 19: return rj2_pick<4, 4, 256, 128>(cl);
    default: return rj2_pick<4, 2, 256, 64>(cl);
  }
}

bool rows_ok(int row, int mr, int nc) {
  const Row& r = kTab[row];
  if (r.kind == 2) return mr <= r.rx * r.nt;
  return mr <= r.rx * r.nt && nc <= r.rv * r.nt;
}

}  // namespace

// Jacobi stage on d.Y = [X ; V] (column-major, ld = ldy).  Returns
// cudaErrorNotSupported when no register-resident variant fits the shape.
cudaError_t svd_rjac_run(cudaStream_t st, const SvdDev& d, int mr, int vofs, int nc, long long ldy, double tol,
                         int* sweeps_dev) {
  static const int prof = [] {  // thread-safe once
    const char* pe = std::getenv("TDVP_SVD_PROF");  // per-phase cycle counts on stderr (diagnostics only)
    return pe ? std::max(1, std::atoi(pe)) : 0;
  }();
  constexpr int full_rounds = 0, fastp = 0;
  int row = -1;
  {
    // latency: measured fastest first (microbench.py --svd, B200); throughput
    // (concurrent SVDs of segment lanes): variant 14 packs two block pairs per
    // CTA, half the CTAs per SVD (c2sat p = 8 lanes: 146 vs 166 ms/step)
    const int prefer[] = {6, 10, 19};
    if (d.throughput && rows_ok(14, mr, nc)) row = 14;
    for (int r : prefer)
      if (row < 0 && rows_ok(r, mr, nc)) { row = r; break; }
  }
  if (row < 0) return cudaErrorNotSupported;
  const int bw = kTab[row].bw, kind = kTab[row].kind, grp = kTab[row].groups;
  const int nt = kind == 2 ? grp * kTab[row].nt + kTab[row].ntv : kTab[row].nt;
  const int nb = (nc + bw - 1) / bw;
  const int nbe = std::max(2, nb + (nb & 1));
  const int P = (nbe / 2 + grp - 1) / grp;  // CTAs
  cudaError_t e;
  bool cluster = P <= 16;
  RjVariant v{};
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  cfg.gridDim = dim3(P);
  cfg.blockDim = dim3(nt);
  cfg.stream = st;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cluster) {
    v = rj_variant(row, true);
    if ((e = set_cluster_nonportable(v.fn)) != cudaSuccess) return e;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, v.fn, &cfg) != cudaSuccess || ncl < 1) {
      cudaGetLastError();
      cluster = false;
    }
  }
  if (!cluster) {
    v = rj_variant(row, false);
    int occ = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, v.fn, nt, 0)) != cudaSuccess) return e;
    if (occ * g_num_sms < P) return cudaErrorNotSupported;
  }
  if ((e = cudaMemsetAsync(d.offmax, 0, 4 * sizeof(double), st)) != cudaSuccess) return e;
  if (prof) {
    unsigned long long z[12] = {0};
    cudaMemcpyToSymbolAsync(g_rj_prof, z, sizeof(z), 0, cudaMemcpyHostToDevice, st);
  }
  int max_sweeps = 60;
  cplx* Yp = d.Y;
  double* offb = d.offmax;
  void* args1[] = {(void*)&Yp,  (void*)&ldy,        (void*)&mr,  (void*)&vofs,  (void*)&nc,   (void*)&nb,
                   (void*)&nbe, (void*)&tol,        (void*)&max_sweeps,  (void*)&full_rounds,
                   (void*)&offb, (void*)&sweeps_dev, (void*)&prof, (void*)&fastp};
  unsigned* flg = nullptr;
  // point-to-point round flags: measured slower than the grid barrier (flag
  // round trips through L2 + fences cost more than cg's barrier at 32 CTAs)
  constexpr int use_flags = 0;
  if (kind == 2 && use_flags && d.flags != nullptr && (size_t)2 * nbe <= d.flags_elems) {
    flg = d.flags;
    if ((e = cudaMemsetAsync(flg, 0, (size_t)2 * nbe * sizeof(unsigned), st)) != cudaSuccess) return e;
  }
  void* args2[] = {(void*)&Yp,  (void*)&ldy, (void*)&mr,         (void*)&vofs, (void*)&nc,         (void*)&nb,
                   (void*)&nbe, (void*)&tol, (void*)&max_sweeps, (void*)&offb, (void*)&sweeps_dev, (void*)&prof,
                   (void*)&flg};
  void** args = kind == 2 ? args2 : args1;
  if (cluster) {
    if ((e = cudaLaunchKernelExC(&cfg, v.fn, args)) != cudaSuccess) return e;
  } else {
    if ((e = cudaLaunchCooperativeKernel(v.fn, dim3(P), dim3(nt), args, 0, st)) != cudaSuccess) return e;
  }
  if (prof) {
    unsigned long long z[12];
    cudaMemcpyFromSymbolAsync(z, g_rj_prof, sizeof(z), 0, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    std::fprintf(stderr,
                 "rjac prof mr=%d nc=%d row=%d bw=%d nt=%d P=%d cluster=%d cycles: load %llu steps %llu store %llu "
                 "barrier %llu | dots %llu reduce %llu sync %llu gather %llu params %llu apply %llu\n",
                 mr, nc, row, bw, nt, P, (int)cluster, z[0], z[1], z[2], z[3], z[4], z[5], z[6], z[8], z[9], z[7]);
  }
  return cudaGetLastError();
}
