// Microbenchmark of the block-Jacobi inner solve (32 x 32 Hermitian two-sided
// Jacobi, one sweep of 31 rounds) in one CTA: variants of the round structure.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
#include "../../paper_1912_06127_b200/csrc/common.cuh"
constexpr int PC = 32, GP = 33, NTB = 256;
__device__ __forceinline__ void rr_pair(int n, int round, int i, int& a, int& b) {
  const int m = n - 1;
  if (i == 0) { a = n - 1; b = round % m; } else { a = (round + i) % m; b = (round - i + m) % m; }
  if (a > b) { const int t = a; a = b; b = t; }
}
__device__ __forceinline__ void params(double ga, double gc, cplx g, double tol2q, double& cs, cplx& sn) {
  cs = 1.0; sn = cmk(0, 0);
  const double ag2 = cabs2(g), gg = ga * gc;
  if (ga > 0.0 && gc > 0.0 && ag2 > 1e-300 && ag2 > tol2q * gg) {
    const double w = gc - ga;
    const double rD = rsqrt(fma(w, w, 4.0 * ag2));
    const double qq = 0.5 * fma(fabs(w), rD, 1.0);
    const double rcs = rsqrt(qq);
    cs = qq * rcs;
    const double f = copysign(rD * rcs, w);
    sn = cmk(f * g.x, f * g.y);
  }
}
__device__ __forceinline__ double frsqrt(double x) {
  // MUFU.RSQ64H seed + 2 Newton steps (the seed is good to ~2^-23)
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  return y * fma(-h * y, y, 1.5);
}
__device__ __forceinline__ void params_fast(double ga, double gc, cplx g, double tol2q, double& cs, cplx& sn) {
  cs = 1.0; sn = cmk(0, 0);
  const double ag2 = cabs2(g), gg = ga * gc;
  if (ga > 0.0 && gc > 0.0 && ag2 > 1e-300 && ag2 > tol2q * gg) {
    const double w = gc - ga;
    const double rD = frsqrt(fma(w, w, 4.0 * ag2));
    const double qq = 0.5 * fma(fabs(w), rD, 1.0);
    const double rcs = frsqrt(qq);
    cs = qq * rcs;
    const double f = copysign(rD * rcs, w);
    sn = cmk(f * g.x, f * g.y);
  }
}
struct Sm { cplx G[PC][GP]; cplx Q[PC][GP]; double cs[16]; cplx sn[16]; int rp[16], rq[16]; unsigned char ua[136], ub[136]; };

template <int VAR>
__global__ void k(const cplx* G0, long long* cyc, cplx* out, int reps) {
  __shared__ Sm sm;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) { int u = 0; for (int a = 0; a < 16; ++a) for (int b = a; b < 16; ++b) { sm.ua[u] = a; sm.ub[u] = b; ++u; } }
  long long t0 = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int e = tid; e < PC * PC; e += NTB) { sm.G[e / PC][e % PC] = G0[e]; sm.Q[e / PC][e % PC] = cmk(e / PC == e % PC, 0); }
    __syncthreads();
    if (rep == 1) t0 = clock64();
    const double tol2q = 1e-30;
    for (int rd = 0; rd < PC - 1; ++rd) {
      if (VAR == 0 || VAR >= 2) {
        if (tid < 16) {
          int p, q; rr_pair(PC, rd, tid, p, q);
          double cs; cplx sn; params(sm.G[p][p].x, sm.G[q][q].x, sm.G[p][q], tol2q, cs, sn);
          sm.rp[tid] = p; sm.rq[tid] = q; sm.cs[tid] = cs; sm.sn[tid] = sn;
        }
        __syncthreads();
      }
      // per-warp params (VAR 1): lanes 0..15 of every warp compute all 16, broadcast by shuffle
      double cs_l = 1.0; cplx sn_l = cmk(0, 0); int p_l = 0, q_l = 0;
      if (VAR == 1) {
        const int i = lane & 15;
        rr_pair(PC, rd, i, p_l, q_l);
        params(sm.G[p_l][p_l].x, sm.G[q_l][q_l].x, sm.G[p_l][q_l], tol2q, cs_l, sn_l);
        __syncthreads();  // everyone read G before anyone writes
      }
      auto get = [&](int r, int& p, int& q, double& cs, cplx& sn) {
        if (VAR != 1) { p = sm.rp[r]; q = sm.rq[r]; cs = sm.cs[r]; sn = sm.sn[r]; }
        else {
          p = __shfl_sync(0xffffffffu, p_l, r); q = __shfl_sync(0xffffffffu, q_l, r);
          cs = __shfl_sync(0xffffffffu, cs_l, r);
          sn.x = __shfl_sync(0xffffffffu, sn_l.x, r); sn.y = __shfl_sync(0xffffffffu, sn_l.y, r);
        }
      };
      {
        const int u = tid;
        const int ra = u < 136 ? sm.ua[u] : 0, rb = u < 136 ? sm.ub[u] : 0;
        int p1, q1, p2, q2; double ca, cb; cplx sa, sb;
        get(ra, p1, q1, ca, sa); get(rb, p2, q2, cb, sb);
        if (u < 136 && VAR != 2 && VAR != 4) {
          const cplx b00 = sm.G[p1][p2], b01 = sm.G[p1][q2], b10 = sm.G[q1][p2], b11 = sm.G[q1][q2];
          const cplx r00 = csub(cscale(b00, ca), cmul(sa, b10));
          const cplx r01 = csub(cscale(b01, ca), cmul(sa, b11));
          const cplx r10 = cadd(cmul(cconj(sa), b00), cscale(b10, ca));
          const cplx r11 = cadd(cmul(cconj(sa), b01), cscale(b11, ca));
          cplx n00 = csub(cscale(r00, cb), cmul(cconj(sb), r01));
          cplx n01 = cadd(cmul(sb, r00), cscale(r01, cb));
          cplx n10 = csub(cscale(r10, cb), cmul(cconj(sb), r11));
          cplx n11 = cadd(cmul(sb, r10), cscale(r11, cb));
          if (ra == rb) { if (sa.x != 0.0 || sa.y != 0.0) n01 = cmk(0, 0); n00.y = n11.y = 0; n10 = cconj(n01); }
          sm.G[p1][p2] = n00; sm.G[p1][q2] = n01; sm.G[q1][p2] = n10; sm.G[q1][q2] = n11;
          if (ra != rb) { sm.G[p2][p1] = cconj(n00); sm.G[q2][p1] = cconj(n01); sm.G[p2][q1] = cconj(n10); sm.G[q2][q1] = cconj(n11); }
        }
        for (int h = 0; h < 2 && VAR != 2 && VAR != 3; ++h) {
          const int v = tid + h * NTB; const int row = v >> 4, r2 = v & 15;
          int p, q; double c; cplx sn; get(r2, p, q, c, sn);
          const cplx qp = sm.Q[row][p], qq = sm.Q[row][q];
          sm.Q[row][p] = csub(cscale(qp, c), cmul(cconj(sn), qq));
          sm.Q[row][q] = cadd(cmul(sn, qp), cscale(qq, c));
        }
      }
      __syncthreads();
    }
  }
  if (tid == 0) *cyc = (clock64() - t0) / (reps - 1);
  for (int e = tid; e < PC * PC; e += NTB) out[e] = sm.Q[e / PC][e % PC];
}
// VAR 5: every thread's round indices by arithmetic (no index loads), the
// G 2x2 block and the Q entries of the round loaded BEFORE the parameter
// barrier (they only depend on the previous round), so after the barrier a
// thread only loads (cs, sn) and does the arithmetic
__global__ void k5(const cplx* G0, long long* cyc, cplx* out, int reps) {
  __shared__ Sm sm;
  const int tid = threadIdx.x;
  int ra = 0, rb = 0;
  if (tid < 136) { int u = tid, a = 0; while (u >= 16 - a) { u -= 16 - a; ++a; } ra = a; rb = a + u; }
  long long t0 = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int e = tid; e < PC * PC; e += NTB) { sm.G[e / PC][e % PC] = G0[e]; sm.Q[e / PC][e % PC] = cmk(e / PC == e % PC, 0); }
    __syncthreads();
    if (rep == 1) t0 = clock64();
    const double tol2q = 1e-30;
    for (int rd = 0; rd < PC - 1; ++rd) {
      int p1, q1, p2, q2;
      rr_pair(PC, rd, ra, p1, q1);
      rr_pair(PC, rd, rb, p2, q2);
      cplx b00, b01, b10, b11;
      if (tid < 136) { b00 = sm.G[p1][p2]; b01 = sm.G[p1][q2]; b10 = sm.G[q1][p2]; b11 = sm.G[q1][q2]; }
      int qr[2], qp_[2], qq_[2], qrb[2];
      cplx qpv[2], qqv[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int v = tid + h * NTB; qr[h] = v >> 4; qrb[h] = v & 15;
        rr_pair(PC, rd, qrb[h], qp_[h], qq_[h]);
        qpv[h] = sm.Q[qr[h]][qp_[h]]; qqv[h] = sm.Q[qr[h]][qq_[h]];
      }
      if (tid < 16) {
        int p, q; rr_pair(PC, rd, tid, p, q);
        double cs; cplx sn; params(sm.G[p][p].x, sm.G[q][q].x, sm.G[p][q], tol2q, cs, sn);
        sm.cs[tid] = cs; sm.sn[tid] = sn;
      }
      __syncthreads();
      if (tid < 136) {
        const double ca = sm.cs[ra], cb = sm.cs[rb];
        const cplx sa = sm.sn[ra], sb = sm.sn[rb];
        const cplx r00 = csub(cscale(b00, ca), cmul(sa, b10));
        const cplx r01 = csub(cscale(b01, ca), cmul(sa, b11));
        const cplx r10 = cadd(cmul(cconj(sa), b00), cscale(b10, ca));
        const cplx r11 = cadd(cmul(cconj(sa), b01), cscale(b11, ca));
        cplx n00 = csub(cscale(r00, cb), cmul(cconj(sb), r01));
        cplx n01 = cadd(cmul(sb, r00), cscale(r01, cb));
        cplx n10 = csub(cscale(r10, cb), cmul(cconj(sb), r11));
        cplx n11 = cadd(cmul(sb, r10), cscale(r11, cb));
        if (ra == rb) { if (sa.x != 0.0 || sa.y != 0.0) n01 = cmk(0, 0); n00.y = n11.y = 0; n10 = cconj(n01); }
        sm.G[p1][p2] = n00; sm.G[p1][q2] = n01; sm.G[q1][p2] = n10; sm.G[q1][q2] = n11;
        if (ra != rb) { sm.G[p2][p1] = cconj(n00); sm.G[q2][p1] = cconj(n01); sm.G[p2][q1] = cconj(n10); sm.G[q2][q1] = cconj(n11); }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double c = sm.cs[qrb[h]]; const cplx sn = sm.sn[qrb[h]];
        sm.Q[qr[h]][qp_[h]] = csub(cscale(qpv[h], c), cmul(cconj(sn), qqv[h]));
        sm.Q[qr[h]][qq_[h]] = cadd(cmul(sn, qpv[h]), cscale(qqv[h], c));
      }
      __syncthreads();
    }
  }
  if (tid == 0) *cyc = (clock64() - t0) / (reps - 1);
  for (int e = tid; e < PC * PC; e += NTB) out[e] = sm.Q[e / PC][e % PC];
}
// VAR 6: as the two-phase kernel, but G kept as its UPPER triangle only
// (an entry below the diagonal is read as the conjugate of its mirror and
// never written): 4 stores per 2x2 block instead of 8
__device__ __forceinline__ cplx gget(const Sm& sm, int i, int j) { return i <= j ? sm.G[i][j] : cconj(sm.G[j][i]); }
__device__ __forceinline__ void gput(Sm& sm, int i, int j, cplx v) {
  if (i <= j) sm.G[i][j] = v;  // i > j: the mirror block (written by its owner) holds it
}
__global__ void k6(const cplx* G0, long long* cyc, cplx* out, int reps) {
  __shared__ Sm sm;
  const int tid = threadIdx.x;
  if (tid == 0) { int u = 0; for (int a = 0; a < 16; ++a) for (int b = a; b < 16; ++b) { sm.ua[u] = a; sm.ub[u] = b; ++u; } }
  long long t0 = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int e = tid; e < PC * PC; e += NTB) { sm.G[e / PC][e % PC] = G0[e]; sm.Q[e / PC][e % PC] = cmk(e / PC == e % PC, 0); }
    __syncthreads();
    if (rep == 1) t0 = clock64();
    const double tol2q = 1e-30;
    for (int rd = 0; rd < PC - 1; ++rd) {
      if (tid < 16) {
        int p, q; rr_pair(PC, rd, tid, p, q);
        double cs; cplx sn; params(sm.G[p][p].x, sm.G[q][q].x, sm.G[p][q], tol2q, cs, sn);
        sm.rp[tid] = p; sm.rq[tid] = q; sm.cs[tid] = cs; sm.sn[tid] = sn;
      }
      __syncthreads();
      if (tid < 136) {
        const int ra = sm.ua[tid], rb = sm.ub[tid];
        const int p1 = sm.rp[ra], q1 = sm.rq[ra], p2 = sm.rp[rb], q2 = sm.rq[rb];
        const double ca = sm.cs[ra], cb = sm.cs[rb];
        const cplx sa = sm.sn[ra], sb = sm.sn[rb];
        const cplx b00 = gget(sm, p1, p2), b01 = gget(sm, p1, q2), b10 = gget(sm, q1, p2), b11 = gget(sm, q1, q2);
        const cplx r00 = csub(cscale(b00, ca), cmul(sa, b10));
        const cplx r01 = csub(cscale(b01, ca), cmul(sa, b11));
        const cplx r10 = cadd(cmul(cconj(sa), b00), cscale(b10, ca));
        const cplx r11 = cadd(cmul(cconj(sa), b01), cscale(b11, ca));
        cplx n00 = csub(cscale(r00, cb), cmul(cconj(sb), r01));
        cplx n01 = cadd(cmul(sb, r00), cscale(r01, cb));
        cplx n10 = csub(cscale(r10, cb), cmul(cconj(sb), r11));
        cplx n11 = cadd(cmul(sb, r10), cscale(r11, cb));
        if (ra == rb) { if (sa.x != 0.0 || sa.y != 0.0) n01 = cmk(0, 0); n00.y = n11.y = 0; n10 = cconj(n01); }
        // block (ra, rb), ra <= rb, holds rows {p1, q1} x columns {p2, q2}; for
        // ra < rb an entry with row > column belongs to the mirror: store its conjugate there
        auto put = [&](int i, int j, cplx v) { if (i <= j) sm.G[i][j] = v; else sm.G[j][i] = cconj(v); };
        put(p1, p2, n00); put(p1, q2, n01); put(q1, p2, n10); put(q1, q2, n11);
      }
      for (int h = 0; h < 2; ++h) {
        const int v = tid + h * NTB; const int row = v >> 4, r2 = v & 15;
        const int p = sm.rp[r2], q = sm.rq[r2]; const double c = sm.cs[r2]; const cplx sn = sm.sn[r2];
        const cplx qp = sm.Q[row][p], qq = sm.Q[row][q];
        sm.Q[row][p] = csub(cscale(qp, c), cmul(cconj(sn), qq));
        sm.Q[row][q] = cadd(cmul(sn, qp), cscale(qq, c));
      }
      __syncthreads();
    }
  }
  if (tid == 0) *cyc = (clock64() - t0) / (reps - 1);
  for (int e = tid; e < PC * PC; e += NTB) out[e] = sm.Q[e / PC][e % PC];
}
__global__ void k7(const cplx* G0, long long* cyc, cplx* out, int reps) {
  __shared__ Sm sm;
  const int tid = threadIdx.x;
  if (tid == 0) { int u = 0; for (int a = 0; a < 16; ++a) for (int b = a; b < 16; ++b) { sm.ua[u] = a; sm.ub[u] = b; ++u; } }
  long long t0 = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int e = tid; e < PC * PC; e += NTB) { sm.G[e / PC][e % PC] = G0[e]; sm.Q[e / PC][e % PC] = cmk(e / PC == e % PC, 0); }
    __syncthreads();
    if (rep == 1) t0 = clock64();
    const double tol2q = 1e-30;
    for (int rd = 0; rd < PC - 1; ++rd) {
      if (tid < 16) {
        int p, q; rr_pair(PC, rd, tid, p, q);
        double cs; cplx sn; params(sm.G[p][p].x, sm.G[q][q].x, sm.G[p][q], tol2q, cs, sn);
        sm.rp[tid] = p; sm.rq[tid] = q; sm.cs[tid] = cs; sm.sn[tid] = sn;
      }
      __syncthreads();
      if (tid < 136) {
        const int ra = sm.ua[tid], rb = sm.ub[tid];
        const int p1 = sm.rp[ra], q1 = sm.rq[ra], p2 = sm.rp[rb], q2 = sm.rq[rb];
        const double ca = sm.cs[ra], cb = sm.cs[rb];
        const cplx sa = sm.sn[ra], sb = sm.sn[rb];
        const cplx b00 = gget(sm, p1, p2), b01 = gget(sm, p1, q2), b10 = gget(sm, q1, p2), b11 = gget(sm, q1, q2);
        const cplx r00 = csub(cscale(b00, ca), cmul(sa, b10));
        const cplx r01 = csub(cscale(b01, ca), cmul(sa, b11));
        const cplx r10 = cadd(cmul(cconj(sa), b00), cscale(b10, ca));
        const cplx r11 = cadd(cmul(cconj(sa), b01), cscale(b11, ca));
        cplx n00 = csub(cscale(r00, cb), cmul(cconj(sb), r01));
        cplx n01 = cadd(cmul(sb, r00), cscale(r01, cb));
        cplx n10 = csub(cscale(r10, cb), cmul(cconj(sb), r11));
        cplx n11 = cadd(cmul(sb, r10), cscale(r11, cb));
        if (ra == rb) { if (sa.x != 0.0 || sa.y != 0.0) n01 = cmk(0, 0); n00.y = n11.y = 0; n10 = cconj(n01); }
        // block (ra, rb), ra <= rb, holds rows {p1, q1} x columns {p2, q2}; for
        // ra < rb an entry with row > column belongs to the mirror: store its conjugate there
        auto put = [&](int i, int j, cplx v) { if (i <= j) sm.G[i][j] = v; else sm.G[j][i] = cconj(v); };
        put(p1, p2, n00); put(p1, q2, n01); put(q1, p2, n10); put(q1, q2, n11);
      }
      // Q units (row, pair) rebalanced: the 136 G threads take one unit each,
      // the other 120 threads the remaining 376 (at most 4 each)
      for (int v = tid < 136 ? tid : tid, h = 0; h < (tid < 136 ? 1 : 4); ++h, v += 120) {
        if (tid >= 136 && h == 0) v = tid;
        if (v >= 512) break;
        const int row = v >> 4, r2 = v & 15;
        const int p = sm.rp[r2], q = sm.rq[r2]; const double c = sm.cs[r2]; const cplx sn = sm.sn[r2];
        const cplx qp = sm.Q[row][p], qq = sm.Q[row][q];
        sm.Q[row][p] = csub(cscale(qp, c), cmul(cconj(sn), qq));
        sm.Q[row][q] = cadd(cmul(sn, qp), cscale(qq, c));
      }
      __syncthreads();
    }
  }
  if (tid == 0) *cyc = (clock64() - t0) / (reps - 1);
  for (int e = tid; e < PC * PC; e += NTB) out[e] = sm.Q[e / PC][e % PC];
}
__global__ void k8(const cplx* G0, long long* cyc, cplx* out, int reps) {
  __shared__ Sm sm;
  const int tid = threadIdx.x;
  if (tid == 0) { int u = 0; for (int a = 0; a < 16; ++a) for (int b = a; b < 16; ++b) { sm.ua[u] = a; sm.ub[u] = b; ++u; } }
  long long t0 = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int e = tid; e < PC * PC; e += NTB) { sm.G[e / PC][e % PC] = G0[e]; sm.Q[e / PC][e % PC] = cmk(e / PC == e % PC, 0); }
    __syncthreads();
    if (rep == 1) t0 = clock64();
    const double tol2q = 1e-30;
    for (int rd = 0; rd < PC - 1; ++rd) {
      if (tid < 16) {
        int p, q; rr_pair(PC, rd, tid, p, q);
        double cs; cplx sn; params_fast(sm.G[p][p].x, sm.G[q][q].x, sm.G[p][q], tol2q, cs, sn);
        sm.rp[tid] = p; sm.rq[tid] = q; sm.cs[tid] = cs; sm.sn[tid] = sn;
      }
      __syncthreads();
      if (tid < 136) {
        const int ra = sm.ua[tid], rb = sm.ub[tid];
        const int p1 = sm.rp[ra], q1 = sm.rq[ra], p2 = sm.rp[rb], q2 = sm.rq[rb];
        const double ca = sm.cs[ra], cb = sm.cs[rb];
        const cplx sa = sm.sn[ra], sb = sm.sn[rb];
        const cplx b00 = gget(sm, p1, p2), b01 = gget(sm, p1, q2), b10 = gget(sm, q1, p2), b11 = gget(sm, q1, q2);
        const cplx r00 = csub(cscale(b00, ca), cmul(sa, b10));
        const cplx r01 = csub(cscale(b01, ca), cmul(sa, b11));
        const cplx r10 = cadd(cmul(cconj(sa), b00), cscale(b10, ca));
        const cplx r11 = cadd(cmul(cconj(sa), b01), cscale(b11, ca));
        cplx n00 = csub(cscale(r00, cb), cmul(cconj(sb), r01));
        cplx n01 = cadd(cmul(sb, r00), cscale(r01, cb));
        cplx n10 = csub(cscale(r10, cb), cmul(cconj(sb), r11));
        cplx n11 = cadd(cmul(sb, r10), cscale(r11, cb));
        if (ra == rb) { if (sa.x != 0.0 || sa.y != 0.0) n01 = cmk(0, 0); n00.y = n11.y = 0; n10 = cconj(n01); }
        // block (ra, rb), ra <= rb, holds rows {p1, q1} x columns {p2, q2}; for
        // ra < rb an entry with row > column belongs to the mirror: store its conjugate there
        auto put = [&](int i, int j, cplx v) { if (i <= j) sm.G[i][j] = v; else sm.G[j][i] = cconj(v); };
        put(p1, p2, n00); put(p1, q2, n01); put(q1, p2, n10); put(q1, q2, n11);
      }
      for (int h = 0; h < 2; ++h) {
        const int v = tid + h * NTB; const int row = v >> 4, r2 = v & 15;
        const int p = sm.rp[r2], q = sm.rq[r2]; const double c = sm.cs[r2]; const cplx sn = sm.sn[r2];
        const cplx qp = sm.Q[row][p], qq = sm.Q[row][q];
        sm.Q[row][p] = csub(cscale(qp, c), cmul(cconj(sn), qq));
        sm.Q[row][q] = cadd(cmul(sn, qp), cscale(qq, c));
      }
      __syncthreads();
    }
  }
  if (tid == 0) *cyc = (clock64() - t0) / (reps - 1);
  for (int e = tid; e < PC * PC; e += NTB) out[e] = sm.Q[e / PC][e % PC];
}
int main() {
  cplx h[PC * PC];
  srand(1);
  for (int i = 0; i < PC; ++i) for (int j = 0; j <= i; ++j) {
    double re = (rand() / (double)RAND_MAX) - 0.5, im = i == j ? 0 : (rand() / (double)RAND_MAX) - 0.5;
    if (i == j) re += 10 + i;
    h[i * PC + j] = cmk(re, im); h[j * PC + i] = cmk(re, -im);
  }
  cplx *dG, *dO; long long* dc; cudaMalloc(&dG, sizeof(h)); cudaMalloc(&dO, sizeof(h)); cudaMalloc(&dc, 8);
  cudaMemcpy(dG, h, sizeof(h), cudaMemcpyHostToDevice);
  long long c0, c1; cplx o0[PC * PC], o1[PC * PC];
  k<0><<<1, NTB>>>(dG, dc, dO, 20); cudaMemcpy(&c0, dc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(o0, dO, sizeof(h), cudaMemcpyDeviceToHost);
  k<1><<<1, NTB>>>(dG, dc, dO, 20); cudaMemcpy(&c1, dc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(o1, dO, sizeof(h), cudaMemcpyDeviceToHost);
  long long c2, c3, c4;
  k<2><<<1, NTB>>>(dG, dc, dO, 20); cudaMemcpy(&c2, dc, 8, cudaMemcpyDeviceToHost);
  k<3><<<1, NTB>>>(dG, dc, dO, 20); cudaMemcpy(&c3, dc, 8, cudaMemcpyDeviceToHost);
  k<4><<<1, NTB>>>(dG, dc, dO, 20); cudaMemcpy(&c4, dc, 8, cudaMemcpyDeviceToHost);
  long long c5; cplx o5[PC * PC];
  k5<<<1, NTB>>>(dG, dc, dO, 20); cudaMemcpy(&c5, dc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(o5, dO, sizeof(h), cudaMemcpyDeviceToHost);
  double d5 = 0; for (int e = 0; e < PC * PC; ++e) d5 = fmax(d5, fabs(o0[e].x - o5[e].x) + fabs(o0[e].y - o5[e].y));
  printf("prefetch variant: %lld (%.0f/round), max |dQ| vs two-phase %.2e\n", c5, c5 / 31.0, d5);
  long long c6; cplx o6[PC * PC];
  k6<<<1, NTB>>>(dG, dc, dO, 20); cudaMemcpy(&c6, dc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(o6, dO, sizeof(h), cudaMemcpyDeviceToHost);
  double d6 = 0; for (int e = 0; e < PC * PC; ++e) d6 = fmax(d6, fabs(o0[e].x - o6[e].x) + fabs(o0[e].y - o6[e].y));
  printf("upper-only variant: %lld (%.0f/round), max |dQ| vs two-phase %.2e\n", c6, c6 / 31.0, d6);
  long long c7; cplx o7[PC * PC];
  k7<<<1, NTB>>>(dG, dc, dO, 20); cudaMemcpy(&c7, dc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(o7, dO, sizeof(h), cudaMemcpyDeviceToHost);
  double d7 = 0; for (int e = 0; e < PC * PC; ++e) d7 = fmax(d7, fabs(o0[e].x - o7[e].x) + fabs(o0[e].y - o7[e].y));
  printf("rebalanced Q variant: %lld (%.0f/round), max |dQ| vs two-phase %.2e\n", c7, c7 / 31.0, d7);
  long long c8; cplx o8[PC * PC];
  k8<<<1, NTB>>>(dG, dc, dO, 20); cudaMemcpy(&c8, dc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(o8, dO, sizeof(h), cudaMemcpyDeviceToHost);
  double d8 = 0; for (int e = 0; e < PC * PC; ++e) d8 = fmax(d8, fabs(o0[e].x - o8[e].x) + fabs(o0[e].y - o8[e].y));
  printf("fast-rsqrt variant: %lld (%.0f/round), max |dQ| vs two-phase %.2e\n", c8, c8 / 31.0, d8);
  printf("params only %.0f/round, params+G %.0f/round, params+Q %.0f/round\n", c2 / 31.0, c3 / 31.0, c4 / 31.0);
  double diff = 0; for (int e = 0; e < PC * PC; ++e) diff = fmax(diff, fabs(o0[e].x - o1[e].x) + fabs(o0[e].y - o1[e].y));
  printf("cycles per inner sweep: two-phase %lld (%.0f/round), per-warp params %lld (%.0f/round); max |dQ| %.2e; err %s\n", c0, c0 / 31.0, c1, c1 / 31.0, diff, cudaGetErrorString(cudaGetLastError()));
}
