// Block one-sided (Hestenes) Jacobi on the FP64 tensor pipe (DMMA) for the
// truncated SVD of the two-site matrix (Fig. 6; SURVEY §8(a) a4,
// K2 "block rotations on DMMA").
//
// Operates on d.Y = [X ; V] (column-major, ld = ldy): X = rows [0, xr) (after
// the QR preconditioner X = R2^H, xr = nc), V = rows [vofs, vofs + nc).  The
// columns are cut into blocks of BB = 16; a sweep is a round-robin tournament
// over the blocks (nbe - 1 rounds of nbe / 2 disjoint block pairs).  For one
// block pair (PC = 32 columns) a round
//   1. forms the PC x PC Gram matrix G = X_p^H X_p on the DMMA pipe (the
//      upper-triangular 8 x 8 tiles; one complex MAC = 4 real DMMA.8x8x4),
//      split over the S CTAs of the pair by rows (deterministic reduction:
//      warps in a fixed tree, CTAs in index order through global memory);
//   2. measures the pair's largest scaled coupling c = |g_ij| / sqrt(g_ii g_jj)
//      (the one-sided convergence test, relative, so tiny columns count);
//   3. if c > tol / 4: rotates G by two-sided Jacobi rotations in shared
//      memory -- every column pair of the matrix exactly once per outer sweep:
//      a full cyclic sweep over the pair's 32 columns in the sweep's round 0,
//      the 16 x 16 cross-block pairs in the other rounds -- accumulating the
//      unitary Q (every S CTA of the pair does this redundantly on the
//      identical G, so no broadcast is needed), and
//   4. applies X_p <- X_p Q on the DMMA pipe over its rows (all 8 warps).
// The inner solve (step 3) runs on warps 0..3 only; meanwhile warps 4..7
// replay the CTA's PREVIOUS round on V (V_p <- V_p Q_prev on its V rows, the
// same DMMA products in the same round order per block, so V is bit-identical
// to an in-round update), ordered by their own per-(block, slice) flags.  The
// V half of the rotation work thus overlaps the latency-bound inner solve
// instead of following it.
// The inner solve only has to produce a unitary Q that orthogonalises the
// pair well; the result's accuracy is set by the outer test, computed from
// the actual columns every round (one-sided Jacobi's relative accuracy).
// Rounds are ordered by point-to-point flags per (block, row slice) -- a pair
// starts as soon as its two blocks finished the previous round on its rows --
// and sweeps by a grid barrier; the sweep loop stops with the rule
// of svd_rjac.cu (c <= tol, or c^2 <= 0.01 tol: the next sweep would rotate
// nothing).  All sweeps run in ONE cooperative launch.
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

__device__ unsigned long long g_bj_prof[8];  // CTA 0 cycles per phase (TDVP_SVD_PROF)

namespace {

constexpr int BB = 16;        // columns per block
constexpr int PC = 2 * BB;    // columns per block pair
constexpr int NTB = 256;      // threads per CTA (8 warps)
constexpr int NIW = 4;        // warps of the inner solve (the other NVW replay V meanwhile)
constexpr int NVW = NTB / 32 - NIW;
constexpr int GP = PC + 1;    // padded row length of the shared PC x PC matrices
constexpr int NUT = 10;       // upper-triangular 8 x 8 tiles of a 32 x 32 Gram matrix
constexpr int NUB = (PC / 2) * (PC / 2 + 1) / 2;  // upper-triangular 2 x 2 blocks of the inner rotation rounds

struct BjArgs {
  cplx* Y;
  long long ldy;
  int xr, vofs, nc, nb, nbe;
  int S, P;  // CTAs per pair, pairs per round
  double tol;
  int max_sweeps;
  cplx* part;      // [2][P][S][PC * PC] partial Gram matrices (double-buffered by round parity)
  unsigned* pcnt;  // [P] monotonic pair counters
  unsigned* gbar;  // [1] monotonic grid-barrier counter (end of every sweep)
  unsigned* done;  // [nbe][S] X-phase rounds completed on row slice s of block b (monotonic)
  unsigned* vdone; // [nbe][S] V-phase rounds completed on row slice s of block b (monotonic)
  double* offb;    // [3] per-sweep max scaled coupling
  int* sweeps_out;
  double* flop_out;  // algorithmic DMMA flops executed (Gram + apply)
  int prof;
  int inner_max;  // inner Jacobi sweeps per block pair and round (at most)
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

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

// upper-triangular tile index t -> (ti, tj), ti <= tj, of the 4 x 4 tile grid
__device__ __forceinline__ void ut_tile(int t, int& ti, int& tj) {
  constexpr int TI[NUT] = {0, 0, 0, 0, 1, 1, 1, 2, 2, 3};
  constexpr int TJ[NUT] = {0, 1, 2, 3, 1, 2, 3, 2, 3, 3};
  ti = TI[t];
  tj = TJ[t];
}

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    while (true) {
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if ((int)(v - target) >= 0) break;
      __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// per-warp cp.async ring: NST stages of 8 rows x PC columns (column-major,
// row index swizzled by sw(col) so both the Gram's and the apply's fragment
// reads are bank-conflict free)
constexpr int NST = 4;
constexpr int STG = 8 * PC;  // complex elements per stage
__device__ __forceinline__ int sw(int col) { return ((col & 1) << 2) | (col & 2); }
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

struct Smem {
  union {
    cplx red[4][PC * GP];       // warp-tree reduction of the Gram tiles
    cplx ring[8][NST][STG];     // cp.async staging of X / V rows (Gram and apply loops)
  };
  cplx G[PC][GP];
  cplx Q[PC][GP];
  cplx Qp[PC][GP];   // the previous round's Q (pending V update)
  double cs[PC / 2];
  cplx sn[PC / 2];
  int rp[PC / 2], rq[PC / 2];
  int col[PC];       // global column of pair column i (-1: absent)
  int colp[PC];      // the previous round's columns (pending V update)
  cplx part[2][PC * PC];  // CL: this CTA's partial Gram (by round parity), read by the pair's cluster
  unsigned char ut_a[136], ut_b[136];  // upper-triangle 2 x 2 block u -> (row pair, column pair)
  double offw[8];
  int any;
};

// CL: the S CTAs of a pair form one thread-block cluster and exchange their
// partial Grams through distributed shared memory (one cluster barrier per
// round); else through global memory and a per-pair counter
template <bool CL>
__global__ void __launch_bounds__(NTB, 1) bjac_kernel(BjArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  Smem& sm = *reinterpret_cast<Smem*>(smraw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int pair = blockIdx.x / a.S, s = blockIdx.x - pair * a.S;
  const unsigned G_ = gridDim.x;
  cplx* __restrict__ Y = a.Y;
  const long long ldy = a.ldy;
  const double tol = a.tol, tol4 = 0.25 * tol;
  // this CTA's row ranges (multiples of 8) of X and of V
  auto split = [&](int n, int& r0, int& r1) {
    const int chunks = (n + 7) / 8;
    const int c0 = (int)((long long)chunks * s / a.S), c1 = (int)((long long)chunks * (s + 1) / a.S);
    r0 = c0 * 8;
    r1 = min(n, c1 * 8);
  };
  int xr0, xr1, vr0, vr1;
  split(a.xr, xr0, xr1);
  split(a.nc, vr0, vr1);
  if (tid == 0) {
    int u = 0;
    for (int ra = 0; ra < PC / 2; ++ra)
      for (int rb = ra; rb < PC / 2; ++rb) {
        sm.ut_a[u] = (unsigned char)ra;
        sm.ut_b[u] = (unsigned char)rb;
        ++u;
      }
  }
  __syncthreads();
  unsigned long long round_g = 0;  // rounds completed (all sweeps), for the monotonic counters
  const bool prof = a.prof && blockIdx.x == 0 && tid == 0;
  unsigned long long pt = clock64();
  auto mark = [&](int i) {
    if (prof) {
      const unsigned long long t = clock64();
      g_bj_prof[i] += t - pt;
      pt = t;
    }
  };
  // Y_p rows [rb0, re0) <- Y_p Q (sm.Q, columns sm.col) on the DMMA pipe:
  // 8-row stages, warp w takes stages w, w+8, ... through its cp.async ring.
  // 3M products: a q = (P1 - P2) + i (P3 - P1 - P2) with P1 = ar qr,
  // P2 = ai qi, P3 = (ar + ai)(qr + qi)
  // Warps wl = 0 .. nw - 1 of the calling group (wl = wid - first warp).
  auto apply_rows = [&](int rb0, int re0, const cplx (*Qm)[GP], const int* colv, int wl, int nw) {
    double bqr[8][4], bqi[8][4], bqs[8][4];  // B fragments of Q: [k-step][j-tile]
#pragma unroll
    for (int ks = 0; ks < 8; ++ks)
#pragma unroll
      for (int jt = 0; jt < 4; ++jt) {
        const cplx q = Qm[ks * 4 + (lane & 3)][jt * 8 + (lane >> 2)];
        bqr[ks][jt] = q.x;
        bqi[ks][jt] = q.y;
        bqs[ks][jt] = q.x + q.y;
      }
    int cs_[4][2];
#pragma unroll
    for (int jt = 0; jt < 4; ++jt)
#pragma unroll
      for (int h = 0; h < 2; ++h) cs_[jt][h] = colv[jt * 8 + 2 * (lane & 3) + h];
    int ccol[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) ccol[k] = colv[(lane >> 3) + 4 * k];
    cplx* ring = &sm.ring[wid][0][0];
    const int nstage = (re0 - rb0 + 7) / 8;
    auto issue = [&](int j, int slot) {
      const int rb = rb0 + 8 * j;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int col = (lane >> 3) + 4 * k, r = lane & 7, row = rb + r;
        const bool v = j < nstage && ccol[k] >= 0 && row < re0;
        cp_async16(ring + slot * STG + col * 8 + (r ^ sw(col)), v ? (const void*)(Y + (long long)ccol[k] * ldy + row)
                                                                  : (const void*)Y, v);
      }
      cp_commit();
    };
#pragma unroll
    for (int i = 0; i < NST - 1; ++i) issue(wl + nw * i, i);
    int slot = 0;
    for (int j = wl; j < nstage; j += nw) {
      cp_wait<NST - 2>();
      __syncwarp();
      issue(j + nw * (NST - 1), slot == 0 ? NST - 1 : slot - 1);
      const cplx* st = ring + slot * STG;
      cplx av[8];
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const int col = ks * 4 + (lane & 3), r = lane >> 2;
        av[ks] = st[col * 8 + (r ^ sw(col))];
      }
      double c1[4][2], c2[4][2], c3[4][2];
#pragma unroll
      for (int jt = 0; jt < 4; ++jt) c1[jt][0] = c1[jt][1] = c2[jt][0] = c2[jt][1] = c3[jt][0] = c3[jt][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const double as = av[ks].x + av[ks].y;
#pragma unroll
        for (int jt = 0; jt < 4; ++jt) {
          dmma(c1[jt][0], c1[jt][1], av[ks].x, bqr[ks][jt]);
          dmma(c2[jt][0], c2[jt][1], av[ks].y, bqi[ks][jt]);
          dmma(c3[jt][0], c3[jt][1], as, bqs[ks][jt]);
        }
      }
      slot = slot + 1 == NST ? 0 : slot + 1;
      const int ro = rb0 + 8 * j + (lane >> 2);
      if (ro < re0) {
#pragma unroll
        for (int jt = 0; jt < 4; ++jt)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (cs_[jt][h] >= 0)
              __stcg(Y + (long long)cs_[jt][h] * ldy + ro,
                     cmk(c1[jt][h] - c2[jt][h], c3[jt][h] - c1[jt][h] - c2[jt][h]));
      }
    }
    cp_wait<0>();
  };
  // V update pending from this CTA's previous round (warps 4..7 replay it
  // during the next round's inner solve): blocks, global round index, whether
  // the pair rotated; its Q and columns wait in sm.Qp / sm.colp
  bool pv = false, pv_rot = false;
  int pvI = 0, pvJ = 0;
  unsigned long long pv_g = 0;
  double vflops = 0.0;
  // V rows [rb0, re0) <- V Q_prev (sm.Qp, columns sm.colp) by warps 4..7
  // (wl = wid - NIW), like apply_rows over the warp's own cp.async ring (an
  // 8-stage ring borrowing the idle inner warp's stages measured the same:
  // the V stream is bound by DMMA issue of one warp per SM sub-partition)
  constexpr int NSV = NST;
  auto v_stream = [&](int rb0, int re0) {
    const int wl = wid - NIW;
    double bqr[8][4], bqi[8][4], bqs[8][4];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks)
#pragma unroll
      for (int jt = 0; jt < 4; ++jt) {
        const cplx q = sm.Qp[ks * 4 + (lane & 3)][jt * 8 + (lane >> 2)];
        bqr[ks][jt] = q.x;
        bqi[ks][jt] = q.y;
        bqs[ks][jt] = q.x + q.y;
      }
    int cs_[4][2];
#pragma unroll
    for (int jt = 0; jt < 4; ++jt)
#pragma unroll
      for (int h = 0; h < 2; ++h) cs_[jt][h] = sm.colp[jt * 8 + 2 * (lane & 3) + h];
    int ccol[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) ccol[k] = sm.colp[(lane >> 3) + 4 * k];
    cplx* const rbase = &sm.ring[wid][0][0];
    auto slot_ptr = [&](int slot) -> cplx* { return rbase + slot * STG; };
    const int nstage = (re0 - rb0 + 7) / 8;
    auto issue = [&](int j, int slot) {
      const int rb = rb0 + 8 * j;
      cplx* dst = slot_ptr(slot);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int col = (lane >> 3) + 4 * k, r = lane & 7, row = rb + r;
        const bool v = j < nstage && ccol[k] >= 0 && row < re0;
        cp_async16(dst + col * 8 + (r ^ sw(col)), v ? (const void*)(Y + (long long)ccol[k] * ldy + row) : (const void*)Y,
                   v);
      }
      cp_commit();
    };
#pragma unroll
    for (int i = 0; i < NSV - 1; ++i) issue(wl + NVW * i, i);
    int slot = 0;
    for (int j = wl; j < nstage; j += NVW) {
      cp_wait<NSV - 2>();
      __syncwarp();
      issue(j + NVW * (NSV - 1), slot == 0 ? NSV - 1 : slot - 1);
      const cplx* st = slot_ptr(slot);
      cplx av[8];
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const int col = ks * 4 + (lane & 3), r = lane >> 2;
        av[ks] = st[col * 8 + (r ^ sw(col))];
      }
      double c1[4][2], c2[4][2], c3[4][2];
#pragma unroll
      for (int jt = 0; jt < 4; ++jt) c1[jt][0] = c1[jt][1] = c2[jt][0] = c2[jt][1] = c3[jt][0] = c3[jt][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const double as = av[ks].x + av[ks].y;
#pragma unroll
        for (int jt = 0; jt < 4; ++jt) {
          dmma(c1[jt][0], c1[jt][1], av[ks].x, bqr[ks][jt]);
          dmma(c2[jt][0], c2[jt][1], av[ks].y, bqi[ks][jt]);
          dmma(c3[jt][0], c3[jt][1], as, bqs[ks][jt]);
        }
      }
      const int ro = rb0 + 8 * j + (lane >> 2);
      if (ro < re0) {
#pragma unroll
        for (int jt = 0; jt < 4; ++jt)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (cs_[jt][h] >= 0)
              __stcg(Y + (long long)cs_[jt][h] * ldy + ro,
                     cmk(c1[jt][h] - c2[jt][h], c3[jt][h] - c1[jt][h] - c2[jt][h]));
      }
      slot = slot + 1 == NSV ? 0 : slot + 1;
    }
    cp_wait<0>();
  };
  // the pending update's blocks finished their previous V round on slice s
  auto v_wait = [&]() {
    for (const int blk : {pvI, pvJ}) {
      const unsigned* f = a.vdone + (long long)blk * a.S + s;
      while (true) {
        unsigned v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if ((int)(v - (unsigned)pv_g) >= 0) break;
        __nanosleep(20);
      }
    }
  };
  auto v_release = [&]() {  // after a __syncthreads that follows every v_stream
    if (tid == NIW * 32) {
      __threadfence();
      for (const int blk : {pvI, pvJ}) {
        unsigned* f = a.vdone + (long long)blk * a.S + s;
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"((unsigned)(pv_g + 1)) : "memory");
      }
      if (s == 0 && pv_rot) vflops += 8.0 * (double)a.nc * PC * PC;
    }
  };
  double flops = 0.0;
  int sweep = 0;
  for (; sweep < a.max_sweeps; ++sweep) {
    double* off_cur = a.offb + (sweep % 3);
    if (blockIdx.x == 0 && tid == 0) a.offb[(sweep + 1) % 3] = 0.0;
    for (int round = 0; round < a.nbe - 1; ++round, ++round_g) {
      int bI, bJ;
      rr_pair(a.nbe, round, pair, bI, bJ);
      // point-to-point dependencies instead of a grid barrier: slice s of
      // blocks I and J must have finished the previous round (their slice s
      // rows are only ever read and written by the slice-s CTA of their pair)
      if (tid == 0) {
        const unsigned need = (unsigned)round_g;
        for (const int blk : {bI, bJ}) {
          const unsigned* f = a.done + (long long)blk * a.S + s;
          while (true) {
            unsigned v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
            if ((int)(v - need) >= 0) break;
            __nanosleep(20);
          }
        }
      }
      if (tid < PC) {
        const int blk = tid < BB ? bI : bJ;
        const int c = blk * BB + (tid & (BB - 1));
        sm.col[tid] = (blk < a.nb && c < a.nc) ? c : -1;
      }
      __syncthreads();
      // ---- 1. partial Gram over rows [xr0, xr1) of X: warp w takes 8-row
      // stages w, w+8, ... streamed through its cp.async ring (NST - 1 stages
      // in flight), two 4-row DMMA k-steps per stage
      // 3M products: conj(a) b = (P1 + P2) + i (P3 - P1 + P2) with P1 = ar br,
      // P2 = ai bi, P3 = (ar - ai)(br + bi): three real DMMAs per complex MAC
      double g1[NUT][2], g2[NUT][2], g3[NUT][2];
#pragma unroll
      for (int t = 0; t < NUT; ++t) g1[t][0] = g1[t][1] = g2[t][0] = g2[t][1] = g3[t][0] = g3[t][1] = 0.0;
      {
        // this lane's cp.async chunks: c = lane + 32 k -> column c >> 3, row c & 7
        int ccol[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) ccol[k] = sm.col[(lane >> 3) + 4 * k];
        cplx* ring = &sm.ring[wid][0][0];
        const int nstage = (xr1 - xr0 + 7) / 8;
        auto issue = [&](int j, int slot) {
          const int rb = xr0 + 8 * j;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int col = (lane >> 3) + 4 * k, r = lane & 7, row = rb + r;
            const bool v = j < nstage && ccol[k] >= 0 && row < xr1;
            cp_async16(ring + slot * STG + col * 8 + (r ^ sw(col)), v ? (const void*)(Y + (long long)ccol[k] * ldy + row)
                                                                      : (const void*)Y, v);
          }
          cp_commit();
        };
#pragma unroll
        for (int i = 0; i < NST - 1; ++i) issue(wid + 8 * i, i);
        int slot = 0;
        for (int j = wid; j < nstage; j += 8) {
          cp_wait<NST - 2>();
          __syncwarp();
          // refill the slot consumed in the previous iteration, NST - 1 stages ahead
          issue(j + 8 * (NST - 1), slot == 0 ? NST - 1 : slot - 1);
          const cplx* st = ring + slot * STG;
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            double xr_[4], xi_[4], xs[4], xd[4];
#pragma unroll
            for (int cb = 0; cb < 4; ++cb) {
              const int col = cb * 8 + (lane >> 2), r = 4 * t + (lane & 3);
              const cplx v = st[col * 8 + (r ^ sw(col))];
              xr_[cb] = v.x;
              xi_[cb] = v.y;
              xs[cb] = v.x + v.y;
              xd[cb] = v.x - v.y;
            }
#pragma unroll
            for (int tt = 0; tt < NUT; ++tt) {
              int ti, tj;
              ut_tile(tt, ti, tj);
              // G[i][j] += conj(x_ki) x_kj : A from x[ti] (row-major 8x4), B from x[tj] (col-major 4x8)
              dmma(g1[tt][0], g1[tt][1], xr_[ti], xr_[tj]);
              dmma(g2[tt][0], g2[tt][1], xi_[ti], xi_[tj]);
              dmma(g3[tt][0], g3[tt][1], xd[ti], xs[tj]);
            }
          }
          slot = slot + 1 == NST ? 0 : slot + 1;
        }
        cp_wait<0>();
      }
      __syncthreads();  // every warp is done with its ring (aliases the reduction buffer)
      double gR[NUT][2], gI[NUT][2];
#pragma unroll
      for (int t = 0; t < NUT; ++t)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          gR[t][h] = g1[t][h] + g2[t][h];
          gI[t][h] = g3[t][h] - g1[t][h] + g2[t][h];
        }
      mark(0);
      // warp tree (fixed order): 4-7 -> 0-3, 2-3 -> 0-1, 1 -> 0
      auto tile_store = [&](cplx* dst) {
#pragma unroll
        for (int t = 0; t < NUT; ++t) {
          int ti, tj;
          ut_tile(t, ti, tj);
          const int r = ti * 8 + (lane >> 2);
#pragma unroll
          for (int h = 0; h < 2; ++h) dst[r * GP + tj * 8 + 2 * (lane & 3) + h] = cmk(gR[t][h], gI[t][h]);
        }
      };
      auto tile_add = [&](const cplx* src) {
#pragma unroll
        for (int t = 0; t < NUT; ++t) {
          int ti, tj;
          ut_tile(t, ti, tj);
          const int r = ti * 8 + (lane >> 2);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const cplx v = src[r * GP + tj * 8 + 2 * (lane & 3) + h];
            gR[t][h] += v.x;
            gI[t][h] += v.y;
          }
        }
      };
      if (wid >= 4) tile_store(sm.red[wid - 4]);
      __syncthreads();
      if (wid < 4) tile_add(sm.red[wid]);
      __syncthreads();
      if (wid == 2 || wid == 3) tile_store(sm.red[wid - 2]);
      __syncthreads();
      if (wid < 2) tile_add(sm.red[wid]);
      __syncthreads();
      if (wid == 1) tile_store(sm.red[0]);
      __syncthreads();
      if (wid == 0) {
        tile_add(sm.red[0]);
        // this CTA's partial -> its slot (upper tiles only)
        cplx* dst = CL ? sm.part[round_g & 1]
                       : a.part + (((long long)(round_g & 1) * a.P + pair) * a.S + s) * (PC * PC);
#pragma unroll
        for (int t = 0; t < NUT; ++t) {
          int ti, tj;
          ut_tile(t, ti, tj);
          const int r = ti * 8 + (lane >> 2);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            cplx* q = dst + r * PC + tj * 8 + 2 * (lane & 3) + h;
            if (CL) *q = cmk(gR[t][h], gI[t][h]);
            else __stcg(q, cmk(gR[t][h], gI[t][h]));
          }
        }
      }
      // pair barrier: all S partials of this pair written
      if (CL) {
        // the partial slots are double-buffered by round parity: a CTA writes
        // round r + 2's only after this barrier of round r + 1, which the
        // others pass only after their reads of round r
        cooperative_groups::this_cluster().sync();
      } else {
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          atomicAdd(a.pcnt + pair, 1u);
          const unsigned target = (unsigned)((round_g + 1) * (unsigned long long)a.S);
          while (true) {
            unsigned v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.pcnt + pair) : "memory");
            if ((int)(v - target) >= 0) break;
            __nanosleep(20);
          }
          __threadfence();
        }
        __syncthreads();
      }
      // ---- sum the S partials in index order -> G (Hermitian, both triangles)
      for (int e = tid; e < PC * PC; e += NTB) {
        const int i = e / PC, j = e - i * PC;
        if (i <= j) {
          cplx v = cmk(0.0, 0.0);
          for (int q = 0; q < a.S; ++q) {
            if (CL) {
              cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
              v = cadd(v, *cl.map_shared_rank(&sm.part[round_g & 1][e], q));
            } else {
              v = cadd(v, __ldcg(a.part + (((long long)(round_g & 1) * a.P + pair) * a.S + q) * (PC * PC) + e));
            }
          }
          if (i == j) v.y = 0.0;
          sm.G[i][j] = v;
          sm.G[j][i] = cconj(v);
        }
      }
      __syncthreads();
      // ---- 2. largest scaled coupling of the pair (one-sided convergence test)
      {
        double m = 0.0;
        for (int e = tid; e < PC * PC; e += NTB) {
          const int i = e / PC, j = e - i * PC;
          if (i < j) {
            const double gi = sm.G[i][i].x, gj = sm.G[j][j].x;
            if (gi > 0.0 && gj > 0.0) m = fmax(m, cabs2(sm.G[i][j]) / (gi * gj));
          }
        }
        m = warp_max(m);
        if (lane == 0) sm.offw[wid] = m;
      }
      __syncthreads();
      double c2 = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) c2 = fmax(c2, sm.offw[w]);
      const double cpair = sqrt(c2);
      mark(1);
      if (s == 0 && tid == 0) {
        atomic_max_nonneg(off_cur, cpair);
        flops += 8.0 * (double)a.xr * PC * PC * (double)NUT / 16.0;
      }
      const bool rotate = cpair > tol4;
      if (wid < NIW) {
        if (rotate) {
        // ---- 3. two-sided cyclic Jacobi on G (shared memory), Q accumulated,
        // by warps 0..3 (named barrier 1) while warps 4..7 replay the previous
        // round's rotation on this CTA's V rows
        for (int e = tid; e < PC * PC; e += NIW * 32) {
          const int i = e / PC, j = e - i * PC;
          sm.Q[i][j] = cmk(i == j ? 1.0 : 0.0, 0.0);
        }
        const double tol2q = tol4 * tol4;
        // Each column pair once per outer sweep (as svd_rjac.cu): in the
        // sweep's round 0 (where every block sits in exactly one pair) a full
        // cyclic sweep over the 32 columns, 31 rotation rounds of 16 disjoint
        // rotations (intra-block and cross pairs); in the other rounds only
        // the 16 cross-block rotation rounds (i, 16 + (i + rd) mod 16).
        // Per rotation round: threads 0..15 compute the parameters (rsqrt
        // only); then the inner warps update the 136 2 x 2 blocks of the upper
        // triangle of G (row pair ra <= column pair rb; the lower triangle is
        // the mirror) and the (row, column pair) entries of Q.
        const int nrd = round == 0 ? PC - 1 : BB;
        for (int rd = 0; rd < nrd; ++rd) {
          if (tid < PC / 2) {
            int p, q;
            if (round == 0) {
              rr_pair(PC, rd, tid, p, q);
            } else {
              p = tid;
              q = BB + ((tid + rd) & (BB - 1));
            }
            double cs = 1.0;
            cplx sn = cmk(0.0, 0.0);
            const double ga = sm.G[p][p].x, gc = sm.G[q][q].x;
            const cplx g = sm.G[p][q];
            const double ag2 = cabs2(g);
            const double gg = ga * gc;
            if (ga > 0.0 && gc > 0.0 && ag2 > 1e-300 && ag2 > tol2q * gg) {
              // zero g = x_p^H x_q by x_p' = cs x_p - conj(sn) x_q, x_q' = sn x_p + cs x_q:
              // cos^2 = (1 + |w| / D) / 2, sn = sgn(w) g / (D cs), D = sqrt(w^2 + 4 |g|^2)
              const double w = gc - ga;
              const double rD = rsqrt(fma(w, w, 4.0 * ag2));
              const double qq = 0.5 * fma(fabs(w), rD, 1.0);
              const double rcs = rsqrt(qq);
              cs = qq * rcs;
              const double f = copysign(rD * rcs, w);
              sn = cmk(f * g.x, f * g.y);
            }
            sm.rp[tid] = p;
            sm.rq[tid] = q;
            sm.cs[tid] = cs;
            sm.sn[tid] = sn;
          }
          named_bar(1, NIW * 32);
          for (int ub = tid; ub < NUB; ub += NIW * 32) {
            const int ra = sm.ut_a[ub], rb = sm.ut_b[ub];
            const int p1 = sm.rp[ra], q1 = sm.rq[ra], p2 = sm.rp[rb], q2 = sm.rq[rb];
            const double ca = sm.cs[ra], cb = sm.cs[rb];
            const cplx sa = sm.sn[ra], sb = sm.sn[rb];
            const cplx b00 = sm.G[p1][p2], b01 = sm.G[p1][q2], b10 = sm.G[q1][p2], b11 = sm.G[q1][q2];
            // B <- J_a^H B J_b ; rows: p' = ca p - sa q, q' = conj(sa) p + ca q
            const cplx r00 = csub(cscale(b00, ca), cmul(sa, b10));
            const cplx r01 = csub(cscale(b01, ca), cmul(sa, b11));
            const cplx r10 = cadd(cmul(cconj(sa), b00), cscale(b10, ca));
            const cplx r11 = cadd(cmul(cconj(sa), b01), cscale(b11, ca));
            // columns: p' = cb p - conj(sb) q ; q' = sb p + cb q
            cplx n00 = csub(cscale(r00, cb), cmul(cconj(sb), r01));
            cplx n01 = cadd(cmul(sb, r00), cscale(r01, cb));
            cplx n10 = csub(cscale(r10, cb), cmul(cconj(sb), r11));
            cplx n11 = cadd(cmul(sb, r10), cscale(r11, cb));
            if (ra == rb) {
              if (sa.x != 0.0 || sa.y != 0.0) n01 = cmk(0.0, 0.0);
              n00.y = n11.y = 0.0;
              n10 = cconj(n01);
            }
            sm.G[p1][p2] = n00;
            sm.G[p1][q2] = n01;
            sm.G[q1][p2] = n10;
            sm.G[q1][q2] = n11;
            if (ra != rb) {  // mirror: G[b][a] = G[a][b]^H
              sm.G[p2][p1] = cconj(n00);
              sm.G[q2][p1] = cconj(n01);
              sm.G[p2][q1] = cconj(n10);
              sm.G[q2][q1] = cconj(n11);
            }
          }
          // Q <- Q J_b: units (row, column pair) = tid + 128 h
#pragma unroll
          for (int h = 0; h < (PC * PC / 2 + NIW * 32 - 1) / (NIW * 32); ++h) {
            const int u = tid + h * NIW * 32;
            if (u >= PC * PC / 2) break;
            const int row = u >> 4, rb = u & 15;
            const int p2 = sm.rp[rb], q2 = sm.rq[rb];
            const double cb = sm.cs[rb];
            const cplx sb = sm.sn[rb];
            const cplx qp = sm.Q[row][p2], qq = sm.Q[row][q2];
            sm.Q[row][p2] = csub(cscale(qp, cb), cmul(cconj(sb), qq));
            sm.Q[row][q2] = cadd(cmul(sb, qp), cscale(qq, cb));
          }
          named_bar(1, NIW * 32);
        }
        }
      } else if (pv) {
        const bool vprof = a.prof && blockIdx.x == 0 && tid == NIW * 32;
        const unsigned long long t0 = vprof ? clock64() : 0;
        if (tid == NIW * 32) v_wait();
        named_bar(2, NVW * 32);
        if (pv_rot) v_stream(a.vofs + vr0, a.vofs + vr1);
        if (vprof) g_bj_prof[5] += clock64() - t0;
      }
      __syncthreads();
      if (pv) v_release();
      if (rotate) {
        if (prof) g_bj_prof[6]++;
        if (prof) g_bj_prof[7]++;
        mark(2);
        // ---- 4. X_p <- X_p Q on the DMMA pipe over this CTA's rows (all warps)
        if (s == 0 && tid == 0) flops += 8.0 * (double)a.xr * PC * PC;
        apply_rows(xr0, xr1, sm.Q, sm.col, wid, 8);
      }
      mark(3);
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        const unsigned v = (unsigned)(round_g + 1);
        for (const int blk : {bI, bJ}) {
          unsigned* f = a.done + (long long)blk * a.S + s;
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
        }
      }
      // this round's V update becomes pending (replayed during the next
      // round's inner solve, or after the last sweep)
      if (rotate)
        for (int e = tid; e < PC * PC; e += NTB) sm.Qp[e / PC][e % PC] = sm.Q[e / PC][e % PC];
      if (tid < PC) sm.colp[tid] = sm.col[tid];
      pv = true;
      pv_rot = rotate;
      pvI = bI;
      pvJ = bJ;
      pv_g = round_g;
      __syncthreads();
    }
    grid_barrier(a.gbar, (unsigned)((sweep + 1) * (unsigned long long)G_));
    mark(4);
    const double off = __ldcg(off_cur);
    if (!(off > tol) || off * off <= 0.01 * tol) break;
  }
  if (pv) {  // the last round's V update
    if (tid == NIW * 32) v_wait();
    __syncthreads();
    if (pv_rot && wid >= NIW) v_stream(a.vofs + vr0, a.vofs + vr1);
    __syncthreads();
    v_release();
  }
  if (blockIdx.x == 0 && tid == 0) *a.sweeps_out = min(sweep + 1, a.max_sweeps);
  if (s == 0 && tid == 0 && flops > 0.0) atomicAdd(a.flop_out, flops);
  if (s == 0 && tid == NIW * 32 && vflops > 0.0) atomicAdd(a.flop_out, vflops);
  if (CL) cooperative_groups::this_cluster().sync();  // partners may still read this CTA's partials
}

}  // namespace

size_t svd_bjac_work_elems(int sms) { return (size_t)2 * sms * PC * PC + 64; }

// Jacobi stage on d.Y = [X ; V]: X rows [0, xr), V rows [vofs, vofs + nc).
// cudaErrorNotSupported when the shape or the workspace does not fit.
cudaError_t svd_bjac_run(cudaStream_t st, const SvdDev& d, int xr, int vofs, int nc, long long ldy, double tol,
                         int* sweeps_dev, double* flop_dev) {
  if (d.bjwork == nullptr || d.flags == nullptr || nc < PC) return cudaErrorNotSupported;
  const int nb = (nc + BB - 1) / BB;
  const int nbe = nb + (nb & 1);
  const int P = nbe / 2;
  const void* fn = reinterpret_cast<const void*>(bjac_kernel<false>);
  const void* fnc = reinterpret_cast<const void*>(bjac_kernel<true>);
  const size_t smem = sizeof(Smem);
  cudaError_t e;
  if ((e = set_smem_attr(fn, (int)smem)) != cudaSuccess) return e;
  if ((e = set_smem_attr(fnc, (int)smem)) != cudaSuccess) return e;
  if ((e = set_cluster_nonportable(fnc)) != cudaSuccess) return e;
  int occ = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bjac_kernel<false>, NTB, smem)) != cudaSuccess) return e;
  if (occ < 1) return cudaErrorNotSupported;
  // S CTAs per pair (row slices) so that the grid fills the SMs once
  const int S = std::max(1, std::min(16, occ * g_num_sms / P));
  if (P * S > occ * g_num_sms) return cudaErrorNotSupported;
  const size_t nfl = (size_t)P + 1 + (size_t)2 * nbe * S;
  const size_t npart = (size_t)2 * P * S * PC * PC;
  if (npart > d.bjwork_elems || nfl > d.flags_elems)
    return cudaErrorNotSupported;
  unsigned* pcnt = d.flags;
  unsigned* gbar = d.flags + P;
  unsigned* done = d.flags + P + 1;
  unsigned* vdone = done + (size_t)nbe * S;
  if ((e = cudaMemsetAsync(d.flags, 0, nfl * sizeof(unsigned), st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(d.offmax, 0, 4 * sizeof(double), st)) != cudaSuccess) return e;
  BjArgs a;
  a.Y = d.Y;
  a.ldy = ldy;
  a.xr = xr;
  a.vofs = vofs;
  a.nc = nc;
  a.nb = nb;
  a.nbe = nbe;
  a.S = S;
  a.P = P;
  a.tol = tol;
  a.max_sweeps = 60;
  a.part = d.bjwork;
  a.vdone = vdone;
  a.pcnt = pcnt;
  a.gbar = gbar;
  a.done = done;
  a.offb = d.offmax;
  a.sweeps_out = sweeps_dev;
  a.flop_out = flop_dev;
  static const int prof = std::getenv("TDVP_SVD_PROF") ? 1 : 0;  // thread-safe once
  a.prof = prof;
  a.inner_max = 1;  // one inner sweep per round (measured fastest: the outer sweep count does not grow)
  if (prof) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbolAsync(g_bj_prof, z, sizeof(z), 0, cudaMemcpyHostToDevice, st);
  }
  void* args[] = {(void*)&a};
  // cluster variant when the P clusters of S CTAs can all be resident at once
  // (a cooperative launch needs every CTA co-resident for the sweep barrier)
  bool cl = false;
  {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    cfg.gridDim = dim3(P * S);
    cfg.blockDim = dim3(NTB);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = S;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    static const int use_cl = [] {  // thread-safe once
      const char* ev = std::getenv("TDVP_BJ_CLUSTER");
      return ev ? std::atoi(ev) : 1;
    }();
    if (use_cl && S > 1 && cudaOccupancyMaxActiveClusters(&ncl, fnc, &cfg) == cudaSuccess && ncl >= P) {
      cfg.numAttrs = 2;
      e = cudaLaunchKernelEx(&cfg, bjac_kernel<true>, a);
      cl = e == cudaSuccess;
      if (!cl) cudaGetLastError();  // not launchable as a cooperative cluster grid: the global-memory exchange
    } else {
      cudaGetLastError();
    }
  }
  if (!cl) e = cudaLaunchCooperativeKernel(fn, dim3(P * S), dim3(NTB), args, smem, st);
  if (e == cudaSuccess && prof) {
    unsigned long long z[8];
    cudaMemcpyFromSymbolAsync(z, g_bj_prof, sizeof(z), 0, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    std::fprintf(stderr,
                 "bjac prof xr=%d nc=%d P=%d S=%d cycles: gram %llu pairsum %llu inner %llu apply %llu gridbar %llu vphase %llu | "
                 "inner sweeps %llu in %llu rounds\n",
                 xr, nc, P, S, z[0], z[1], z[2], z[3], z[4], z[5], z[6], z[7]);
  }
  return e;
}
