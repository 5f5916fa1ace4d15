// Internal kernel launchers of libtdvp (not part of the public C-ABI).
#pragma once
#include <cuda_runtime.h>
#include <algorithm>
#include <cstddef>
#include "common.cuh"

extern int g_num_sms;

// ---------------------------------------------------------------- zgemm.cu
// C[b] = alpha * op(A[b]) op(B[b]) + beta * C[b], row-major complex128.
// op: 0 = N, 1 = T, 2 = C (conj-transpose), 3 = R (conj, no transpose).
// op(A) is M x K (A stored M x K for N/R, K x M for T/C); op(B) is K x N.
// `work` (optional) enables deterministic split-K for small M x N.
enum { OP_N = 0, OP_T = 1, OP_C = 2, OP_R = 3 };
// Structural block masks of op(A) (M x K) and op(B) (K x N) for block-sparse
// operands (U(1) charge blocks): a[(m/32) * ldA + k/8] != 0 when the
// 32-row x 8-column block of op(A) may be nonzero, b[(k/8) * ldB + n/32]
// likewise for op(B); a CTA visits only the k-chunks where both its A rows
// and its B columns may be nonzero (exact zeros elsewhere, so the product is
// unchanged).  Device pointers; nullptr = dense.
struct GemmMask {
  const unsigned char* a = nullptr;
  const unsigned char* b = nullptr;
  int ldA = 0, ldB = 0;
};
cudaError_t zgemm(cudaStream_t st, int opA, int opB, int M, int N, int K, cplx alpha, const cplx* A, long long lda,
                  const cplx* B, long long ldb, cplx beta, cplx* C, long long ldc, int batch = 1, long long sA = 0,
                  long long sB = 0, long long sC = 0, cplx* work = nullptr, size_t work_elems = 0,
                  const double* skip = nullptr, const GemmMask* mask = nullptr);

// -------------------------------------------------------------- chanmix.cu
// Sparse MPO-channel contraction:
//   out[o*so_out + off_out(oc) + i*si_out] = sum_{e in row oc} coef[e] * in[o*so_in + off_in(e) + i*si_in]
// with off(.) = c0*s0 + c1*s1 + c2*s2 from per-channel index triples.
struct ChanMix {
  int n_oc = 0, nnz = 0;
  int* rowptr = nullptr;   // device [n_oc+1]
  int4* oc_idx = nullptr;  // device [n_oc]   (c0, c1, c2, -)
  int4* ic_idx = nullptr;  // device [nnz]    (c0, c1, c2, -)
  cplx* coef = nullptr;    // device [nnz]
  int n_ic = 0;            // distinct input channels
  int4* icu_idx = nullptr; // device [n_ic]  (c0, c1, c2, -)
  int* slot = nullptr;     // device [nnz]   entry -> distinct input channel
};
struct Strides3 {
  long long s0, s1, s2;
};
// skip: device flag, != 0 -> the kernel returns at once (converged Lanczos, krylov_tol > 0)
cudaError_t chanmix(cudaStream_t st, const ChanMix& cm, int n_outer, int n_inner, const cplx* in, long long so_in,
                    long long si_in, Strides3 in_ch, cplx* out, long long so_out, long long si_out, Strides3 out_ch,
                    const double* skip = nullptr);

// ---------------------------------------------------------------- vec.cu
cudaError_t scale_rows(cudaStream_t st, cplx* out, const cplx* in, const double* v, int rows, long long cols);
cudaError_t scale_cols(cudaStream_t st, cplx* out, const cplx* in, const double* v, long long rows, int cols);
cudaError_t copy_cplx(cudaStream_t st, cplx* dst, const cplx* src, long long n);
cudaError_t fill_cplx(cudaStream_t st, cplx* dst, cplx v, long long n);
// result (device cplx) = sum_i x_i * y_i (no conjugation), deterministic.
cudaError_t sum_products(cudaStream_t st, const cplx* x, const cplx* y, long long n, cplx* result, double* partials,
                         unsigned* counter);
cudaError_t any_nonfinite(cudaStream_t st, const cplx* x, long long n, int* flag);

// ------------------------------------------------------------- lanczos.cu
constexpr int KMAX = 16;
struct LanczosDev {
  double* scal;       // [ALPHA 0..KMAX) [BETA KMAX..2KMAX) [N0 2KMAX] [BRK 2KMAX+1]
  cplx* coef;         // [2][KMAX+1] multi-dot results
  cplx* y;            // [KMAX] exp(tau T) e1 * n0
  double* partials;   // reduction scratch [nblk_max * 2 * (KMAX+1)]
  unsigned* counter;  // last-block counter (self-resetting)
  int* brk_count;     // number of Lanczos runs that hit breakdown
};
enum { LZ_N0 = 2 * KMAX, LZ_BRK = 2 * KMAX + 1, LZ_SKIP = 2 * KMAX + 2, LZ_KEFF = 2 * KMAX + 3, LZ_E0 = 2 * KMAX + 4 };
int lanczos_nblk(long long n);
cudaError_t lz_start(cudaStream_t st, const LanczosDev& d, const cplx* x, cplx* v0, long long n);
// one cooperative launch for a whole Lanczos iteration after the matvec (see lanczos.cu)
// tol > 0 (paper mode, "convergence tolerance 1e-6"): after
// beta_k, block 0 estimates the error n0 beta_k |(exp(tau T_{k+1}) e1)_k| and,
// below tol, sets scal[LZ_SKIP] (every later kernel of this Lanczos returns at
// once) and scal[LZ_KEFF] = k + 1 (the Krylov dimension used by the final exp
// and combination)
cudaError_t lz_iter(cudaStream_t st, const LanczosDev& d, const cplx* V, long long ldv, int nv, cplx* w, cplx* vnext,
                    long long n, int k, int last, double tol = 0.0, double tau_re = 0.0, double tau_im = 0.0);
cudaError_t lz_tridiag_exp(cudaStream_t st, const LanczosDev& d, int K, double tau_re, double tau_im);
// ground state of the K x K Lanczos tridiagonal (two-site DMRG):
// restricted to the Krylov dimension before a breakdown, the lowest eigenpair
// (mu_0, y) by cyclic Jacobi; y normalised with y_0 >= 0 into d.y (zeros beyond),
// mu_0 into scal[LZ_E0]
cudaError_t lz_tridiag_ground(cudaStream_t st, const LanczosDev& d, int K);
cudaError_t lz_combine(cudaStream_t st, const LanczosDev& d, const cplx* V, long long ldv, int K, cplx* out,
                       long long n);

// ----------------------------------------------------------------- svd.cu
struct SvdDev {
  cplx* Y;            // (mr + nc) x nc, column-major, ld = ldy
  long long ldy;
  double* sigma;      // [nc]
  int* order;         // [nc]
  double* offmax;     // [1]
  int* ires;          // [4] : chi, chi_eps, nonfinite, r
  double* dres;       // [4] : w (discarded weight), sigma_1
  double* h_buf;      // pinned host mirror [8] (offmax, dres..)
  int* h_ibuf;        // pinned host mirror [4]
  cudaEvent_t ev_jac[2];  // optional: recorded around the Jacobi kernel (timing)
  cplx* qrbuf;            // QR preconditioning workspace (svd_qr_work_elems), nullptr = off
  size_t qrbuf_elems;
  unsigned* flags;        // Jacobi per-block round counters (2 per column block), nullptr = grid barriers
  size_t flags_elems;
  int throughput;         // 1: several SVDs run concurrently (segment lanes): prefer fewer CTAs per SVD
  int* perm;              // [2 nc]: column presort permutation and its inverse (QR path), nullptr = off
  cplx* bjwork;           // block-Jacobi partial Gram matrices (svd_bjac_work_elems), nullptr = off
  size_t bjwork_elems;
};
size_t svd_qr_work_elems(int m, int n);
struct TruncParams {
  int chi_max;
  double eps, w_max, delta;
};
// Full SVD by blocked one-sided Jacobi, then truncation (SURVEY O-7) and the split
// Psi_L = U S, Lambda = S, V = 1/S, Psi_R = S W^dagger.  theta is m x n row-major.
// Returns chi via *chi_out (host), discarded weight via *w_out (host).
// *jac_flop_out (optional): algorithmic flops of the Jacobi stage as executed
// (block-Jacobi DMMA path; 0 for the SIMT paths, whose count the caller derives
// from the sweeps)
cudaError_t svd_truncate_split(cudaStream_t st, const SvdDev& d, const cplx* theta, int m, int n,
                               const TruncParams& tp, cplx* psiL, cplx* psiR, double* lam, double* vinv,
                               int* chi_out, double* w_out, int* r_out, int* chi_eps_out, int* sweeps_out,
                               float* jac_ms_out = nullptr, double* jac_flop_out = nullptr);
size_t svd_work_elems(int m, int n);
// ------------------------------------------------------------------ qr.cu
// Blocked Householder QR workspace (column-major A, m x n, m >= n).
struct QrWork {
  cplx* Vc;        // reflectors as rows, n x ldv (ldv >= m)
  long long ldv;
  cplx* T;         // per-panel kb x kb triangular factors
  cplx* tau;       // [n]
  cplx* W1;        // [max(n, nc) * kb]
  cplx* W2;
  int kb;          // panel width = qr_kb_for(m)
  cplx* gw;        // split-K workspace of the V^H C products (nullptr: no split)
  size_t gw_elems;
};
int qr_kb_for(int m);  // panel width 32 (one CTA for <= 256 rows, a cluster beyond), 0 = unsupported
cudaError_t qr_factor(cudaStream_t st, const QrWork& w, cplx* A, long long lda, int m, int n);
// C (column-major m x nc, ld ldc) <- Q C with Q from qr_factor (m x n reflectors)
cudaError_t qr_apply_q(cudaStream_t st, const QrWork& w, int m, int n, cplx* C, long long ldc, int nc);
// X[0:rows_total, 0:n] = [R^H ; 0] from the upper triangle of the factored A
cudaError_t qr_r_conjtrans(cudaStream_t st, const cplx* A, long long lda, int n, cplx* X, long long ldx,
                           int rows_total);

// cluster-resident QR (n <= 16 columns per CTA band fitting shared memory;
// cudaErrorNotSupported otherwise): A overwritten by R and the reflector
// tails, tau[n]; optionally [R^H ; 0] (rh_rows x n, ld ldrh) written to RH.
cudaError_t qr_factor_cluster(cudaStream_t st, cplx* A, long long lda, int m, int n, cplx* tau, cplx* RH,
                              long long ldrh, int rh_rows);
// the same over a cooperative grid (bands up to one CTA per SM), counter in global memory
cudaError_t qr_factor_grid(cudaStream_t st, cplx* A, long long lda, int m, int n, cplx* tau, cplx* RH, long long ldrh,
                           int rh_rows, unsigned* gcnt);
// C (m x nc) <- H_0 ... H_{n-1} C with qr_factor_cluster's reflectors
cudaError_t qr_apply_refl(cudaStream_t st, const cplx* A, long long lda, const cplx* tau, int m, int n, cplx* C,
                          long long ldc, int nc);
// two independent applications in one launch
cudaError_t qr_apply_refl2(cudaStream_t st, const cplx* A0, long long lda0, const cplx* tau0, int m0, int n0, cplx* C0,
                           long long ldc0, int nc0, const cplx* A1, long long lda1, const cplx* tau1, int m1, int n1,
                           cplx* C1, long long ldc1, int nc1);

// svd_bjac.cu: block one-sided Jacobi on the DMMA pipe (blocks of 16 columns,
// pairs spread over S CTAs by rows, one cooperative launch).  X rows [0, xr),
// V rows [vofs, vofs + nc) of d.Y.  *flop_dev += executed DMMA flops.
size_t svd_bjac_work_elems(int sms);
cudaError_t svd_bjac_run(cudaStream_t st, const SvdDev& d, int xr, int vofs, int nc, long long ldy, double tol,
                         int* sweeps_dev, double* flop_dev);

// Opt a kernel into `bytes` of dynamic shared memory on the CURRENT device,
// once per (device, kernel), thread-safe (lanes and handles on several devices).
cudaError_t set_smem_attr(const void* fn, int bytes);
// Allow non-portable cluster sizes (up to 16 CTAs) for a kernel, once per device.
cudaError_t set_cluster_nonportable(const void* fn);

// svd_rjac.cu: register-resident Jacobi stage on d.Y = [X ; V]; returns
// cudaErrorNotSupported for shapes it does not cover (svd.cu falls back).
cudaError_t svd_rjac_run(cudaStream_t st, const SvdDev& d, int mr, int vofs, int nc, long long ldy, double tol,
                         int* sweeps_dev);
