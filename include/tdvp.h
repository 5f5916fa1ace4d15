/*
 * libtdvp — B200-native hot path of the parallel two-site TDVP (p2TDVP) for
 * matrix product states, Secular et al., arXiv:1912.06127.
 *
 * C-ABI boundary.  Plain pointers and sizes only.
 *
 * Conventions (SURVEY.md §8 "Conventions"):
 *   - complex numbers are interleaved (re, im) doubles (= numpy complex128);
 *   - all tensors are row-major;
 *   - site tensor Psi_j: (chi_j, d, chi_{j+1}) where chi[] has L+1 entries,
 *     chi[0] = chi[L] = 1 (chi[b+1] is the bond between sites b and b+1);
 *   - MPO tensor W_j: (D[j], d_out, d_in, D[j+1]) with W[w,s,t,w'] = <s|O|t>,
 *     D[] has L+1 entries with D[0] = D[L] = 1;
 *   - Lambda_b (bond b between sites b, b+1, b = 0..L-2): chi[b+1] float64,
 *     descending, strictly positive; V_b = 1/Lambda_b.
 *
 * Ownership: every input is copied; the caller keeps its buffers.  Outputs
 * go to caller-allocated buffers.  A handle owns all device memory it
 * allocates and is not thread-safe; distinct handles are independent.
 *
 * Errors: functions return 0 on success or a negative code, with a message
 * in tdvp_last_error(handle).  No C++ exception crosses the ABI.
 */
#ifndef TDVP_H
#define TDVP_H

#ifdef __cplusplus
extern "C" {
#endif

#define TDVP_OK 0
#define TDVP_EARG -1      /* bad argument: L<2, d<2, chi_max<1, dims mismatch, ends != 1 */
#define TDVP_ENONFINITE -2 /* non-finite input or Lambda <= 0 */
#define TDVP_EPARTITION -3 /* n_segments not 1 or even with 2 <= p <= L/2, segment < 2 sites,
                              or p != world size in multi-process mode */
#define TDVP_ECUDA -4     /* CUDA / NCCL failure (incl. no device) */
#define TDVP_ENUMERIC -5  /* NaN after exp or SVD, or all singular values zero */
#define TDVP_ESTATE -6    /* call order: MPO/MPS not set */

typedef struct tdvp_ctx* tdvp_t;

/* Truncation and Krylov knobs; defaults mirror PAPER.md:100 (S-IV). */
typedef struct {
  double eps;             /* relative SV cutoff epsilon, drop sigma < eps*sigma_1; default 1e-12 */
  double w_max;           /* max discarded weight per SVD; 0 = off (default) */
  int krylov_k;           /* Krylov vectors K, 1..15 ("maximum of 8"); default 8 */
  double krylov_tol;      /* 0 (default): always krylov_k vectors (parity mode, SURVEY AMB-5);
                             > 0 (paper mode, "tolerance 1e-6"): stop after iteration k
                             once n0 beta_k |(exp(tau T_{k+1}) e1)_k| < krylov_tol, decided on
                             the device (the oracle's rule); a timing variant */
  double multiplet_delta; /* AMB-9 multiplet guard at the chi_max cut; default 1e-6 */
  int timing;             /* 1: record CUDA events around every H_eff matvec and SVD (stats) */
  /* Multi-GPU in ONE process (SURVEY §8(b) "one process drives devices 0..p-1";
   * PAPER.md:470 one segment per processor): n_devices > 1 spreads the p segments
   * of tdvp_step(h, dt, p) over device_ids[0..n_devices-1] (segment q on
   * device_ids[q * n_devices / p]); each segment runs on its own host thread and
   * stream, boundary messages travel as cudaMemcpyPeerAsync
   * (NVLink P2P; peer access is enabled where supported); measurements and
   * tdvp_get_mps gather onto device_ids[0].  device_ids[0] must be the device the
   * handle was created on; ids may repeat (several segments per device).  The
   * array is copied.  n_devices <= 1: all segments on the handle's device.
   * tdvp_get_params returns the handle's copy. */
  int n_devices;
  const int* device_ids;
  /* Dynamic load balancing ("dynamic load balancer",
   * :237 load imbalance limits the scaling): 0 = off (default); in (0, 1):
   * before every tdvp_step with n_segments = p > 1 the chi-weighted min-max
   * partition (tdvp_partition_balanced of the current bond dimensions) replaces
   * the current one when its largest segment cost is below (1 - rebalance) x
   * the current partition's.  The state is kept; the environments are rebuilt
   * (the sequential section).  Single-process handles only. */
  double rebalance;
  /* U(1) block-sparse splits ("symmetric
   * block-sparse tensors"): 0 = off (default); 1 = the MPO conserves S^z_tot and
   * the MPS has definite S^z_tot (d = 2).  Bond charges (2 S^z of the left part)
   * are inferred from the MPS's nonzero pattern at the next layout (TDVP_EARG if
   * it is not charge-definite) and tracked through every split and boundary
   * message; every SVD (tdvp_step, tdvp_dmrg, tdvp_reorthonormalize) then runs
   * sector by sector with the truncation rule applied to the union of all
   * sectors' singular values (identical kept spectrum to the dense split), and
   * every tensor keeps exact zeros outside its charge blocks.  Single-process. */
  int u1;
} tdvp_params;

typedef struct {
  double w_step;          /* discarded weight summed over all SVDs of the last step (eq:discweight) */
  double w_total;         /* cumulative over all steps */
  int trunc_active;       /* chi_max / w_max / multiplet guard cut something in the last step */
  int n_pair, n_back;     /* two-site and one-site updates in the last step */
  int krylov_breakdowns;  /* cumulative Lanczos breakdowns (invariant subspace found) */
  int svd_sweeps_max;     /* max Jacobi sweeps of any SVD in the last step */
  double step_ms;         /* device time of the last step (CUDA events) */
  double heff2_ms;        /* summed device time of all H_eff^(2) matvecs in the last step (timing=1) */
  double heff2_flop;      /* algorithmic real flops of those matvecs */
  int heff2_calls;
  double heff1_ms, heff1_flop;
  double svd_ms;          /* summed SVD time (timing=1) */
  long long gemm_launches; /* DMMA GEMM kernel launches in the last step */
  long long kernel_launches; /* all kernel launches of this library in the last step */
  double svd_jac_ms;      /* summed device time of the Jacobi kernel of every SVD (timing=1) */
  double svd_jac_flop;    /* its algorithmic real flops: sweeps * nc(nc-1)/2 * (16 mr + 24 (mr + nc)) */
  int svd_sweeps_total;   /* Jacobi sweeps summed over the SVDs of the last step */
  double lanczos2_ms;     /* whole two-site Krylov exponentials incl. their H_eff^(2) matvecs (timing=1) */
  double lanczos1_ms;     /* whole one-site backward exponentials (timing=1) */
  double env_ms;          /* environment updates after the splits (timing=1) */
  /* H_eff^(2) matvec time and algorithmic flops binned by max(chi_L, chi_R) of the
   * pair: [0] <= 128, [1] <= 256, [2] <= 512, [3] > 512 (timing=1) */
  double heff2_ms_bin[4];
  double heff2_flop_bin[4];
  /* algorithmic HBM bytes of the Lanczos vector passes of the last step (timing=1;
   * their time is lanczos2_ms + lanczos1_ms - heff2_ms - heff1_ms) */
  double lz_vec_bytes;
  int rebalances;         /* cumulative dynamic re-partitionings (tdvp_params.rebalance) */
  /* the block-Jacobi (DMMA) SVD kernel alone (more than 1024 columns): device time
   * (timing=1), the flops it executed (Gram + rotation products, 8 per complex
   * MAC, counted on the device), launches */
  double svd_bj_ms, svd_bj_flop;
  int svd_bj_calls;
  /* the Lanczos vector passes (everything of the Krylov exponentials but the
   * matvecs) binned like heff2_*_bin by max(chi_L, chi_R): device time and
   * algorithmic bytes (timing=1) */
  double lz_ms_bin[4];
  double lz_bytes_bin[4];
  /* the flops the H_eff^(2) / H_eff^(1) matvecs executed (timing=1): the
   * algorithmic counts heff2_flop / heff1_flop (every MPO
   * channel) minus the environments' identity channels, which are copied
   * instead of contracted (MpoSite::lid / rid) */
  double heff2_flop_exec, heff1_flop_exec;
} tdvp_stats;

/* Create a handle for an L-site chain of local dimension d, MPO bond dimension
 * up to D_mpo and bond dimension cap chi_max, on the current CUDA device.
 * Allocates per-site buffers at chi_j^max = min(d^j, d^(L-j), chi_max). */
int tdvp_create(int L, int d, int D_mpo, int chi_max, tdvp_t* out);

int tdvp_set_params(tdvp_t h, const tdvp_params* p);
int tdvp_get_params(tdvp_t h, tdvp_params* p);

/* Copy the MPO.  D: L+1 bond dims (ends 1, each <= D_mpo); W[j] points to
 * D[j]*d*d*D[j+1] complex values (interleaved). */
int tdvp_set_mpo(tdvp_t h, const int* D, const double* const* W);

/* Copy an inverse-canonical MPS (must be exactly
 * inverse-canonical).  chi: L+1 bond dims (ends 1,
 * chi[b] <= chi_j^max); Psi[j]: chi[j]*d*chi[j+1] complex; Lambda[b]:
 * chi[b+1] doubles > 0 for b = 0..L-2.  Environments are rebuilt at the next
 * tdvp_step (sequential initialisation). */
int tdvp_set_mps(tdvp_t h, const int* chi, const double* const* Psi, const double* const* Lambda);

/* One full timestep dt (two half-sweeps) with n_segments
 * partitions (SURVEY App. A protocol).  n_segments = 1 is
 * serial 2TDVP.  In single-process mode all segments run on this handle's
 * device (BSP-equivalent order); after tdvp_comm_init each rank runs
 * segment q = rank and n_segments must equal the world size.  Changing
 * n_segments rebuilds the environments (sequential section). */
int tdvp_step(tdvp_t h, double dt, int n_segments);

/* One one-site TDVP step dt with n_segments partitions: the integrator of
 * the hybrid scheme PAPER.md:697 describes ("starts with 2TDVP and switches
 * to 1TDVP when chi_max is saturated"), and its segment-parallel form p1TDVP
 * ("could be developed using the same approach"; the paper gives no
 * algorithm: readings R-1TDVP / R-P1TDVP in DESIGN.md).  n_segments = 1:
 * serial 1TDVP -- left-to-right then right-to-left sweep with tau = dt/2:
 * forward one-site steps exp(-i tau H_eff^(1)) (the last site once by dt, the
 * turnaround merge of PAPER.md:430), each bond split by the truncated SVD of
 * tdvp_step (O-7; interior bond dimensions never grow) and
 * evolved backwards by exp(+i tau H_eff^(0)), H_eff^(0) C[a,b] =
 * sum L[a,w,a'] R[b,w,b'] C[a',b'].  n_segments = p > 1: the p2TDVP
 * half-step programs of tdvp_step with their boundary phases unchanged (the
 * two-site Lambda^-1-merged boundary pair updates, which may
 * grow the boundary bonds up to chi_max) and one-site segment interiors.
 * The state stays in the inverse-canonical product form of tdvp_set_mps.
 * Partition, executors and devices as for tdvp_step; dense mode only
 * (TDVP_EARG with u1 = 1).  Stats as for tdvp_step. */
int tdvp_step1(tdvp_t h, double dt, int n_segments);

/* One step of the hybrid scheme: tdvp_step1(h, dt,
 * n_segments) when the handle is single-process dense and every bond j is
 * saturated (chi_j = min(chi_max, d^(j+1), d^(L-j-1))); tdvp_step(h, dt,
 * n_segments) otherwise.  *used (may be NULL) = 1 or 2, the integrator run. */
int tdvp_step_hybrid(tdvp_t h, double dt, int n_segments, int* used);

/* Full-zipper measurements of Psi_0 V_0 Psi_1 ... Psi_{L-1} (any gauge,
 * normalised by <psi|psi>).  Not on the timed path. */
int tdvp_measure_sz(tdvp_t h, double* sz /* [L] */);
int tdvp_measure_energy(tdvp_t h, double* E);
int tdvp_measure_norm(tdvp_t h, double* norm2 /* <psi|psi> */);

/* <psi_a|psi_b> of two handles' current states (same L, d, device; local
 * mode).  Used for the infidelity I = 1 - |<a|b>| / sqrt(<a|a><b|b>) between
 * a serial and a segment-parallel run (PAPER.md, benchmark section: "the
 * infidelity between the states obtained serially and in parallel").  Reads
 * both states, modifies neither; synchronises both handles' streams.
 * Errors: TDVP_EARG (null / mismatched handles), TDVP_ESTATE (no MPO/MPS, or the
 * state is distributed across ranks). */
int tdvp_overlap(tdvp_t a, tdvp_t b, double* re, double* im);
/* I = 1 - |<a|b>| / sqrt(<a|a><b|b>) (PAPER.md benchmark section "the infidelity
 * between the states obtained serially and in parallel"), computed by the
 * library from tdvp_overlap and the two norms.  Errors as tdvp_overlap. */
int tdvp_infidelity(tdvp_t a, tdvp_t b, double* infidelity);

/* Reorthonormalisation: re-gauge the current MPS into
 * inverse-canonical form by an SVD sweep left->right and one right->left on
 * the device (singular values below 1e-14 sigma_1 are dropped, the state is
 * normalised to 1), then rebuild the environments at the next tdvp_step.  The
 * physical state is unchanged up to that floor and the normalisation; the
 * Lambda_j afterwards are its exact Schmidt values.  Serial; local mode only.
 * Errors: TDVP_ESTATE (no MPO/MPS, distributed), TDVP_ENUMERIC (zero norm). */
int tdvp_reorthonormalize(tdvp_t h);

/* Two-site DMRG ground-state sweeps on the handle's MPO, starting from its
 * current MPS (every quench
 * starts from a DMRG ground state).  A sweep = pairs j = 0..L-2 left->right,
 * then j = L-3..0 right->left; each pair update merges Theta,
 * replaces it by the lowest eigenvector of H_eff^(2) from
 * `restarts` restarted Lanczos runs of tdvp_params.krylov_k vectors, and splits
 * it with the same truncated SVD as tdvp_step.
 * energies[s] (optional, n_sweeps entries) = the Ritz value of the last update
 * of sweep s.  The final state is re-gauged into exactly inverse-canonical
 * form (as tdvp_reorthonormalize; "important to ensure the
 * initial state is orthonormal") and stays in the handle: set another MPO with
 * tdvp_set_mpo and call tdvp_step for a quench.  Serial, one device.
 * Errors: TDVP_EARG, TDVP_ESTATE (no MPO/MPS, multi-rank), TDVP_ENUMERIC. */
int tdvp_dmrg(tdvp_t h, int n_sweeps, int restarts, double* energies);

int tdvp_get_stats(tdvp_t h, tdvp_stats* s);
/* Current bond dimensions (owner view): chi[L+1]. */
int tdvp_get_chi(tdvp_t h, int* chi);
/* Copy the current MPS (owner copies) into caller buffers sized by
 * tdvp_get_chi (or at chi_j^max). */
int tdvp_get_mps(tdvp_t h, double** Psi, double** Lambda);

const char* tdvp_last_error(tdvp_t h);
void tdvp_destroy(tdvp_t h);

/* ---- multi-process (one rank per GPU, NCCL point-to-point over NVLink) ---- */
/* Writes a 128-byte ncclUniqueId (call on rank 0, broadcast the bytes). */
int tdvp_nccl_unique_id(unsigned char* id128);
/* Join the rank group; afterwards tdvp_step(h, dt, world) runs segment `rank`. */
int tdvp_comm_init(tdvp_t h, int rank, int world, const unsigned char* id128);

/* ---- host-only schedule (no GPU needed; used by the CPU protocol tests) ----
 * Writes the op list of segment q in half h (1 or 2) of a p-segment step
 * into ops[4*i .. 4*i+3] = {kind, j, tau_full, build} and returns the number of
 * ops (or a negative error).  kind: 1 PAIR(j,j+1), 2 BACK(j), 3 SEND_R
 * (Psi_{e+1}, Lambda_e, beta_{e+1} -> q+1), 4 RECV_L, 5 SEND_L (Psi_s,
 * gamma_s -> q-1), 6 RECV_R.  build: bit0 beta_{j+1}, bit1 gamma_j. */
int tdvp_plan(int L, int p, int h, int q, int* ops, int max_ops);
/* The same for the p1TDVP programs of tdvp_step1 (reading R-P1TDVP): kinds
 * additionally 7 = SITE_R, 8 = SITE_L, 9 = FWD (schedule.h). */
int tdvp_plan1(int L, int p, int h, int q, int* ops, int max_ops);
/* Segment bounds [s, e] of segment q (SURVEY O-3). */
int tdvp_partition(int L, int p, int* s, int* e);

/* Load balancing ("load imbalance is the
 * limiter").  tdvp_set_partition: use the explicit contiguous partition with
 * segment q starting at site s[q] (s[0] = 0, p even, 2 <= p <= L/2, every
 * segment >= 2 sites) whenever tdvp_step is called with
 * n_segments = p; p = 0 restores the uniform rule.  The state is kept; the
 * next step re-lays it out and rebuilds the environments.  In multi-process
 * mode every rank must set the same partition.  Errors: TDVP_EARG,
 * TDVP_EPARTITION.
 * tdvp_partition_balanced (host only): the contiguous partition into p
 * segments (each >= 2 sites) minimising the largest segment cost, site cost
 * chi_j chi_{j+1} (chi_j + chi_{j+1}) from the bond dimensions chi[L+1]
 * (e.g. tdvp_get_chi): exact dynamic programme, deterministic (smallest split
 * index on ties).  Writes s[p], e[p]. */
int tdvp_set_partition(tdvp_t h, int p, const int* s);
int tdvp_partition_balanced(int L, int p, const int* chi, int* s, int* e);
/* The partition the handle's segments currently use: *p segments, segment q
 * = sites [s[q], e[q]] (caller arrays of >= *p entries; NULL s/e: count only). */
int tdvp_get_partition(tdvp_t h, int* p, int* s, int* e);

/* ---- kernel-level entry points (host buffers; copies inside) -------------
 * For parity tests of the individual contractions against the oracle.
 * H_eff^(2) theta: Lenv (cl, Dl, cl), W1 (Dl, d, d, Dm),
 * W2 (Dm, d, d, Dr), Renv (cr, Dr, cr), theta/out (cl, d, d, cr). */
int tdvp_apply_heff2(int cl, int cr, int d, int Dl, int Dm, int Dr, const double* Lenv, const double* W1,
                     const double* W2, const double* Renv, const double* theta, double* out);
/* H_eff^(1) psi: psi/out (cl, d, cr). */
int tdvp_apply_heff1(int cl, int cr, int d, int Dl, int Dr, const double* Lenv, const double* W, const double* Renv,
                     const double* psi, double* out);
/* beta' = env_left(beta, A, W): beta (cl,Dl,cl), A (cl,d,cr) -> (cr,Dr,cr).
 * gamma' = env_right(gamma, B, W): gamma (cr,Dr,cr), B (cl,d,cr) -> (cl,Dl,cl). */
int tdvp_env_left(int cl, int cr, int d, int Dl, int Dr, const double* beta, const double* A, const double* W,
                  double* out);
int tdvp_env_right(int cl, int cr, int d, int Dl, int Dr, const double* gamma, const double* B, const double* W,
                   double* out);
/* exp(tau H) v for a dense Hermitian n x n H by the device Lanczos (K vectors). */
int tdvp_expm_lanczos_dense(int n, const double* H, const double* v, double tau_re, double tau_im, int K,
                            double* out);
/* Truncated SVD split of an m x n matrix:
 * writes chi, w, Psi_L (m x chi), Lambda (chi), Psi_R (chi x n). */
int tdvp_svd_split(int m, int n, const double* M, int chi_max, double eps, double w_max, double delta, int* chi,
                   double* w, double* psiL, double* lam, double* psiR);
/* C = op(A) op(B) complex GEMM on the DMMA path (op 0 N, 1 T, 2 C, 3 conj). */
int tdvp_zgemm(int opA, int opB, int M, int N, int K, const double* A, const double* B, double* C);

/* ---- microbenchmarks (device-resident operands, CUDA-event / wall timed) ---- */
/* Mean device time (ms) of one H_eff^(2) matvec at chi_L = chi_R = chi with the
 * given MPO site tensors, and its algorithmic real flop count. */
int tdvp_bench_heff2(int chi, int Dl, int Dm, int Dr, const double* W1, const double* W2, int reps, double* ms,
                     double* flop);
/* Mean wall time (ms, includes the host read of chi) of one truncated SVD split
 * of the m x n matrix M; *sweeps = Jacobi sweeps of the last run. */
int tdvp_bench_svd(int m, int n, const double* M, int reps, double* ms, int* sweeps);

#ifdef __cplusplus
}
#endif
#endif /* TDVP_H */
