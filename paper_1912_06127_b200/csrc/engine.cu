// libtdvp engine: device state, local updates, sweep executor, C-ABI.
//
// Hot path per two-site update:
//   a1 merge   Theta = Psi_j diag(V_j) Psi_{j+1}            (row scale + DMMA GEMM)
//   a2 H_eff   L.theta (DMMA GEMM) -> W_j, W_{j+1} (sparse channel mix) -> .R^T (DMMA GEMM)
//   a3 Lanczos device-resident K-vector Krylov exp (lanczos.cu)
//   a4 SVD     blocked one-sided Jacobi + truncation (svd.cu)
//   a5 env     beta_{j+1} / gamma_j (GEMM, channel mix, GEMM)
// a6 one-site backward update, a7 schedule (schedule.h), a8 boundary exchange
// (device copies in single-process mode, NCCL send/recv across ranks).
#include <dlfcn.h>
#include <nccl.h>

#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <exception>
#include <mutex>
#include <thread>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <limits>
#include <algorithm>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tdvp.h"
#include "common.cuh"
#include "kernels.h"
#include "schedule.h"

// Page-locked host storage for the full-state host copy: tdvp_set_mps /
// upload_state / download_state move up to d chi_max^2 L complex values per
// call, which DMA straight from pinned pages (no staging through the driver's
// bounce buffers); the pages are kept while the shapes stay (assign / resize
// of an equal size does not reallocate).
template <class T>
struct PinnedAlloc {
  using value_type = T;
  PinnedAlloc() = default;
  template <class U>
  PinnedAlloc(const PinnedAlloc<U>&) {}
  T* allocate(size_t n) {
    void* p = nullptr;
    if (n == 0) n = 1;
    if (cudaHostAlloc(&p, n * sizeof(T), cudaHostAllocPortable) != cudaSuccess || !p) {
      cudaGetLastError();
      throw std::bad_alloc();
    }
    return static_cast<T*>(p);
  }
  void deallocate(T* p, size_t) { cudaFreeHost(p); }
  template <class U>
  bool operator==(const PinnedAlloc<U>&) const { return true; }
  template <class U>
  bool operator!=(const PinnedAlloc<U>&) const { return false; }
};
using hvec = std::vector<double, PinnedAlloc<double>>;

// f(k, i0, i1) over the concatenated element ranges [0, sizes[k]), split
// evenly over up to 8 host threads (the full-state validation and copy of
// tdvp_set_mps: d chi_max^2 L doubles, memory-bandwidth bound on one core)
template <class F>
void host_parallel(const std::vector<size_t>& sizes, F f) {
  size_t total = 0;
  for (size_t n : sizes) total += n;
  const unsigned hc = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  const int T = (int)std::max<size_t>(1, std::min<size_t>(hc, total >> 20));
  auto work = [&](int t) {
    const size_t lo = total * t / T, hi = total * (t + 1) / T;
    size_t base = 0;
    for (size_t k = 0; k < sizes.size() && base < hi; base += sizes[k], ++k) {
      const size_t a = std::max(lo, base), b = std::min(hi, base + sizes[k]);
      if (a < b) f(k, a - base, b - base);
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < T; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
}

namespace {

// ------------------------------------------------------------------ errors
struct TdvpError : std::runtime_error {
  int code;
  TdvpError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
#define CK(expr)                                                                                          \
  do {                                                                                                    \
    cudaError_t _e = (expr);                                                                              \
    if (_e != cudaSuccess)                                                                                \
      throw TdvpError(TDVP_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e) + " @" +             \
                                      std::to_string(__LINE__));                                          \
  } while (0)
#define NK(expr)                                                                                          \
  do {                                                                                                    \
    if (!nccl().ok) throw TdvpError(TDVP_ECUDA, "libnccl.so.2 could not be loaded");                      \
    ncclResult_t _r = (expr);                                                                             \
    if (_r != ncclSuccess) throw TdvpError(TDVP_ECUDA, std::string(#expr) + ": " + nccl().GetErrorString(_r)); \
  } while (0)

// NCCL is resolved at run time (dlopen) so that the library never pins a
// libnccl.so.2 different from the one torch.distributed already loaded.
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi& nccl() {
  // resolved once, thread-safe (function-local static initialisation)
  static NcclApi api = [] {
    NcclApi a;
    void* hd = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!hd) hd = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!hd) return a;
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(hd, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(hd, "ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(hd, "ncclCommDestroy");
    a.Send = (decltype(a.Send))dlsym(hd, "ncclSend");
    a.Recv = (decltype(a.Recv))dlsym(hd, "ncclRecv");
    a.GroupStart = (decltype(a.GroupStart))dlsym(hd, "ncclGroupStart");
    a.GroupEnd = (decltype(a.GroupEnd))dlsym(hd, "ncclGroupEnd");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(hd, "ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.Send && a.Recv && a.GroupStart && a.GroupEnd &&
           a.GetErrorString;
    return a;
  }();
  return api;
}

// ------------------------------------------------------------------ buffers
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  void alloc(size_t b) {
    release();
    if (b == 0) b = 16;
    CK(cudaMalloc(&p, b));
    bytes = b;
  }
  cplx* c() const { return reinterpret_cast<cplx*>(p); }
  double* d() const { return reinterpret_cast<double*>(p); }
  int* i() const { return reinterpret_cast<int*>(p); }
};
using BufPtr = std::unique_ptr<DevBuf>;

// RAII: make `dev` current for the scope (multi-device handles allocate and
// launch per segment device), restore the previous device afterwards
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev != prev) CK(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
// device-to-device copy on `st` (a stream of the current device); across
// devices by cudaMemcpyPeerAsync (NVLink P2P when peer access is enabled)
inline void d2d(void* dst, int ddev, const void* src, int sdev, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  if (ddev == sdev) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st));
  else CK(cudaMemcpyPeerAsync(dst, ddev, src, sdev, bytes, st));
}
BufPtr make_buf(size_t bytes) {
  BufPtr b(new DevBuf());
  b->alloc(bytes);
  return b;
}

// MPO site: CSR tables for the sparse channel stages (values copied from W)
struct MpoSite {
  int Dl = 1, Dr = 1;
  ChanMix cmL;  // (w,t) -> (s,w'): H1, H2 stages, env_left
  ChanMix cmR;  // (t,w') -> (w,s): env_right
  // pair (j, j+1): (w,t1,t2) -> (s1,s2,w''), coef sum_w' W_j[w,s1,t1,w'] W_{j+1}[w',s2,t2,w''];
  // H_eff^(2)'s two channel stages in one pass when its inputs fit the gather kernel
  ChanMix cm12;
  bool has12 = false;
  // identity channels of the environments at this site (build_mpo_tables):
  // lid: beta_j[:, Dl-1, :] = A^dag A = I (the "not started" channel: beta_0 = 1
  // and every W_k, k < j, feeds column Dr-1 only from row Dl-1 with the
  // identity); rid: gamma_j[:, 0, :] = B B^dag = I (the "done" channel, rows 0
  // of every W_k, k > j).  Exact for the canonical A = U, B = W^dag of every
  // split; H_eff then copies instead of contracting those channels
  bool lid = false, rid = false;
  std::vector<BufPtr> store;
};

// Segment: everything one process owns
struct Segment {
  int q = 0, s = 0, e = 0;
  int dev = 0;          // device holding this segment's tensors (multi-device handles)
  std::vector<int> cb;  // bond dims, L+1 (own view)
  std::vector<BufPtr> psi, beta, gamma;  // per site (null if not held)
  std::vector<BufPtr> lam, vinv;         // per bond
  // U(1) mode (tdvp_params.u1): charges 2 S^z of the left part for every index
  // of bond position k (bond left of site k), k = 0..L; kept for the bonds
  // this segment's updates touch (host side: chi is host-known anyway)
  std::vector<std::vector<int>> qb;
};

// One boundary message between segment lanes (SEND_R: Psi'_{e+1}, Lambda'_e,
// V_e, beta_{e+1}; SEND_L: Psi_s, gamma_s): the sender copies
// into the staging buffers on its stream and records `posted`; the receiver
// waits for it on its stream, copies out and records `consumed`, which the
// next send on this channel waits for.  Depth 1: per half-step every channel
// carries at most one message, and the receiver consumes it within the same
// half (segment_program), so a blocked sender never closes a cycle.
struct LaneMsg {
  std::mutex m;
  std::condition_variable cv;
  int ready = 0;
  int meta[2] = {0, 0};
  int sdev = 0, rdev = 0;  // sender / receiver device (staging lives on rdev)
  cudaEvent_t posted = nullptr, consumed = nullptr;
  bool consumed_rec = false;
  BufPtr psi, lam, vinv, env;
  std::vector<int> q;  // U(1) mode: charges of the bond the message updates
  ~LaneMsg() {
    if (posted) cudaEventDestroy(posted);
    if (consumed) cudaEventDestroy(consumed);
  }
};

}  // namespace

struct tdvp_ctx {
  tdvp_ctx() : mpo(mpo_own) {}
  // a segment lane: own stream and workspace, the parent's MPO
  explicit tdvp_ctx(tdvp_ctx* par, bool own_mpo = false) : mpo(own_mpo ? mpo_own : par->mpo_own), parent(par) {}
  tdvp_ctx(const tdvp_ctx&) = delete;
  tdvp_ctx& operator=(const tdvp_ctx&) = delete;
  int L = 0, d = 0, Dmpo = 0, chi_max = 0;
  tdvp_params prm{};
  const double* cur_skip = nullptr;  // inside a paper-mode Lanczos: its device "converged" flag
  // U(1) mode: block masks of the first and last GEMM of the H_eff matvec in
  // progress (set around a Lanczos exponential, nullptr otherwise)
  const GemmMask* cur_mask[2] = {nullptr, nullptr};
  struct MaskSet {
    std::vector<unsigned char> ha, hb;
    BufPtr da, db;
    GemmMask g;
  } masks[2];
  std::vector<std::vector<int>> h_r;  // MPO channel charges per bond position (U(1)); empty = not conserving
  int dev = 0;
  // devices of a multi-device handle (tdvp_params.n_devices / device_ids):
  // segment q of a p-segment step lives on devs[q * n / p]; devs[0] = dev
  std::vector<int> devs;
  bool multi_dev = false;
  std::vector<int> h_D;                       // MPO bond dims (host copy, per-device MPO tables)
  std::vector<std::vector<cplx>> h_W;         // MPO tensors (host copy)
  cudaStream_t st = nullptr;
  std::string err;
  std::vector<int> cbmax;  // L+1
  std::vector<MpoSite> mpo_own;
  std::vector<MpoSite>& mpo;  // lanes: the parent's sites
  MpoSite mpo_id, mpo_sz;  // D = 1 identity / S^z (measurement)
  bool have_mpo = false, have_mps = false, envs_valid = false;
  bool evolved = false;  // stepped since the last tdvp_set_mps (the host copy h_psi is stale in rank mode)
  int layout_p = 0;  // segments currently laid out (0: the host copy h_psi/h_lam is authoritative)
  // the step in progress runs the p1TDVP programs (tdvp_step1; reading
  // R-P1TDVP) instead of the p2TDVP ones; msites: chain-end sites evolved by dt
  // at the end of its half 1
  bool one_site = false;
  std::set<int> msites;
  int alloc_p = 0;   // segments whose device buffers are allocated (kept across tdvp_set_mps)
  std::vector<std::pair<int, int>> bounds;
  std::vector<std::pair<int, int>> custom;  // tdvp_set_partition: explicit bounds for n_segments = custom.size()
  std::vector<Segment> segs;
  // full-state host copy (multi-process initialisation)
  std::vector<hvec> h_psi;  // pinned
  std::vector<std::vector<double>> h_lam;
  std::vector<int> h_chi;
  std::vector<std::vector<int>> h_q;  // U(1) mode: bond charges of the host copy (positions 0..L)
  BufPtr u1_idx, u1_lam, u1_vinv;     // U(1) split: sector index lists, per-sector spectra
  // workspace
  long long n2max = 0, n1max = 0, scratch = 0, svdmax = 0, work_elems = 0;
  BufPtr theta, krylov, wvec, T1, T2, tmpA, tmpB, svdY, svdQ, svdF, gemm_work, partials;
  BufPtr lz_scal, lz_coef, lz_y, lz_counter, lz_brk;
  BufPtr lz_brk_own;  // a multi-device lane's breakdown counter (on its device)
  BufPtr svd_sigma, svd_order, svd_perm, svd_bj, svd_off, svd_ires, svd_dres, red_res, envA, envB;
  double* h_pin = nullptr;
  int* h_ipin = nullptr;
  LanczosDev lz{};
  SvdDev sv{};
  // stats
  tdvp_stats stats{};
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<std::pair<int, int>> ev_h2, ev_h1, ev_svd, ev_lz2, ev_lz1, ev_env;
  std::vector<int> ev_h2_bin;  // chi bin of every ev_h2 entry (tdvp_stats.heff2_*_bin)
  // one record per timed Krylov exponential: its whole span, its chi bin and
  // the range of its matvec events in ev_h2 (which = 2) or ev_h1 (which = 1)
  struct LzRec {
    int ea, eb, bin, which;
    size_t mv0, mv1;
  };
  std::vector<LzRec> ev_lzrec;
  int cur_bin = 0;             // chi bin of the pair update in progress
  cudaEvent_t ev_step0 = nullptr, ev_step1 = nullptr;
  // NCCL
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  BufPtr hdr;
  // Segment lanes (single process, p > 1): segment q runs on lane q -- its
  // own host thread, stream and workspace (lane 0 = this handle) -- so the p
  // segments' sweeps run concurrently on one GPU; boundary messages go
  // through staging buffers ordered by events (LaneMsg).  TDVP_LANES=0: the
  // round-robin executor on one stream.
  tdvp_ctx* parent = nullptr;
  bool lanes_on = true;
  // U(1) split: workers that run the sector SVDs concurrently (own stream and
  // SVD workspace each; allocated on the first U(1) split)
  struct U1Worker {
    cudaStream_t st = nullptr;
    BufPtr Y, Q, F, sigma, order, perm, bj, off, ires, dres;
    double* h_pin = nullptr;
    int* h_ipin = nullptr;
    SvdDev sv{};
    ~U1Worker() {
      if (st) cudaStreamSynchronize(st);
      if (h_pin) cudaFreeHost(h_pin);
      if (h_ipin) cudaFreeHost(h_ipin);
      if (st) cudaStreamDestroy(st);
    }
  };
  std::vector<std::unique_ptr<U1Worker>> u1w;
  std::vector<std::unique_ptr<tdvp_ctx>> lanes;  // lanes 1 .. p-1
  std::vector<std::unique_ptr<LaneMsg>> msg_r, msg_l;  // per segment: to q+1, to q-1
  ~tdvp_ctx();
};

std::atomic<long long> g_launch_count{0};
std::atomic<long long> g_gemm_count{0};

tdvp_ctx::~tdvp_ctx() {
  int prev = -1;
  cudaGetDevice(&prev);
  if (prev != dev) cudaSetDevice(dev);  // this context's stream, events and buffers live on `dev`
  if (st) cudaStreamSynchronize(st);
  lanes.clear();
  u1w.clear();
  msg_r.clear();
  msg_l.clear();
  segs.clear();
  mpo_own.clear();
  for (auto e : ev_pool) cudaEventDestroy(e);
  if (ev_step0) cudaEventDestroy(ev_step0);
  if (ev_step1) cudaEventDestroy(ev_step1);
  for (auto e : sv.ev_jac)
    if (e) cudaEventDestroy(e);
  if (h_pin) cudaFreeHost(h_pin);
  if (h_ipin) cudaFreeHost(h_ipin);
  if (comm && nccl().ok) nccl().CommDestroy(comm);
  if (st) cudaStreamDestroy(st);
  if (prev >= 0 && prev != dev) cudaSetDevice(prev);
}

namespace {

constexpr cplx ONE = {1.0, 0.0}, ZERO = {0.0, 0.0};

// ------------------------------------------------------------ small helpers
cudaEvent_t ev_get(tdvp_ctx* h) {
  if (h->ev_used == h->ev_pool.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    h->ev_pool.push_back(e);
  }
  return h->ev_pool[h->ev_used++];
}
int ev_record(tdvp_ctx* h) {
  const int idx = (int)h->ev_used;
  CK(cudaEventRecord(ev_get(h), h->st));
  return idx;
}

void gemm(tdvp_ctx* h, int opA, int opB, int M, int N, int K, const cplx* A, long long lda, const cplx* B,
          long long ldb, cplx* C, long long ldc, const GemmMask* mask = nullptr) {
  CK(zgemm(h->st, opA, opB, M, N, K, ONE, A, lda, B, ldb, ZERO, C, ldc, 1, 0, 0, 0, h->gemm_work->c(),
           (size_t)h->work_elems, h->cur_skip, mask));
  g_gemm_count++;
  g_launch_count++;
}
void cmix(tdvp_ctx* h, const ChanMix& cm, int n_outer, int n_inner, const cplx* in, long long so_in, long long si_in,
          Strides3 ich, cplx* out, long long so_out, long long si_out, Strides3 och) {
  CK(chanmix(h->st, cm, n_outer, n_inner, in, so_in, si_in, ich, out, so_out, si_out, och, h->cur_skip));
  g_launch_count++;
}

// build CSR tables of one MPO site tensor W (Dl, d, d, Dr) (host structure pass;
// the values are copied, not computed)
void upload_mix(MpoSite& ms, ChanMix& cm, const std::vector<int>& rowptr, const std::vector<int4>& oc,
                const std::vector<int4>& ic, const std::vector<cplx>& coef) {
  cm.n_oc = (int)oc.size();
  cm.nnz = (int)ic.size();
  BufPtr b1 = make_buf(rowptr.size() * sizeof(int));
  BufPtr b2 = make_buf(std::max<size_t>(1, oc.size()) * sizeof(int4));
  BufPtr b3 = make_buf(std::max<size_t>(1, ic.size()) * sizeof(int4));
  BufPtr b4 = make_buf(std::max<size_t>(1, coef.size()) * sizeof(cplx));
  CK(cudaMemcpy(b1->p, rowptr.data(), rowptr.size() * sizeof(int), cudaMemcpyHostToDevice));
  if (!oc.empty()) CK(cudaMemcpy(b2->p, oc.data(), oc.size() * sizeof(int4), cudaMemcpyHostToDevice));
  if (!ic.empty()) CK(cudaMemcpy(b3->p, ic.data(), ic.size() * sizeof(int4), cudaMemcpyHostToDevice));
  if (!coef.empty()) CK(cudaMemcpy(b4->p, coef.data(), coef.size() * sizeof(cplx), cudaMemcpyHostToDevice));
  cm.rowptr = b1->i();
  cm.oc_idx = reinterpret_cast<int4*>(b2->p);
  cm.ic_idx = reinterpret_cast<int4*>(b3->p);
  cm.coef = b4->c();
  // distinct input channels: the gather kernel loads each once per point
  std::vector<int4> icu;
  std::vector<int> slot(ic.size());
  for (size_t e = 0; e < ic.size(); ++e) {
    size_t k = 0;
    while (k < icu.size() && !(icu[k].x == ic[e].x && icu[k].y == ic[e].y && icu[k].z == ic[e].z)) ++k;
    if (k == icu.size()) icu.push_back(ic[e]);
    slot[e] = (int)k;
  }
  cm.n_ic = (int)icu.size();
  BufPtr b5 = make_buf(std::max<size_t>(1, icu.size()) * sizeof(int4));
  BufPtr b6 = make_buf(std::max<size_t>(1, slot.size()) * sizeof(int));
  if (!icu.empty()) CK(cudaMemcpy(b5->p, icu.data(), icu.size() * sizeof(int4), cudaMemcpyHostToDevice));
  if (!slot.empty()) CK(cudaMemcpy(b6->p, slot.data(), slot.size() * sizeof(int), cudaMemcpyHostToDevice));
  cm.icu_idx = reinterpret_cast<int4*>(b5->p);
  cm.slot = b6->i();
  ms.store.push_back(std::move(b1));
  ms.store.push_back(std::move(b2));
  ms.store.push_back(std::move(b3));
  ms.store.push_back(std::move(b4));
  ms.store.push_back(std::move(b5));
  ms.store.push_back(std::move(b6));
}

void build_site(MpoSite& ms, int Dl, int Dr, int d, const std::vector<cplx>& W) {
  ms.Dl = Dl;
  ms.Dr = Dr;
  ms.store.clear();
  auto at = [&](int w, int s, int t, int w2) { return W[(((size_t)w * d + s) * d + t) * Dr + w2]; };
  auto nz = [](cplx v) { return v.x != 0.0 || v.y != 0.0; };
  auto upload = [&](ChanMix& cm, const std::vector<int>& rowptr, const std::vector<int4>& oc,
                    const std::vector<int4>& ic, const std::vector<cplx>& coef) { upload_mix(ms, cm, rowptr, oc, ic, coef); };
  {  // cmL: out (s, w') <- in (w, t), coef W[w,s,t,w']
    std::vector<int> rp{0};
    std::vector<int4> oc, ic;
    std::vector<cplx> cf;
    for (int s = 0; s < d; ++s)
      for (int w2 = 0; w2 < Dr; ++w2) {
        oc.push_back(make_int4(s, w2, 0, 0));
        for (int w = 0; w < Dl; ++w)
          for (int t = 0; t < d; ++t)
            if (nz(at(w, s, t, w2))) {
              ic.push_back(make_int4(w, t, 0, 0));
              cf.push_back(at(w, s, t, w2));
            }
        rp.push_back((int)ic.size());
      }
    upload(ms.cmL, rp, oc, ic, cf);
  }
  {  // cmR: out (w, s) <- in (t, w'), coef W[w,s,t,w']
    std::vector<int> rp{0};
    std::vector<int4> oc, ic;
    std::vector<cplx> cf;
    for (int w = 0; w < Dl; ++w)
      for (int s = 0; s < d; ++s) {
        oc.push_back(make_int4(w, s, 0, 0));
        for (int t = 0; t < d; ++t)
          for (int w2 = 0; w2 < Dr; ++w2)
            if (nz(at(w, s, t, w2))) {
              ic.push_back(make_int4(t, w2, 0, 0));
              cf.push_back(at(w, s, t, w2));
            }
        rp.push_back((int)ic.size());
      }
    upload(ms.cmR, rp, oc, ic, cf);
  }
}

// H_eff^(2) pair table of sites (j, j+1) (host structure pass over the two
// MPO tensors; only used when the (w, t1, t2) inputs fit the gather kernel)
void build_pair(MpoSite& ms, int Dl, int Dm, int Dr, int d, const std::vector<cplx>& W1,
                const std::vector<cplx>& W2) {
  ms.has12 = false;
  if (Dl * d * d > 32) return;
  auto a1 = [&](int w, int s, int t, int w2) { return W1[(((size_t)w * d + s) * d + t) * Dm + w2]; };
  auto a2 = [&](int w, int s, int t, int w2) { return W2[(((size_t)w * d + s) * d + t) * Dr + w2]; };
  std::vector<int> rp{0};
  std::vector<int4> oc, ic;
  std::vector<cplx> cf;
  for (int s1 = 0; s1 < d; ++s1)
    for (int s2 = 0; s2 < d; ++s2)
      for (int w3 = 0; w3 < Dr; ++w3) {
        oc.push_back(make_int4(s1, s2, w3, 0));
        for (int w = 0; w < Dl; ++w)
          for (int t1 = 0; t1 < d; ++t1)
            for (int t2 = 0; t2 < d; ++t2) {
              cplx v = ZERO;
              for (int w2 = 0; w2 < Dm; ++w2) v = cadd(v, cmul(a1(w, s1, t1, w2), a2(w2, s2, t2, w3)));
              if (v.x != 0.0 || v.y != 0.0) {
                ic.push_back(make_int4(w, t1, t2, 0));
                cf.push_back(v);
              }
            }
        rp.push_back((int)ic.size());
      }
  upload_mix(ms, ms.cm12, rp, oc, ic, cf);
  ms.has12 = ms.cm12.n_ic <= 32;
}

size_t nnz_of(const MpoSite& ms) { return (size_t)ms.cmL.nnz; }

// ---------------------------------------------------------- contractions
// H_eff^(2) x: x, y (cl, d, d, cr)
// stage 1 of the H_eff matvecs: T1[(a, w), :] = L[(a, w), a'] x[a', :] (n
// columns); with the left identity channel (lid) its rows w = Dl-1 are x
// itself (a strided copy) and the GEMM runs over the other Dl-1 channels
// (batched by channel)
void heff_stage1(tdvp_ctx* h, const cplx* Lenv, int Dl, bool lid, int cl, long long n, const cplx* x, cplx* T1) {
  if (!lid || h->cur_mask[0] != nullptr) {
    gemm(h, OP_N, OP_N, cl * Dl, (int)n, cl, Lenv, cl, x, n, T1, n, h->cur_mask[0]);
    return;
  }
  CK(cudaMemcpy2DAsync(T1 + (long long)(Dl - 1) * n, (size_t)Dl * n * sizeof(cplx), x, (size_t)n * sizeof(cplx),
                       (size_t)n * sizeof(cplx), cl, cudaMemcpyDeviceToDevice, h->st));
  if (Dl > 1) {
    CK(zgemm(h->st, OP_N, OP_N, cl, (int)n, cl, ONE, Lenv, (long long)Dl * cl, x, n, ZERO, T1, (long long)Dl * n,
             Dl - 1, cl, 0, n, h->gemm_work->c(), (size_t)h->work_elems, h->cur_skip, nullptr));
    g_gemm_count++;
    g_launch_count++;
  }
}

// last stage: y[r, b] = sum_{(w, b')} T[r, (w, b')] R[b, (w, b')] (rows r);
// with the right identity channel (rid) the w = 0 term is T[r, (0, b)] (a
// strided copy into y) and the GEMM accumulates the other Dr-1 channels
void heff_stage_last(tdvp_ctx* h, const cplx* T, int rows, int Dr, bool rid, int cr, const cplx* Renv, cplx* y) {
  const long long K = (long long)Dr * cr;
  if (!rid || h->cur_mask[1] != nullptr) {
    gemm(h, OP_N, OP_T, rows, cr, (int)K, T, K, Renv, K, y, cr, h->cur_mask[1]);
    return;
  }
  CK(cudaMemcpy2DAsync(y, (size_t)cr * sizeof(cplx), T, (size_t)K * sizeof(cplx), (size_t)cr * sizeof(cplx), rows,
                       cudaMemcpyDeviceToDevice, h->st));
  if (Dr > 1) {
    CK(zgemm(h->st, OP_N, OP_T, rows, cr, (int)(K - cr), ONE, T + cr, K, Renv + cr, K, ONE, y, cr, 1, 0, 0, 0,
             h->gemm_work->c(), (size_t)h->work_elems, h->cur_skip, nullptr));
    g_gemm_count++;
    g_launch_count++;
  }
}

// H_eff^(2) x: x, y (cl, d, d, cr)
void heff2(tdvp_ctx* h, const cplx* Lenv, const MpoSite& W1, const MpoSite& W2, const cplx* Renv, int cl, int cr,
           const cplx* x, cplx* y) {
  const int d = h->d, Dl = W1.Dl, Dm = W1.Dr, Dr = W2.Dr;
  cplx* T1 = h->T1->c();
  cplx* T2 = h->T2->c();
  // stage 1: T1[(a,w),(t1,t2,b')] = L[(a,w),a'] x[a',(t1,t2,b')]
  heff_stage1(h, Lenv, Dl, W1.lid, cl, (long long)d * d * cr, x, T1);
  if (W1.has12) {
    // stages 2+3 in one pass: T3[a][s1][s2][w''][b'] = sum W12[(w,t1,t2) -> (s1,s2,w'')] T1[a][w][t1][t2][b']
    cmix(h, W1.cm12, cl, cr, T1, (long long)Dl * d * d * cr, 1,
         Strides3{(long long)d * d * cr, (long long)d * cr, (long long)cr}, T2, (long long)d * d * Dr * cr, 1,
         Strides3{(long long)d * Dr * cr, (long long)Dr * cr, (long long)cr});
    heff_stage_last(h, T2, cl * d * d, Dr, W2.rid, cr, Renv, y);
    return;
  }
  // stage 2: T2[a][s1][w'][(t2,b')] = sum W1[w,s1,t1,w'] T1[a][w][t1][(t2,b')]
  cmix(h, W1.cmL, cl, d * cr, T1, (long long)Dl * d * d * cr, 1, Strides3{(long long)d * d * cr, (long long)d * cr, 0},
       T2, (long long)d * Dm * d * cr, 1, Strides3{(long long)Dm * d * cr, (long long)d * cr, 0});
  // stage 3: T3[(a,s1)][s2][w''][b'] = sum W2[w',s2,t2,w''] T2[(a,s1)][w'][t2][b']   (T3 reuses T1)
  cmix(h, W2.cmL, cl * d, cr, T2, (long long)Dm * d * cr, 1, Strides3{(long long)d * cr, (long long)cr, 0}, T1,
       (long long)d * Dr * cr, 1, Strides3{(long long)Dr * cr, (long long)cr, 0});
  // stage 4: y[(a,s1,s2), b] = T3[(a,s1,s2),(w'',b')] R[b,(w'',b')]^T
  heff_stage_last(h, T1, cl * d * d, Dr, W2.rid, cr, Renv, y);
}

// H_eff^(1) x: x, y (cl, d, cr)
void heff1(tdvp_ctx* h, const cplx* Lenv, const MpoSite& W, const cplx* Renv, int cl, int cr, const cplx* x, cplx* y) {
  const int d = h->d, Dl = W.Dl, Dr = W.Dr;
  cplx* T1 = h->T1->c();
  cplx* T2 = h->T2->c();
  heff_stage1(h, Lenv, Dl, W.lid, cl, (long long)d * cr, x, T1);
  cmix(h, W.cmL, cl, cr, T1, (long long)Dl * d * cr, 1, Strides3{(long long)d * cr, (long long)cr, 0}, T2,
       (long long)d * Dr * cr, 1, Strides3{(long long)Dr * cr, (long long)cr, 0});
  heff_stage_last(h, T2, cl * d, Dr, W.rid, cr, Renv, y);
}

// beta'[b,w',b'] = sum conj(A[a,s,b]) beta[a,w,a'] W[w,s,t,w'] A[a',t,b']
void env_left(tdvp_ctx* h, const cplx* beta, const cplx* A, const MpoSite& W, int cl, int cr, cplx* out) {
  const int d = h->d, Dl = W.Dl, Dr = W.Dr;
  cplx* X = h->T1->c();
  cplx* Y = h->T2->c();
  gemm(h, OP_N, OP_N, cl * Dl, d * cr, cl, beta, cl, A, (long long)d * cr, X, (long long)d * cr);
  cmix(h, W.cmL, cl, cr, X, (long long)Dl * d * cr, 1, Strides3{(long long)d * cr, (long long)cr, 0}, Y,
       (long long)d * Dr * cr, 1, Strides3{(long long)Dr * cr, (long long)cr, 0});
  gemm(h, OP_C, OP_N, cr, Dr * cr, cl * d, A, cr, Y, (long long)Dr * cr, out, (long long)Dr * cr);
}

// gamma'[a,w,a'] = sum conj(B[a,s,b]) W[w,s,t,w'] B[a',t,b'] gamma[b,w',b']
void env_right(tdvp_ctx* h, const cplx* gamma, const cplx* B, const MpoSite& W, int cl, int cr, cplx* out) {
  const int d = h->d, Dl = W.Dl, Dr = W.Dr;
  cplx* X = h->T1->c();
  cplx* Y = h->T2->c();
  // X[(a',t),(b,w')] = B[(a',t),b'] gamma[(b,w'),b']
  gemm(h, OP_N, OP_T, cl * d, cr * Dr, cr, B, cr, gamma, cr, X, (long long)cr * Dr);
  // Y[w][a'][s][b] = sum W[w,s,t,w'] X[a'][t][b][w']
  cmix(h, W.cmR, cl, cr, X, (long long)d * cr * Dr, Dr, Strides3{(long long)cr * Dr, 1, 0}, Y, (long long)d * cr, 1,
       Strides3{(long long)cl * d * cr, (long long)cr, 0});
  // out[a,(w,a')] = conj(B)[a,(s,b)] Y[(w,a'),(s,b)]^T
  gemm(h, OP_R, OP_T, cl, Dl * cl, d * cr, B, (long long)d * cr, Y, (long long)d * cr, out, (long long)Dl * cl);
}

double flops_heff2(int cl, int cr, int d, int Dl, int Dr, size_t nnz1, size_t nnz2) {
  // 8 [d^2 cl cr (Dl cl + Dr cr) + d cl cr (nnz W_j + nnz W_{j+1})]
  return 8.0 * ((double)d * d * cl * cr * ((double)Dl * cl + (double)Dr * cr) +
                (double)d * cl * cr * (double)(nnz1 + nnz2));
}
// flops the H_eff matvecs execute: the identity channels (MpoSite::lid/rid)
// are copied, not contracted
double flops_heff2_exec(int cl, int cr, int d, int Dl, int Dr, size_t nnz1, size_t nnz2, bool lid, bool rid) {
  return 8.0 * ((double)d * d * cl * cr * ((double)(Dl - (lid ? 1 : 0)) * cl + (double)(Dr - (rid ? 1 : 0)) * cr) +
                (double)d * cl * cr * (double)(nnz1 + nnz2));
}
double flops_heff1_exec(int cl, int cr, int d, int Dl, int Dr, size_t nnz, bool lid, bool rid) {
  return 8.0 * ((double)d * cl * cr * ((double)(Dl - (lid ? 1 : 0)) * cl + (double)(Dr - (rid ? 1 : 0)) * cr) +
                (double)cl * cr * (double)nnz);
}
double flops_heff1(int cl, int cr, int d, int Dl, int Dr, size_t nnz) {
  return 8.0 * ((double)d * cl * cr * ((double)Dl * cl + (double)Dr * cr) + (double)cl * cr * (double)nnz);
}

// exp(tau H) x -> out, device-resident Lanczos (SURVEY O-10)
void expm_lanczos(tdvp_ctx* h, const std::function<void(const cplx*, cplx*)>& matvec, const cplx* x, cplx* out,
                  long long n, double tre, double tim, int K, int which /*2: heff2 1: heff1 0: other*/, double mv_flop,
                  double mv_flop_exec = -1.0) {
  if (mv_flop_exec < 0.0) mv_flop_exec = mv_flop;
  cplx* V = h->krylov->c();
  cplx* w = h->wvec->c();
  const bool tm = h->prm.timing && which;
  const int lz_ea = tm ? ev_record(h) : -1;
  const size_t lz_mv0 = which == 2 ? h->ev_h2.size() : h->ev_h1.size();
  CK(lz_start(h->st, h->lz, x, V, n));
  g_launch_count += 2;
  // paper mode (krylov_tol > 0): the convergence test runs on
  // the device; once it passes, every later kernel of this exponential
  // (matvec GEMMs and channel mixes, Lanczos iterations) returns at once
  const double ktol = h->prm.krylov_tol;
  const bool paper = ktol > 0.0;
  h->cur_skip = paper ? h->lz.scal + LZ_SKIP : nullptr;
  for (int k = 0; k < K; ++k) {
    int e0 = -1;
    if (h->prm.timing && which) e0 = ev_record(h);
    matvec(V + (long long)k * n, w);
    if (e0 >= 0) {
      const int e1 = ev_record(h);
      (which == 2 ? h->ev_h2 : h->ev_h1).emplace_back(e0, e1);
      if (which == 2) {
        h->stats.heff2_flop += mv_flop;
        h->stats.heff2_flop_exec += mv_flop_exec;
        h->stats.heff2_calls++;
        h->stats.heff2_flop_bin[h->cur_bin] += mv_flop;
        h->ev_h2_bin.push_back(h->cur_bin);
      } else {
        h->stats.heff1_flop += mv_flop;
        h->stats.heff1_flop_exec += mv_flop_exec;
      }
    }
    CK(lz_iter(h->st, h->lz, V, n, k + 1, w, V + (long long)(k + 1) * n, n, k, k + 1 == K ? 1 : 0, ktol, tre, tim));
    g_launch_count++;
  }
  h->cur_skip = nullptr;
  if (h->prm.timing && which) {
    // algorithmic bytes of the vector passes: start 3 passes over n,
    // iteration k < K-1 with nv = k+1 basis vectors (3 nv + 6) (dots; update + dots;
    // update + norm; scale), the last (nv + 1) (dots only), combination K + 1
    double units = 3.0 + (double)(K + 1) + (double)(K + 1);
    for (int k = 0; k + 1 < K; ++k) units += 3.0 * (k + 1) + 6.0;
    h->stats.lz_vec_bytes += units * 16.0 * (double)n;
    h->stats.lz_bytes_bin[h->cur_bin] += units * 16.0 * (double)n;
  }
  CK(lz_tridiag_exp(h->st, h->lz, K, tre, tim));
  CK(lz_combine(h->st, h->lz, V, n, K, out, n));
  g_launch_count += 2;
  if (tm)
    h->ev_lzrec.push_back({lz_ea, ev_record(h), h->cur_bin, which, lz_mv0,
                           which == 2 ? h->ev_h2.size() : h->ev_h1.size()});
}

// --------------------------------------------------------- local updates
inline cplx* P(const BufPtr& b) { return b ? b->c() : nullptr; }

void require_held(const Segment& g, int j) {
  if (!g.psi[j] || !g.beta[j] || !g.gamma[j]) throw TdvpError(TDVP_ECUDA, "internal: site not held by segment");
}

// ------------------------------------------------------------ U(1) split
// (PAPER.md:643-651 symmetric block-sparse tensors).  With an
// S^z-conserving MPO and a state of definite S^z every bond index carries a
// charge q = 2 S^z of the sites to its left; the matrix to split is block
// diagonal in the charge of the new bond (rows and columns carry it), so its
// SVD is the union of the sector SVDs.  Each sector is gathered and split by
// the dense path (svd_truncate_split, untruncated), the truncation rule O-7
// (incl. AMB-9 / R-9b) is applied on the host to the union of all sectors'
// singular values in descending order, exactly as the dense kernel does, and
// the kept columns / rows are scattered into Psi_L / Psi_R, which keep exact
// zeros outside their blocks.  Oracle: oracle/u1.py.
constexpr int U1_C[2] = {1, -1};  // 2 S^z of the basis states (0 = up, 1 = down)

__global__ void u1_gather_kernel(const cplx* __restrict__ M, long long ldm, const int* __restrict__ rows,
                                 const int* __restrict__ cols, int mq, int nq, cplx* out) {
  const long long total = (long long)mq * nq;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / nq), k = (int)(e - (long long)i * nq);
    out[e] = M[(long long)rows[i] * ldm + cols[k]];
  }
}
// dst[rows[i]][kmap[k]] = src[i][k] (kmap[k] < 0: dropped), src mq x kq, dst ld ldd
__global__ void u1_scatter_cols_kernel(const cplx* __restrict__ src, int mq, int kq, const int* __restrict__ rows,
                                       const int* __restrict__ kmap, cplx* dst, long long ldd) {
  const long long total = (long long)mq * kq;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / kq), k = (int)(e - (long long)i * kq);
    const int c = kmap[k];
    if (c >= 0) dst[(long long)rows[i] * ldd + c] = src[e];
  }
}
// dst[kmap[k]][cols[i]] = src[k][i], src kq x nq, dst ld ldd
__global__ void u1_scatter_rows_kernel(const cplx* __restrict__ src, int kq, int nq, const int* __restrict__ cols,
                                       const int* __restrict__ kmap, cplx* dst, long long ldd) {
  const long long total = (long long)kq * nq;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(e / nq), i = (int)(e - (long long)k * nq);
    const int c = kmap[k];
    if (c >= 0) dst[(long long)c * ldd + cols[i]] = src[e];
  }
}

// bond charges of the host MPS copy from its nonzero pattern (q[0] = {0});
// TDVP_EARG if an index is reachable with two charges or none
std::vector<std::vector<int>> infer_charges(const tdvp_ctx* h) {
  const int L = h->L, d = h->d;
  std::vector<std::vector<int>> q(L + 1);
  q[0] = {0};
  const int UNSET = std::numeric_limits<int>::min();
  for (int j = 0; j < L; ++j) {
    const int cl = h->h_chi[j], cr = h->h_chi[j + 1];
    const hvec& t = h->h_psi[j];
    q[j + 1].assign(cr, UNSET);
    for (int a = 0; a < cl; ++a)
      for (int s = 0; s < d; ++s)
        for (int b = 0; b < cr; ++b) {
          const size_t e = (((size_t)a * d + s) * cr + b) * 2;
          if (t[e] == 0.0 && t[e + 1] == 0.0) continue;
          const int v = q[j][a] + U1_C[s];
          if (q[j + 1][b] == UNSET) q[j + 1][b] = v;
          else if (q[j + 1][b] != v)
            throw TdvpError(TDVP_EARG, "u1: the MPS is not of definite charge (bond " + std::to_string(j + 1) + ")");
        }
    for (int b = 0; b < cr; ++b)
      if (q[j + 1][b] == UNSET) throw TdvpError(TDVP_EARG, "u1: a bond index with no nonzero entry");
  }
  return q;
}

int owner_of(tdvp_ctx* h, int j);
// the bond charges of the current (laid-out) state, owner view
std::vector<std::vector<int>> assemble_charges(tdvp_ctx* h) {
  const int L = h->L;
  std::vector<std::vector<int>> q(L + 1);
  q[0] = {0};
  for (int k = 1; k < L; ++k) q[k] = h->segs[owner_of(h, k - 1)].qb[k];
  q[L] = h->segs[owner_of(h, L - 1)].qb[L];
  return q;
}

inline int u1_grid(long long n) { return (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, 4LL * g_num_sms)); }

// Split the m x n row-major matrix M (device) with row charges rq and column
// charges cq: Psi_L (m x chi), Psi_R (chi x n), Lambda / V (chi), q_mid (chi).
void u1_svd_split(tdvp_ctx* h, const cplx* M, int m, int n, const std::vector<int>& rq, const std::vector<int>& cq,
                  const TruncParams& tp, cplx* psiL, cplx* psiR, double* lam, double* vinv, int& chi, double& w,
                  int& r, int& chi_eps, std::vector<int>& q_mid, int& sweeps_sum) {
  std::map<int, std::pair<std::vector<int>, std::vector<int>>> sec;
  for (int i = 0; i < m; ++i) sec[rq[i]].first.push_back(i);
  for (int k = 0; k < n; ++k) sec[cq[k]].second.push_back(k);
  struct Sector {
    int Q, mq, nq, kq = 0, idx_off = 0;
    long long offL = 0, offR = 0, goff = 0, koff = 0;
    std::vector<double> sig;
  };
  std::vector<Sector> ss;
  std::vector<int> idx;  // rows then cols of every sector
  for (auto& kv : sec) {
    if (kv.second.first.empty() || kv.second.second.empty()) continue;
    Sector t;
    t.Q = kv.first;
    t.mq = (int)kv.second.first.size();
    t.nq = (int)kv.second.second.size();
    t.idx_off = (int)idx.size();
    idx.insert(idx.end(), kv.second.first.begin(), kv.second.first.end());
    idx.insert(idx.end(), kv.second.second.begin(), kv.second.second.end());
    ss.push_back(std::move(t));
  }
  if (ss.empty()) throw TdvpError(TDVP_ENUMERIC, "U(1) split: no charge sector carries weight");
  if (idx.size() * sizeof(int) > h->u1_idx->bytes / 2) throw TdvpError(TDVP_ECUDA, "internal: U(1) index buffer");
  int* didx = h->u1_idx->i();
  CK(cudaMemcpyAsync(didx, idx.data(), idx.size() * sizeof(int), cudaMemcpyHostToDevice, h->st));
  const TruncParams full{std::max(m, n), 0.0, 0.0, 0.0};
  cplx* stL = h->T1->c();
  cplx* stR = h->T2->c();
  // every sector gets its own regions: the gathered block in tmpA, its factors
  // in T1 / T2 and its spectrum in u1_lam / u1_vinv, sized by kmax = min(mq, nq)
  // (sum mq nq <= m n and sum kmax <= min(m, n): the sectors partition rows and columns)
  {
    long long go = 0, lo = 0, ro = 0, ko = 0;
    for (auto& t : ss) {
      const int kmax = std::min(t.mq, t.nq);
      t.offL = lo;
      t.offR = ro;
      t.goff = go;
      t.koff = ko;
      go += (long long)t.mq * t.nq;
      lo += (long long)t.mq * kmax;
      ro += (long long)kmax * t.nq;
      ko += kmax;
    }
  }
  // sector SVDs run concurrently: NW worker threads, each with its own stream
  // and SVD workspace (svd_truncate_split reads chi back on the host), sectors
  // handed out largest first; the workers wait on the index upload
  constexpr int NW = 4;
  if (h->u1w.empty()) {
    const long long ncmax = (long long)h->d * h->chi_max;
    const size_t nflags = (size_t)4 * ncmax + 64;
    for (int w = 0; w < NW; ++w) {
      auto u = std::make_unique<tdvp_ctx::U1Worker>();
      CK(cudaStreamCreateWithFlags(&u->st, cudaStreamNonBlocking));
      u->Y = make_buf((size_t)h->svdmax * sizeof(cplx));
      u->Q = make_buf(h->svdQ->bytes);
      u->F = make_buf(nflags * sizeof(unsigned));
      u->sigma = make_buf(ncmax * sizeof(double) + 64);
      u->order = make_buf(ncmax * sizeof(int) + 64);
      u->perm = make_buf(2 * ncmax * sizeof(int) + 64);
      u->bj = make_buf(svd_bjac_work_elems(g_num_sms) * sizeof(cplx));
      u->off = make_buf(64);
      u->ires = make_buf(64);
      u->dres = make_buf(64);
      CK(cudaMallocHost(&u->h_pin, 16 * sizeof(double)));
      CK(cudaMallocHost(&u->h_ipin, 16 * sizeof(int)));
      u->sv = SvdDev{u->Y->c(), 0, u->sigma->d(), u->order->i(), u->off->d(), u->ires->i(), u->dres->d(),
                     u->h_pin, u->h_ipin, {nullptr, nullptr}, u->Q->c(), h->svdQ->bytes / sizeof(cplx),
                     reinterpret_cast<unsigned*>(u->F->p), nflags, 1, u->perm->i(), u->bj->c(),
                     svd_bjac_work_elems(g_num_sms)};
      h->u1w.push_back(std::move(u));
    }
  }
  cudaEvent_t ev_in = ev_get(h);
  CK(cudaEventRecord(ev_in, h->st));
  std::vector<int> order(ss.size());
  for (size_t i = 0; i < ss.size(); ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(), [&](int a_, int b_) {
    return (long long)ss[a_].mq * ss[a_].nq > (long long)ss[b_].mq * ss[b_].nq;
  });
  std::atomic<int> next{0};
  std::vector<int> sws(ss.size(), 0);
  std::vector<std::string> errs(NW);
  std::vector<int> errc(NW, 0);
  const int dev = h->dev;
  auto work = [&](int w) {
    try {
      DeviceGuard dg(dev);
      tdvp_ctx::U1Worker& u = *h->u1w[w];
      CK(cudaStreamWaitEvent(u.st, ev_in, 0));
      for (int i = next.fetch_add(1); i < (int)ss.size(); i = next.fetch_add(1)) {
        Sector& t = ss[order[i]];
        cplx* blk = h->tmpA->c() + t.goff;
        u1_gather_kernel<<<u1_grid((long long)t.mq * t.nq), 256, 0, u.st>>>(M, n, didx + t.idx_off,
                                                                          didx + t.idx_off + t.mq, t.mq, t.nq, blk);
        CK(cudaGetLastError());
        int k = 0, rr = 0, ce = 0, sw = 0;
        double ww = 0.0;
        cudaError_t se = svd_truncate_split(u.st, u.sv, blk, t.mq, t.nq, full, stL + t.offL, stR + t.offR,
                                            h->u1_lam->d() + t.koff, h->u1_vinv->d() + t.koff, &k, &ww, &rr, &ce,
                                            &sw);
        if (se == cudaErrorUnknown) throw TdvpError(TDVP_ENUMERIC, "non-finite or zero spectrum in a U(1) sector");
        CK(se);
        sws[order[i]] = std::max(sw, 0);
        t.kq = k;
        t.sig.resize(k);
        CK(cudaMemcpyAsync(t.sig.data(), h->u1_lam->d() + t.koff, k * sizeof(double), cudaMemcpyDeviceToHost, u.st));
        CK(cudaStreamSynchronize(u.st));
      }
    } catch (const TdvpError& e) {
      errc[w] = e.code;
      errs[w] = e.what();
    } catch (const std::exception& e) {
      errc[w] = TDVP_ECUDA;
      errs[w] = e.what();
    }
  };
  {
    std::vector<std::thread> th;
    for (int w = 1; w < NW; ++w) th.emplace_back(work, w);
    work(0);
    for (auto& x : th) x.join();
  }
  for (int w = 0; w < NW; ++w)
    if (errc[w]) throw TdvpError(errc[w], errs[w]);
  sweeps_sum = 0;
  for (int x : sws) sweeps_sum += x;
  g_launch_count += 2 * (long long)ss.size();
  // global order: descending sigma, ties by sector charge then index (oracle/u1.py)
  struct Ent { double s; int sec, k; };
  std::vector<Ent> all;
  for (int si = 0; si < (int)ss.size(); ++si)
    for (int k = 0; k < ss[si].kq; ++k) all.push_back(Ent{ss[si].sig[k], si, k});
  std::stable_sort(all.begin(), all.end(), [&](const Ent& a, const Ent& b) {
    if (a.s != b.s) return a.s > b.s;
    if (ss[a.sec].Q != ss[b.sec].Q) return ss[a.sec].Q < ss[b.sec].Q;
    return a.k < b.k;
  });
  r = (int)all.size();
  const double s1 = all[0].s;
  if (!(s1 > 0.0) || !std::isfinite(s1)) throw TdvpError(TDVP_ENUMERIC, "U(1) split: zero or non-finite spectrum");
  // the truncation rule O-7 with AMB-9 / R-9b (as svd_truncate_kernel)
  const double eps = tp.eps > 0.0 ? tp.eps : 1e-14;
  int nz = 0;
  chi_eps = 0;
  for (auto& e : all) {
    chi_eps += (e.s >= eps * s1);
    nz += (e.s > 0.0);
  }
  int chi_w = nz;
  if (tp.w_max > 0.0) {
    std::vector<double> tail(r + 1, 0.0);
    for (int k = r - 1; k >= 0; --k) tail[k] = tail[k + 1] + all[k].s * all[k].s;
    for (int c = 0; c <= r; ++c)
      if (tail[c] <= tp.w_max) { chi_w = c; break; }
    chi_w = std::max(chi_w, 1);
  }
  chi = std::max(1, std::min(std::min(chi_eps, chi_w), tp.chi_max));
  while (chi > 1 && chi < r && all[chi - 1].s - all[chi].s <= tp.delta * all[chi - 1].s + 1e-13 * s1) --chi;
  w = 0.0;
  for (int k = chi; k < r; ++k) w += all[k].s * all[k].s;
  // the kept triplets ordered by charge (ascending), then sigma (descending):
  // every bond basis stays sorted by charge, so the U(1) blocks of the next
  // contractions are contiguous and the GEMM block masks skip them whole
  std::stable_sort(all.begin(), all.begin() + chi, [&](const Ent& a, const Ent& b) {
    if (ss[a.sec].Q != ss[b.sec].Q) return ss[a.sec].Q < ss[b.sec].Q;
    return a.s > b.s;
  });
  // scatter the kept triplets; lam / V / charges in that order
  CK(cudaMemsetAsync(psiL, 0, (size_t)m * chi * sizeof(cplx), h->st));
  CK(cudaMemsetAsync(psiR, 0, (size_t)chi * n * sizeof(cplx), h->st));
  std::vector<std::vector<int>> km(ss.size());
  for (int si = 0; si < (int)ss.size(); ++si) km[si].assign(ss[si].kq, -1);
  std::vector<double> hl(chi), hv(chi);
  q_mid.assign(chi, 0);
  for (int c = 0; c < chi; ++c) {
    km[all[c].sec][all[c].k] = c;
    hl[c] = all[c].s;
    hv[c] = 1.0 / all[c].s;
    q_mid[c] = ss[all[c].sec].Q;
  }
  std::vector<int> kflat;
  std::vector<int> koff(ss.size());
  for (int si = 0; si < (int)ss.size(); ++si) {
    koff[si] = (int)kflat.size();
    kflat.insert(kflat.end(), km[si].begin(), km[si].end());
  }
  int* dk = didx + (h->u1_idx->bytes / 2) / sizeof(int);  // second half of the index buffer
  CK(cudaMemcpyAsync(dk, kflat.data(), std::max<size_t>(1, kflat.size()) * sizeof(int), cudaMemcpyHostToDevice, h->st));
  for (int si = 0; si < (int)ss.size(); ++si) {
    const Sector& t = ss[si];
    if (t.kq == 0) continue;
    u1_scatter_cols_kernel<<<u1_grid((long long)t.mq * t.kq), 256, 0, h->st>>>(stL + t.offL, t.mq, t.kq,
                                                                               didx + t.idx_off, dk + koff[si], psiL,
                                                                               chi);
    u1_scatter_rows_kernel<<<u1_grid((long long)t.kq * t.nq), 256, 0, h->st>>>(stR + t.offR, t.kq, t.nq,
                                                                               didx + t.idx_off + t.mq,
                                                                               dk + koff[si], psiR, n);
  }
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(lam, hl.data(), chi * sizeof(double), cudaMemcpyHostToDevice, h->st));
  CK(cudaMemcpyAsync(vinv, hv.data(), chi * sizeof(double), cudaMemcpyHostToDevice, h->st));
  CK(cudaStreamSynchronize(h->st));  // host vectors go out of scope
}

// row / column charges of the two-site matrix of pair (j, j+1): rows (a, s1),
// columns (s2, b) (AMB-17)
void u1_pair_charges(const Segment& g, int j, int d, std::vector<int>& rq, std::vector<int>& cq) {
  const std::vector<int>& qa = g.qb[j];
  const std::vector<int>& qc = g.qb[j + 2];
  const int cl = g.cb[j], cr = g.cb[j + 2];
  if ((int)qa.size() != cl || (int)qc.size() != cr) throw TdvpError(TDVP_ECUDA, "internal: U(1) charges out of date");
  rq.resize((size_t)cl * d);
  cq.resize((size_t)d * cr);
  for (int a = 0; a < cl; ++a)
    for (int s = 0; s < d; ++s) rq[(size_t)a * d + s] = qa[a] + U1_C[s];
  for (int s = 0; s < d; ++s)
    for (int b = 0; b < cr; ++b) cq[(size_t)s * cr + b] = qc[b] - U1_C[s];
}

// Block masks of op(A) = rows x k and op(B) = k x cols for a U(1)-blocked
// product: an element of op(A) can be nonzero only if its row charge equals
// its k charge, of op(B) only if its k charge equals its column charge
// (charges in one common frame; INT_MIN = unknown = matches every charge).
// 32-row / 8-k / 32-column blocks as GemmMask expects; uploaded on h->st.
void build_mask(tdvp_ctx* h, tdvp_ctx::MaskSet& ms, const std::vector<int>& rq, const std::vector<int>& kq,
                const std::vector<int>& cq) {
  const int M = (int)rq.size(), K = (int)kq.size(), N = (int)cq.size();
  const int mb = (M + 31) / 32, kb = (K + 7) / 8, nb = (N + 31) / 32;
  int lo = 0, hi = 0;
  bool first = true;
  for (const auto* v : {&rq, &kq, &cq})
    for (int x : *v)
      if (x != std::numeric_limits<int>::min()) {
        lo = first ? x : std::min(lo, x);
        hi = first ? x : std::max(hi, x);
        first = false;
      }
  const int W = (hi - lo) / 64 + 1;
  auto sets = [&](const std::vector<int>& q, int blk, int nblk) {
    std::vector<uint64_t> out((size_t)nblk * W, 0);
    for (int i = 0; i < (int)q.size(); ++i) {
      uint64_t* w = out.data() + (size_t)(i / blk) * W;
      if (q[i] == std::numeric_limits<int>::min()) {
        for (int k = 0; k < W; ++k) w[k] = ~0ull;
      } else {
        const int o = q[i] - lo;
        w[o / 64] |= 1ull << (o % 64);
      }
    }
    return out;
  };
  const std::vector<uint64_t> sr = sets(rq, 32, mb), sk = sets(kq, 8, kb), sc = sets(cq, 32, nb);
  auto meet = [&](const uint64_t* a, const uint64_t* b) {
    for (int k = 0; k < W; ++k)
      if (a[k] & b[k]) return 1;
    return 0;
  };
  ms.ha.assign((size_t)mb * kb, 0);
  ms.hb.assign((size_t)kb * nb, 0);
  for (int r = 0; r < mb; ++r)
    for (int k = 0; k < kb; ++k) ms.ha[(size_t)r * kb + k] = (unsigned char)meet(&sr[(size_t)r * W], &sk[(size_t)k * W]);
  for (int k = 0; k < kb; ++k)
    for (int c = 0; c < nb; ++c) ms.hb[(size_t)k * nb + c] = (unsigned char)meet(&sk[(size_t)k * W], &sc[(size_t)c * W]);
  if (!ms.da || ms.da->bytes < ms.ha.size()) ms.da = make_buf(ms.ha.size() + 64);
  if (!ms.db || ms.db->bytes < ms.hb.size()) ms.db = make_buf(ms.hb.size() + 64);
  CK(cudaMemcpyAsync(ms.da->p, ms.ha.data(), ms.ha.size(), cudaMemcpyHostToDevice, h->st));
  CK(cudaMemcpyAsync(ms.db->p, ms.hb.data(), ms.hb.size(), cudaMemcpyHostToDevice, h->st));
  ms.g.a = reinterpret_cast<const unsigned char*>(ms.da->p);
  ms.g.b = reinterpret_cast<const unsigned char*>(ms.db->p);
  ms.g.ldA = kb;
  ms.g.ldB = nb;
}

// the masks of the two dense GEMMs of H_eff^(2) (pair j) or H_eff^(1) (site j)
// in U(1) mode (charge frames derived in DESIGN.md §N1): stage 1
// beta[(a,w),a'] theta[a',(t..,b')]: rows q(a) - r(w), k q(a'), columns
// q(b') - sum c(t); last stage T[(a,s..),(w',b')] R^T[(w',b'),b]: rows
// q(a) + sum c(s), k q(b') + r(w'), columns q(b).  Returns false (dense) when
// the MPO's channel charges are unknown.
bool set_heff_masks(tdvp_ctx* h, const Segment& g, int j, int nsite) {
  const int d = h->d, L = h->L;
  const tdvp_ctx* root = h->parent ? h->parent : h;
  if (!h->prm.u1 || (int)root->h_r.size() != L + 1) return false;
  const std::vector<int>& qa = g.qb[j];
  const std::vector<int>& qb = g.qb[j + nsite];
  const std::vector<int>& rl = root->h_r[j];
  const std::vector<int>& rr = root->h_r[j + nsite];
  const int cl = g.cb[j], cr = g.cb[j + nsite], Dl = (int)rl.size(), Dr = (int)rr.size();
  if ((int)qa.size() != cl || (int)qb.size() != cr) return false;
  const int UNK = std::numeric_limits<int>::min();
  const int ns = nsite == 2 ? d * d : d;
  auto csum = [&](int idx) { return nsite == 2 ? U1_C[idx / d] + U1_C[idx % d] : U1_C[idx]; };
  std::vector<int> rq((size_t)cl * Dl), kq(qa.begin(), qa.end()), cq((size_t)ns * cr);
  for (int a = 0; a < cl; ++a)
    for (int w = 0; w < Dl; ++w) rq[(size_t)a * Dl + w] = rl[w] == UNK ? UNK : qa[a] - rl[w];
  for (int t = 0; t < ns; ++t)
    for (int b = 0; b < cr; ++b) cq[(size_t)t * cr + b] = qb[b] - csum(t);
  build_mask(h, h->masks[0], rq, kq, cq);
  std::vector<int> rq2((size_t)cl * ns), kq2((size_t)Dr * cr);
  for (int a = 0; a < cl; ++a)
    for (int t = 0; t < ns; ++t) rq2[(size_t)a * ns + t] = qa[a] + csum(t);
  for (int w = 0; w < Dr; ++w)
    for (int b = 0; b < cr; ++b) kq2[(size_t)w * cr + b] = rr[w] == UNK ? UNK : qb[b] + rr[w];
  build_mask(h, h->masks[1], rq2, kq2, qb);
  h->cur_mask[0] = &h->masks[0].g;
  h->cur_mask[1] = &h->masks[1].g;
  return true;
}

// the split of a two-site update: dense or sector-wise (U(1))
cudaError_t split_theta(tdvp_ctx* h, Segment& g, int j, const cplx* th2, int cl, int cr, const TruncParams& tp,
                        int& chi, double& w, int& r, int& chi_eps, int& sweeps, float* jac_ms, double* jac_flop) {
  const int d = h->d;
  if (!h->prm.u1)
    return svd_truncate_split(h->st, h->sv, th2, cl * d, d * cr, tp, P(g.psi[j]), P(g.psi[j + 1]), g.lam[j]->d(),
                              g.vinv[j]->d(), &chi, &w, &r, &chi_eps, &sweeps, jac_ms, jac_flop);
  std::vector<int> rq, cq, qm;
  u1_pair_charges(g, j, d, rq, cq);
  u1_svd_split(h, th2, cl * d, d * cr, rq, cq, tp, P(g.psi[j]), P(g.psi[j + 1]), g.lam[j]->d(), g.vinv[j]->d(), chi, w,
               r, chi_eps, qm, sweeps);
  g.qb[j + 1] = qm;
  if (jac_flop) *jac_flop = 0.0;
  if (jac_ms) *jac_ms = 0.f;
  return cudaSuccess;
}

// two-site forward update of (j, j+1) (SURVEY O-6)
void pair_update(tdvp_ctx* h, Segment& g, int j, double dt, int full, int build) {
  const int d = h->d;
  const int cl = g.cb[j], cm = g.cb[j + 1], cr = g.cb[j + 2];
  const MpoSite& W1 = h->mpo[j];
  const MpoSite& W2 = h->mpo[j + 1];
  cplx* th = h->theta->c();
  // a1: Theta = Psi_j diag(V_j) Psi_{j+1}
  CK(scale_rows(h->st, h->tmpA->c(), P(g.psi[j + 1]), g.vinv[j]->d(), cm, (long long)d * cr));
  g_launch_count++;
  gemm(h, OP_N, OP_N, cl * d, d * cr, cm, P(g.psi[j]), cm, h->tmpA->c(), (long long)d * cr, th, (long long)d * cr);
  // a2/a3: Theta' = exp(-i tau H_eff^(2)) Theta
  const long long n = (long long)cl * d * d * cr;
  const cplx* Lenv = P(g.beta[j]);
  const cplx* Renv = P(g.gamma[j + 1]);
  const double tau = full ? dt : 0.5 * dt;
  const double fl = flops_heff2(cl, cr, d, W1.Dl, W2.Dr, nnz_of(W1), nnz_of(W2));
  {
    const int cx = std::max(cl, cr);
    h->cur_bin = cx <= 128 ? 0 : cx <= 256 ? 1 : cx <= 512 ? 2 : 3;
  }
  cplx* th2 = h->tmpB->c();
  const int el0 = h->prm.timing ? ev_record(h) : -1;
  set_heff_masks(h, g, j, 2);
  expm_lanczos(
      h, [&](const cplx* x, cplx* y) { heff2(h, Lenv, W1, W2, Renv, cl, cr, x, y); }, th, th2, n, 0.0, -tau,
      h->prm.krylov_k, 2, fl,
      h->prm.u1 ? fl : flops_heff2_exec(cl, cr, d, W1.Dl, W2.Dr, nnz_of(W1), nnz_of(W2), W1.lid, W2.rid));
  h->cur_mask[0] = h->cur_mask[1] = nullptr;
  if (el0 >= 0) h->ev_lz2.emplace_back(el0, ev_record(h));
  // a4: truncated SVD split
  int e0 = -1;
  if (h->prm.timing) e0 = ev_record(h);
  TruncParams tp{h->chi_max, h->prm.eps, h->prm.w_max, h->prm.multiplet_delta};
  int chi = 0, r = 0, chi_eps = 0, sweeps = 0;
  double w = 0.0;
  float jac_ms = 0.f;
  double jac_flop = 0.0;
  cudaError_t se = split_theta(h, g, j, th2, cl, cr, tp, chi, w, r, chi_eps, sweeps, h->prm.timing ? &jac_ms : nullptr,
                               &jac_flop);
  if (se == cudaErrorUnknown) throw TdvpError(TDVP_ENUMERIC, "non-finite or zero spectrum in SVD at bond " + std::to_string(j));
  CK(se);
  g_launch_count += 5;
  if (e0 >= 0) h->ev_svd.emplace_back(e0, ev_record(h));
  if (chi > h->cbmax[j + 1]) throw TdvpError(TDVP_ECUDA, "internal: chi exceeds allocation");
  g.cb[j + 1] = chi;
  h->stats.w_step += w;
  h->stats.n_pair++;
  h->stats.svd_sweeps_max = std::max(h->stats.svd_sweeps_max, sweeps);
  h->stats.svd_sweeps_total += sweeps;
  {
    const double mr = std::max(cl * d, d * cr), nc = std::min(cl * d, d * cr);
    h->stats.svd_jac_ms += jac_ms;
    // block-Jacobi (DMMA) path: the flops it executed; SIMT paths: the scalar count per sweep
    h->stats.svd_jac_flop += jac_flop > 0.0 ? jac_flop
                                            : (double)sweeps * nc * (nc - 1) / 2 * (16.0 * mr + 24.0 * (mr + nc));
    if (jac_flop > 0.0) {  // the block-Jacobi (DMMA) kernel alone: the dominant kernel at chi = 1024
      h->stats.svd_bj_ms += jac_ms;
      h->stats.svd_bj_flop += jac_flop;
      h->stats.svd_bj_calls++;
    }
  }
  if (chi < std::min(chi_eps, r)) h->stats.trunc_active = 1;
  // a5: environments for the next update
  const int ee0 = h->prm.timing ? ev_record(h) : -1;
  if (build & BUILD_BETA) {
    CK(scale_cols(h->st, h->tmpA->c(), P(g.psi[j]), g.vinv[j]->d(), (long long)cl * d, chi));
    g_launch_count++;
    env_left(h, P(g.beta[j]), h->tmpA->c(), W1, cl, chi, P(g.beta[j + 1]));
  }
  if (build & BUILD_GAMMA) {
    CK(scale_rows(h->st, h->tmpA->c(), P(g.psi[j + 1]), g.vinv[j]->d(), chi, (long long)d * cr));
    g_launch_count++;
    env_right(h, P(g.gamma[j + 1]), h->tmpA->c(), W2, chi, cr, P(g.gamma[j]));
  }
  if (ee0 >= 0) h->ev_env.emplace_back(ee0, ev_record(h));
}

// ----------------------------------------------------------- two-site DMRG
// (SURVEY N3; PAPER.md:100 ARPACK with 8 Krylov vectors, :122, :130, :178 the
// ground states every quench starts from).  Lowest eigenvector of H_eff^(2)
// by restarted Lanczos on the device: `restarts` times, the K-vector basis of
// the fused Lanczos iterations from the current vector, the lowest eigenpair
// of the tridiagonal (one thread, Jacobi; y_0 >= 0), x <- V y.  Reading
// R-DMRG in DESIGN.md; the oracle is oracle/dmrg.py.
void ground_lanczos(tdvp_ctx* h, const std::function<void(const cplx*, cplx*)>& matvec, const cplx* x, cplx* out,
                    long long n, int K, int restarts) {
  cplx* V = h->krylov->c();
  cplx* w = h->wvec->c();
  const cplx* cur = x;
  for (int r = 0; r < restarts; ++r) {
    CK(lz_start(h->st, h->lz, cur, V, n));
    g_launch_count += 2;
    for (int k = 0; k < K; ++k) {
      matvec(V + (long long)k * n, w);
      CK(lz_iter(h->st, h->lz, V, n, k + 1, w, V + (long long)(k + 1) * n, n, k, k + 1 == K ? 1 : 0));
      g_launch_count++;
    }
    CK(lz_tridiag_ground(h->st, h->lz, K));
    CK(lz_combine(h->st, h->lz, V, n, K, out, n));
    g_launch_count += 2;
    cur = out;
  }
}

// DMRG pair update of (j, j+1): merge, ground state of H_eff^(2), the same
// truncated SVD split as the TDVP pair update, environments `build`
void dmrg_pair(tdvp_ctx* h, Segment& g, int j, int build, int restarts) {
  const int d = h->d;
  const int cl = g.cb[j], cm = g.cb[j + 1], cr = g.cb[j + 2];
  const MpoSite& W1 = h->mpo[j];
  const MpoSite& W2 = h->mpo[j + 1];
  cplx* th = h->theta->c();
  CK(scale_rows(h->st, h->tmpA->c(), P(g.psi[j + 1]), g.vinv[j]->d(), cm, (long long)d * cr));
  gemm(h, OP_N, OP_N, cl * d, d * cr, cm, P(g.psi[j]), cm, h->tmpA->c(), (long long)d * cr, th, (long long)d * cr);
  const long long n = (long long)cl * d * d * cr;
  const cplx* Lenv = P(g.beta[j]);
  const cplx* Renv = P(g.gamma[j + 1]);
  cplx* th2 = h->tmpB->c();
  set_heff_masks(h, g, j, 2);
  ground_lanczos(
      h, [&](const cplx* x, cplx* y) { heff2(h, Lenv, W1, W2, Renv, cl, cr, x, y); }, th, th2, n, h->prm.krylov_k,
      restarts);
  h->cur_mask[0] = h->cur_mask[1] = nullptr;
  TruncParams tp{h->chi_max, h->prm.eps, h->prm.w_max, h->prm.multiplet_delta};
  int chi = 0, r = 0, chi_eps = 0, sweeps = 0;
  double w = 0.0;
  cudaError_t se = split_theta(h, g, j, th2, cl, cr, tp, chi, w, r, chi_eps, sweeps, nullptr, nullptr);
  if (se == cudaErrorUnknown) throw TdvpError(TDVP_ENUMERIC, "non-finite or zero spectrum in SVD at bond " + std::to_string(j));
  CK(se);
  if (chi > h->cbmax[j + 1]) throw TdvpError(TDVP_ECUDA, "internal: chi exceeds allocation");
  g.cb[j + 1] = chi;
  h->stats.w_step += w;
  h->stats.n_pair++;
  if (chi < std::min(chi_eps, r)) h->stats.trunc_active = 1;
  if (build & BUILD_BETA) {
    CK(scale_cols(h->st, h->tmpA->c(), P(g.psi[j]), g.vinv[j]->d(), (long long)cl * d, chi));
    env_left(h, P(g.beta[j]), h->tmpA->c(), W1, cl, chi, P(g.beta[j + 1]));
  }
  if (build & BUILD_GAMMA) {
    CK(scale_rows(h->st, h->tmpA->c(), P(g.psi[j + 1]), g.vinv[j]->d(), chi, (long long)d * cr));
    env_right(h, P(g.gamma[j + 1]), h->tmpA->c(), W2, chi, cr, P(g.gamma[j]));
  }
}

// one-site backward update Psi_j <- exp(+i dt/2 H_eff^(1)) Psi_j
void back_update(tdvp_ctx* h, Segment& g, int j, double dt) {
  const int d = h->d, cl = g.cb[j], cr = g.cb[j + 1];
  const MpoSite& W = h->mpo[j];
  const long long n = (long long)cl * d * cr;
  const cplx* Lenv = P(g.beta[j]);
  const cplx* Renv = P(g.gamma[j]);
  CK(copy_cplx(h->st, h->tmpB->c(), P(g.psi[j]), n));
  g_launch_count++;
  const double fl = flops_heff1(cl, cr, d, W.Dl, W.Dr, nnz_of(W));
  {
    const int cx = std::max(cl, cr);
    h->cur_bin = cx <= 128 ? 0 : cx <= 256 ? 1 : cx <= 512 ? 2 : 3;
  }
  const int el0 = h->prm.timing ? ev_record(h) : -1;
  set_heff_masks(h, g, j, 1);
  expm_lanczos(
      h, [&](const cplx* x, cplx* y) { heff1(h, Lenv, W, Renv, cl, cr, x, y); }, h->tmpB->c(), P(g.psi[j]), n, 0.0,
      0.5 * dt, h->prm.krylov_k, 1, fl,
      h->prm.u1 ? fl : flops_heff1_exec(cl, cr, d, W.Dl, W.Dr, nnz_of(W), W.lid, W.rid));
  h->cur_mask[0] = h->cur_mask[1] = nullptr;
  if (el0 >= 0) h->ev_lz1.emplace_back(el0, ev_record(h));
  h->stats.n_back++;
}

// ------------------------------------------------------ one-site TDVP
// Serial 1TDVP, the integrator the hybrid scheme of PAPER.md:697 switches to
// once chi_max is saturated (reading R-1TDVP in DESIGN.md; oracle/tdvp1.py
// step1 is the same algorithm step by step).  Storage stays the paper's
// inverse-canonical product Psi_0 V_0 Psi_1 ...; every
// bond split is the 2TDVP truncated SVD (O-7).

// H_eff^(0) C (bond matrix): y[a, b] = sum L[a, w, a'] R[b, w, b'] x[a', b']
// (the one-site Fig 5b contraction, without a site tensor):
// two DMMA GEMMs, T[(a, w), b'] = L[(a, w), a'] x[a', b'], y = T R^T over (w, b')
void heff0(tdvp_ctx* h, const cplx* Lenv, const cplx* Renv, int D, int cl, int cr, const cplx* x, cplx* y) {
  cplx* T1 = h->T1->c();
  gemm(h, OP_N, OP_N, cl * D, cr, cl, Lenv, cl, x, cr, T1, cr);
  gemm(h, OP_N, OP_T, cl, cr, D * cr, T1, (long long)D * cr, Renv, (long long)D * cr, y, cr);
}

double flops_heff0(int cl, int cr, int D) { return 8.0 * ((double)D * cl * cl * cr + (double)D * cl * cr * cr); }

// forward one-site step Psi_j <- exp(-i t H_eff^(1)) Psi_j
void site_forward(tdvp_ctx* h, Segment& g, int j, double t) {
  const int d = h->d, cl = g.cb[j], cr = g.cb[j + 1];
  const MpoSite& W = h->mpo[j];
  const long long n = (long long)cl * d * cr;
  const cplx* Lenv = P(g.beta[j]);
  const cplx* Renv = P(g.gamma[j]);
  CK(copy_cplx(h->st, h->tmpB->c(), P(g.psi[j]), n));
  g_launch_count++;
  expm_lanczos(
      h, [&](const cplx* x, cplx* y) { heff1(h, Lenv, W, Renv, cl, cr, x, y); }, h->tmpB->c(), P(g.psi[j]), n, 0.0,
      -t, h->prm.krylov_k, 0, flops_heff1(cl, cr, d, W.Dl, W.Dr, nnz_of(W)));
}

// truncated SVD of an m x n matrix into (U S, S W^dag), Lambda / V of bond b
int split_bond(tdvp_ctx* h, Segment& g, int b, const cplx* M, int m, int n, cplx* US, cplx* SWh) {
  TruncParams tp{h->chi_max, h->prm.eps, h->prm.w_max, h->prm.multiplet_delta};
  int chi = 0, r = 0, chi_eps = 0, sweeps = 0;
  double w = 0.0;
  cudaError_t se = svd_truncate_split(h->st, h->sv, M, m, n, tp, US, SWh, g.lam[b]->d(), g.vinv[b]->d(), &chi, &w, &r,
                                      &chi_eps, &sweeps);
  if (se == cudaErrorUnknown) throw TdvpError(TDVP_ENUMERIC, "non-finite or zero spectrum in SVD at bond " + std::to_string(b));
  CK(se);
  g_launch_count += 5;
  if (chi > h->cbmax[b + 1]) throw TdvpError(TDVP_ECUDA, "internal: chi exceeds allocation");
  h->stats.w_step += w;
  h->stats.svd_sweeps_max = std::max(h->stats.svd_sweeps_max, sweeps);
  h->stats.svd_sweeps_total += sweeps;
  if (chi < std::min(chi_eps, r)) h->stats.trunc_active = 1;
  return chi;
}

// one-site interior operations of the p1TDVP programs (schedule.h
// OP_SITE_R / OP_SITE_L / OP_FWD; oracle/tdvp1.py _site_right/_site_left)
// bond matrix C in theta (<= max chi_b^2 <= the two-site buffer), its evolved
// copy C2 in tmpB (free between the environment update and the next site step)
void site_right(tdvp_ctx* h, Segment& g, int j, bool done, double dt) {
  const int d = h->d, K = h->prm.krylov_k;
  const double tau = 0.5 * dt;
  if (!done) site_forward(h, g, j, tau);
  cplx* C = h->theta->c();
  cplx* C2 = h->tmpB->c();
  const int cl = g.cb[j], cr = g.cb[j + 1], cr2 = g.cb[j + 2];
  const MpoSite& W = h->mpo[j];
  // B = diag(V_j) Psi_{j+1} (right-canonical), before V_j is replaced
  CK(scale_rows(h->st, h->tmpA->c(), P(g.psi[j + 1]), g.vinv[j]->d(), cr, (long long)d * cr2));
  CK(copy_cplx(h->st, h->tmpB->c(), P(g.psi[j]), (long long)cl * d * cr));
  g_launch_count += 2;
  const int chi = split_bond(h, g, j, h->tmpB->c(), cl * d, cr, P(g.psi[j]), C);
  g.cb[j + 1] = chi;
  // beta_{j+1} from U = Psi_j diag(V_j)
  CK(scale_cols(h->st, h->tmpB->c(), P(g.psi[j]), g.vinv[j]->d(), (long long)cl * d, chi));
  g_launch_count++;
  env_left(h, P(g.beta[j]), h->tmpB->c(), W, cl, chi, P(g.beta[j + 1]));
  // C <- exp(+i tau H_eff^(0)(beta_{j+1}, gamma_j)) C
  const cplx* Le = P(g.beta[j + 1]);
  const cplx* Re = P(g.gamma[j]);
  expm_lanczos(
      h, [&](const cplx* x, cplx* y) { heff0(h, Le, Re, W.Dr, chi, cr, x, y); }, C, C2, (long long)chi * cr, 0.0,
      tau, K, 0, flops_heff0(chi, cr, W.Dr));
  // Psi_{j+1} = C B
  gemm(h, OP_N, OP_N, chi, d * cr2, cr, C2, cr, h->tmpA->c(), (long long)d * cr2, P(g.psi[j + 1]),
       (long long)d * cr2);
}

void site_left(tdvp_ctx* h, Segment& g, int j, bool done, double dt) {
  const int d = h->d, K = h->prm.krylov_k;
  const double tau = 0.5 * dt;
  if (!done) site_forward(h, g, j, tau);
  cplx* C = h->theta->c();
  cplx* C2 = h->tmpB->c();
  const int cl2 = g.cb[j - 1], cl = g.cb[j], cr = g.cb[j + 1];
  const MpoSite& W = h->mpo[j];
  // A = Psi_{j-1} diag(V_{j-1}) (left-canonical), before V_{j-1} is replaced
  CK(scale_cols(h->st, h->tmpA->c(), P(g.psi[j - 1]), g.vinv[j - 1]->d(), (long long)cl2 * d, cl));
  CK(copy_cplx(h->st, h->tmpB->c(), P(g.psi[j]), (long long)cl * d * cr));
  g_launch_count += 2;
  const int chi = split_bond(h, g, j - 1, h->tmpB->c(), cl, d * cr, C, P(g.psi[j]));
  g.cb[j] = chi;
  // gamma_{j-1} from W^dag = diag(V_{j-1}) Psi_j
  CK(scale_rows(h->st, h->tmpB->c(), P(g.psi[j]), g.vinv[j - 1]->d(), chi, (long long)d * cr));
  g_launch_count++;
  env_right(h, P(g.gamma[j]), h->tmpB->c(), W, chi, cr, P(g.gamma[j - 1]));
  // C <- exp(+i tau H_eff^(0)(beta_j, gamma_{j-1})) C
  const cplx* Le = P(g.beta[j]);
  const cplx* Re = P(g.gamma[j - 1]);
  expm_lanczos(
      h, [&](const cplx* x, cplx* y) { heff0(h, Le, Re, W.Dl, cl, chi, x, y); }, C, C2, (long long)cl * chi, 0.0,
      tau, K, 0, flops_heff0(cl, chi, W.Dl));
  // Psi_{j-1} = A C
  gemm(h, OP_N, OP_N, cl2 * d, chi, cl, h->tmpA->c(), cl, C2, chi, P(g.psi[j - 1]), chi);
}

// hybrid switch rule: every bond at min(chi_max, d^(j+1), d^(L-j-1))
int owner_of(tdvp_ctx* h, int j);
bool chi_saturated(tdvp_ctx* h) {
  for (int j = 0; j + 1 < h->L; ++j) {
    long long cap = 1;
    const int k = std::min(j + 1, h->L - j - 1);
    for (int i = 0; i < k && cap < h->chi_max; ++i) cap *= h->d;
    if (h->segs[owner_of(h, j)].cb[j + 1] < std::min<long long>(cap, h->chi_max)) return false;
  }
  return true;
}

// ------------------------------------------------------------ layout / init
void alloc_segment(tdvp_ctx* h, Segment& g, int q, int s, int e, int dev) {
  const int L = h->L, d = h->d;
  DeviceGuard dg(dev);
  g.dev = dev;
  g.q = q;
  g.s = s;
  g.e = e;
  g.cb.assign(L + 1, 1);
  g.psi.clear();
  g.beta.clear();
  g.gamma.clear();
  g.lam.clear();
  g.vinv.clear();
  g.psi.resize(L);
  g.beta.resize(L);
  g.gamma.resize(L);
  g.lam.resize(L - 1);
  g.vinv.resize(L - 1);
  const int hi = std::min(e + 1, L - 1);
  for (int j = s; j <= hi; ++j) {
    g.psi[j] = make_buf((size_t)h->cbmax[j] * d * h->cbmax[j + 1] * sizeof(cplx));
    g.beta[j] = make_buf((size_t)h->cbmax[j] * h->mpo[j].Dl * h->cbmax[j] * sizeof(cplx));
    g.gamma[j] = make_buf((size_t)h->cbmax[j + 1] * h->mpo[j].Dr * h->cbmax[j + 1] * sizeof(cplx));
  }
  for (int b = std::max(s - 1, 0); b <= std::min(e, L - 2); ++b) {
    g.lam[b] = make_buf((size_t)h->cbmax[b + 1] * sizeof(double));
    g.vinv[b] = make_buf((size_t)h->cbmax[b + 1] * sizeof(double));
  }
}

__global__ void recip_kernel(const double* lam, double* vinv, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) vinv[i] = 1.0 / lam[i];
}

// owner segment of site j (single-process layout)
int owner_of(tdvp_ctx* h, int j) {
  for (size_t q = 0; q < h->bounds.size(); ++q)
    if (j >= h->bounds[q].first && j <= h->bounds[q].second) return (int)q;
  return -1;
}
bool local_mode(tdvp_ctx* h) { return h->world == 1; }

// device of segment q in a p-segment layout: contiguous groups of segments per
// device (neighbouring segments share a device when p > n_devices)
int seg_device(tdvp_ctx* h, int q, int p) {
  if (!h->multi_dev || h->devs.empty()) return h->dev;
  const int n = (int)h->devs.size();
  return h->devs[std::min(n - 1, (int)((long long)q * n / p))];
}

tdvp_ctx* lane_of(tdvp_ctx* h, int q);

// upload the full host MPS copy into the current layout
void upload_state(tdvp_ctx* h) {
  const int L = h->L;
  for (auto& g : h->segs) {
    // the segment's own device and a stream of it (its lane's, when on another device)
    DeviceGuard dg(g.dev);
    cudaStream_t st = g.dev == h->dev ? h->st : lane_of(h, g.q)->st;
    g.cb = h->h_chi;
    if (h->prm.u1) {
      if ((int)h->h_q.size() != L + 1) h->h_q = infer_charges(h);
      g.qb = h->h_q;
    } else {
      g.qb.clear();
    }
    const int hi = std::min(g.e + 1, L - 1);
    for (int j = g.s; j <= hi; ++j)
      CK(cudaMemcpyAsync(g.psi[j]->p, h->h_psi[j].data(), h->h_psi[j].size() * sizeof(double), cudaMemcpyHostToDevice,
                         st));
    for (int b = std::max(g.s - 1, 0); b <= std::min(g.e, L - 2); ++b) {
      CK(cudaMemcpyAsync(g.lam[b]->p, h->h_lam[b].data(), h->h_lam[b].size() * sizeof(double),
                         cudaMemcpyHostToDevice, st));
      const int n = (int)h->h_lam[b].size();
      recip_kernel<<<(n + 255) / 256, 256, 0, st>>>(g.lam[b]->d(), g.vinv[b]->d(), n);
      CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(st));
  }
  CK(cudaStreamSynchronize(h->st));
}

// download owner copies into the host MPS copy
void download_state(tdvp_ctx* h) {
  const int L = h->L, d = h->d;
  if (!local_mode(h)) throw TdvpError(TDVP_ESTATE, "state download across ranks is not supported");
  std::vector<int> chi(L + 1, 1);
  for (int b = 0; b < L - 1; ++b) chi[b + 1] = h->segs[owner_of(h, b)].cb[b + 1];  // left owner owns bond b
  h->h_chi = chi;
  CK(cudaStreamSynchronize(h->st));  // every lane's work was joined into h->st by the step
  if (h->prm.u1 && !h->segs.empty() && !h->segs[0].qb.empty()) h->h_q = assemble_charges(h);
  for (int j = 0; j < L; ++j) {
    Segment& g = h->segs[owner_of(h, j)];
    const size_t n = (size_t)chi[j] * d * chi[j + 1] * 2;
    h->h_psi[j].resize(n);
    DeviceGuard dg(g.dev);
    CK(cudaMemcpy(h->h_psi[j].data(), g.psi[j]->p, n * sizeof(double), cudaMemcpyDeviceToHost));
  }
  for (int b = 0; b < L - 1; ++b) {
    Segment& g = h->segs[owner_of(h, b)];
    h->h_lam[b].resize(chi[b + 1]);
    DeviceGuard dg(g.dev);
    CK(cudaMemcpy(h->h_lam[b].data(), g.lam[b]->p, chi[b + 1] * sizeof(double), cudaMemcpyDeviceToHost));
  }
}

// Sequential initial environments (O-2) from the host
// MPS copy: beta_{j+1} = env_left(beta_j, Psi_j V_j, W_j),
// gamma_{j-1} = env_right(gamma_j, V_{j-1} Psi_j, W_j), stored wherever held.
void build_envs(tdvp_ctx* h) {
  const int L = h->L, d = h->d;
  const std::vector<int>& chi = h->h_chi;
  bool on_lead = local_mode(h);
  for (const auto& g : h->segs) on_lead = on_lead && g.dev == h->dev;
  if (on_lead) {
    // every segment on this handle's device: the state was just uploaded
    // (upload_state), so the chains read the owners' device tensors -- no
    // second host upload, no host synchronisation per site
    const cplx one = ONE;
    cplx* cur = h->envA->c();
    cplx* nxt = h->envB->c();
    auto store = [&](bool left, int j, const cplx* src, long long n) {
      for (auto& g : h->segs) {
        const BufPtr& b = left ? g.beta[j] : g.gamma[j];
        if (b) CK(cudaMemcpyAsync(b->p, src, n * sizeof(cplx), cudaMemcpyDeviceToDevice, h->st));
      }
    };
    CK(cudaMemcpyAsync(cur, &one, sizeof(cplx), cudaMemcpyHostToDevice, h->st));
    store(true, 0, cur, 1);
    // serial layout: every step, DMRG sweep and 1TDVP step starts with a
    // left-to-right sweep, which rebuilds beta_1..beta_{L-1} as it goes
    // (the initial envs a sweep needs are the ones ahead of it)
    const int left_end = h->layout_p == 1 ? 0 : L - 1;
    for (int j = 0; j < left_end; ++j) {
      const Segment& o = h->segs[owner_of(h, j)];
      CK(scale_cols(h->st, h->tmpA->c(), P(o.psi[j]), o.vinv[j]->d(), (long long)chi[j] * d, chi[j + 1]));
      env_left(h, cur, h->tmpA->c(), h->mpo[j], chi[j], chi[j + 1], nxt);
      std::swap(cur, nxt);
      store(true, j + 1, cur, (long long)chi[j + 1] * h->mpo[j].Dr * chi[j + 1]);
    }
    cur = h->envA->c();
    nxt = h->envB->c();
    CK(cudaMemcpyAsync(cur, &one, sizeof(cplx), cudaMemcpyHostToDevice, h->st));
    store(false, L - 1, cur, 1);
    for (int j = L - 1; j > 0; --j) {
      const Segment& o = h->segs[owner_of(h, j)];
      CK(scale_rows(h->st, h->tmpA->c(), P(o.psi[j]), o.vinv[j - 1]->d(), chi[j], (long long)d * chi[j + 1]));
      env_right(h, cur, h->tmpA->c(), h->mpo[j], chi[j], chi[j + 1], nxt);
      std::swap(cur, nxt);
      store(false, j - 1, cur, (long long)chi[j] * h->mpo[j].Dl * chi[j]);
    }
    CK(cudaStreamSynchronize(h->st));
    return;
  }
  // scratch: running env (envA/envB ping-pong), site tensor upload (T2 reused), scaled tensor (tmpA)
  DevBuf psi_tmp, lam_tmp, vinv_tmp;
  psi_tmp.alloc((size_t)h->n1max * sizeof(cplx));
  lam_tmp.alloc((size_t)h->chi_max * sizeof(double) + 64);
  vinv_tmp.alloc((size_t)h->chi_max * sizeof(double) + 64);
  auto upload_site = [&](int j) {
    CK(cudaMemcpyAsync(psi_tmp.p, h->h_psi[j].data(), h->h_psi[j].size() * sizeof(double), cudaMemcpyHostToDevice,
                       h->st));
  };
  auto upload_bond = [&](int b) {
    const int n = (int)h->h_lam[b].size();
    CK(cudaMemcpyAsync(lam_tmp.p, h->h_lam[b].data(), n * sizeof(double), cudaMemcpyHostToDevice, h->st));
    recip_kernel<<<(n + 255) / 256, 256, 0, h->st>>>(lam_tmp.d(), vinv_tmp.d(), n);
    CK(cudaGetLastError());
  };
  const cplx one = ONE;
  // left chain
  cplx* cur = h->envA->c();
  cplx* nxt = h->envB->c();
  CK(cudaMemcpyAsync(cur, &one, sizeof(cplx), cudaMemcpyHostToDevice, h->st));
  auto store = [&](bool left, int j, const cplx* src, long long n) {
    for (auto& g : h->segs) {
      const BufPtr& b = left ? g.beta[j] : g.gamma[j];
      if (b) d2d(b->p, g.dev, src, h->dev, n * sizeof(cplx), h->st);
    }
  };
  store(true, 0, cur, 1);
  for (int j = 0; j < L - 1; ++j) {
    upload_site(j);
    upload_bond(j);
    CK(scale_cols(h->st, h->tmpA->c(), psi_tmp.c(), vinv_tmp.d(), (long long)chi[j] * d, chi[j + 1]));
    env_left(h, cur, h->tmpA->c(), h->mpo[j], chi[j], chi[j + 1], nxt);
    std::swap(cur, nxt);
    store(true, j + 1, cur, (long long)chi[j + 1] * h->mpo[j].Dr * chi[j + 1]);
    CK(cudaStreamSynchronize(h->st));  // host tmp buffers are reused
  }
  cur = h->envA->c();
  nxt = h->envB->c();
  CK(cudaMemcpyAsync(cur, &one, sizeof(cplx), cudaMemcpyHostToDevice, h->st));
  store(false, L - 1, cur, 1);
  for (int j = L - 1; j > 0; --j) {
    upload_site(j);
    upload_bond(j - 1);
    CK(scale_rows(h->st, h->tmpA->c(), psi_tmp.c(), vinv_tmp.d(), chi[j], (long long)d * chi[j + 1]));
    env_right(h, cur, h->tmpA->c(), h->mpo[j], chi[j], chi[j + 1], nxt);
    std::swap(cur, nxt);
    store(false, j - 1, cur, (long long)chi[j] * h->mpo[j].Dl * chi[j]);
    CK(cudaStreamSynchronize(h->st));
  }
  CK(cudaStreamSynchronize(h->st));
}

void layout(tdvp_ctx* h, int p) {
  std::vector<std::pair<int, int>> b;
  std::string err;
  if ((int)h->custom.size() == p && p > 1) b = h->custom;
  else if (!plan_partition(h->L, p, b, err)) throw TdvpError(TDVP_EPARTITION, err);
  if (!local_mode(h) && p != h->world)
    throw TdvpError(TDVP_EPARTITION, "n_segments must equal the world size in multi-process mode");
  if (h->layout_p != 0 && h->have_mps && local_mode(h)) download_state(h);  // keep the current state
  if (h->layout_p != 0 && !local_mode(h) && h->evolved)
    throw TdvpError(TDVP_ESTATE,
                    "re-layout of an evolved state is not supported in multi-process mode (each rank holds only its "
                    "segment); call tdvp_set_mps first");
  if (h->alloc_p != p || h->segs.empty() || h->bounds != b) {
    // (re)allocate; the same partition reuses its buffers (a new state from
    // tdvp_set_mps is uploaded into them: no cudaMalloc/cudaFree per call)
    h->segs.clear();
    h->bounds = b;
    if (local_mode(h)) {
      h->segs.resize(p);
      for (int q = 0; q < p; ++q) alloc_segment(h, h->segs[q], q, b[q].first, b[q].second, seg_device(h, q, p));
    } else {
      h->segs.resize(1);
      alloc_segment(h, h->segs[0], h->rank, b[h->rank].first, b[h->rank].second, h->dev);
    }
    h->msg_r.clear();
    h->msg_l.clear();
    h->alloc_p = p;
  }
  h->layout_p = p;
  upload_state(h);
  build_envs(h);
  h->envs_valid = true;
}

// ------------------------------------------------------------ exchanges
// local mode: copy boundary data between segments (device to device)
void copy_buf(tdvp_ctx* h, const BufPtr& dst, const BufPtr& src, size_t bytes) {
  CK(cudaMemcpyAsync(dst->p, src->p, bytes, cudaMemcpyDeviceToDevice, h->st));
}

// SEND_R: Psi'_{e+1}, Lambda'_e (and V), beta_{e+1} from q to q+1
void send_right_local(tdvp_ctx* h, Segment& a, Segment& b) {
  const int e = a.e, d = h->d;
  const int chi = a.cb[e + 1], cr = a.cb[e + 2];
  b.cb[e + 1] = chi;
  if (h->prm.u1) b.qb[e + 1] = a.qb[e + 1];
  copy_buf(h, b.psi[e + 1], a.psi[e + 1], (size_t)chi * d * cr * sizeof(cplx));
  copy_buf(h, b.lam[e], a.lam[e], (size_t)chi * sizeof(double));
  copy_buf(h, b.vinv[e], a.vinv[e], (size_t)chi * sizeof(double));
  copy_buf(h, b.beta[e + 1], a.beta[e + 1], (size_t)chi * h->mpo[e + 1].Dl * chi * sizeof(cplx));
}
// SEND_L: Psi_s, gamma_s from q to q-1
void send_left_local(tdvp_ctx* h, Segment& b, Segment& a) {
  const int s = b.s, d = h->d;
  const int cl = b.cb[s], cr = b.cb[s + 1];
  a.cb[s + 1] = cr;
  a.cb[s] = cl;
  if (h->prm.u1) a.qb[s + 1] = b.qb[s + 1];
  copy_buf(h, a.psi[s], b.psi[s], (size_t)cl * d * cr * sizeof(cplx));
  copy_buf(h, a.gamma[s], b.gamma[s], (size_t)cr * h->mpo[s].Dr * cr * sizeof(cplx));
}

// NCCL mode
// The header (chi) is host-known on the sender: stream-ordered, no host
// synchronisation (a pageable-memory H2D copy has consumed `v` when it
// returns; the next header's copy is ordered after this send on the stream).
// The receiver needs chi on the host to size its receives, so it waits.
void nccl_send_ints(tdvp_ctx* h, const int* v, int n, int peer) {
  CK(cudaMemcpyAsync(h->hdr->p, v, n * sizeof(int), cudaMemcpyHostToDevice, h->st));
  NK(nccl().Send(h->hdr->p, n, ncclInt32, peer, h->comm, h->st));
}
void nccl_recv_ints(tdvp_ctx* h, int* v, int n, int peer) {
  NK(nccl().Recv(h->hdr->p, n, ncclInt32, peer, h->comm, h->st));
  CK(cudaMemcpyAsync(v, h->hdr->p, n * sizeof(int), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
}
void send_right_nccl(tdvp_ctx* h, Segment& a) {
  const int e = a.e, d = h->d, peer = a.q + 1;
  const int chi = a.cb[e + 1], cr = a.cb[e + 2];
  int hd[2] = {chi, cr};
  nccl_send_ints(h, hd, 2, peer);
  NK(nccl().GroupStart());
  NK(nccl().Send(a.psi[e + 1]->p, (size_t)chi * d * cr * 2, ncclFloat64, peer, h->comm, h->st));
  NK(nccl().Send(a.lam[e]->p, (size_t)chi, ncclFloat64, peer, h->comm, h->st));
  NK(nccl().Send(a.beta[e + 1]->p, (size_t)chi * h->mpo[e + 1].Dl * chi * 2, ncclFloat64, peer, h->comm, h->st));
  NK(nccl().GroupEnd());
}
void recv_left_nccl(tdvp_ctx* h, Segment& b) {
  const int s = b.s, d = h->d, peer = b.q - 1;
  int hd[2];
  nccl_recv_ints(h, hd, 2, peer);
  const int chi = hd[0], cr = hd[1];
  b.cb[s] = chi;
  b.cb[s + 1] = cr;
  NK(nccl().GroupStart());
  NK(nccl().Recv(b.psi[s]->p, (size_t)chi * d * cr * 2, ncclFloat64, peer, h->comm, h->st));
  NK(nccl().Recv(b.lam[s - 1]->p, (size_t)chi, ncclFloat64, peer, h->comm, h->st));
  NK(nccl().Recv(b.beta[s]->p, (size_t)chi * h->mpo[s].Dl * chi * 2, ncclFloat64, peer, h->comm, h->st));
  NK(nccl().GroupEnd());
  recip_kernel<<<(chi + 255) / 256, 256, 0, h->st>>>(b.lam[s - 1]->d(), b.vinv[s - 1]->d(), chi);
  CK(cudaGetLastError());
}
void send_left_nccl(tdvp_ctx* h, Segment& b) {
  const int s = b.s, d = h->d, peer = b.q - 1;
  const int cl = b.cb[s], cr = b.cb[s + 1];
  int hd[2] = {cl, cr};
  nccl_send_ints(h, hd, 2, peer);
  NK(nccl().GroupStart());
  NK(nccl().Send(b.psi[s]->p, (size_t)cl * d * cr * 2, ncclFloat64, peer, h->comm, h->st));
  NK(nccl().Send(b.gamma[s]->p, (size_t)cr * h->mpo[s].Dr * cr * 2, ncclFloat64, peer, h->comm, h->st));
  NK(nccl().GroupEnd());
}
void recv_right_nccl(tdvp_ctx* h, Segment& a) {
  const int e = a.e, d = h->d, peer = a.q + 1;
  int hd[2];
  nccl_recv_ints(h, hd, 2, peer);
  const int cl = hd[0], cr = hd[1];
  a.cb[e + 1] = cl;
  a.cb[e + 2] = cr;
  NK(nccl().GroupStart());
  NK(nccl().Recv(a.psi[e + 1]->p, (size_t)cl * d * cr * 2, ncclFloat64, peer, h->comm, h->st));
  NK(nccl().Recv(a.gamma[e + 1]->p, (size_t)cr * h->mpo[e + 1].Dr * cr * 2, ncclFloat64, peer, h->comm, h->st));
  NK(nccl().GroupEnd());
}

void exec_compute(tdvp_ctx* h, Segment& g, const SchedOp& op, double dt) {
  if (op.kind == OP_PAIR) pair_update(h, g, op.j, dt, op.full, op.build);
  else if (op.kind == OP_BACK) back_update(h, g, op.j, dt);
  else if (op.kind == OP_SITE_R) site_right(h, g, op.j, op.full != 0, dt);
  else if (op.kind == OP_SITE_L) site_left(h, g, op.j, op.full != 0, dt);
  else if (op.kind == OP_FWD) site_forward(h, g, op.j, op.full ? dt : 0.5 * dt);
}

// the program of segment q in half hh of the step in progress (p2TDVP, or
// p1TDVP when h->one_site)
std::vector<SchedOp> program_of(tdvp_ctx* h, int hh, int q, const std::set<int>& merged) {
  const int L = h->L, p = h->layout_p;
  return h->one_site ? segment_program1(L, p, hh, q, h->bounds[q], merged, h->msites)
                     : segment_program(L, p, hh, q, h->bounds[q], merged);
}

// one half-step
void run_half(tdvp_ctx* h, int hh, double dt, const std::set<int>& merged) {
  const int L = h->L, p = h->layout_p;
  if (!local_mode(h)) {
    Segment& g = h->segs[0];
    for (const SchedOp& op : program_of(h, hh, g.q, merged)) {
      switch (op.kind) {
        case OP_SEND_R: send_right_nccl(h, g); break;
        case OP_RECV_L: recv_left_nccl(h, g); break;
        case OP_SEND_L: send_left_nccl(h, g); break;
        case OP_RECV_R: recv_right_nccl(h, g); break;
        default: exec_compute(h, g, op, dt);
      }
    }
    return;
  }
  // single process: cooperative round-robin executor over the segment
  // programs; a SEND copies immediately, a RECV waits for its message.
  std::vector<std::vector<SchedOp>> prog(p);
  std::vector<size_t> pc(p, 0);
  std::vector<int> msg_from_left(p, 0), msg_from_right(p, 0);
  for (int q = 0; q < p; ++q) prog[q] = program_of(h, hh, q, merged);
  size_t done = 0;
  while (done < (size_t)p) {
    bool progress = false;
    done = 0;
    for (int q = 0; q < p; ++q) {
      while (pc[q] < prog[q].size()) {
        const SchedOp& op = prog[q][pc[q]];
        Segment& g = h->segs[q];
        if (op.kind == OP_RECV_L) {
          if (!msg_from_left[q]) break;
          msg_from_left[q]--;
        } else if (op.kind == OP_RECV_R) {
          if (!msg_from_right[q]) break;
          msg_from_right[q]--;
        } else if (op.kind == OP_SEND_R) {
          send_right_local(h, g, h->segs[q + 1]);
          msg_from_left[q + 1]++;
        } else if (op.kind == OP_SEND_L) {
          send_left_local(h, g, h->segs[q - 1]);
          msg_from_right[q - 1]++;
        } else {
          exec_compute(h, g, op, dt);
        }
        pc[q]++;
        progress = true;
      }
      if (pc[q] == prog[q].size()) done++;
    }
    if (done < (size_t)p && !progress) throw TdvpError(TDVP_ECUDA, "internal: schedule deadlock");
  }
}

// ------------------------------------------------------------ segment lanes
void alloc_workspace(tdvp_ctx* h);

void build_mpo_tables(std::vector<MpoSite>& mpo, int L, int d, const std::vector<int>& D,
                      const std::vector<std::vector<cplx>>& W);

// lane q (1..p-1): own host thread, stream and workspace, on the device of
// segment q.  In a multi-device handle every lane also holds its own copy of
// the MPO tables (device pointers) on its device; a lane whose device no
// longer matches the layout is rebuilt.
tdvp_ctx* lane_of(tdvp_ctx* h, int q) {
  if (q == 0) return h;
  const int p = std::max(h->layout_p, q + 1);
  const int want = seg_device(h, q, p);
  if ((int)h->lanes.size() >= q && h->lanes[q - 1]->dev != want) {
    CK(cudaStreamSynchronize(h->lanes[q - 1]->st));
    h->lanes.resize(q - 1);  // rebuild this lane and the later ones
  }
  while ((int)h->lanes.size() < q) {
    const int lq = (int)h->lanes.size() + 1;
    const int ldev = seg_device(h, lq, p);
    DeviceGuard dg(ldev);
    std::unique_ptr<tdvp_ctx> ln(new tdvp_ctx(h, h->multi_dev));
    ln->L = h->L;
    ln->d = h->d;
    ln->Dmpo = h->Dmpo;
    ln->chi_max = h->chi_max;
    ln->cbmax = h->cbmax;
    ln->dev = ldev;
    CK(cudaStreamCreateWithFlags(&ln->st, cudaStreamNonBlocking));
    alloc_workspace(ln.get());
    if (h->multi_dev) {
      CK(cudaMalloc(&ln->lz.brk_count, 64));
      ln->lz_brk_own.reset(new DevBuf());
      ln->lz_brk_own->p = ln->lz.brk_count;
      ln->lz_brk_own->bytes = 64;
      CK(cudaMemset(ln->lz.brk_count, 0, 64));
      if (h->have_mpo) build_mpo_tables(ln->mpo_own, h->L, h->d, h->h_D, h->h_W);
    } else {
      ln->lz.brk_count = h->lz_brk->i();  // one breakdown counter per handle
    }
    CK(cudaEventCreate(&ln->sv.ev_jac[0]));
    CK(cudaEventCreate(&ln->sv.ev_jac[1]));
    h->lanes.push_back(std::move(ln));
  }
  return h->lanes[q - 1].get();
}

// staging buffers for the boundary messages of the current layout
void alloc_msgs(tdvp_ctx* h) {
  const int p = h->layout_p, d = h->d;
  h->msg_r.clear();
  h->msg_l.clear();
  h->msg_r.resize(p);
  h->msg_l.resize(p);
  // staging buffers on the RECEIVER's device (the sender's copy crosses
  // NVLink); `posted` recorded by the sender's stream, `consumed` by the
  // receiver's, each created on its recording device
  auto mk = [&](std::unique_ptr<LaneMsg>& m, int sdev, int rdev, size_t psi, size_t lam, size_t env) {
    m.reset(new LaneMsg());
    m->sdev = sdev;
    m->rdev = rdev;
    {
      DeviceGuard dg(sdev);
      CK(cudaEventCreateWithFlags(&m->posted, cudaEventDisableTiming));
    }
    DeviceGuard dg(rdev);
    CK(cudaEventCreateWithFlags(&m->consumed, cudaEventDisableTiming));
    m->psi = make_buf(psi * sizeof(cplx));
    m->env = make_buf(env * sizeof(cplx));
    if (lam) {
      m->lam = make_buf(lam * sizeof(double));
      m->vinv = make_buf(lam * sizeof(double));
    }
  };
  for (int q = 0; q < p; ++q) {
    const int s = h->bounds[q].first, e = h->bounds[q].second;
    if (q + 1 < p) {
      const size_t c1 = h->cbmax[e + 1], c2 = h->cbmax[e + 2];
      mk(h->msg_r[q], h->segs[q].dev, h->segs[q + 1].dev, c1 * d * c2, c1, c1 * h->mpo[e + 1].Dl * c1);
    }
    if (q > 0) {
      const size_t c0 = h->cbmax[s], c1 = h->cbmax[s + 1];
      mk(h->msg_l[q], h->segs[q].dev, h->segs[q - 1].dev, c0 * d * c1, 0, c1 * h->mpo[s].Dr * c1);
    }
  }
}

void lane_wait(LaneMsg& m, int want, const std::atomic<bool>& abort) {
  std::unique_lock<std::mutex> lk(m.m);
  m.cv.wait(lk, [&] { return m.ready == want || abort.load(); });
  if (m.ready != want) throw TdvpError(TDVP_ECUDA, "segment lane aborted");
}
void lane_post(LaneMsg& m, int ready, bool consumed) {
  {
    std::lock_guard<std::mutex> lk(m.m);
    m.ready = ready;
    if (consumed) m.consumed_rec = true;
  }
  m.cv.notify_all();
}
void lane_copy(tdvp_ctx* ln, void* dst, const void* src, size_t bytes) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ln->st));
}

// SEND_R / RECV_L: Psi'_{e+1}, Lambda'_e, V_e, beta_{e+1}
void lane_send_right(tdvp_ctx* ln, Segment& a, LaneMsg& m, const std::atomic<bool>& abort) {
  lane_wait(m, 0, abort);
  if (m.consumed_rec) CK(cudaStreamWaitEvent(ln->st, m.consumed, 0));
  const int e = a.e, d = ln->d, chi = a.cb[e + 1], cr = a.cb[e + 2];
  d2d(m.psi->p, m.rdev, a.psi[e + 1]->p, m.sdev, (size_t)chi * d * cr * sizeof(cplx), ln->st);
  d2d(m.lam->p, m.rdev, a.lam[e]->p, m.sdev, (size_t)chi * sizeof(double), ln->st);
  d2d(m.vinv->p, m.rdev, a.vinv[e]->p, m.sdev, (size_t)chi * sizeof(double), ln->st);
  d2d(m.env->p, m.rdev, a.beta[e + 1]->p, m.sdev, (size_t)chi * ln->mpo[e + 1].Dl * chi * sizeof(cplx), ln->st);
  CK(cudaEventRecord(m.posted, ln->st));
  m.meta[0] = chi;
  m.meta[1] = cr;
  if (ln->prm.u1) m.q = a.qb[e + 1];
  lane_post(m, 1, false);
}
void lane_recv_left(tdvp_ctx* ln, Segment& b, LaneMsg& m, const std::atomic<bool>& abort) {
  lane_wait(m, 1, abort);
  CK(cudaStreamWaitEvent(ln->st, m.posted, 0));
  const int e = b.s - 1, d = ln->d, chi = m.meta[0], cr = m.meta[1];
  b.cb[e + 1] = chi;
  if (ln->prm.u1) b.qb[e + 1] = m.q;
  lane_copy(ln, b.psi[e + 1]->p, m.psi->p, (size_t)chi * d * cr * sizeof(cplx));
  lane_copy(ln, b.lam[e]->p, m.lam->p, (size_t)chi * sizeof(double));
  lane_copy(ln, b.vinv[e]->p, m.vinv->p, (size_t)chi * sizeof(double));
  lane_copy(ln, b.beta[e + 1]->p, m.env->p, (size_t)chi * ln->mpo[e + 1].Dl * chi * sizeof(cplx));
  CK(cudaEventRecord(m.consumed, ln->st));
  lane_post(m, 0, true);
}
// SEND_L / RECV_R: Psi_s, gamma_s
void lane_send_left(tdvp_ctx* ln, Segment& b, LaneMsg& m, const std::atomic<bool>& abort) {
  lane_wait(m, 0, abort);
  if (m.consumed_rec) CK(cudaStreamWaitEvent(ln->st, m.consumed, 0));
  const int s = b.s, d = ln->d, cl = b.cb[s], cr = b.cb[s + 1];
  d2d(m.psi->p, m.rdev, b.psi[s]->p, m.sdev, (size_t)cl * d * cr * sizeof(cplx), ln->st);
  d2d(m.env->p, m.rdev, b.gamma[s]->p, m.sdev, (size_t)cr * ln->mpo[s].Dr * cr * sizeof(cplx), ln->st);
  CK(cudaEventRecord(m.posted, ln->st));
  m.meta[0] = cl;
  m.meta[1] = cr;
  if (ln->prm.u1) m.q = b.qb[s + 1];
  lane_post(m, 1, false);
}
void lane_recv_right(tdvp_ctx* ln, Segment& a, LaneMsg& m, const std::atomic<bool>& abort) {
  lane_wait(m, 1, abort);
  CK(cudaStreamWaitEvent(ln->st, m.posted, 0));
  const int s = a.e + 1, d = ln->d, cl = m.meta[0], cr = m.meta[1];
  a.cb[s] = cl;
  a.cb[s + 1] = cr;
  if (ln->prm.u1) a.qb[s + 1] = m.q;
  lane_copy(ln, a.psi[s]->p, m.psi->p, (size_t)cl * d * cr * sizeof(cplx));
  lane_copy(ln, a.gamma[s]->p, m.env->p, (size_t)cr * ln->mpo[s].Dr * cr * sizeof(cplx));
  CK(cudaEventRecord(m.consumed, ln->st));
  lane_post(m, 0, true);
}

void reset_step_stats(tdvp_ctx* h) {
  h->stats.w_step = 0.0;
  h->stats.trunc_active = 0;
  h->stats.n_pair = h->stats.n_back = 0;
  h->stats.svd_sweeps_max = 0;
  h->stats.svd_sweeps_total = 0;
  h->stats.svd_jac_ms = h->stats.svd_jac_flop = 0.0;
  h->stats.svd_bj_ms = h->stats.svd_bj_flop = 0.0;
  h->stats.svd_bj_calls = 0;
  h->stats.heff2_flop = h->stats.heff1_flop = 0.0;
  h->stats.heff2_flop_exec = h->stats.heff1_flop_exec = 0.0;
  h->stats.heff2_calls = 0;
  h->stats.lz_vec_bytes = 0.0;
  for (int i = 0; i < 4; ++i) h->stats.heff2_ms_bin[i] = h->stats.heff2_flop_bin[i] = 0.0;
  for (int i = 0; i < 4; ++i) h->stats.lz_ms_bin[i] = h->stats.lz_bytes_bin[i] = 0.0;
  h->ev_lzrec.clear();
  h->ev_used = 0;
  h->ev_h2.clear();
  h->ev_h2_bin.clear();
  h->ev_h1.clear();
  h->ev_svd.clear();
  h->ev_lz2.clear();
  h->ev_lz1.clear();
  h->ev_env.clear();
}

// both half-steps of segment q on its lane (the per-rank program of the NCCL
// executor, with lane messages in place of send/recv)
void lane_program(tdvp_ctx* h, int q, double dt, const std::set<int>& merged, const std::atomic<bool>& abort) {
  tdvp_ctx* ln = q == 0 ? h : h->lanes[q - 1].get();
  Segment& g = h->segs[q];
  const int L = h->L, p = h->layout_p;
  for (int hh = 1; hh <= 2; ++hh)
    for (const SchedOp& op : program_of(h, hh, q, merged)) {
      if (abort.load()) throw TdvpError(TDVP_ECUDA, "segment lane aborted");
      switch (op.kind) {
        case OP_SEND_R: lane_send_right(ln, g, *h->msg_r[q], abort); break;
        case OP_RECV_L: lane_recv_left(ln, g, *h->msg_r[q - 1], abort); break;
        case OP_SEND_L: lane_send_left(ln, g, *h->msg_l[q], abort); break;
        case OP_RECV_R: lane_recv_right(ln, g, *h->msg_l[q + 1], abort); break;
        default: exec_compute(ln, g, op, dt);
      }
    }
}

// one step with p concurrent lanes; the caller recorded ev_step0 on h->st
void run_step_lanes(tdvp_ctx* h, double dt, const std::set<int>& merged) {
  const int p = h->layout_p;
  h->sv.throughput = 1;
  for (int q = 1; q < p; ++q) {
    tdvp_ctx* ln = lane_of(h, q);
    ln->sv.throughput = 1;
    ln->prm = h->prm;
    reset_step_stats(ln);
    CK(cudaStreamWaitEvent(ln->st, h->ev_step0, 0));
  }
  std::atomic<bool> abort{false};
  std::vector<std::exception_ptr> errs(p);
  auto body = [&](int q) {
    try {
      // lanes were created (and their devices checked) above, on this thread:
      // the workers only read h->lanes
      CK(cudaSetDevice(q == 0 ? h->dev : h->lanes[q - 1]->dev));
      lane_program(h, q, dt, merged, abort);
    } catch (...) {
      errs[q] = std::current_exception();
      abort.store(true);
      for (auto* v : {&h->msg_r, &h->msg_l})
        for (auto& m : *v)
          if (m) {
            std::lock_guard<std::mutex> lk(m->m);
            m->cv.notify_all();
          }
    }
  };
  std::vector<std::thread> th;
  th.reserve(p - 1);
  for (int q = 1; q < p; ++q) th.emplace_back(body, q);
  body(0);
  for (auto& t : th) t.join();
  for (int q = 0; q < p; ++q)
    if (errs[q]) {
      for (int r = 1; r < p; ++r) cudaStreamSynchronize(h->lanes[r - 1]->st);
      for (auto* v : {&h->msg_r, &h->msg_l})
        for (auto& m : *v)
          if (m) m->ready = 0, m->consumed_rec = false;
      std::rethrow_exception(errs[q]);
    }
  for (int q = 1; q < p; ++q) {
    tdvp_ctx* ln = h->lanes[q - 1].get();
    int ev;
    {
      DeviceGuard dg(ln->dev);
      ev = ev_record(ln);
    }
    CK(cudaStreamWaitEvent(h->st, ln->ev_pool[ev], 0));
    tdvp_stats& a = h->stats;
    const tdvp_stats& b = ln->stats;
    a.w_step += b.w_step;
    a.trunc_active |= b.trunc_active;
    a.n_pair += b.n_pair;
    a.n_back += b.n_back;
    a.svd_sweeps_max = std::max(a.svd_sweeps_max, b.svd_sweeps_max);
    a.svd_sweeps_total += b.svd_sweeps_total;
    a.svd_jac_ms += b.svd_jac_ms;
    a.svd_jac_flop += b.svd_jac_flop;
    a.svd_bj_ms += b.svd_bj_ms;
    a.svd_bj_flop += b.svd_bj_flop;
    a.svd_bj_calls += b.svd_bj_calls;
    a.heff2_flop += b.heff2_flop;
    a.heff2_calls += b.heff2_calls;
    a.heff1_flop += b.heff1_flop;
    a.heff2_flop_exec += b.heff2_flop_exec;
    a.heff1_flop_exec += b.heff1_flop_exec;
    a.lz_vec_bytes += b.lz_vec_bytes;
    for (int i = 0; i < 4; ++i) a.heff2_flop_bin[i] += b.heff2_flop_bin[i];
    for (int i = 0; i < 4; ++i) a.lz_bytes_bin[i] += b.lz_bytes_bin[i];
  }
}

void finish_timing(tdvp_ctx* h) {
  auto sum = [&](const std::vector<std::pair<int, int>>& v) {
    double t = 0.0;
    for (auto& pr : v) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, h->ev_pool[pr.first], h->ev_pool[pr.second]));
      t += ms;
    }
    return t;
  };
  h->stats.heff2_ms = sum(h->ev_h2);
  for (size_t i = 0; i < h->ev_h2.size() && i < h->ev_h2_bin.size(); ++i) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev_pool[h->ev_h2[i].first], h->ev_pool[h->ev_h2[i].second]));
    h->stats.heff2_ms_bin[h->ev_h2_bin[i]] += ms;
  }
  h->stats.heff1_ms = sum(h->ev_h1);
  h->stats.svd_ms = sum(h->ev_svd);
  h->stats.lanczos2_ms = sum(h->ev_lz2);
  h->stats.lanczos1_ms = sum(h->ev_lz1);
  h->stats.env_ms = sum(h->ev_env);
  for (const auto& r : h->ev_lzrec) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev_pool[r.ea], h->ev_pool[r.eb]));
    double t = ms;
    const auto& mv = r.which == 2 ? h->ev_h2 : h->ev_h1;
    for (size_t i = r.mv0; i < r.mv1 && i < mv.size(); ++i) {
      CK(cudaEventElapsedTime(&ms, h->ev_pool[mv[i].first], h->ev_pool[mv[i].second]));
      t -= ms;
    }
    h->stats.lz_ms_bin[r.bin] += t;
  }
}

int balanced_partition(int L, int p, const int* chi, int* s, int* e, double* best);
double partition_cost(int L, const int* chi, const std::vector<std::pair<int, int>>& bounds);
void reorthonormalize(tdvp_ctx* h);

void do_step(tdvp_ctx* h, double dt, int p, bool one_site = false) {
  if (!h->have_mpo || !h->have_mps) throw TdvpError(TDVP_ESTATE, "MPO and MPS must be set before tdvp_step");
  if (!std::isfinite(dt)) throw TdvpError(TDVP_EARG, "dt must be finite");
  if (one_site && h->prm.u1) throw TdvpError(TDVP_EARG, "tdvp_step1 runs in dense mode (u1 = 0)");
  if (h->prm.u1 && !local_mode(h)) throw TdvpError(TDVP_EARG, "u1 is not supported across ranks (use one process)");
  // dynamic load balancing ("dynamic load balancer"):
  // before the step, re-partition when the chi-weighted optimum beats the
  // current partition's largest segment cost by the relative margin
  // prm.rebalance (state kept; the environments are rebuilt, a serial section)
  if (h->prm.rebalance > 0.0 && p > 1 && local_mode(h) && h->layout_p == p && h->envs_valid) {
    std::vector<int> chi(h->L + 1, 1), ss(p), ee(p);
    for (int b = 0; b < h->L - 1; ++b) chi[b + 1] = h->segs[owner_of(h, b)].cb[b + 1];
    double best = 0.0;
    if (balanced_partition(h->L, p, chi.data(), ss.data(), ee.data(), &best) == TDVP_OK) {
      const double cur = partition_cost(h->L, chi.data(), h->bounds);
      if (best < (1.0 - h->prm.rebalance) * cur) {
        std::vector<std::pair<int, int>> nb(p);
        for (int q = 0; q < p; ++q) nb[q] = {ss[q], ee[q]};
        if (nb != h->bounds) {
          // Moving a boundary turns a gauge-broken boundary bond (both sides
          // evolved independently) into an interior bond whose
          // next merge Psi_b V_b Psi_{b+1} would amplify the mismatch by
          // V = 1/Lambda: re-gauge the state exactly first
          // (reorthonormalisation), then lay it out anew.
          reorthonormalize(h);
          h->custom = nb;
          h->envs_valid = false;
          h->stats.rebalances++;
        }
      }
    }
  }
  if (p != h->layout_p || !h->envs_valid) layout(h, p);
  reset_step_stats(h);
  h->evolved = true;
  const long long l0 = g_launch_count, g0 = g_gemm_count;
  CK(cudaEventRecord(h->ev_step0, h->st));
  std::set<int> merged;
  h->one_site = one_site;
  if (one_site) merged1(h->L, p, h->bounds, merged, h->msites);
  else merged = merged_pairs(h->L, p, h->bounds);
  struct OneSiteReset {
    tdvp_ctx* h;
    ~OneSiteReset() { h->one_site = false; }
  } reset_one_site{h};
  const bool lanes = local_mode(h) && p > 1 && (h->lanes_on || h->multi_dev);
  if (lanes) {
    if ((int)h->msg_r.size() != p) alloc_msgs(h);
    run_step_lanes(h, dt, merged);
    h->sv.throughput = 0;
  } else {
    run_half(h, 1, dt, merged);
    run_half(h, 2, dt, merged);
  }
  CK(cudaEventRecord(h->ev_step1, h->st));
  CK(cudaStreamSynchronize(h->st));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, h->ev_step0, h->ev_step1));
  h->stats.step_ms = ms;
  h->stats.w_total += h->stats.w_step;
  h->stats.kernel_launches = g_launch_count - l0;
  h->stats.gemm_launches = g_gemm_count - g0;
  if (h->prm.timing) {
    finish_timing(h);
    if (lanes)
      for (int q = 1; q < p; ++q) {
        // summed device time over lanes (concurrent: may exceed step_ms)
        tdvp_ctx* ln = h->lanes[q - 1].get();
        DeviceGuard dg(ln->dev);  // its events live on its device
        finish_timing(ln);
        h->stats.heff2_ms += ln->stats.heff2_ms;
        h->stats.heff1_ms += ln->stats.heff1_ms;
        h->stats.svd_ms += ln->stats.svd_ms;
        h->stats.lanczos2_ms += ln->stats.lanczos2_ms;
        h->stats.lanczos1_ms += ln->stats.lanczos1_ms;
        h->stats.env_ms += ln->stats.env_ms;
        for (int i = 0; i < 4; ++i) h->stats.lz_ms_bin[i] += ln->stats.lz_ms_bin[i];
        for (int i = 0; i < 4; ++i) h->stats.heff2_ms_bin[i] += ln->stats.heff2_ms_bin[i];
      }
  }
}

// ------------------------------------------------------------ measurement
// Full zipper over M_j = Psi_j V_j (j < L-1), M_{L-1} = Psi_{L-1} (AMB-10).
struct MeasureOut {
  double norm = 0.0, energy = 0.0;
  std::vector<double> sz;
};
void measure(tdvp_ctx* h, bool want_sz, bool want_E, MeasureOut& out) {
  if (!h->have_mps || !h->have_mpo) throw TdvpError(TDVP_ESTATE, "MPO and MPS must be set");
  if (!local_mode(h)) throw TdvpError(TDVP_ESTATE, "measurement across ranks: gather the MPS to one rank");
  if (h->layout_p == 0) layout(h, 1);
  const int L = h->L, d = h->d;
  std::vector<int> chi(L + 1, 1);
  for (int j = 1; j < L; ++j) chi[j] = h->segs[owner_of(h, j - 1)].cb[j];
  // chain tensors M_j into a contiguous scratch set (owner copies)
  std::vector<BufPtr> M(L);
  for (int j = 0; j < L; ++j) {
    Segment& g = h->segs[owner_of(h, j)];
    const long long n = (long long)chi[j] * d * chi[j + 1];
    M[j] = make_buf(n * sizeof(cplx));
    if (j < L - 1) CK(scale_cols(h->st, M[j]->c(), P(g.psi[j]), g.vinv[j]->d(), (long long)chi[j] * d, chi[j + 1]));
    else CK(copy_cplx(h->st, M[j]->c(), P(g.psi[j]), n));
  }
  const cplx one = ONE;
  // left norm envs E_j (j = 0..L) and right envs F_j (j = 0..L-1)
  std::vector<BufPtr> E(L + 1), F(L);
  E[0] = make_buf(sizeof(cplx));
  CK(cudaMemcpyAsync(E[0]->p, &one, sizeof(cplx), cudaMemcpyHostToDevice, h->st));
  for (int j = 0; j < L; ++j) {
    E[j + 1] = make_buf((size_t)chi[j + 1] * chi[j + 1] * sizeof(cplx));
    env_left(h, E[j]->c(), M[j]->c(), h->mpo_id, chi[j], chi[j + 1], E[j + 1]->c());
  }
  F[L - 1] = make_buf(sizeof(cplx));
  CK(cudaMemcpyAsync(F[L - 1]->p, &one, sizeof(cplx), cudaMemcpyHostToDevice, h->st));
  for (int j = L - 1; j > 0; --j) {
    F[j - 1] = make_buf((size_t)chi[j] * chi[j] * sizeof(cplx));
    env_right(h, F[j]->c(), M[j]->c(), h->mpo_id, chi[j], chi[j + 1], F[j - 1]->c());
  }
  cplx nrm;
  CK(cudaMemcpyAsync(&nrm, E[L]->p, sizeof(cplx), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  out.norm = nrm.x;
  if (!(out.norm > 0.0) || !std::isfinite(out.norm)) throw TdvpError(TDVP_ENUMERIC, "non-positive norm");
  if (want_sz) {
    out.sz.assign(L, 0.0);
    BufPtr X = make_buf((size_t)h->chi_max * h->chi_max * sizeof(cplx) + 64);
    BufPtr R = make_buf(sizeof(cplx) * L);
    for (int j = 0; j < L; ++j) {
      env_left(h, E[j]->c(), M[j]->c(), h->mpo_sz, chi[j], chi[j + 1], X->c());
      CK(sum_products(h->st, X->c(), F[j]->c(), (long long)chi[j + 1] * chi[j + 1], R->c() + j, h->partials->d(),
                      reinterpret_cast<unsigned*>(h->lz_counter->p)));
    }
    std::vector<cplx> r(L);
    CK(cudaMemcpyAsync(r.data(), R->p, L * sizeof(cplx), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    for (int j = 0; j < L; ++j) out.sz[j] = r[j].x / out.norm;
  }
  if (want_E) {
    BufPtr A = make_buf(h->envA->bytes), B = make_buf(h->envA->bytes);
    cplx* cur = A->c();
    cplx* nxt = B->c();
    CK(cudaMemcpyAsync(cur, &one, sizeof(cplx), cudaMemcpyHostToDevice, h->st));
    for (int j = 0; j < L; ++j) {
      env_left(h, cur, M[j]->c(), h->mpo[j], chi[j], chi[j + 1], nxt);
      std::swap(cur, nxt);
    }
    cplx e;
    CK(cudaMemcpyAsync(&e, cur, sizeof(cplx), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    out.energy = e.x / out.norm;
  }
}

// CSR tables of every MPO site and the pair tables W_j W_{j+1} (H_eff^(2)'s
// fused channel pass) on the current device
void build_mpo_tables(std::vector<MpoSite>& mpo, int L, int d, const std::vector<int>& D,
                      const std::vector<std::vector<cplx>>& W) {
  mpo.clear();
  mpo.resize(L);
  for (int j = 0; j < L; ++j) build_site(mpo[j], D[j], D[j + 1], d, W[j]);
  for (int j = 0; j + 1 < L; ++j) build_pair(mpo[j], D[j], D[j + 1], D[j + 2], d, W[j], W[j + 1]);
  // identity-channel structure (MpoSite::lid / rid)
  auto at = [&](int j, int w, int s, int t, int w2) { return W[j][(((size_t)w * d + s) * d + t) * D[j + 1] + w2]; };
  auto is = [](cplx v, double x) { return v.x == x && v.y == 0.0; };
  auto col_last_identity = [&](int j) {  // column D_{j+1}-1 fed only by row D_j-1 with the identity
    for (int w = 0; w < D[j]; ++w)
      for (int s = 0; s < d; ++s)
        for (int t = 0; t < d; ++t)
          if (!is(at(j, w, s, t, D[j + 1] - 1), (w == D[j] - 1 && s == t) ? 1.0 : 0.0)) return false;
    return true;
  };
  auto row0_identity = [&](int j) {  // row 0 feeds only column 0 with the identity
    for (int w2 = 0; w2 < D[j + 1]; ++w2)
      for (int s = 0; s < d; ++s)
        for (int t = 0; t < d; ++t)
          if (!is(at(j, 0, s, t, w2), (w2 == 0 && s == t) ? 1.0 : 0.0)) return false;
    return true;
  };
  mpo[0].lid = true;
  for (int j = 1; j < L; ++j) mpo[j].lid = mpo[j - 1].lid && col_last_identity(j - 1);
  mpo[L - 1].rid = true;
  for (int j = L - 2; j >= 0; --j) mpo[j].rid = mpo[j + 1].rid && row0_identity(j + 1);
}

// ------------------------------------------------------------ workspace
void alloc_workspace(tdvp_ctx* h) {
  const int L = h->L, d = h->d, D = h->Dmpo;
  long long n2 = 1, n1 = 1, scr = 1, svd = 1, env = 1, svq = 1;
  for (int j = 0; j < L; ++j) {
    const long long cl = h->cbmax[j], cr1 = h->cbmax[j + 1];
    n1 = std::max(n1, cl * d * cr1);
    env = std::max(env, std::max(cl * cl, cr1 * cr1) * D);
    scr = std::max(scr, cl * d * cr1 * D * d);
    if (j + 1 < L) {
      const long long cr = h->cbmax[j + 2];
      n2 = std::max(n2, cl * d * d * cr);
      scr = std::max(scr, cl * d * d * cr * D);
      svd = std::max(svd, (long long)svd_work_elems((int)(cl * d), (int)(d * cr)));
      svq = std::max(svq, (long long)svd_qr_work_elems((int)(cl * d), (int)(d * cr)));
    }
  }
  h->n2max = n2;
  h->n1max = n1;
  h->scratch = scr;
  h->svdmax = svd;
  h->work_elems = std::max<long long>(1 << 20, std::min<long long>(4 * scr, 1 << 23));
  const int K = KMAX;
  h->theta = make_buf(n2 * sizeof(cplx));
  h->krylov = make_buf((size_t)K * n2 * sizeof(cplx));
  h->wvec = make_buf(n2 * sizeof(cplx));
  h->T1 = make_buf(scr * sizeof(cplx));
  h->T2 = make_buf(scr * sizeof(cplx));
  h->tmpA = make_buf(std::max(n2, n1) * sizeof(cplx));
  h->tmpB = make_buf(std::max(n2, n1) * sizeof(cplx));
  h->svdY = make_buf(svd * sizeof(cplx));
  h->svdQ = make_buf(svq * sizeof(cplx));
  // the SVD has nc = min(cl d, d cr) <= d chi_max columns: every per-column
  // buffer below is sized by d chi_max (2 Jacobi counters per column block,
  // blocks >= 2 columns)
  const long long ncmax = (long long)h->d * h->chi_max;
  const size_t nflags = (size_t)4 * ncmax + 64;
  h->svdF = make_buf(nflags * sizeof(unsigned));
  h->gemm_work = make_buf(h->work_elems * sizeof(cplx));
  h->envA = make_buf(env * sizeof(cplx));
  h->envB = make_buf(env * sizeof(cplx));
  const int nblk = 4 * g_num_sms;
  h->partials = make_buf((size_t)nblk * 2 * (KMAX + 1) * sizeof(double));
  h->lz_scal = make_buf((2 * KMAX + 8) * sizeof(double));
  h->lz_coef = make_buf(2 * (KMAX + 1) * sizeof(cplx));
  h->lz_y = make_buf(KMAX * sizeof(cplx));
  h->lz_counter = make_buf(64);
  h->lz_brk = make_buf(64);
  CK(cudaMemset(h->lz_counter->p, 0, 64));
  CK(cudaMemset(h->lz_brk->p, 0, 64));
  h->svd_sigma = make_buf(ncmax * sizeof(double) + 64);
  h->svd_order = make_buf(ncmax * sizeof(int) + 64);
  h->svd_perm = make_buf(2 * ncmax * sizeof(int) + 64);
  h->svd_bj = make_buf(svd_bjac_work_elems(g_num_sms) * sizeof(cplx));
  h->u1_idx = make_buf((size_t)2 * (4 * ncmax + 64) * sizeof(int));
  h->u1_lam = make_buf(ncmax * sizeof(double) + 64);
  h->u1_vinv = make_buf(ncmax * sizeof(double) + 64);
  h->svd_off = make_buf(64);
  h->svd_ires = make_buf(64);
  h->svd_dres = make_buf(64);
  h->hdr = make_buf(64);
  CK(cudaMallocHost(&h->h_pin, 16 * sizeof(double)));
  CK(cudaMallocHost(&h->h_ipin, 16 * sizeof(int)));
  h->lz = LanczosDev{h->lz_scal->d(), h->lz_coef->c(), h->lz_y->c(), h->partials->d(),
                     reinterpret_cast<unsigned*>(h->lz_counter->p), h->lz_brk->i()};
  h->sv = SvdDev{h->svdY->c(), 0, h->svd_sigma->d(), h->svd_order->i(), h->svd_off->d(), h->svd_ires->i(),
                 h->svd_dres->d(), h->h_pin, h->h_ipin, {nullptr, nullptr}, h->svdQ->c(), (size_t)svq,
                 reinterpret_cast<unsigned*>(h->svdF->p), nflags, 0, h->svd_perm->i(), h->svd_bj->c(),
                 svd_bjac_work_elems(g_num_sms)};
}

// chi-weighted min-max contiguous partition:
// exact DP, smallest split index on ties; *best = its largest segment cost
int balanced_partition(int L, int p, const int* chi, int* s, int* e, double* best) {
  if (p == 1) {
    s[0] = 0;
    e[0] = L - 1;
    return TDVP_OK;
  }
  if (p < 2 || p % 2 != 0 || p > L / 2) return TDVP_EPARTITION;
  // site cost ~ the one-site update / half a pair update: chi_j chi_{j+1} (chi_j + chi_{j+1})
  std::vector<double> pre(L + 1, 0.0);
  for (int j = 0; j < L; ++j) {
    const double a = chi[j], b = chi[j + 1];
    if (!(a >= 1.0) || !(b >= 1.0)) return TDVP_EARG;
    pre[j + 1] = pre[j] + a * b * (a + b);
  }
  // f[q][i]: min over partitions of sites [0, i) into q segments (each >= 2) of the max segment cost
  const double INF = 1e300;
  std::vector<std::vector<double>> f(p + 1, std::vector<double>(L + 1, INF));
  std::vector<std::vector<int>> arg(p + 1, std::vector<int>(L + 1, -1));
  f[0][0] = 0.0;
  for (int q = 1; q <= p; ++q)
    for (int i = 2 * q; i <= L - 2 * (p - q); ++i)
      for (int k = 2 * (q - 1); k <= i - 2; ++k) {
        if (f[q - 1][k] >= INF) continue;
        const double v = std::max(f[q - 1][k], pre[i] - pre[k]);
        if (v < f[q][i]) {
          f[q][i] = v;
          arg[q][i] = k;
        }
      }
  if (f[p][L] >= INF) return TDVP_EPARTITION;
  if (best) *best = f[p][L];
  for (int q = p, i = L; q >= 1; --q) {
    const int k = arg[q][i];
    s[q - 1] = k;
    e[q - 1] = i - 1;
    i = k;
  }
  return TDVP_OK;
}

// largest segment cost of the contiguous partition `bounds` (site cost as above)
double partition_cost(int L, const int* chi, const std::vector<std::pair<int, int>>& bounds) {
  double worst = 0.0;
  for (const auto& sg : bounds) {
    double c = 0.0;
    for (int j = sg.first; j <= sg.second && j < L; ++j) {
      const double a = chi[j], b = chi[j + 1];
      c += a * b * (a + b);
    }
    worst = std::max(worst, c);
  }
  return worst;
}

// chain tensors M_j = Psi_j diag(V_j) (j < L-1), M_{L-1} = Psi_{L-1} of a local-mode handle
std::vector<BufPtr> chain_tensors(tdvp_ctx* h, std::vector<int>& chi) {
  const int L = h->L, d = h->d;
  if (h->layout_p == 0) layout(h, 1);
  chi.assign(L + 1, 1);
  for (int j = 1; j < L; ++j) chi[j] = h->segs[owner_of(h, j - 1)].cb[j];
  std::vector<BufPtr> M(L);
  CK(cudaStreamSynchronize(h->st));
  BufPtr tv = make_buf((size_t)h->chi_max * sizeof(double) + 64);
  for (int j = 0; j < L; ++j) {
    Segment& g = h->segs[owner_of(h, j)];
    const long long n = (long long)chi[j] * d * chi[j + 1];
    M[j] = make_buf(n * sizeof(cplx));
    // a multi-device handle gathers the chain onto the lead device (NVLink peer copies)
    d2d(M[j]->p, h->dev, g.psi[j]->p, g.dev, (size_t)n * sizeof(cplx), h->st);
    if (j < L - 1) {
      d2d(tv->p, h->dev, g.vinv[j]->p, g.dev, (size_t)chi[j + 1] * sizeof(double), h->st);
      CK(scale_cols(h->st, M[j]->c(), M[j]->c(), tv->d(), (long long)chi[j] * d, chi[j + 1]));
      CK(cudaStreamSynchronize(h->st));  // tv is reused
    }
  }
  return M;
}

void reorthonormalize(tdvp_ctx* h) {
  {
    if (!h->have_mps || !h->have_mpo) throw TdvpError(TDVP_ESTATE, "MPO and MPS must be set");
    if (!local_mode(h)) throw TdvpError(TDVP_ESTATE, "reorthonormalisation across ranks: gather the MPS first");
    const int L = h->L, d = h->d;
    std::vector<int> chi;
    std::vector<BufPtr> A = chain_tensors(h, chi);
    long long big = 1;
    for (int j = 0; j < L; ++j) big = std::max(big, (long long)h->cbmax[j] * d * h->cbmax[j + 1]);
    BufPtr pl = make_buf(big * sizeof(cplx)), pr = make_buf(big * sizeof(cplx)), tmp = make_buf(big * sizeof(cplx));
    BufPtr lam = make_buf((size_t)(2 * h->chi_max + 8) * sizeof(double));
    BufPtr vin = make_buf((size_t)(2 * h->chi_max + 8) * sizeof(double));
    std::vector<std::vector<double>> hlam(L - 1);
    const TruncParams tp{h->chi_max, 0.0, 0.0, 0.0};
    std::vector<std::vector<int>> q;
    if (h->prm.u1) q = assemble_charges(h);
    // U(1) mode: rq / cq are the row / column charges, the kept vectors' charges come back in qm
    auto svd = [&](const cplx* M, int m, int n, int& k, const std::vector<int>* rq, const std::vector<int>* cq,
                   std::vector<int>* qm) {
      int r = 0, ce = 0, sw = 0;
      double w = 0.0;
      if (h->prm.u1) {
        u1_svd_split(h, M, m, n, *rq, *cq, tp, pl->c(), pr->c(), lam->d(), vin->d(), k, w, r, ce, *qm, sw);
        return;
      }
      cudaError_t se = svd_truncate_split(h->st, h->sv, M, m, n, tp, pl->c(), pr->c(), lam->d(), vin->d(), &k, &w, &r,
                                          &ce, &sw);
      if (se == cudaErrorUnknown) throw TdvpError(TDVP_ENUMERIC, "SVD numerical failure in reorthonormalisation");
      CK(se);
    };
    std::vector<int> rq, cq, qm;
    // L -> R: A_j = U S W^dagger  ->  A_j = U,  A_{j+1} = (S W^dagger) A_{j+1}
    for (int j = 0; j + 1 < L; ++j) {
      int k = 0;
      if (h->prm.u1) {
        rq.resize((size_t)chi[j] * d);
        for (int a = 0; a < chi[j]; ++a)
          for (int s2 = 0; s2 < d; ++s2) rq[(size_t)a * d + s2] = q[j][a] + U1_C[s2];
        cq = q[j + 1];
      }
      svd(A[j]->c(), chi[j] * d, chi[j + 1], k, &rq, &cq, &qm);
      if (h->prm.u1) q[j + 1] = qm;
      if (k > h->cbmax[j + 1]) throw TdvpError(TDVP_ECUDA, "internal: reorthonormalisation rank");
      BufPtr U = make_buf((size_t)chi[j] * d * k * sizeof(cplx));
      CK(scale_cols(h->st, U->c(), pl->c(), vin->d(), (long long)chi[j] * d, k));
      gemm(h, OP_N, OP_N, k, d * chi[j + 2], chi[j + 1], pr->c(), chi[j + 1], A[j + 1]->c(), (long long)d * chi[j + 2],
           tmp->c(), (long long)d * chi[j + 2]);
      BufPtr An = make_buf((size_t)k * d * chi[j + 2] * sizeof(cplx));
      CK(copy_cplx(h->st, An->c(), tmp->c(), (long long)k * d * chi[j + 2]));
      A[j] = std::move(U);
      A[j + 1] = std::move(An);
      chi[j + 1] = k;
    }
    // R -> L: A_j = U S W^dagger  ->  B_j = W^dagger, Lambda_{j-1} = S, A_{j-1} = A_{j-1} (U S)
    for (int j = L - 1; j >= 1; --j) {
      int k = 0;
      if (h->prm.u1) {
        rq = q[j];
        cq.resize((size_t)d * chi[j + 1]);
        for (int s2 = 0; s2 < d; ++s2)
          for (int b = 0; b < chi[j + 1]; ++b) cq[(size_t)s2 * chi[j + 1] + b] = q[j + 1][b] - U1_C[s2];
      }
      svd(A[j]->c(), chi[j], d * chi[j + 1], k, &rq, &cq, &qm);
      if (h->prm.u1) q[j] = qm;
      BufPtr B = make_buf((size_t)k * d * chi[j + 1] * sizeof(cplx));
      CK(scale_rows(h->st, B->c(), pr->c(), vin->d(), k, (long long)d * chi[j + 1]));
      gemm(h, OP_N, OP_N, chi[j - 1] * d, k, chi[j], A[j - 1]->c(), chi[j], pl->c(), k, tmp->c(), k);
      BufPtr An = make_buf((size_t)chi[j - 1] * d * k * sizeof(cplx));
      CK(copy_cplx(h->st, An->c(), tmp->c(), (long long)chi[j - 1] * d * k));
      hlam[j - 1].resize(k);
      CK(cudaMemcpyAsync(hlam[j - 1].data(), lam->p, k * sizeof(double), cudaMemcpyDeviceToHost, h->st));
      CK(cudaStreamSynchronize(h->st));
      A[j] = std::move(B);
      A[j - 1] = std::move(An);
      chi[j] = k;
    }
    // download, normalise, Psi_0 = A_0 / n, Lambda /= n, Psi_j = Lambda_{j-1} B_j
    std::vector<hvec> hpsi(L);
    for (int j = 0; j < L; ++j) {
      hpsi[j].resize((size_t)chi[j] * d * chi[j + 1] * 2);
      CK(cudaMemcpyAsync(hpsi[j].data(), A[j]->p, hpsi[j].size() * sizeof(double), cudaMemcpyDeviceToHost, h->st));
    }
    CK(cudaStreamSynchronize(h->st));
    double nrm = 0.0;
    for (double v : hpsi[0]) nrm += v * v;
    nrm = std::sqrt(nrm);
    if (!(nrm > 0.0) || !std::isfinite(nrm)) throw TdvpError(TDVP_ENUMERIC, "zero or non-finite norm");
    for (double& v : hpsi[0]) v /= nrm;
    for (auto& l : hlam)
      for (double& v : l) v /= nrm;
    for (int j = 1; j < L; ++j) {
      const int cl = chi[j], rest = d * chi[j + 1];
      for (int a = 0; a < cl; ++a)
        for (int e = 0; e < 2 * rest; ++e) hpsi[j][(size_t)a * 2 * rest + e] *= hlam[j - 1][a];
    }
    h->h_psi = std::move(hpsi);
    h->h_lam = std::move(hlam);
    h->h_chi = chi;
    if (h->prm.u1) h->h_q = q;
    h->envs_valid = false;
    h->layout_p = 0;  // re-layout: upload + sequential environment build at the next call
  }
}


int fail(tdvp_ctx* h, const TdvpError& e) {
  if (h) h->err = e.what();
  return e.code;
}

void init_device_globals() {
  static std::atomic<bool> done{false};
  if (done.load()) return;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0) g_num_sms = sms;
  }
  done = true;
}

std::vector<cplx> to_cplx(const double* p, size_t n) {
  std::vector<cplx> v(n);
  for (size_t i = 0; i < n; ++i) v[i] = cmk(p[2 * i], p[2 * i + 1]);
  return v;
}

// ------------------------------------------------------------ standalone kernels context
tdvp_ctx* scratch_ctx(int maxchi, int D) {
  // a small context for the kernel-level test entry points
  static tdvp_ctx* sc = nullptr;
  static int cap = 0, capD = 0;
  if (sc && cap >= maxchi && capD >= D) return sc;
  delete sc;
  sc = new tdvp_ctx();
  init_device_globals();
  CK(cudaStreamCreateWithFlags(&sc->st, cudaStreamNonBlocking));
  sc->L = 2;
  sc->d = 2;
  sc->Dmpo = D;
  sc->chi_max = maxchi;
  sc->cbmax = {1, maxchi, 1};
  // size the workspace for a (maxchi, d, d, maxchi) problem
  sc->cbmax = {maxchi, maxchi, maxchi};
  alloc_workspace(sc);
  cap = maxchi;
  capD = D;
  return sc;
}

}  // namespace

// =================================================================== C-ABI
extern "C" {

int tdvp_create(int L, int d, int D_mpo, int chi_max, tdvp_t* out) {
  if (!out) return TDVP_EARG;
  *out = nullptr;
  if (L < 2 || d < 2 || D_mpo < 1 || chi_max < 1) return TDVP_EARG;
  tdvp_ctx* h = new tdvp_ctx();
  try {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) throw TdvpError(TDVP_ECUDA, "no CUDA device");
    init_device_globals();
    CK(cudaGetDevice(&h->dev));
    h->L = L;
    h->d = d;
    h->Dmpo = D_mpo;
    h->chi_max = chi_max;
    h->prm.eps = 1e-12;
    h->prm.w_max = 0.0;
    h->prm.krylov_k = 8;
    h->prm.krylov_tol = 0.0;
    h->prm.multiplet_delta = 1e-6;
    h->prm.timing = 0;
    h->devs = {h->dev};
    h->prm.n_devices = 1;
    h->prm.device_ids = h->devs.data();
    if (const char* ev = std::getenv("TDVP_LANES")) h->lanes_on = std::atoi(ev) != 0;
    h->cbmax.assign(L + 1, 1);
    for (int j = 0; j <= L; ++j) {
      double a = std::pow((double)d, std::min(j, 62)), b = std::pow((double)d, std::min(L - j, 62));
      h->cbmax[j] = (int)std::min<double>(std::min(a, b), (double)chi_max);
    }
    CK(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
    CK(cudaEventCreate(&h->ev_step0));
    CK(cudaEventCreate(&h->ev_step1));
    alloc_workspace(h);
    CK(cudaEventCreate(&h->sv.ev_jac[0]));
    CK(cudaEventCreate(&h->sv.ev_jac[1]));
    // measurement MPOs (D = 1): identity and S^z (d = 2 spin-1/2 convention)
    std::vector<cplx> Id(d * d, ZERO), Sz(d * d, ZERO);
    for (int s = 0; s < d; ++s) Id[s * d + s] = ONE;
    Sz[0] = cmk(0.5, 0);
    Sz[d * d - 1] = cmk(-0.5, 0);
    build_site(h->mpo_id, 1, 1, d, Id);
    build_site(h->mpo_sz, 1, 1, d, Sz);
    h->h_psi.resize(L);
    h->h_lam.resize(L - 1);
  } catch (const TdvpError& e) {
    std::fprintf(stderr, "tdvp_create: %s\n", e.what());
    const int c = e.code;
    tdvp_destroy(h);
    return c;
  }
  *out = h;
  return TDVP_OK;
}

int tdvp_set_params(tdvp_t h, const tdvp_params* p) {
  if (!h || !p) return TDVP_EARG;
  if (p->krylov_k < 1 || p->krylov_k >= KMAX || !(p->eps >= 0.0) || p->eps >= 1.0 || !(p->w_max >= 0.0) ||
      !(p->multiplet_delta >= 0.0) || !(p->krylov_tol >= 0.0) || p->krylov_tol >= 1.0 || !(p->rebalance >= 0.0) ||
      p->rebalance >= 1.0) {
    h->err = "invalid params (krylov_k in 1..15, 0 <= eps < 1, w_max >= 0, 0 <= krylov_tol < 1)";
    return TDVP_EARG;
  }
  try {
    std::vector<int> devs;
    if (p->n_devices > 1) {
      if (!p->device_ids) throw TdvpError(TDVP_EARG, "n_devices > 1 needs device_ids");
      int ndev = 0;
      CK(cudaGetDeviceCount(&ndev));
      for (int i = 0; i < p->n_devices; ++i) {
        const int dv = p->device_ids[i];
        if (dv < 0 || dv >= ndev) throw TdvpError(TDVP_EARG, "device id out of range");
        devs.push_back(dv);
      }
      if (devs[0] != h->dev)
        throw TdvpError(TDVP_EARG, "device_ids[0] must be the device the handle was created on");
      if (!local_mode(h)) throw TdvpError(TDVP_ESTATE, "a multi-device handle cannot also be a rank of a group");
    }
    const bool multi = devs.size() > 1;
    if (multi != h->multi_dev || (multi && devs != h->devs)) {
      // new device map: keep the state, re-lay it out at the next step
      if (h->layout_p != 0 && h->have_mps) download_state(h);
      h->layout_p = 0;
      h->alloc_p = 0;
      h->segs.clear();
      h->msg_r.clear();
      h->msg_l.clear();
      h->lanes.clear();
      h->multi_dev = multi;
      h->devs = multi ? devs : std::vector<int>{h->dev};
      if (multi)
        for (int a : h->devs)
          for (int b : h->devs)
            if (a != b) {
              int ok = 0;
              if (cudaDeviceCanAccessPeer(&ok, a, b) == cudaSuccess && ok) {
                DeviceGuard dg(a);
                const cudaError_t pe = cudaDeviceEnablePeerAccess(b, 0);
                if (pe != cudaSuccess) cudaGetLastError();  // already enabled: fine
              }
            }
    }
  } catch (const TdvpError& e) {
    return fail(h, e);
  }
  if (p->u1 && h->d != 2) {
    h->err = "u1 needs d = 2 (spin-1/2 charges)";
    return TDVP_EARG;
  }
  if (!!p->u1 != !!h->prm.u1 && h->layout_p != 0) {
    // switching the U(1) mode re-lays the state out (charges inferred / dropped)
    try {
      if (h->have_mps && local_mode(h)) download_state(h);
    } catch (const TdvpError& e) {
      return fail(h, e);
    }
    h->layout_p = 0;
    h->envs_valid = false;
    h->h_q.clear();
  }
  h->prm = *p;
  h->prm.n_devices = (int)h->devs.size();
  h->prm.device_ids = h->devs.data();
  return TDVP_OK;
}

int tdvp_get_params(tdvp_t h, tdvp_params* p) {
  if (!h || !p) return TDVP_EARG;
  *p = h->prm;
  return TDVP_OK;
}

int tdvp_set_mpo(tdvp_t h, const int* D, const double* const* W) {
  if (!h || !D || !W) return TDVP_EARG;
  try {
    const int L = h->L, d = h->d;
    if (D[0] != 1 || D[L] != 1) throw TdvpError(TDVP_EARG, "MPO boundary bond dims must be 1");
    for (int j = 0; j <= L; ++j)
      if (D[j] < 1 || D[j] > h->Dmpo) throw TdvpError(TDVP_EARG, "MPO bond dim out of range");
    std::vector<std::vector<cplx>> hw(L);
    for (int j = 0; j < L; ++j) {
      if (!W[j]) throw TdvpError(TDVP_EARG, "null MPO tensor");
      const size_t n = (size_t)D[j] * d * d * D[j + 1];
      for (size_t i = 0; i < 2 * n; ++i)
        if (!std::isfinite(W[j][i])) throw TdvpError(TDVP_ENONFINITE, "non-finite MPO entry");
      hw[j] = to_cplx(W[j], n);
    }
    std::vector<MpoSite> mpo;
    h->h_D.assign(D, D + L + 1);
    build_mpo_tables(mpo, L, d, h->h_D, hw);
    h->h_W = std::move(hw);
    h->mpo = std::move(mpo);
    // U(1): channel charges r(w') = r(w) + c(s) - c(t) over the nonzero W[w,s,t,w'];
    // inconsistent -> the MPO does not conserve S^z (masks off; u1 steps still exact)
    h->h_r.clear();
    if (d == 2) {
      const int UNK = std::numeric_limits<int>::min();
      std::vector<std::vector<int>> r(L + 1);
      r[0] = {0};
      bool ok = true;
      for (int j = 0; j < L && ok; ++j) {
        r[j + 1].assign(D[j + 1], UNK);
        const auto& Wj = h->h_W[j];
        for (int w = 0; w < D[j] && ok; ++w) {
          if (r[j][w] == UNK) continue;
          for (int s2 = 0; s2 < 2; ++s2)
            for (int t = 0; t < 2; ++t)
              for (int w2 = 0; w2 < D[j + 1]; ++w2) {
                const cplx v = Wj[(((size_t)w * 2 + s2) * 2 + t) * D[j + 1] + w2];
                if (v.x == 0.0 && v.y == 0.0) continue;
                const int val = r[j][w] + U1_C[s2] - U1_C[t];
                if (r[j + 1][w2] == UNK) r[j + 1][w2] = val;
                else if (r[j + 1][w2] != val) ok = false;
              }
        }
      }
      if (ok) h->h_r = std::move(r);
    }
    h->lanes.clear();  // lanes of a multi-device handle hold per-device copies of the tables
    h->have_mpo = true;
    h->envs_valid = false;
    if (h->layout_p != 0 && h->have_mps && local_mode(h)) download_state(h);
    h->layout_p = 0;
    h->alloc_p = 0;
    h->segs.clear();
  } catch (const TdvpError& e) {
    return fail(h, e);
  }
  return TDVP_OK;
}

int tdvp_set_mps(tdvp_t h, const int* chi, const double* const* Psi, const double* const* Lambda) {
  if (!h || !chi || !Psi || (h->L > 1 && !Lambda)) return TDVP_EARG;
  try {
    const int L = h->L, d = h->d;
    if (chi[0] != 1 || chi[L] != 1) throw TdvpError(TDVP_EARG, "MPS boundary bond dims must be 1");
    for (int j = 1; j < L; ++j)
      if (chi[j] < 1 || chi[j] > h->cbmax[j]) throw TdvpError(TDVP_EARG, "bond dim exceeds min(d^j, d^(L-j), chi_max)");
    // validate everything first (the handle keeps its state on error), then
    // copy into the existing host vectors (their pages are reused: no
    // allocation or page faults per call for the same shapes)
    std::vector<size_t> sz(L);
    for (int j = 0; j < L; ++j) {
      if (!Psi[j]) throw TdvpError(TDVP_EARG, "null Psi");
      sz[j] = (size_t)chi[j] * d * chi[j + 1] * 2;
    }
    std::atomic<bool> bad{false};
    host_parallel(sz, [&](size_t j, size_t i0, size_t i1) {
      const double* src = Psi[j];
      bool fin = true;
      for (size_t i = i0; i < i1; ++i) fin &= std::isfinite(src[i]);
      if (!fin) bad = true;
    });
    if (bad) throw TdvpError(TDVP_ENONFINITE, "non-finite Psi entry");
    for (int b = 0; b < L - 1; ++b) {
      if (!Lambda[b]) throw TdvpError(TDVP_EARG, "null Lambda");
      for (int i = 0; i < chi[b + 1]; ++i)
        if (!std::isfinite(Lambda[b][i]) || !(Lambda[b][i] > 0.0))
          throw TdvpError(TDVP_ENONFINITE, "Lambda must be finite and > 0");
    }
    h->h_psi.resize(L);
    h->h_lam.resize(L - 1);
    for (int j = 0; j < L; ++j)
      if (h->h_psi[j].size() != sz[j]) {
        h->h_psi[j].clear();
        h->h_psi[j].resize(sz[j]);
      }
    host_parallel(sz, [&](size_t j, size_t i0, size_t i1) {
      std::memcpy(h->h_psi[j].data() + i0, Psi[j] + i0, (i1 - i0) * sizeof(double));
    });
    for (int b = 0; b < L - 1; ++b) h->h_lam[b].assign(Lambda[b], Lambda[b] + chi[b + 1]);
    h->h_chi.assign(chi, chi + L + 1);
    h->h_q.clear();  // U(1) charges are re-inferred at the next layout
    h->have_mps = true;
    h->evolved = false;
    h->envs_valid = false;
    h->layout_p = 0;  // re-layout (upload + env build) at the next step, same buffers
  } catch (const TdvpError& e) {
    return fail(h, e);
  }
  return TDVP_OK;
}

int tdvp_step(tdvp_t h, double dt, int n_segments) {
  if (!h) return TDVP_EARG;
  try {
    do_step(h, dt, n_segments);
  } catch (const TdvpError& e) {
    return fail(h, e);
  }
  return TDVP_OK;
}

int tdvp_step1(tdvp_t h, double dt, int n_segments) {
  if (!h) return TDVP_EARG;
  try {
    do_step(h, dt, n_segments, true);
  } catch (const TdvpError& e) {
    return fail(h, e);
  }
  return TDVP_OK;
}

int tdvp_step_hybrid(tdvp_t h, double dt, int n_segments, int* used) {
  if (!h) return TDVP_EARG;
  try {
    bool one = false;
    if (h->have_mps && h->have_mpo && local_mode(h) && !h->prm.u1) {
      if (h->layout_p == 0) {
        // nothing laid out yet: the host copy's bond dimensions
        one = true;
        for (int j = 0; j + 1 < h->L; ++j) {
          long long cap = 1;
          const int k = std::min(j + 1, h->L - j - 1);
          for (int i = 0; i < k && cap < h->chi_max; ++i) cap *= h->d;
          if (h->h_chi[j + 1] < std::min<long long>(cap, h->chi_max)) one = false;
        }
      } else {
        one = chi_saturated(h);
      }
    }
    do_step(h, dt, n_segments, one);
    if (used) *used = one ? 1 : 2;
  } catch (const TdvpError& e) {
    return fail(h, e);
  }
  return TDVP_OK;
}

int tdvp_measure_sz(tdvp_t h, double* sz) {
  if (!h || !sz) return TDVP_EARG;
  try {
    MeasureOut m;
    measure(h, true, false, m);
    for (int j = 0; j < h->L; ++j) sz[j] = m.sz[j];
  } catch (const TdvpError& e) {
    return fail(h, e);
  }
  return TDVP_OK;
}

int tdvp_measure_energy(tdvp_t h, double* E) {
  if (!h || !E) return TDVP_EARG;
  try {
    MeasureOut m;
    measure(h, false, true, m);
    *E = m.energy;
  } catch (const TdvpError& e) {
    return fail(h, e);
  }
  return TDVP_OK;
}

int tdvp_measure_norm(tdvp_t h, double* n) {
  if (!h || !n) return TDVP_EARG;
  try {
    MeasureOut m;
    measure(h, false, false, m);
    *n = m.norm;
  } catch (const TdvpError& e) {
    return fail(h, e);
  }
  return TDVP_OK;
}


// <psi_a | psi_b> by a two-state zipper (PAPER.md Sec. benchmarks, infidelity
// I = 1 - |<1|2>| / sqrt(<1|1><2|2>)): E_{j+1} = M1_j^H (E_j M2_j)
int tdvp_overlap(tdvp_t a, tdvp_t b, double* re, double* im) {
  if (!a || !b || !re || !im) return TDVP_EARG;
  try {
    if (a->L != b->L || a->d != b->d) throw TdvpError(TDVP_EARG, "overlap: handles differ in L or d");
    if (!a->have_mps || !b->have_mps || !a->have_mpo || !b->have_mpo)
      throw TdvpError(TDVP_ESTATE, "overlap: MPO and MPS must be set on both handles");
    if (!local_mode(a) || !local_mode(b)) throw TdvpError(TDVP_ESTATE, "overlap across ranks: gather the MPS first");
    if (a->dev != b->dev) throw TdvpError(TDVP_EARG, "overlap: handles on different devices");
    const int L = a->L, d = a->d;
    std::vector<int> ca, cb;
    std::vector<BufPtr> Ma = chain_tensors(a, ca);
    std::vector<BufPtr> Mb = chain_tensors(b, cb);
    CK(cudaStreamSynchronize(b->st));  // b's tensors are read on a's stream
    long long tmax = 1, emax = 1;
    for (int j = 0; j <= L; ++j) emax = std::max(emax, (long long)ca[j] * cb[j]);
    for (int j = 0; j < L; ++j) tmax = std::max(tmax, (long long)ca[j] * d * cb[j + 1]);
    BufPtr E0 = make_buf(emax * sizeof(cplx)), E1 = make_buf(emax * sizeof(cplx)), T = make_buf(tmax * sizeof(cplx));
    const cplx one = ONE;
    CK(cudaMemcpyAsync(E0->p, &one, sizeof(cplx), cudaMemcpyHostToDevice, a->st));
    for (int j = 0; j < L; ++j) {
      // T[a1][(s,b2)] = sum_a2 E[a1][a2] M2[a2][(s,b2)]
      gemm(a, OP_N, OP_N, ca[j], d * cb[j + 1], cb[j], E0->c(), cb[j], Mb[j]->c(), (long long)d * cb[j + 1], T->c(),
           (long long)d * cb[j + 1]);
      // E'[b1][b2] = sum_{(a1,s)} conj(M1[(a1,s)][b1]) T[(a1,s)][b2]
      gemm(a, OP_C, OP_N, ca[j + 1], cb[j + 1], ca[j] * d, Ma[j]->c(), ca[j + 1], T->c(), cb[j + 1], E1->c(),
           cb[j + 1]);
      std::swap(E0, E1);
    }
    cplx r;
    CK(cudaMemcpyAsync(&r, E0->p, sizeof(cplx), cudaMemcpyDeviceToHost, a->st));
    CK(cudaStreamSynchronize(a->st));
    *re = r.x;
    *im = r.y;
  } catch (const TdvpError& e) {
    return fail(a, e);
  }
  return TDVP_OK;
}

// infidelity I = 1 - |<a|b>| / sqrt(<a|a><b|b>) between two handles' states
// (PAPER.md benchmark section: serial vs parallel)
int tdvp_infidelity(tdvp_t a, tdvp_t b, double* inf) {
  if (!a || !b || !inf) return TDVP_EARG;
  double re = 0.0, im = 0.0;
  int rc = tdvp_overlap(a, b, &re, &im);
  if (rc != TDVP_OK) return rc;
  try {
    MeasureOut ma, mb;
    measure(a, false, false, ma);
    measure(b, false, false, mb);
    *inf = 1.0 - std::hypot(re, im) / std::sqrt(ma.norm * mb.norm);
  } catch (const TdvpError& e) {
    return fail(a, e);
  }
  return TDVP_OK;
}

// Reorthonormalisation (Fig. reorth): exact re-gauging of the
// current chain into inverse-canonical form on the device -- an SVD sweep L->R
// (A_j <- U, A_{j+1} <- S W^dagger A_{j+1}) and one R->L (B_j = W^dagger,
// Lambda_{j-1} = S, A_{j-1} <- A_{j-1} U S), singular values below 1e-14
// sigma_1 dropped, the state normalised -- then the environments are rebuilt
// at the next step (a serial procedure, as in the paper).
int tdvp_reorthonormalize(tdvp_t h) {
  if (!h) return TDVP_EARG;
  try {
    reorthonormalize(h);
  } catch (const TdvpError& e) {
    return fail(h, e);
  }
  return TDVP_OK;
}

int tdvp_dmrg(tdvp_t h, int n_sweeps, int restarts, double* energies) {
  if (!h || n_sweeps < 0 || restarts < 1) return TDVP_EARG;
  try {
    if (!h->have_mpo || !h->have_mps) throw TdvpError(TDVP_ESTATE, "MPO and MPS must be set before tdvp_dmrg");
    if (!local_mode(h)) throw TdvpError(TDVP_ESTATE, "tdvp_dmrg runs on a single-process handle");
    const int L = h->L;
    if (h->layout_p != 1 || !h->envs_valid) layout(h, 1);
    Segment& g = h->segs[0];
    reset_step_stats(h);
    for (int sw = 0; sw < n_sweeps; ++sw) {
      for (int j = 0; j + 1 < L; ++j) dmrg_pair(h, g, j, BUILD_BETA | (j == L - 2 ? BUILD_GAMMA : 0), restarts);
      for (int j = L - 3; j >= 0; --j) dmrg_pair(h, g, j, BUILD_GAMMA | (j == 0 ? BUILD_BETA : 0), restarts);
      double e = 0.0;
      CK(cudaMemcpyAsync(&e, h->lz.scal + LZ_E0, sizeof(double), cudaMemcpyDeviceToHost, h->st));
      CK(cudaStreamSynchronize(h->st));
      if (energies) energies[sw] = e;
    }
    // a DMRG state is a valid factorisation but not exactly inverse-canonical
    // (each Lambda_j dates from the last update of bond j, the state changed
    // since); 2TDVP needs exactly inverse-canonical input, so
    // re-gauge it (reorthonormalisation)
    if (n_sweeps > 0) reorthonormalize(h);
    h->evolved = true;
  } catch (const TdvpError& e) {
    return fail(h, e);
  }
  return TDVP_OK;
}

int tdvp_get_stats(tdvp_t h, tdvp_stats* s) {
  if (!h || !s) return TDVP_EARG;
  int brk = 0;
  if (h->lz_brk && cudaMemcpy(&brk, h->lz_brk->p, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess)
    h->stats.krylov_breakdowns = brk;
  *s = h->stats;
  return TDVP_OK;
}

int tdvp_get_chi(tdvp_t h, int* chi) {
  if (!h || !chi) return TDVP_EARG;
  try {
    if (!h->have_mps) throw TdvpError(TDVP_ESTATE, "MPS not set");
    if (h->layout_p == 0) {
      for (int j = 0; j <= h->L; ++j) chi[j] = h->h_chi[j];
      return TDVP_OK;
    }
    if (!local_mode(h)) throw TdvpError(TDVP_ESTATE, "not available across ranks");
    chi[0] = chi[h->L] = 1;
    for (int j = 1; j < h->L; ++j) chi[j] = h->segs[owner_of(h, j - 1)].cb[j];
  } catch (const TdvpError& e) {
    return fail(h, e);
  }
  return TDVP_OK;
}

int tdvp_get_mps(tdvp_t h, double** Psi, double** Lambda) {
  if (!h || !Psi) return TDVP_EARG;
  try {
    if (!h->have_mps) throw TdvpError(TDVP_ESTATE, "MPS not set");
    if (h->prm.u1) {
      // U(1) mode keeps every bond basis sorted by charge; the ABI returns
      // descending Lambda: permute each bond on the host copy on the way out
      const int L = h->L, d = h->d;
      if (h->layout_p != 0) download_state(h);
      std::vector<std::vector<double>> ps;
      for (const hvec& v : h->h_psi) ps.emplace_back(v.begin(), v.end());
      std::vector<std::vector<double>> lm = h->h_lam;
      const std::vector<int>& chi = h->h_chi;
      for (int b = 0; b + 1 < L; ++b) {
        const int n = chi[b + 1];
        std::vector<int> perm(n);
        for (int i = 0; i < n; ++i) perm[i] = i;
        std::stable_sort(perm.begin(), perm.end(), [&](int x, int y) { return lm[b][x] > lm[b][y]; });
        std::vector<double> nl(n);
        for (int i = 0; i < n; ++i) nl[i] = lm[b][perm[i]];
        lm[b] = nl;
        // Psi_b: right index; Psi_{b+1}: left index
        const int cl = chi[b], cr2 = chi[b + 2];
        std::vector<double> a2(ps[b].size()), b2(ps[b + 1].size());
        for (int a = 0; a < cl * d; ++a)
          for (int i = 0; i < n; ++i) {
            a2[((size_t)a * n + i) * 2] = ps[b][((size_t)a * n + perm[i]) * 2];
            a2[((size_t)a * n + i) * 2 + 1] = ps[b][((size_t)a * n + perm[i]) * 2 + 1];
          }
        const size_t row = (size_t)d * cr2 * 2;
        for (int i = 0; i < n; ++i) std::memcpy(&b2[i * row], &ps[b + 1][perm[i] * row], row * sizeof(double));
        ps[b] = std::move(a2);
        ps[b + 1] = std::move(b2);
      }
      for (int j = 0; j < L; ++j) std::memcpy(Psi[j], ps[j].data(), ps[j].size() * sizeof(double));
      if (Lambda)
        for (int b = 0; b + 1 < L; ++b) std::memcpy(Lambda[b], lm[b].data(), lm[b].size() * sizeof(double));
      return TDVP_OK;
    }
    if (h->layout_p != 0 && local_mode(h)) {
      // device state authoritative: straight into the caller's buffers (no host staging copy)
      const int L = h->L, d = h->d;
      std::vector<int> chi(L + 1, 1);
      for (int b = 0; b < L - 1; ++b) chi[b + 1] = h->segs[owner_of(h, b)].cb[b + 1];
      CK(cudaStreamSynchronize(h->st));
      for (int j = 0; j < L; ++j) {
        const Segment& g = h->segs[owner_of(h, j)];
        DeviceGuard dg(g.dev);
        CK(cudaMemcpy(Psi[j], g.psi[j]->p, (size_t)chi[j] * d * chi[j + 1] * sizeof(cplx), cudaMemcpyDeviceToHost));
      }
      if (Lambda)
        for (int b = 0; b < L - 1; ++b) {
          const Segment& g = h->segs[owner_of(h, b)];
          DeviceGuard dg(g.dev);
          CK(cudaMemcpy(Lambda[b], g.lam[b]->p, (size_t)chi[b + 1] * sizeof(double), cudaMemcpyDeviceToHost));
        }
      return TDVP_OK;
    }
    if (h->layout_p != 0) download_state(h);
    for (int j = 0; j < h->L; ++j) std::memcpy(Psi[j], h->h_psi[j].data(), h->h_psi[j].size() * sizeof(double));
    if (Lambda)
      for (int b = 0; b < h->L - 1; ++b) std::memcpy(Lambda[b], h->h_lam[b].data(), h->h_lam[b].size() * sizeof(double));
  } catch (const TdvpError& e) {
    return fail(h, e);
  }
  return TDVP_OK;
}

const char* tdvp_last_error(tdvp_t h) { return h ? h->err.c_str() : "null handle"; }

void tdvp_destroy(tdvp_t h) { delete h; }

int tdvp_nccl_unique_id(unsigned char* id128) {
  if (!id128) return TDVP_EARG;
  ncclUniqueId id;
  if (!nccl().ok || nccl().GetUniqueId(&id) != ncclSuccess) return TDVP_ECUDA;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(id128, &id, 128);
  return TDVP_OK;
}

int tdvp_comm_init(tdvp_t h, int rank, int world, const unsigned char* id128) {
  if (!h || !id128 || world < 1 || rank < 0 || rank >= world) return TDVP_EARG;
  try {
    ncclUniqueId id;
    std::memcpy(&id, id128, 128);
    NK(nccl().CommInitRank(&h->comm, world, id, rank));
    h->rank = rank;
    h->world = world;
    h->layout_p = 0;
    h->alloc_p = 0;
    h->segs.clear();
  } catch (const TdvpError& e) {
    return fail(h, e);
  }
  return TDVP_OK;
}

int tdvp_plan(int L, int p, int hh, int q, int* ops, int max_ops) {
  std::vector<std::pair<int, int>> b;
  std::string err;
  if (!plan_partition(L, p, b, err)) return TDVP_EPARTITION;
  if (hh < 1 || hh > 2 || q < 0 || q >= p) return TDVP_EARG;
  const std::set<int> merged = merged_pairs(L, p, b);
  const std::vector<SchedOp> prog = segment_program(L, p, hh, q, b[q], merged);
  if ((int)prog.size() > max_ops) return TDVP_EARG;
  for (size_t i = 0; i < prog.size(); ++i) {
    ops[4 * i] = prog[i].kind;
    ops[4 * i + 1] = prog[i].j;
    ops[4 * i + 2] = prog[i].full;
    ops[4 * i + 3] = prog[i].build;
  }
  return (int)prog.size();
}

int tdvp_plan1(int L, int p, int hh, int q, int* ops, int max_ops) {
  std::vector<std::pair<int, int>> b;
  std::string err;
  if (!plan_partition(L, p, b, err)) return TDVP_EPARTITION;
  if (hh < 1 || hh > 2 || q < 0 || q >= p) return TDVP_EARG;
  std::set<int> pairs, sites;
  merged1(L, p, b, pairs, sites);
  const std::vector<SchedOp> prog = segment_program1(L, p, hh, q, b[q], pairs, sites);
  if ((int)prog.size() > max_ops) return TDVP_EARG;
  for (size_t i = 0; i < prog.size(); ++i) {
    ops[4 * i] = prog[i].kind;
    ops[4 * i + 1] = prog[i].j;
    ops[4 * i + 2] = prog[i].full;
    ops[4 * i + 3] = prog[i].build;
  }
  return (int)prog.size();
}

int tdvp_set_partition(tdvp_t h, int p, const int* s) {
  if (!h) return TDVP_EARG;
  try {
    if (p == 0) {
      h->custom.clear();
    } else {
      if (!s) throw TdvpError(TDVP_EARG, "null segment starts");
      const int L = h->L;
      if (p < 2 || p % 2 != 0 || p > L / 2) throw TdvpError(TDVP_EPARTITION, "p must be even, 2 <= p <= L/2");
      if (s[0] != 0) throw TdvpError(TDVP_EPARTITION, "the first segment must start at site 0");
      std::vector<std::pair<int, int>> b(p);
      for (int q = 0; q < p; ++q) {
        const int e = q + 1 < p ? s[q + 1] - 1 : L - 1;
        if (e - s[q] + 1 < 2) throw TdvpError(TDVP_EPARTITION, "segment shorter than two sites (PAPER.md:470)");
        b[q] = {s[q], e};
      }
      h->custom = b;
    }
    h->envs_valid = false;  // re-layout (state kept) at the next step
  } catch (const TdvpError& e) {
    return fail(h, e);
  }
  return TDVP_OK;
}

int tdvp_partition_balanced(int L, int p, const int* chi, int* s, int* e) {
  if (L < 2 || !chi || !s || !e) return TDVP_EARG;
  return balanced_partition(L, p, chi, s, e, nullptr);
}

int tdvp_get_partition(tdvp_t h, int* p, int* s, int* e) {
  if (!h || !p) return TDVP_EARG;
  *p = (int)h->bounds.size();
  if (s && e)
    for (size_t q = 0; q < h->bounds.size(); ++q) {
      s[q] = h->bounds[q].first;
      e[q] = h->bounds[q].second;
    }
  return TDVP_OK;
}

int tdvp_partition(int L, int p, int* s, int* e) {
  std::vector<std::pair<int, int>> b;
  std::string err;
  if (!plan_partition(L, p, b, err)) return TDVP_EPARTITION;
  for (int q = 0; q < p; ++q) {
    s[q] = b[q].first;
    e[q] = b[q].second;
  }
  return TDVP_OK;
}

// ----------------------------------------------------- kernel-level entries
static int upload_run_download(const std::function<void(tdvp_ctx*)>& fn) {
  try {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) throw TdvpError(TDVP_ECUDA, "no CUDA device");
    fn(nullptr);
  } catch (const TdvpError& e) {
    std::fprintf(stderr, "libtdvp: %s\n", e.what());
    return e.code;
  }
  return TDVP_OK;
}

static BufPtr up(const double* p, size_t ncplx, cudaStream_t st) {
  BufPtr b = make_buf(ncplx * sizeof(cplx));
  CK(cudaMemcpyAsync(b->p, p, ncplx * sizeof(cplx), cudaMemcpyHostToDevice, st));
  return b;
}

int tdvp_apply_heff2(int cl, int cr, int d, int Dl, int Dm, int Dr, const double* Lenv, const double* W1,
                     const double* W2, const double* Renv, const double* theta, double* out) {
  if (d != 2) return TDVP_EARG;
  return upload_run_download([&](tdvp_ctx*) {
    tdvp_ctx* h = scratch_ctx(std::max(cl, cr), std::max(Dl, std::max(Dm, Dr)));
    MpoSite w1, w2;
    build_site(w1, Dl, Dm, d, to_cplx(W1, (size_t)Dl * d * d * Dm));
    build_site(w2, Dm, Dr, d, to_cplx(W2, (size_t)Dm * d * d * Dr));
    build_pair(w1, Dl, Dm, Dr, d, to_cplx(W1, (size_t)Dl * d * d * Dm), to_cplx(W2, (size_t)Dm * d * d * Dr));
    BufPtr L_ = up(Lenv, (size_t)cl * Dl * cl, h->st), R_ = up(Renv, (size_t)cr * Dr * cr, h->st);
    const size_t n = (size_t)cl * d * d * cr;
    BufPtr x = up(theta, n, h->st), y = make_buf(n * sizeof(cplx));
    heff2(h, L_->c(), w1, w2, R_->c(), cl, cr, x->c(), y->c());
    CK(cudaMemcpyAsync(out, y->p, n * sizeof(cplx), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
  });
}

int tdvp_apply_heff1(int cl, int cr, int d, int Dl, int Dr, const double* Lenv, const double* W, const double* Renv,
                     const double* psi, double* out) {
  if (d != 2) return TDVP_EARG;
  return upload_run_download([&](tdvp_ctx*) {
    tdvp_ctx* h = scratch_ctx(std::max(cl, cr), std::max(Dl, Dr));
    MpoSite w;
    build_site(w, Dl, Dr, d, to_cplx(W, (size_t)Dl * d * d * Dr));
    BufPtr L_ = up(Lenv, (size_t)cl * Dl * cl, h->st), R_ = up(Renv, (size_t)cr * Dr * cr, h->st);
    const size_t n = (size_t)cl * d * cr;
    BufPtr x = up(psi, n, h->st), y = make_buf(n * sizeof(cplx));
    heff1(h, L_->c(), w, R_->c(), cl, cr, x->c(), y->c());
    CK(cudaMemcpyAsync(out, y->p, n * sizeof(cplx), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
  });
}

int tdvp_env_left(int cl, int cr, int d, int Dl, int Dr, const double* beta, const double* A, const double* W,
                  double* out) {
  if (d != 2) return TDVP_EARG;
  return upload_run_download([&](tdvp_ctx*) {
    tdvp_ctx* h = scratch_ctx(std::max(cl, cr), std::max(Dl, Dr));
    MpoSite w;
    build_site(w, Dl, Dr, d, to_cplx(W, (size_t)Dl * d * d * Dr));
    BufPtr b = up(beta, (size_t)cl * Dl * cl, h->st), a = up(A, (size_t)cl * d * cr, h->st);
    const size_t n = (size_t)cr * Dr * cr;
    BufPtr y = make_buf(n * sizeof(cplx));
    env_left(h, b->c(), a->c(), w, cl, cr, y->c());
    CK(cudaMemcpyAsync(out, y->p, n * sizeof(cplx), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
  });
}

int tdvp_env_right(int cl, int cr, int d, int Dl, int Dr, const double* gamma, const double* B, const double* W,
                   double* out) {
  if (d != 2) return TDVP_EARG;
  return upload_run_download([&](tdvp_ctx*) {
    tdvp_ctx* h = scratch_ctx(std::max(cl, cr), std::max(Dl, Dr));
    MpoSite w;
    build_site(w, Dl, Dr, d, to_cplx(W, (size_t)Dl * d * d * Dr));
    BufPtr g = up(gamma, (size_t)cr * Dr * cr, h->st), b = up(B, (size_t)cl * d * cr, h->st);
    const size_t n = (size_t)cl * Dl * cl;
    BufPtr y = make_buf(n * sizeof(cplx));
    env_right(h, g->c(), b->c(), w, cl, cr, y->c());
    CK(cudaMemcpyAsync(out, y->p, n * sizeof(cplx), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
  });
}

int tdvp_expm_lanczos_dense(int n, const double* H, const double* v, double tau_re, double tau_im, int K, double* out) {
  if (n < 1 || K < 1 || K >= KMAX) return TDVP_EARG;
  return upload_run_download([&](tdvp_ctx*) {
    const int chi = std::max(1, (int)std::ceil(std::sqrt(n / 4.0)) + 1);
    tdvp_ctx* h = scratch_ctx(std::max(chi, 8), 1);
    if ((long long)n > h->n2max) throw TdvpError(TDVP_EARG, "n too large for scratch context");
    BufPtr Hd = up(H, (size_t)n * n, h->st), x = up(v, n, h->st), y = make_buf((size_t)n * sizeof(cplx));
    expm_lanczos(
        h,
        [&](const cplx* a, cplx* b) {
          gemm(h, OP_N, OP_N, n, 1, n, Hd->c(), n, a, 1, b, 1);
        },
        x->c(), y->c(), n, tau_re, tau_im, K, 0, 0.0);
    CK(cudaMemcpyAsync(out, y->p, (size_t)n * sizeof(cplx), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
  });
}

int tdvp_svd_split(int m, int n, const double* M, int chi_max, double eps, double w_max, double delta, int* chi,
                   double* w, double* psiL, double* lam, double* psiR) {
  if (m < 1 || n < 1 || chi_max < 1) return TDVP_EARG;
  int rc = upload_run_download([&](tdvp_ctx*) {
    tdvp_ctx* h = scratch_ctx(std::max(8, (std::max(m, n) + 1) / 2 + 1), 1);
    if ((long long)svd_work_elems(m, n) > h->svdmax || (long long)m * n > h->n2max)
      throw TdvpError(TDVP_EARG, "matrix too large for scratch context");
    BufPtr a = up(M, (size_t)m * n, h->st);
    const int k = std::min(m, n);
    BufPtr pl = make_buf((size_t)m * k * sizeof(cplx)), pr = make_buf((size_t)k * n * sizeof(cplx));
    BufPtr l = make_buf(k * sizeof(double)), vi = make_buf(k * sizeof(double));
    TruncParams tp{chi_max, eps, w_max, delta};
    int c = 0, r = 0, ce = 0, sw = 0;
    double ww = 0.0;
    cudaError_t se = svd_truncate_split(h->st, h->sv, a->c(), m, n, tp, pl->c(), pr->c(), l->d(), vi->d(), &c, &ww, &r,
                                        &ce, &sw);
    if (se == cudaErrorUnknown) throw TdvpError(TDVP_ENUMERIC, "SVD numerical failure");
    CK(se);
    CK(cudaMemcpyAsync(psiL, pl->p, (size_t)m * c * sizeof(cplx), cudaMemcpyDeviceToHost, h->st));
    CK(cudaMemcpyAsync(psiR, pr->p, (size_t)c * n * sizeof(cplx), cudaMemcpyDeviceToHost, h->st));
    CK(cudaMemcpyAsync(lam, l->p, c * sizeof(double), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    *chi = c;
    *w = ww;
  });
  return rc;
}

int tdvp_zgemm(int opA, int opB, int M, int N, int K, const double* A, const double* B, double* C) {
  if (M < 1 || N < 1 || K < 1 || opA < 0 || opA > 3 || opB < 0 || opB > 3) return TDVP_EARG;
  return upload_run_download([&](tdvp_ctx*) {
    init_device_globals();
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    BufPtr a = up(A, (size_t)M * K, st), b = up(B, (size_t)K * N, st), c = make_buf((size_t)M * N * sizeof(cplx));
    const bool ta = (opA == 1 || opA == 2), tb = (opB == 1 || opB == 2);
    BufPtr work = make_buf((size_t)(1 << 22) * sizeof(cplx));
    CK(zgemm(st, opA, opB, M, N, K, ONE, a->c(), ta ? M : K, b->c(), tb ? K : N, ZERO, c->c(), N, 1, 0, 0, 0,
             work->c(), (size_t)1 << 22));
    CK(cudaMemcpyAsync(C, c->p, (size_t)M * N * sizeof(cplx), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaStreamDestroy(st));
  });
}


// ----------------------------------------------------- microbenchmarks (device-resident operands)
int tdvp_bench_heff2(int chi, int Dl, int Dm, int Dr, const double* W1, const double* W2, int reps, double* ms,
                     double* flop) {
  if (chi < 1 || reps < 1) return TDVP_EARG;
  return upload_run_download([&](tdvp_ctx*) {
    tdvp_ctx* h = scratch_ctx(chi, std::max(Dl, std::max(Dm, Dr)));
    const int d = 2;
    MpoSite w1, w2;
    build_site(w1, Dl, Dm, d, to_cplx(W1, (size_t)Dl * d * d * Dm));
    build_site(w2, Dm, Dr, d, to_cplx(W2, (size_t)Dm * d * d * Dr));
    build_pair(w1, Dl, Dm, Dr, d, to_cplx(W1, (size_t)Dl * d * d * Dm), to_cplx(W2, (size_t)Dm * d * d * Dr));
    const size_t nL = (size_t)chi * Dl * chi, nR = (size_t)chi * Dr * chi, n = (size_t)chi * d * d * chi;
    BufPtr L_ = make_buf(nL * sizeof(cplx)), R_ = make_buf(nR * sizeof(cplx)), x = make_buf(n * sizeof(cplx)),
           y = make_buf(n * sizeof(cplx));
    CK(fill_cplx(h->st, L_->c(), cmk(0.01, -0.02), (long long)nL));
    CK(fill_cplx(h->st, R_->c(), cmk(-0.03, 0.01), (long long)nR));
    CK(fill_cplx(h->st, x->c(), cmk(0.5, 0.25), (long long)n));
    heff2(h, L_->c(), w1, w2, R_->c(), chi, chi, x->c(), y->c());  // warm-up
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, h->st));
    for (int r = 0; r < reps; ++r) heff2(h, L_->c(), w1, w2, R_->c(), chi, chi, (r & 1) ? y->c() : x->c(), (r & 1) ? x->c() : y->c());
    CK(cudaEventRecord(e1, h->st));
    CK(cudaEventSynchronize(e1));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, e0, e1));
    *ms = t / reps;
    *flop = flops_heff2(chi, chi, d, Dl, Dr, nnz_of(w1), nnz_of(w2));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

int tdvp_bench_svd(int m, int n, const double* M, int reps, double* ms, int* sweeps) {
  if (m < 1 || n < 1 || reps < 1) return TDVP_EARG;
  return upload_run_download([&](tdvp_ctx*) {
    tdvp_ctx* h = scratch_ctx(std::max(8, (std::max(m, n) + 1) / 2 + 1), 1);
    BufPtr a = up(M, (size_t)m * n, h->st);
    const int k = std::min(m, n);
    BufPtr pl = make_buf((size_t)m * k * sizeof(cplx)), pr = make_buf((size_t)k * n * sizeof(cplx));
    BufPtr l = make_buf(k * sizeof(double)), vi = make_buf(k * sizeof(double));
    TruncParams tp{k, 1e-12, 0.0, 1e-6};
    int c = 0, r = 0, ce = 0, sw = 0;
    double ww = 0.0;
    CK(svd_truncate_split(h->st, h->sv, a->c(), m, n, tp, pl->c(), pr->c(), l->d(), vi->d(), &c, &ww, &r, &ce, &sw));
    CK(cudaStreamSynchronize(h->st));
    const auto t0 = std::chrono::high_resolution_clock::now();
    for (int i = 0; i < reps; ++i)
      CK(svd_truncate_split(h->st, h->sv, a->c(), m, n, tp, pl->c(), pr->c(), l->d(), vi->d(), &c, &ww, &r, &ce, &sw));
    CK(cudaStreamSynchronize(h->st));
    const auto t1 = std::chrono::high_resolution_clock::now();
    *ms = std::chrono::duration<double, std::milli>(t1 - t0).count() / reps;
    *sweeps = sw;
  });
}

}  // extern "C"
