// ksvd.cu -- C ABI (include/ksvd.h) over the sm_100a kernels in kernels.cuh.
//
// One context per GPU / process.  The GK loop (bidiag.py:111-184) is driven
// from here: the host enqueues whole steps on the context stream, keeps all
// scalars (alpha, beta) and the halting status on the device, and only
// waits on the status of step i-kLag before enqueueing step i, so the GPU
// never idles on a host round trip.  The stop rule depends only on device
// status words that are identical on every rank, so all ranks issue the
// same NCCL collectives in the same order.
#include <cuda_runtime.h>
#include <nccl.h>

#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <map>
#include <mutex>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "gen.cuh"
#include "pair.cuh"
#include "kernels.cuh"
#include "klrm.cuh"
#include "resident.cuh"
#include "peer.cuh"
#include "ksvd.h"

using namespace ksvd;

// ---------------------------------------------------------------------------
// errors
static thread_local std::string g_err;

static int set_err(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess)                                                     \
      return set_err(KSVD_ERUNTIME, "%s failed: %s (%s:%d)", #x,              \
                     cudaGetErrorString(e_), __FILE__, __LINE__);              \
  } while (0)
#define NK(x)                                                                  \
  do {                                                                         \
    ncclResult_t r_ = (x);                                                     \
    if (r_ != ncclSuccess)                                                     \
      return set_err(KSVD_ERUNTIME, "%s failed: %s", #x,                      \
                     ncclGetErrorString(r_));                                  \
  } while (0)
#define TRY(x)                                                                 \
  do {                                                                         \
    int rc_ = (x);                                                             \
    if (rc_) return rc_;                                                       \
  } while (0)

int ksvd_set_error_from_host(int code, const char* msg) { return set_err(code, "%s", msg); }

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
static inline int64_t rup(int64_t a, int64_t b) { return cdiv(a, b) * b; }

// cudaFuncAttributeMaxDynamicSharedMemorySize applies per device: set it
// once per (kernel, device) -- a context on a second GPU of the process gets
// its own -- and check the return code.
static int smem_attr(const void* kern, int device, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(kern, device);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return 0;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done[key] = bytes;
  return 0;
}

// ---------------------------------------------------------------------------
// context
enum KClass {
  KC_GEMV_N = 0, KC_GEMV_T = 1, KC_CGS = 2, KC_OTHER = 3, KC_FIN = 4, KC_RESIDENT = 5, KC_NUM = 6
};

struct ksvd_ctx {
  int device = 0, rank = 0, nranks = 1, sms = 148;
  cudaStream_t stream = nullptr;
  ncclComm_t comm = nullptr;
  // NVLink peer exchange (peer.cuh): replaces ncclAllReduce once opened
  bool px = false;
  int64_t px_slot = 0;
  void* px_local = nullptr;  // this rank's receive area + counters (IPC-exported)
  double* px_recv[kPxMaxRanks] = {};
  unsigned long long* px_cnt[kPxMaxRanks] = {};
  void* px_mapped[kPxMaxRanks] = {};  // opened IPC mappings (to close)
  unsigned long long px_seq = 0;
  unsigned long long px_arrivals = 0;  // cumulative CTAs each sender has pushed (same on all ranks)
  int* px_err = nullptr;
  int64_t launches = 0;
  bool profiling = false;
  struct Prof {
    cudaEvent_t a, b;
    int cls;
  };
  std::vector<Prof> pending;
  std::vector<cudaEvent_t> pool;
  double prof_ms[KC_NUM] = {};
  int64_t prof_n[KC_NUM] = {};
  cudaEvent_t marks[8] = {};
  // GK-loop pacing (one loop at a time per context)
  HostProg* hprog = nullptr;  // mapped host memory (host view)
  HostProg* dprog = nullptr;  // device view of the same memory
  cudaEvent_t ring_ev[8] = {};
  unsigned long long* tdbg = nullptr;  // KSVD_PHASE_TIMES: CGS phase timing
  // pinned staging ring for pageable host <-> device matrix transfers
  void* stage[2] = {nullptr, nullptr};
  size_t stage_bytes = 0;
  cudaEvent_t stage_ev[2] = {};
  // grid-barrier kernels: regular launches (all CTAs resident, probed at
  // creation) or, where residency is not guaranteed, cooperative launches
  bool coop_cgs = false;
};

static int get_event(ksvd_ctx* c, cudaEvent_t* ev) {
  if (!c->pool.empty()) {
    *ev = c->pool.back();
    c->pool.pop_back();
    return 0;
  }
  CK(cudaEventCreate(ev));
  return 0;
}

static int collect_profile(ksvd_ctx* c) {
  if (c->pending.empty()) return 0;
  CK(cudaStreamSynchronize(c->stream));
  for (auto& p : c->pending) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, p.a, p.b));
    c->prof_ms[p.cls] += ms;
    c->prof_n[p.cls] += 1;
    c->pool.push_back(p.a);
    c->pool.push_back(p.b);
  }
  c->pending.clear();
  return 0;
}

// Programmatic dependent launch for the GK step kernels: the next kernel's
// CTAs are scheduled while the current one drains and run their prologue
// (k_cgs2_tile2 / k_cgs_tile_phase: the TMA load of the basis tile) before
// griddepcontrol.wait.  Every kernel launched this way calls pdl_wait() in
// every CTA before touching its predecessor's outputs (kernels.cuh).
// Multi-rank: only our own step kernels carry the attribute; the kernels
// that trigger early (k_gemv_n, k_gemv_t2) are always followed by one of
// ours, never directly by a collective, so an NCCL kernel never starts
// before its input is complete (KSVD_PDL_MULTI=0 disables PDL there).
static bool pdl_enabled(const ksvd_ctx* c) {
  static const bool off = [] {
    const char* e = getenv("KSVD_PDL");
    return e && strcmp(e, "0") == 0;
  }();
  static const bool multi_off = [] {
    const char* e = getenv("KSVD_PDL_MULTI");
    return e && strcmp(e, "0") == 0;
  }();
  return !off && (c->comm == nullptr || !multi_off);
}

template <typename... KArgs, typename... Args>
static int launch_impl(ksvd_ctx* c, int cls, bool pdl, void (*kernel)(KArgs...), dim3 grid,
                       dim3 block, size_t smem, Args... args) {
  cudaEvent_t a = nullptr, b = nullptr;
  if (c->profiling) {
    TRY(get_event(c, &a));
    TRY(get_event(c, &b));
    CK(cudaEventRecord(a, c->stream));
  }
  if (pdl) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
  } else {
    kernel<<<grid, block, smem, c->stream>>>(args...);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return set_err(KSVD_ERUNTIME, "kernel launch failed: %s", cudaGetErrorString(e));
  if (c->profiling) {
    CK(cudaEventRecord(b, c->stream));
    c->pending.push_back({a, b, cls});
  }
  c->launches++;
  return 0;
}
template <typename... KArgs, typename... Args>
static int launch(ksvd_ctx* c, int cls, void (*kernel)(KArgs...), dim3 grid, dim3 block,
                  size_t smem, Args... args) {
  return launch_impl(c, cls, false, kernel, grid, block, smem, args...);
}
template <typename... KArgs, typename... Args>
static int launch_step(ksvd_ctx* c, int cls, void (*kernel)(KArgs...), dim3 grid, dim3 block,
                       size_t smem, Args... args) {
  return launch_impl(c, cls, pdl_enabled(c), kernel, grid, block, smem, args...);
}

static PxArgs px_args(ksvd_ctx* c, double* buf, size_t count, int64_t* grid) {
  PxArgs a{};
  a.buf = buf;
  a.L = (int64_t)count;
  for (int r = 0; r < c->nranks; ++r) {
    a.recv[r] = c->px_recv[r];
    a.cnt[r] = c->px_cnt[r];
  }
  a.my_recv = c->px_recv[c->rank];
  a.my_cnt = c->px_cnt[c->rank];
  a.rank = c->rank;
  a.N = c->nranks;
  a.seq = ++c->px_seq;
  a.slot = c->px_slot;
  a.err = c->px_err;
  // a few CTAs (each spins until all peers' CTAs pushed: far below a wave)
  const int64_t G = std::max<int64_t>(1, std::min<int64_t>(16, cdiv((int64_t)count, 2048)));
  c->px_arrivals += (unsigned long long)G;  // counters are cumulative over collectives
  a.want = c->px_arrivals;
  *grid = G;
  return a;
}

static int px_allreduce(ksvd_ctx* c, double* buf, size_t count) {
  int64_t G = 1;
  const PxArgs a = px_args(c, buf, count, &G);
  k_px_allreduce<<<(unsigned)G, kThreads, 0, c->stream>>>(a);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(KSVD_ERUNTIME, "peer all-reduce: %s", cudaGetErrorString(e));
  c->launches++;
  return 0;
}

static int allreduce(ksvd_ctx* c, double* buf, size_t count) {
  if (!c->comm || count == 0) return 0;
  if (c->px && (int64_t)count <= c->px_slot) return px_allreduce(c, buf, count);
  NK(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, c->comm, c->stream));
  return 0;
}

// ---------------------------------------------------------------------------
// matrices
struct GemvNPlan {
  int V, U, nchunks, ngroups;  // ngroups: partial sums per row (chunk groups of 8)
  int64_t nvec, nseg, blocks;
};
struct GemvTPlan {
  int64_t ncoltiles, nsplit, rows_per_split;
  int rg;  // row groups per CTA (k_gemv_t RG)
};

constexpr int kUnrollN = 2;  // U of k_gemv_n (32*U 16-byte vectors per warp chunk)
constexpr int kUnrollT = 16;   // U of k_gemv_t
constexpr int kGemvTCtasPerSm = 4;

struct ksvd_mat {
  ksvd_ctx* ctx = nullptr;
  int64_t m = 0, n = 0, row0 = 0, mloc = 0, lda = 0;
  int64_t n_pad = 0, m_pad = 0;  // vector lengths (512 B multiples)
  int dtype = KSVD_F64;
  void* A = nullptr;
  GemvNPlan pn{};
  GemvTPlan pt{};
  double* part_n = nullptr;  // ngroups x mloc: k_gemv_n partial row sums
  unsigned* seg_cnt = nullptr;  // nseg arrival counters (k_gemv_n<FIN>)
  double* part_t = nullptr;  // nsplit x n_pad
  // plain-product scratch
  double *dx = nullptr, *dy = nullptr;
  DevState* st0 = nullptr;  // always-running state for plain products
  // generator factors (ksvd_matrix_generate): Ps = P diag(s) local rows, Q
  double *gen_ps = nullptr, *gen_q = nullptr;
  int gen_r = 0;
  // factored operator L C R^T (ksvd_matrix_from_factors, reference
  // linops.py:176-205): L = this rank's rows (mloc x s1), R replicated
  // (n x s2), both dense sub-matrices; C (s1 x s2) and two vectors on device
  struct Factored {
    ksvd_mat *L = nullptr, *R = nullptr;
    double *C = nullptr, *t1 = nullptr, *t2 = nullptr;
    int64_t s1 = 0, s2 = 0;
  }* fac = nullptr;
};

static size_t esize(int dtype) { return dtype == KSVD_F32 ? 4 : 8; }

template <typename TA>
static int occupancy_n(int* out) {
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, k_gemv_n<TA, kUnrollN, false>, kThreads, 0));
  return 0;
}

static int plan_matrix(ksvd_mat* M) {
  ksvd_ctx* c = M->ctx;
  const int64_t bytes = esize(M->dtype);
  GemvNPlan& pn = M->pn;
  pn.V = (int)(16 / bytes);
  pn.U = kUnrollN;
  pn.nvec = cdiv(M->n, pn.V);
  pn.nchunks = (int)cdiv(pn.nvec, 32 * pn.U);
  pn.ngroups = (int)cdiv(pn.nchunks, kWarps);
  int occ = 1;
  if (M->dtype == KSVD_F32)
    TRY(occupancy_n<float>(&occ));
  else
    TRY(occupancy_n<double>(&occ));
  occ = std::max(occ, 1);
  // row segments: one wave of CTAs (ngroups per segment), capped by the
  // 8-row blocks
  pn.nseg = std::max<int64_t>(1, std::min<int64_t>((int64_t)c->sms * occ / pn.ngroups,
                                                   cdiv(std::max<int64_t>(M->mloc, 1), 8)));
  pn.blocks = pn.nseg * pn.ngroups;

  GemvTPlan& pt = M->pt;
  // RG row groups: narrower column tiles -> fewer row splits -> a short
  // partial-sum finalisation (KSVD_GEMVT_RG overrides, for experiments)
  pt.rg = 8;
  if (const char* e = getenv("KSVD_GEMVT_RG")) pt.rg = atoi(e);
  if (pt.rg != 1 && pt.rg != 2 && pt.rg != 4 && pt.rg != 8) pt.rg = 8;
  pt.ncoltiles = cdiv(pn.nvec, kThreads / pt.rg);
  const int64_t target = (int64_t)c->sms * kGemvTCtasPerSm;
  int64_t nsplit = std::max<int64_t>(1, cdiv(target, pt.ncoltiles));
  int64_t rps = std::max<int64_t>(64, cdiv(std::max<int64_t>(M->mloc, 1), nsplit));
  pt.rows_per_split = rps;
  pt.nsplit = std::max<int64_t>(1, cdiv(M->mloc, rps));
  return 0;
}

// Leading dimension of A on the device: rows padded to a 16-byte multiple
// only (what the 16-byte vector loads and bulk copies need), so a
// contiguous host matrix uploads as ONE DMA.  KSVD_LDA_BYTES=512 restores
// 512-byte row alignment (measured equivalent for the streaming kernels).
static int64_t lda_for(int64_t n, int64_t es) {
  static const int64_t align = [] {
    const char* e = getenv("KSVD_LDA_BYTES");
    const long v = e ? atol(e) : 16;
    return (int64_t)(v >= 16 && (v & (v - 1)) == 0 ? v : 16);
  }();
  return rup(n, align / es);
}

// All matrix buffers come from the stream-ordered pool (no device-wide
// synchronisation on allocation or free; the pool keeps its memory).
static int alloc_matrix_buffers(ksvd_mat* M) {
  cudaStream_t s = M->ctx->stream;
  const size_t abytes = (size_t)M->mloc * M->lda * esize(M->dtype);
  CK(cudaMallocAsync(&M->A, std::max<size_t>(abytes, 16), s));
  TRY(plan_matrix(M));
  const size_t vec = sizeof(double) * std::max(M->n_pad, M->m_pad);
  CK(cudaMallocAsync((void**)&M->part_n,
                     sizeof(double) * M->pn.ngroups * std::max<int64_t>(M->mloc, 1), s));
  CK(cudaMallocAsync((void**)&M->part_t, sizeof(double) * M->pt.nsplit * M->n_pad, s));
  CK(cudaMallocAsync((void**)&M->seg_cnt, sizeof(unsigned) * M->pn.nseg, s));
  CK(cudaMemsetAsync(M->seg_cnt, 0, sizeof(unsigned) * M->pn.nseg, s));
  CK(cudaMallocAsync((void**)&M->dx, vec, s));
  CK(cudaMallocAsync((void**)&M->dy, vec, s));
  CK(cudaMemsetAsync(M->dx, 0, vec, s));
  CK(cudaMemsetAsync(M->dy, 0, vec, s));
  CK(cudaMallocAsync((void**)&M->st0, sizeof(DevState), s));
  CK(cudaMemsetAsync(M->st0, 0, sizeof(DevState), s));
  return 0;
}

static int free_matrix(ksvd_mat* M) {
  if (!M) return 0;
  cudaStream_t s = M->ctx->stream;
  cudaSetDevice(M->ctx->device);
  if (M->fac) {
    free_matrix(M->fac->L);
    free_matrix(M->fac->R);
    for (double* p : {M->fac->C, M->fac->t1, M->fac->t2})
      if (p) cudaFreeAsync(p, s);
    delete M->fac;
    M->fac = nullptr;
  }
  for (void* p : {(void*)M->A, (void*)M->part_n, (void*)M->part_t, (void*)M->dx, (void*)M->dy,
                  (void*)M->st0, (void*)M->seg_cnt})
    if (p) cudaFreeAsync(p, s);
  cudaFree(M->gen_ps);
  cudaFree(M->gen_q);
  delete M;
  return 0;
}

// w = A p (- alpha q): partial row sums per chunk group (k_gemv_n), then
// the group sums + epilogue (k_gemv_n_finalize) unless the caller fuses the
// finalisation into its k_cgs2_* launch (finalize = false).
// L2 evict_first for A's loads (kernels.cuh a_policy) when A exceeds 2 GB
// (16 L2 capacities): same box, configs 3 / 4: k_gemv_n +1.3 / +0.6 %,
// k_gemv_t2 +0.5 / +0.7 %; on config 2 (0.8 GB) it costs k_gemv_t2 2.5 % of
// the rows k_gemv_n leaves in L2 (profiles/r02/a_evict_first_ab.txt).
// KSVD_A_EVICT_FIRST=0/1 forces it.
static int a_evict_first(const ksvd_mat* M) {
  static const int force = [] {
    const char* e = getenv("KSVD_A_EVICT_FIRST");
    return e ? (strcmp(e, "1") == 0 ? 1 : 0) : -1;
  }();
  if (force >= 0) return force;
  return (size_t)M->mloc * M->lda * esize(M->dtype) >= ((size_t)2 << 30) ? 1 : 0;
}

// tail_fin (the paired step): the finalisation runs in k_gemv_n's tail
// (FIN instantiation, per-segment arrival counters M->seg_cnt) instead.
static int dense_gemv_n(ksvd_mat* M, const double* p_src, const double* p_scale,
                        double* p_dst, const double* qprev, const double* alpha,
                        double* w, DevState* st, int step, bool finalize = true,
                        bool tail_fin = false) {
  ksvd_ctx* c = M->ctx;
  const GemvNPlan& pn = M->pn;
  if (M->mloc == 0) return 0;
  const dim3 grid((unsigned)pn.blocks);
  const GemvNFin nf{M->seg_cnt, qprev, alpha, w};
  // named-barrier CTA row sums (KSVD_GEMVN_NB=0: one __syncthreads per block);
  // same box: k_gemv_n 6,396-6,401 -> 6,444-6,449 GB/s on config 4, 6,804-6,823 ->
  // 6,847-6,855 on config 2 (profiles/r02/gemv_n_nb_ab.txt)
  static const bool nb = [] {
    const char* e = getenv("KSVD_GEMVN_NB");
    return !(e && strcmp(e, "0") == 0);
  }();
#define KSVD_GN(TA, F, B)                                                                   \
  launch_step(c, KC_GEMV_N, k_gemv_n<TA, kUnrollN, F, B>, grid, dim3(kThreads), 0,           \
              (const TA*)M->A, M->lda, M->mloc, pn.nvec, pn.nchunks, pn.ngroups, pn.nseg,    \
              p_src, p_scale, p_dst, M->n, M->part_n, (const DevState*)st, nf, a_evict_first(M))
  if (M->dtype == KSVD_F32) {
    if (nb) TRY(tail_fin ? KSVD_GN(float, true, true) : KSVD_GN(float, false, true));
    else TRY(tail_fin ? KSVD_GN(float, true, false) : KSVD_GN(float, false, false));
  } else {
    if (nb) TRY(tail_fin ? KSVD_GN(double, true, true) : KSVD_GN(double, false, true));
    else TRY(tail_fin ? KSVD_GN(double, true, false) : KSVD_GN(double, false, false));
  }
#undef KSVD_GN
  if (tail_fin) return 0;
  if (finalize)
    TRY(launch(c, KC_FIN, k_gemv_n_finalize, dim3((unsigned)cdiv(M->mloc, kThreads)),
               dim3(kThreads), 0, (const double*)M->part_n, M->mloc, pn.ngroups, M->mloc,
               qprev, alpha, w, st, step));
  return 0;
}

template <typename TA>
static int launch_gemv_t(ksvd_mat* M, dim3 grid, const double* q_src, const double* q_scale,
                         double* q_dst, DevState* st) {
  ksvd_ctx* c = M->ctx;
  const GemvTPlan& pt = M->pt;
  // band-ordered variant (k_gemv_t2): 256-row blocks when A is within a few
  // L2 capacities (the band starts on what k_gemv_n left in L2), 1024-row
  // blocks otherwise (same access granularity as contiguous splits)
  const size_t abytes = (size_t)M->mloc * M->lda * esize(M->dtype);
  if (pt.rg == 8) {
    if (abytes < ((size_t)2 << 30))
      return launch_step(c, KC_GEMV_T, k_gemv_t2<TA, kUnrollT, 8, 2>, grid, dim3(kThreads), 0,
                    (const TA*)M->A, M->lda, M->mloc, M->pn.nvec, pt.rows_per_split, q_src,
                    q_scale, q_dst, M->part_t, M->n_pad, (const DevState*)st, a_evict_first(M));
    return launch_step(c, KC_GEMV_T, k_gemv_t2<TA, kUnrollT, 8, 8>, grid, dim3(kThreads), 0,
                  (const TA*)M->A, M->lda, M->mloc, M->pn.nvec, pt.rows_per_split, q_src,
                  q_scale, q_dst, M->part_t, M->n_pad, (const DevState*)st, a_evict_first(M));
  }
#define KSVD_GT(RG)                                                                    \
  launch_step(c, KC_GEMV_T, k_gemv_t<TA, kUnrollT, RG>, grid, dim3(kThreads), 0,             \
         (const TA*)M->A, M->lda, M->mloc, M->pn.nvec, pt.rows_per_split, q_src, q_scale, \
         q_dst, M->part_t, M->n_pad, (const DevState*)st)
  switch (pt.rg) {
    case 1: return KSVD_GT(1);
    case 2: return KSVD_GT(2);
    default: return KSVD_GT(4);
  }
#undef KSVD_GT
}

// z = sum_ranks A^T q (- beta p): q_src/q_scale/q_dst per k_gemv_t.
static int dense_gemv_t(ksvd_mat* M, const double* q_src, const double* q_scale,
                        double* q_dst, const double* beta, const double* pprev,
                        double* z, DevState* st, int step, bool check,
                        bool finalize = true, bool axpy = true) {
  ksvd_ctx* c = M->ctx;
  const GemvTPlan& pt = M->pt;
  if (M->mloc > 0) {
    dim3 grid((unsigned)pt.ncoltiles, (unsigned)pt.nsplit);
    if (M->dtype == KSVD_F32)
      TRY(launch_gemv_t<float>(M, grid, q_src, q_scale, q_dst, st));
    else
      TRY(launch_gemv_t<double>(M, grid, q_src, q_scale, q_dst, st));
  } else {
    CK(cudaMemsetAsync(M->part_t, 0, sizeof(double) * M->n_pad, c->stream));
  }
  const int nsplit = M->mloc > 0 ? (int)pt.nsplit : 1;
  const bool multi = c->comm != nullptr;
  if (!finalize && !multi) return 0;  // fused into the caller's k_cgs2_tile2
  if (multi && c->px && M->n_pad <= c->px_slot) {
    // split sums + peer exchange + (- beta p) + check in one kernel
    int64_t G = 1;
    const PxArgs a = px_args(c, z, (size_t)M->n_pad, &G);
    k_gemv_t_fin_px<<<(unsigned)G, kThreads, 0, c->stream>>>(
        a, (const double*)M->part_t, M->n_pad, nsplit, M->n, beta, pprev, st, step,
        (int)check);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
      return set_err(KSVD_ERUNTIME, "A^T q exchange: %s", cudaGetErrorString(e));
    c->launches++;
    return 0;
  }
  TRY(launch(c, KC_FIN, k_gemv_t_finalize, dim3((unsigned)cdiv(M->n_pad, 32)),
             dim3(kThreads), 0, (const double*)M->part_t, M->n_pad, nsplit, M->n,
             M->n_pad, multi ? (const double*)nullptr : beta,
             multi ? (const double*)nullptr : pprev, z, st, step,
             (int)(check && !multi)));
  if (multi) {
    TRY(allreduce(c, z, (size_t)M->n_pad));
    if (axpy && (check || pprev))
      TRY(launch(c, KC_FIN, k_axpy_check, dim3((unsigned)cdiv(M->n, kThreads)),
                 dim3(kThreads), 0, z, beta, pprev, M->n, st, step));
  }
  return 0;
}

struct FinArgs {  // deferred gemv_t finalisation (phase 0 of k_cgs2_tile2)
  const double* part = nullptr;
  int64_t ld = 0;
  int nsplit = 0;
  const double* beta = nullptr;
  const double* p = nullptr;
};

// ---------------------------------------------------------------------------
// Factored operator products (reference linops.py:192-202):
//   A p   = L (C (R^T p))      A^T q = R (C^T (L^T q))
// built from the dense kernels on the sub-matrices plus an s x s core
// product; the last stage's partial sums have the k_gemv_n layout, so the
// CGS kernels fuse their finalisation exactly as for a dense A.  Multi-rank:
// L^T q is the only sharded reduction (an s-length all-reduce); R and C are
// replicated, so z is identical on every rank without another collective.
static int local_gemv_t(ksvd_mat* S, const double* q_src, const double* q_scale,
                        double* q_dst, double* out, DevState* st, int step) {
  ksvd_ctx* c = S->ctx;
  const GemvTPlan& pt = S->pt;
  if (S->mloc > 0) {
    dim3 grid((unsigned)pt.ncoltiles, (unsigned)pt.nsplit);
    TRY(launch_gemv_t<double>(S, grid, q_src, q_scale, q_dst, st));
  } else {
    CK(cudaMemsetAsync(S->part_t, 0, sizeof(double) * S->n_pad, c->stream));
  }
  return launch(c, KC_FIN, k_gemv_t_finalize, dim3((unsigned)cdiv(S->n_pad, 32)),
                dim3(kThreads), 0, (const double*)S->part_t, S->n_pad,
                S->mloc > 0 ? (int)pt.nsplit : 1, S->n, S->n_pad, (const double*)nullptr,
                (const double*)nullptr, out, st, step, 0);
}

static int core_gemv(ksvd_mat* M, int trans, const double* x, double* y, DevState* st) {
  const auto* F = M->fac;
  const int64_t outs = trans ? F->s2 : F->s1;
  return launch(M->ctx, KC_OTHER, k_core_gemv, dim3((unsigned)cdiv(outs, kWarps)),
                dim3(kThreads), 0, (const double*)F->C, F->s1, F->s2, trans, x, y,
                (const DevState*)st);
}

static int enqueue_gemv_n(ksvd_mat* M, const double* p_src, const double* p_scale,
                          double* p_dst, const double* qprev, const double* alpha,
                          double* w, DevState* st, int step, bool finalize = true) {
  if (!M->fac) return dense_gemv_n(M, p_src, p_scale, p_dst, qprev, alpha, w, st, step, finalize);
  auto* F = M->fac;
  TRY(local_gemv_t(F->R, p_src, p_scale, p_dst, F->t1, st, step));
  TRY(core_gemv(M, 0, F->t1, F->t2, st));
  return dense_gemv_n(F->L, F->t2, nullptr, nullptr, qprev, alpha, w, st, step, finalize);
}

static int enqueue_gemv_t(ksvd_mat* M, const double* q_src, const double* q_scale,
                          double* q_dst, const double* beta, const double* pprev,
                          double* z, DevState* st, int step, bool check,
                          bool finalize = true) {
  if (!M->fac)
    return dense_gemv_t(M, q_src, q_scale, q_dst, beta, pprev, z, st, step, check, finalize);
  auto* F = M->fac;
  TRY(local_gemv_t(F->L, q_src, q_scale, q_dst, F->t1, st, step));
  TRY(allreduce(M->ctx, F->t1, (size_t)F->s1));
  TRY(core_gemv(M, 1, F->t1, F->t2, st));
  return dense_gemv_n(F->R, F->t2, nullptr, nullptr, pprev, beta, z, st, step, finalize);
}

// where the CGS kernels find the last product's partial sums
static FinArgs fin_left(ksvd_mat* M, const double* alpha, const double* qprev) {
  ksvd_mat* S = M->fac ? M->fac->L : M;
  return FinArgs{S->part_n, S->mloc, S->mloc > 0 ? S->pn.ngroups : 0, alpha, qprev};
}
static FinArgs fin_right(ksvd_mat* M, const double* beta, const double* pprev) {
  if (M->fac) {
    ksvd_mat* S = M->fac->R;
    return FinArgs{S->part_n, S->mloc, S->pn.ngroups, beta, pprev};
  }
  return FinArgs{M->part_t, M->n_pad, M->mloc > 0 ? (int)M->pt.nsplit : 0, beta, pprev};
}

// ---------------------------------------------------------------------------
// CGS2 against a basis (bidiag.py:77-87, 154-156, 171-173)
struct CgsWork {
  double* part = nullptr;  // nrb x cap
  double* c = nullptr;     // cap
  double* red = nullptr;   // 2
  unsigned* bar = nullptr; // grid barrier {count, generation}
  int64_t part_elems = 0;
  int cap = 0;
};

static int choose_rpl(int64_t L) {
  // rows per lane of k_cgs_rows: keep >= ~600 row blocks for parallelism,
  // but fewer, fatter blocks for long vectors (shorter partial reductions)
  if (L >= 128 * 600) return 4;
  if (L >= 64 * 600) return 2;
  return 1;
}

// Grow-only, geometric, stream-ordered (cudaFree would synchronise the
// device inside the GK loop).
static int ensure_cgs(cudaStream_t s, CgsWork* w, int64_t nrb, int cols) {
  const int64_t need = nrb * std::max(cols, 1);
  if (need > w->part_elems) {
    const int64_t n = std::max(need, 2 * w->part_elems);
    if (w->part) CK(cudaFreeAsync(w->part, s));
    CK(cudaMallocAsync(&w->part, sizeof(double) * n, s));
    w->part_elems = n;
  }
  if (cols > w->cap || !w->c) {
    const int n = std::max(std::max(cols, 64), 2 * w->cap);
    if (w->c) CK(cudaFreeAsync(w->c, s));
    CK(cudaMallocAsync(&w->c, sizeof(double) * n, s));
    w->cap = n;
  }
  if (!w->red) CK(cudaMallocAsync(&w->red, sizeof(double) * 4, s));
  if (!w->bar) {
    CK(cudaMallocAsync((void**)&w->bar, sizeof(unsigned) * 2, s));
    CK(cudaMemsetAsync(w->bar, 0, sizeof(unsigned) * 2, s));
  }
  return 0;
}

template <int RPL>
static int cgs_impl(ksvd_ctx* c, CgsWork* W, const double* B, int64_t ldb, int ncols,
                    double* x, int64_t L, int passes, bool sharded, double eps,
                    double* slot, DevState* st, int step, int code, HostProg* hp,
                    int side) {
  const int64_t nrb = std::max<int64_t>(1, cdiv(L, 32 * RPL));
  TRY(ensure_cgs(c->stream, W, nrb, ncols));
  const bool multi = sharded && c->comm != nullptr;
  double* part = W->part;
  const dim3 grid((unsigned)nrb), block(kThreads);
  auto rows = k_cgs_rows<RPL>;
  if (ncols == 0) {
    TRY(launch(c, KC_CGS, rows, grid, block, 0, B, ldb, 0, (const double*)nullptr, x, L,
               kNorm, part, (int)nrb, (const DevState*)st));
  } else {
    // pass 1 coefficients
    TRY(launch(c, KC_CGS, rows, grid, block, 0, B, ldb, ncols, (const double*)nullptr, x, L,
               kDot, part, (int)nrb, (const DevState*)st));
    for (int pass = 1; pass <= passes; ++pass) {
      TRY(launch(c, KC_CGS, k_reduce_part, dim3((unsigned)ncols), block, 0,
                 (const double*)part, (int)nrb, W->c, (const DevState*)st));
      if (multi) TRY(allreduce(c, W->c, ncols));
      // update, fused with the next pass's coefficients or the final norm
      const int mode = kUpdate | (pass < passes ? kDot : kNorm);
      TRY(launch(c, KC_CGS, rows, grid, block, 0, B, ldb, ncols, (const double*)W->c, x, L,
                 mode, part, (int)nrb, (const DevState*)st));
    }
  }
  if (multi) {
    TRY(launch(c, KC_CGS, k_norm_prep, dim3(1), block, 0, (const double*)part, (int)nrb,
               W->red, (const DevState*)st));
    TRY(allreduce(c, W->red, 2));
    TRY(launch(c, KC_CGS, k_norm_test, dim3(1), block, 0, (const double*)nullptr, 0,
               (const double*)W->red, eps, slot, st, step, code, hp, side));
  } else {
    TRY(launch(c, KC_CGS, k_norm_test, dim3(1), block, 0, (const double*)part, (int)nrb,
               (const double*)nullptr, eps, slot, st, step, code, hp, side));
  }
  return 0;
}

// ---- single-rank fused CGS2 (k_cgs2_tile2) ----
constexpr size_t kTileSmemMax = 200 * 1024;  // basis tile budget of k_cgs2_tile2

// The fused single-kernel CGS2 is used where its basis tile fits in shared
// memory (one CTA per SM): there it beats the multi-kernel path by its
// launches; for long vectors (configs 3-5, left side) the multi-kernel path
// with ~L/128 CTAs streams the basis (measured: a one-wave cooperative grid
// streaming it from L2/HBM was slower, config 3 600 vs 581 ms per call).
// KSVD_COOP=0 forces the multi-kernel path (tests).
static bool coop_enabled(const ksvd_ctx* c, int64_t L, int ncols, bool sharded) {
  static const bool off = [] {
    const char* e = getenv("KSVD_COOP");
    return e && strcmp(e, "0") == 0;
  }();
  // a sharded basis needs all-reduces between the passes (multi-kernel path);
  // the replicated right basis takes the fused kernel at any rank count
  if (off || (sharded && c->comm != nullptr)) return false;
  const int64_t G = std::min<int64_t>(c->sms, std::max<int64_t>(1, cdiv(L, 32)));
  const int64_t rows = rup(cdiv(std::max<int64_t>(L, 1), G), 2);
  return rows <= 256 && sizeof(double) * (size_t)ncols * (size_t)(rows + 1) + 16 <= kTileSmemMax;
}

template <int MAXE>
static int tile_attr(int device) {
  return smem_attr((const void*)k_cgs2_tile2<MAXE>, device, (int)kTileSmemMax);
}

static int cgs_coop(ksvd_ctx* c, CgsWork* W, const double* B, int64_t ldb, int ncols, double* x,
                    int64_t L, int passes, double eps, double* slot, DevState* st, int step,
                    int code, HostProg* hp, int side, const FinArgs& fin) {
  CgsCoopArgs a{};
  a.B = B;
  a.ldb = ldb;
  a.ncols = ncols;
  a.x = x;
  a.L = L;
  a.passes = ncols > 0 ? passes : 0;
  a.eps = eps;
  a.slot = slot;
  a.st = st;
  a.step = step;
  a.code = code;
  a.hp = hp;
  a.side = side;
  a.fpart = fin.part;
  a.fld = fin.ld;
  a.fnsplit = fin.nsplit;
  a.fbeta = fin.beta;
  a.fp = fin.p;
  a.tdbg = c->tdbg;
  void* args[] = {&a};

  // tile-resident variant: one CTA per SM, each CTA's basis tile in smem
  // at least kCgsMinRows rows per CTA (KSVD_CGS_MINROWS overrides): fewer
  // CTAs make the cross-CTA reductions and barriers cheaper, more rows per
  // CTA make the shared-memory sweeps longer
  static const int64_t min_rows = [] {
    const char* e = getenv("KSVD_CGS_MINROWS");
    return e ? std::max<int64_t>(2, atoll(e)) : (int64_t)32;
  }();
  int64_t G = std::min<int64_t>(c->sms, std::max<int64_t>(1, cdiv(L, min_rows)));
  int64_t rows = rup(cdiv(std::max<int64_t>(L, 1), G), 2);
  G = std::max<int64_t>(1, cdiv(L, rows));
  const size_t tile_bytes = sizeof(double) * (size_t)ncols * (size_t)(rows + 1);
  const void* kern = nullptr;
  size_t smem = 0;
  if (!(rows <= 256 && tile_bytes + 16 <= kTileSmemMax))
    return set_err(KSVD_ERUNTIME, "internal: CGS2 tile of %lld rows x %d columns does not fit",
                   (long long)rows, ncols);
  smem = tile_bytes + 16;  // + the (ncols + 1)-th reduced sum
  switch ((int)cdiv(rows, 32)) {
#define KSVD_TILE_CASE(E)                  \
  case E:                                  \
    TRY(tile_attr<E>(c->device));          \
    kern = (const void*)k_cgs2_tile2<E>;   \
    break;
    KSVD_TILE_CASE(1)
    KSVD_TILE_CASE(2)
    KSVD_TILE_CASE(3)
    KSVD_TILE_CASE(4)
    KSVD_TILE_CASE(5)
    KSVD_TILE_CASE(6)
    KSVD_TILE_CASE(7)
    default:
      TRY(tile_attr<8>(c->device));
      kern = (const void*)k_cgs2_tile2<8>;
#undef KSVD_TILE_CASE
  }
  a.rows_per_cta = (int)rows;
  // k_cgs2_tile2 reduction mode: every CTA reads all G x (ncols + 1) partials
  // while that is cheaper than a second grid barrier (KSVD_RED_MAX doubles)
  static const int64_t red_max = [] {
    const char* e = getenv("KSVD_RED_MAX");
    return e ? (int64_t)atoll(e) : (int64_t)148 * 16;  // measured: configs 1-2
  }();
  a.redundant = G <= 160 && (int64_t)(ncols + 1) * G <= red_max;
  TRY(ensure_cgs(c->stream, W, G, 2 * (ncols + 1)));  // k_cgs2_tile2: ping-pong + norm row
  a.part = W->part;
  a.c = W->c;
  a.bar = W->bar;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->profiling) {
    TRY(get_event(c, &e0));
    TRY(get_event(c, &e1));
    CK(cudaEventRecord(e0, c->stream));
  }
  {
    // A regular launch with the flip barrier of grid_barrier, so
    // programmatic dependent launch starts the grid while the product
    // drains: its CTAs are scheduled only once every CTA of the product has
    // started, and all G <= #SMs of them are resident once the product's
    // CTAs retire (one CTA per SM).  Measured on config 2: 3692 vs 3624 GK
    // steps/s for a cooperative launch, whose ~6 us launch cannot overlap
    // the product's tail -- which stays the fallback where residency is not
    // guaranteed (ctx->coop_cgs, see residency_probe).
    const bool reg = !c->coop_cgs && G <= c->sms;
    if (!reg) a.bar = nullptr;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)G);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (!reg) {
      at[na].id = cudaLaunchAttributeCooperative;
      at[na].val.cooperative = 1;
      ++na;
    }
    if (pdl_enabled(c)) {
      at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    CK(cudaLaunchKernelExC(&cfg, kern, args));
  }
  if (c->profiling) {
    CK(cudaEventRecord(e1, c->stream));
    c->pending.push_back({e0, e1, KC_CGS});
  }
  c->launches++;
  return 0;
}

// x <- x orthogonalised `passes` times against B[:, :ncols]; *slot = ||x||;
// ||x|| < eps sets status `code` at `step`.
static int cgs(ksvd_ctx* c, CgsWork* W, const double* B, int64_t ldb, int ncols,
               double* x, int64_t L, int passes, bool sharded, double eps,
               double* slot, DevState* st, int step, int code, HostProg* hp = nullptr,
               int side = 0) {
  switch (choose_rpl(L)) {
    case 4:
      return cgs_impl<4>(c, W, B, ldb, ncols, x, L, passes, sharded, eps, slot, st, step, code,
                         hp, side);
    case 2:
      return cgs_impl<2>(c, W, B, ldb, ncols, x, L, passes, sharded, eps, slot, st, step, code,
                         hp, side);
    default:
      return cgs_impl<1>(c, W, B, ldb, ncols, x, L, passes, sharded, eps, slot, st, step, code,
                         hp, side);
  }
}

// ---- multi-rank CGS2 of a row-sharded basis, tile in shared memory ----
// k_cgs_tile_phase: 3 launches (2 with one pass) and k_norm_test around the
// 3 all-reduces, instead of the multi-kernel path's 8 launches.  Applies when
// this rank's rows give <= 256 rows per CTA and the tile fits shared memory
// (KSVD_MTILE=0 keeps the multi-kernel path).
struct TileGeom {
  int64_t G = 0, rows = 0;
  size_t smem = 0;
  bool ok = false;
};
static TileGeom tile_geom(const ksvd_ctx* c, int64_t L, int ncols) {
  TileGeom g;
  g.G = std::min<int64_t>(c->sms, std::max<int64_t>(1, cdiv(L, 32)));
  g.rows = rup(cdiv(std::max<int64_t>(L, 1), g.G), 2);
  g.G = std::max<int64_t>(1, cdiv(L, g.rows));
  const size_t tile_bytes = sizeof(double) * (size_t)ncols * (size_t)(g.rows + 1);
  g.smem = tile_bytes + 16;
  g.ok = L > 0 && ncols > 0 && g.rows <= 256 && g.smem <= kTileSmemMax;
  return g;
}
static bool multi_tile_enabled(const ksvd_ctx* c, int64_t L, int ncols) {
  static const bool off = [] {
    const char* e = getenv("KSVD_MTILE");
    return e && strcmp(e, "0") == 0;
  }();
  return !off && c->comm != nullptr && tile_geom(c, L, ncols).ok;
}

template <int E>
static const void* phase_kernel(int device) {
  const void* k = (const void*)k_cgs_tile_phase<E>;
  return smem_attr(k, device, (int)kTileSmemMax) == 0 ? k : nullptr;
}

static int cgs_tile_multi(ksvd_ctx* c, CgsWork* W, const double* B, int64_t ldb, int ncols,
                          double* x, int64_t L, int passes, double eps, double* slot,
                          DevState* st, int step, int code, HostProg* hp, int side,
                          const FinArgs& fin) {
  const TileGeom g = tile_geom(c, L, ncols);
  const void* kern = nullptr;
  switch ((int)cdiv(g.rows, 32)) {
    case 1: kern = phase_kernel<1>(c->device); break;
    case 2: kern = phase_kernel<2>(c->device); break;
    case 3: kern = phase_kernel<3>(c->device); break;
    case 4: kern = phase_kernel<4>(c->device); break;
    case 5: kern = phase_kernel<5>(c->device); break;
    case 6: kern = phase_kernel<6>(c->device); break;
    case 7: kern = phase_kernel<7>(c->device); break;
    default: kern = phase_kernel<8>(c->device); break;
  }
  if (!kern) return set_err(KSVD_ERUNTIME, "k_cgs_tile_phase: shared-memory attribute");
  TRY(ensure_cgs(c->stream, W, g.G, 2 * (ncols + 1)));
  CgsCoopArgs a{};
  a.B = B;
  a.ldb = ldb;
  a.ncols = ncols;
  a.x = x;
  a.L = L;
  a.rows_per_cta = (int)g.rows;
  a.st = st;
  a.step = step;
  a.part = W->part;
  a.c = W->c;
  // regular launch with the flip barrier (one CTA per SM, G <= #SMs), or a
  // cooperative launch where residency is not guaranteed (ctx->coop_cgs)
  a.bar = c->coop_cgs ? nullptr : W->bar;
  a.tdbg = nullptr;
  const int phases[3] = {0, 1, 2};
  for (int k = 0; k < 3; ++k) {
    int phase = phases[k];
    if (phase == 1 && passes < 2) continue;
    if (phase == 0) {
      a.fpart = fin.part;
      a.fld = fin.ld;
      a.fnsplit = fin.nsplit;
      a.fbeta = fin.beta;
      a.fp = fin.p;
    } else {
      a.fpart = nullptr;
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->profiling) {
      TRY(get_event(c, &e0));
      TRY(get_event(c, &e1));
      CK(cudaEventRecord(e0, c->stream));
    }
    void* args[] = {&a, &phase};
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)g.G);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = g.smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (c->coop_cgs) {
      at[na].id = cudaLaunchAttributeCooperative;
      at[na].val.cooperative = 1;
      ++na;
    }
    if (pdl_enabled(c)) {
      at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    CK(cudaLaunchKernelExC(&cfg, kern, args));
    if (c->profiling) {
      CK(cudaEventRecord(e1, c->stream));
      c->pending.push_back({e0, e1, KC_CGS});
    }
    c->launches++;
    TRY(allreduce(c, W->c, phase < 2 ? (size_t)ncols : 2));
  }
  return launch(c, KC_CGS, k_norm_test, dim3(1), dim3(kThreads), 0, (const double*)nullptr, 0,
                (const double*)W->c, eps, slot, st, step, code, hp, side);
}

// ---- both CGS2 of a step in one kernel (k_cgs2_pair, pair.cuh) ----
struct PairGeom {
  int64_t G[2] = {0, 0}, rows[2] = {0, 0};
  size_t smem = 0;
  int maxe = 0;
  bool ok = false;
};
static PairGeom pair_geom(const ksvd_ctx* c, int64_t L0, int64_t L1, int ncols) {
  PairGeom g;
  const int64_t Gt = c->sms;
  if (L0 <= 0 || L1 <= 0 || ncols <= 0 || Gt < 2) return g;
  // CTAs in proportion to the rows (equal rows per CTA on both sides), at
  // least 32 rows per CTA (k_cgs2_tile2's rule)
  int64_t G0 = std::llround((double)Gt * (double)L0 / (double)(L0 + L1));
  G0 = std::min<int64_t>(std::max<int64_t>(G0, 1), Gt - 1);
  const int64_t L[2] = {L0, L1};
  const int64_t Gs[2] = {G0, Gt - G0};
  for (int s = 0; s < 2; ++s) {
    int64_t Gi = std::min<int64_t>(Gs[s], std::max<int64_t>(1, cdiv(L[s], 32)));
    g.rows[s] = rup(cdiv(L[s], Gi), 2);
    g.G[s] = cdiv(L[s], g.rows[s]);
  }
  const int64_t rmax = std::max(g.rows[0], g.rows[1]);
  g.smem = sizeof(double) * ((size_t)ncols * (size_t)rmax + 2 * (size_t)(ncols + 1)) + 16;
  g.maxe = (int)cdiv(rmax, 32);
  g.ok = rmax <= 256 && g.smem <= kTileSmemMax && g.G[0] + g.G[1] <= c->sms;
  return g;
}
// KSVD_PAIR=0 restores the serialised step (two CGS2 kernels).
static bool pair_enabled(const ksvd_ctx* c, const ksvd_mat* M) {
  static const bool off = [] {
    const char* e = getenv("KSVD_PAIR");
    return e && strcmp(e, "0") == 0;
  }();
  return !off && c->comm == nullptr && !M->fac && M->mloc > 0;
}

template <int MAXE>
static const void* pair_kernel(int device) {
  const void* k = (const void*)k_cgs2_pair<MAXE>;
  return smem_attr(k, device, (int)kTileSmemMax) == 0 ? k : nullptr;
}

// ---------------------------------------------------------------------------
// runs
constexpr int kLag = 3;   // steps enqueued ahead of the last completed one
constexpr int kRing = 8;  // event ring (kRing > kLag)

struct ksvd_run {
  ksvd_mat* M = nullptr;
  int k_max = 0, reorth = 2, cap = 0;
  double eps = 1e-8;
  double *Q = nullptr, *P = nullptr;  // column-major bases
  int64_t ldq = 0, ldp = 0;
  double *w = nullptr, *z = nullptr;
  double *alpha = nullptr, *beta = nullptr;  // 1-based: alpha[i] = alpha_i
  DevState* st = nullptr;
  DevState* st_aux = nullptr;  // terminal column / Ritz filter
  CgsWork left, right;
  double* slot = nullptr;  // scratch scalars
  int kprime = 0, flags = 0, status = 0;
  bool pair_prev = false;  // the last step was paired: p_i is normalised in P[:, i-1]
  // Ritz
  double *G = nullptr, *V = nullptr, *U = nullptr, *sig = nullptr;
};

static int grow_bases(ksvd_run* R, int need_cols) {
  // Q needs need_cols+1 columns, P need_cols columns.
  if (need_cols <= R->cap) return 0;
  ksvd_ctx* c = R->M->ctx;
  int ncap = std::max(need_cols, std::min(R->k_max, std::max(2 * R->cap, 64)));
  ncap = std::min(ncap, R->k_max);
  double *Qn = nullptr, *Pn = nullptr;
  CK(cudaMallocAsync(&Qn, sizeof(double) * R->ldq * (ncap + 1), c->stream));
  CK(cudaMallocAsync(&Pn, sizeof(double) * R->ldp * ncap, c->stream));
  CK(cudaMemsetAsync(Qn, 0, sizeof(double) * R->ldq * (ncap + 1), c->stream));
  CK(cudaMemsetAsync(Pn, 0, sizeof(double) * R->ldp * ncap, c->stream));
  if (R->Q) {
    CK(cudaMemcpyAsync(Qn, R->Q, sizeof(double) * R->ldq * (R->cap + 1),
                       cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(Pn, R->P, sizeof(double) * R->ldp * R->cap,
                       cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaFreeAsync(R->Q, c->stream));
    CK(cudaFreeAsync(R->P, c->stream));
  }
  R->Q = Qn;
  R->P = Pn;
  R->cap = ncap;
  return 0;
}

static void free_run(ksvd_run* R) {
  if (!R) return;
  ksvd_ctx* c = R->M->ctx;
  cudaSetDevice(c->device);
  // stream-ordered frees back to the (non-trimming) pool: no device sync
  for (void* p : {(void*)R->Q, (void*)R->P, (void*)R->w, (void*)R->z, (void*)R->alpha,
                  (void*)R->beta, (void*)R->slot, (void*)R->G, (void*)R->V, (void*)R->U,
                  (void*)R->sig, (void*)R->left.part, (void*)R->left.c, (void*)R->left.red,
                  (void*)R->left.bar, (void*)R->right.part, (void*)R->right.c,
                  (void*)R->right.red, (void*)R->right.bar, (void*)R->st, (void*)R->st_aux})
    if (p) cudaFreeAsync(p, c->stream);
  delete R;
}

static double* Qcol(ksvd_run* R, int j) { return R->Q + (int64_t)j * R->ldq; }
static double* Pcol(ksvd_run* R, int j) { return R->P + (int64_t)j * R->ldp; }

// CGS2 of w against Q[:, :i] and of y = A^T w (the split partials of the
// last k_gemv_t2) against P[:, :i]; beta_{i+1}, alpha_{i+1}, q_{i+1} -> Q[:, i],
// p_{i+1} -> P[:, i], breakdown status -- one launch.
static int cgs_pair(ksvd_run* R, int i, const PairGeom& g) {
  ksvd_mat* M = R->M;
  ksvd_ctx* c = M->ctx;
  PairArgs a{};
  CgsWork* W[2] = {&R->left, &R->right};
  const double* B[2] = {R->Q, R->P};
  const int64_t ldb[2] = {R->ldq, R->ldp};
  const int64_t L[2] = {M->mloc, M->n};
  double* out[2] = {Qcol(R, i), Pcol(R, i)};
  for (int s = 0; s < 2; ++s) {
    TRY(ensure_cgs(c->stream, W[s], g.G[s], 2 * (i + 1)));
    PairSide& S = a.s[s];
    S.B = B[s];
    S.ldb = ldb[s];
    S.ncols = i;
    S.L = L[s];
    S.rows = (int)g.rows[s];
    S.G = (int)g.G[s];
    S.part = W[s]->part;
    S.c = W[s]->c;
    S.out = out[s];
  }
  a.s[0].x = R->w;
  a.s[1].fpart = M->part_t;
  a.s[1].fld = M->n_pad;
  a.s[1].fnsplit = (int)M->pt.nsplit;
  a.passes = R->reorth;
  a.eps = R->eps;
  a.beta_slot = R->beta + i + 1;
  a.alpha_slot = R->alpha + i + 1;
  a.st = R->st;
  a.step = i;
  a.hp = c->dprog;
  const int64_t G = g.G[0] + g.G[1];
  static const int64_t red_max = [] {
    const char* e = getenv("KSVD_RED_MAX");
    return e ? (int64_t)atoll(e) : (int64_t)148 * 16;
  }();
  a.redundant = std::max(g.G[0], g.G[1]) <= 160 && (int64_t)(i + 1) * G <= red_max;
  const void* kern = nullptr;
  switch (g.maxe) {
    case 1: kern = pair_kernel<1>(c->device); break;
    case 2: kern = pair_kernel<2>(c->device); break;
    case 3: kern = pair_kernel<3>(c->device); break;
    case 4: kern = pair_kernel<4>(c->device); break;
    case 5: kern = pair_kernel<5>(c->device); break;
    case 6: kern = pair_kernel<6>(c->device); break;
    case 7: kern = pair_kernel<7>(c->device); break;
    default: kern = pair_kernel<8>(c->device); break;
  }
  if (!kern) return set_err(KSVD_ERUNTIME, "k_cgs2_pair: shared-memory attribute");
  const bool reg = !c->coop_cgs;
  a.bar = reg ? R->left.bar : nullptr;
  void* args[] = {&a};
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->profiling) {
    TRY(get_event(c, &e0));
    TRY(get_event(c, &e1));
    CK(cudaEventRecord(e0, c->stream));
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)G);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = g.smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (!reg) {
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    ++na;
  }
  if (pdl_enabled(c)) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  CK(cudaLaunchKernelExC(&cfg, kern, args));
  if (c->profiling) {
    CK(cudaEventRecord(e1, c->stream));
    c->pending.push_back({e0, e1, KC_CGS});
  }
  c->launches++;
  return 0;
}

// One GK iteration i (1-based), bidiag.py:151-178.
// host-side enqueue timing per section (KSVD_DEBUG_HOST)
static double g_tsec[6];
struct SecTimer {
  int k;
  std::chrono::steady_clock::time_point t0;
  explicit SecTimer(int k_) : k(k_), t0(std::chrono::steady_clock::now()) {}
  ~SecTimer() {
    g_tsec[k] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
};

static int enqueue_step(ksvd_run* R, int i) {
  ksvd_mat* M = R->M;
  ksvd_ctx* c = M->ctx;
  {
    SecTimer t(0);
    TRY(grow_bases(R, i + 1 <= R->k_max ? i + 1 : i));
  }
  SecTimer t_all(5);
  // paired step (pair.cuh): A^T runs on the finalised w, then ONE kernel
  // orthogonalises both sides
  PairGeom pg;
  // (two CGS passes: the right pass must remove beta^2 p_i and A^T Q d, which a
  // single classical pass against a not quite orthonormal basis leaves behind)
  if (i < R->k_max && R->reorth == 2 && pair_enabled(c, M)) pg = pair_geom(c, M->mloc, M->n, i);
  // w = A p_i - alpha_i q_i, with p_i = z / alpha_i stored to P[:, i-1]
  // (after a paired step p_i is already there, normalised)
  {
    SecTimer t(1);
    const bool fin = pg.ok || (!coop_enabled(c, M->mloc, i, true) &&
                               !multi_tile_enabled(c, M->mloc, i));
    // paired: w finalised in k_gemv_n's tail (KSVD_TAILFIN=0: its own kernel)
    static const bool tail_off = [] {
      const char* e = getenv("KSVD_TAILFIN");
      return e && strcmp(e, "0") == 0;
    }();
    const double* p_src = R->pair_prev ? Pcol(R, i - 1) : R->z;
    const double* p_scale = R->pair_prev ? nullptr : R->alpha + i;
    double* p_dst = R->pair_prev ? nullptr : Pcol(R, i - 1);
    if (pg.ok)
      TRY(dense_gemv_n(M, p_src, p_scale, p_dst, Qcol(R, i - 1), R->alpha + i, R->w, R->st, i,
                       true, /*tail_fin=*/!tail_off));
    else
      TRY(enqueue_gemv_n(M, p_src, p_scale, p_dst, Qcol(R, i - 1), R->alpha + i, R->w, R->st, i,
                         fin));
  }
  R->pair_prev = false;
  if (pg.ok) {
    TRY(dense_gemv_t(M, R->w, nullptr, nullptr, nullptr, nullptr, R->z, R->st, i, true,
                     /*finalize=*/false));
    TRY(cgs_pair(R, i, pg));
    R->pair_prev = true;
    return 0;
  }
  SecTimer t_cgs(2);
  // CGS2 against Q[:, :i]; beta_{i+1} = ||w||; beta < eps -> breakdown
  if (multi_tile_enabled(c, M->mloc, i)) {
    const FinArgs fin = fin_left(M, R->alpha + i, Qcol(R, i - 1));
    TRY(cgs_tile_multi(c, &R->left, R->Q, R->ldq, i, R->w, M->mloc, R->reorth, R->eps,
                       R->beta + i + 1, R->st, i, ST_BETA_BREAK, R->M->ctx->dprog, 0, fin));
  } else if (coop_enabled(c, M->mloc, i, true)) {
    const FinArgs fin = fin_left(M, R->alpha + i, Qcol(R, i - 1));
    TRY(cgs_coop(c, &R->left, R->Q, R->ldq, i, R->w, M->mloc, R->reorth, R->eps,
                 R->beta + i + 1, R->st, i, ST_BETA_BREAK, R->M->ctx->dprog, 0, fin));
  } else {
    TRY(cgs(c, &R->left, R->Q, R->ldq, i, R->w, M->mloc, R->reorth, true, R->eps,
            R->beta + i + 1, R->st, i, ST_BETA_BREAK, R->M->ctx->dprog, 0));
  }
  if (i == R->k_max) {
    // q_{k+1} = w / beta; stop before alpha_{k+1} (bidiag.py:165-168)
    TRY(launch(c, KC_OTHER, k_scale, dim3((unsigned)cdiv(std::max<int64_t>(M->mloc, 1), kThreads)),
               dim3(kThreads), 0, (const double*)R->w, (const double*)(R->beta + i + 1),
               Qcol(R, i), M->mloc, (const DevState*)R->st));
    return 0;
  }
  // z = A^T q_{i+1} - beta_{i+1} p_i, q_{i+1} = w / beta stored to Q[:, i];
  // then CGS2 against P[:, :i] (replicated, no collective); alpha_{i+1} = ||z||
  if (coop_enabled(c, M->n, i, false)) {
    FinArgs fin;
    if (c->comm != nullptr && !M->fac) {
      // multi-rank dense A: z = all-reduce of the split sums first; the CGS
      // kernel's finalisation applies - beta p and the non-finite check
      // (the peer-exchange epilogue kernel already did both)
      TRY(dense_gemv_t(M, R->w, R->beta + i + 1, Qcol(R, i), R->beta + i + 1,
                       Pcol(R, i - 1), R->z, R->st, i, true, /*finalize=*/true,
                       /*axpy=*/false));
      if (!(c->px && M->n_pad <= c->px_slot))
        fin = FinArgs{R->z, M->n_pad, 1, R->beta + i + 1, Pcol(R, i - 1)};
    } else {
      TRY(enqueue_gemv_t(M, R->w, R->beta + i + 1, Qcol(R, i), R->beta + i + 1,
                         Pcol(R, i - 1), R->z, R->st, i, true, /*finalize=*/false));
      fin = fin_right(M, R->beta + i + 1, Pcol(R, i - 1));
    }
    TRY(cgs_coop(c, &R->right, R->P, R->ldp, i, R->z, M->n, R->reorth, R->eps,
                 R->alpha + i + 1, R->st, i, ST_ALPHA_BREAK, R->M->ctx->dprog, 1, fin));
  } else {
    TRY(enqueue_gemv_t(M, R->w, R->beta + i + 1, Qcol(R, i), R->beta + i + 1, Pcol(R, i - 1),
                       R->z, R->st, i, true));
    TRY(cgs(c, &R->right, R->P, R->ldp, i, R->z, M->n, R->reorth, false, R->eps,
            R->alpha + i + 1, R->st, i, ST_ALPHA_BREAK, R->M->ctx->dprog, 1));
  }
  return 0;
}

static int read_state(ksvd_run* R) {
  ksvd_ctx* c = R->M->ctx;
  DevState h{};
  CK(cudaMemcpyAsync(&h, R->st, sizeof h, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (c->px) {
    int err = 0;
    CK(cudaMemcpy(&err, c->px_err, sizeof err, cudaMemcpyDeviceToHost));
    if (err) return set_err(KSVD_ERUNTIME, "peer exchange: a peer never arrived (timeout)");
  }
  R->status = h.status;
  R->flags = 0;
  switch (h.status) {
    case ST_RUNNING:
      R->kprime = R->k_max;
      break;
    case ST_DEGENERATE:
      R->kprime = 0;
      R->flags = KSVD_RUN_EARLY | KSVD_RUN_DEGENERATE;
      break;
    case ST_BETA_BREAK:
      R->kprime = h.kprime;
      R->flags = KSVD_RUN_EARLY | KSVD_RUN_BETA_BREAK;
      break;
    case ST_ALPHA_BREAK:
      R->kprime = h.kprime;
      R->flags = KSVD_RUN_EARLY | KSVD_RUN_ALPHA_BREAK;
      break;
    case ST_NONFINITE:
    default:
      R->kprime = h.kprime;
      return set_err(KSVD_ENUMERIC, "non-finite values encountered in the GK step %d "
                     "(A p_i or A^T q_i)", h.where);
  }
  return 0;
}

static int run_steps(ksvd_run* R, int i0);

static int run_loop(ksvd_run* R, const double* q1_local) {
  ksvd_mat* M = R->M;
  ksvd_ctx* c = M->ctx;
  TRY(grow_bases(R, std::min(R->k_max, 64)));
  if (M->mloc > 0)
    CK(cudaMemcpyAsync(R->Q, q1_local, sizeof(double) * M->mloc, cudaMemcpyHostToDevice,
                       c->stream));
  // z = A^T q_1; alpha_1 = ||z||; alpha_1 < eps -> degenerate (bidiag.py:139-145)
  TRY(enqueue_gemv_t(M, R->Q, nullptr, nullptr, nullptr, nullptr, R->z, R->st, 0, true));
  TRY(cgs(c, &R->right, R->P, R->ldp, 0, R->z, M->n, 0, false, R->eps, R->alpha + 1, R->st,
          0, ST_DEGENERATE, R->M->ctx->dprog, 1));
  return run_steps(R, 1);
}

// GK steps i0..k_max (step i: A p_i and A^T q_{i+1} with their CGS2)
static int run_steps(ksvd_run* R, int i0) {
  ksvd_mat* M = R->M;
  ksvd_ctx* c = M->ctx;
  // Pacing: the host enqueues step i only once step i-kLag has finished,
  // waiting on a ring of events (which also flushes the launch queue).  The
  // stop decision is "the run halted at a step <= i-kLag", which depends only
  // on values identical on every rank, so all ranks enqueue the same steps.
  // (Polling a per-step progress word in mapped memory instead measured no
  // faster: its system-scope release store sat on the step's critical path.)
  static const bool dbg = getenv("KSVD_DEBUG_HOST") != nullptr;
  using clk = std::chrono::steady_clock;
  double t_launch = 0, t_wait = 0;
  R->pair_prev = false;  // callers leave z = A^T q_{i0} unnormalised
  for (int i = i0; i <= R->k_max; ++i) {
    auto t0 = clk::now();
    if (i - i0 >= kLag) {
      const int s = i - kLag;
      CK(cudaEventSynchronize(c->ring_ev[s % kRing]));
      std::atomic_thread_fence(std::memory_order_acquire);
      if (*(volatile int*)&c->hprog->halt_step <= s) break;
    }
    auto t1 = clk::now();
    TRY(enqueue_step(R, i));
    CK(cudaEventRecord(c->ring_ev[i % kRing], c->stream));
    auto t2 = clk::now();
    t_wait += std::chrono::duration<double, std::milli>(t1 - t0).count();
    t_launch += std::chrono::duration<double, std::milli>(t2 - t1).count();
  }
  if (c->tdbg) {
    unsigned long long t[16];
    CK(cudaMemcpyAsync(t, c->tdbg, sizeof t, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    fprintf(stderr, "[ksvd] cgs phases (us, CTA 0, cumulative): entry->setup %.1f (entry->fin "
            "%.1f) copy %.1f sweeps %.1f barriers %.1f reductions %.1f (dist sums %.1f, their "
            "barrier %.1f) | tile kernels %llu, in-kernel total %.1f\n",
            t[5] * 1e-3, t[8] * 1e-3, t[1] * 1e-3, t[2] * 1e-3, t[3] * 1e-3, t[4] * 1e-3,
            t[10] * 1e-3, t[11] * 1e-3, t[7], t[6] * 1e-3);
    CK(cudaMemsetAsync(c->tdbg, 0, sizeof t, c->stream));
  }
  if (dbg)
    fprintf(stderr, "[ksvd] gk host: %d steps, enqueue %.3f ms (grow %.1f, gemv_n %.1f, "
            "rest %.1f), wait %.3f ms, launches %lld\n", R->k_max, t_launch, g_tsec[0],
            g_tsec[1], g_tsec[5] - g_tsec[1], t_wait, (long long)c->launches);
  for (double& v : g_tsec) v = 0;
  return read_state(R);
}

constexpr size_t kResidentSmemMax = 200 * 1024;  // single-CTA / resident kernels

// Y = B[:, :kp] G (k_basis_combine_dmma): Ritz vectors and restart bases
static int basis_combine(ksvd_ctx* c, const double* B, int64_t ldb, int64_t L, int kp,
                         const double* G, int take, double* Y, int64_t ldy) {
  if (L <= 0 || take <= 0) return 0;
  return launch(c, KC_OTHER, k_basis_combine_dmma,
                dim3((unsigned)cdiv(L, kBCR), (unsigned)cdiv(take, 32)), dim3(kThreads), 0, B, ldb,
                L, kp, G, take, Y, ldy);
}

template <typename TA>
static int enqueue_multi_rhs(ksvd_mat* M, const double* X, int64_t ldx, int k,
                             const double* sigma, double* Y, int64_t ldy) {
  if (M->mloc == 0 || k == 0) return 0;
  const size_t xs_bytes = sizeof(double) * (size_t)std::min(k, 32) * ldx;
  if (cdiv(M->mloc, kMR) * cdiv(k, kMC) < M->ctx->sms && xs_bytes <= kResidentSmemMax) {
    // too few 256-row tiles to fill the GPU: one CTA per SM, X in shared
    // memory, one warp per row
    TRY(smem_attr((const void*)k_multi_rhs_rows<TA>, M->ctx->device, (int)kResidentSmemMax));
    const int64_t G = std::min<int64_t>(M->ctx->sms, cdiv(M->mloc, kWarps));
    const int rpc = (int)cdiv(M->mloc, G);
    for (int t0 = 0; t0 < k; t0 += 32) {
      const int kk = std::min(32, k - t0);
      TRY(launch(M->ctx, KC_OTHER, k_multi_rhs_rows<TA>, dim3((unsigned)cdiv(M->mloc, rpc)),
                 dim3(kThreads), sizeof(double) * (size_t)kk * ldx, (const TA*)M->A, M->lda,
                 M->mloc, M->n, X + (int64_t)t0 * ldx, ldx, kk,
                 sigma ? sigma + t0 : (const double*)nullptr, Y + (int64_t)t0 * ldy, ldy, rpc));
    }
    return 0;
  }
  TRY(smem_attr((const void*)k_multi_rhs<TA>, M->ctx->device, (int)multi_rhs_smem<TA>()));
  dim3 grid((unsigned)cdiv(M->mloc, kMR), (unsigned)cdiv(k, kMC));
  return launch(M->ctx, KC_OTHER, k_multi_rhs<TA>, grid, dim3(kThreads), multi_rhs_smem<TA>(),
                (const TA*)M->A, M->lda, M->mloc, M->n, X, ldx, k, sigma, Y, ldy);
}

static int multi_rhs(ksvd_mat* M, const double* X, int64_t ldx, int k, const double* sigma,
                     double* Y, int64_t ldy) {
  if (M->fac) {  // small and latency-bound: one factored product per column
    CK(cudaMemsetAsync(M->st0, 0, sizeof(DevState), M->ctx->stream));
    for (int j = 0; j < k; ++j) {
      double* y = Y + (int64_t)j * ldy;
      TRY(enqueue_gemv_n(M, X + (int64_t)j * ldx, nullptr, nullptr, nullptr, nullptr, y,
                         M->st0, 0));
      if (sigma && M->mloc > 0)
        TRY(launch(M->ctx, KC_OTHER, k_scale, dim3((unsigned)cdiv(M->mloc, kThreads)),
                   dim3(kThreads), 0, (const double*)y, sigma + j, y, M->mloc,
                   (const DevState*)M->st0));
    }
    return 0;
  }
  if (M->dtype == KSVD_F32) return enqueue_multi_rhs<float>(M, X, ldx, k, sigma, Y, ldy);
  return enqueue_multi_rhs<double>(M, X, ldx, k, sigma, Y, ldy);
}


// ---------------------------------------------------------------------------
// synthetic matrices (BASELINE.json configs 3-5)

// Cholesky G = L L^T (lower) and R^{-1} = (L^T)^{-1} (upper, row-major).
static int chol_rinv(int r, const std::vector<double>& G, std::vector<double>& Rinv) {
  std::vector<double> L((size_t)r * r, 0.0);
  for (int j = 0; j < r; ++j) {
    double d = G[(size_t)j * r + j];
    for (int k = 0; k < j; ++k) d -= L[(size_t)j * r + k] * L[(size_t)j * r + k];
    if (!(d > 0)) return set_err(KSVD_ENUMERIC, "generator: Gram matrix not positive definite");
    const double ljj = std::sqrt(d);
    L[(size_t)j * r + j] = ljj;
    for (int i = j + 1; i < r; ++i) {
      double v = G[(size_t)i * r + j];
      for (int k = 0; k < j; ++k) v -= L[(size_t)i * r + k] * L[(size_t)j * r + k];
      L[(size_t)i * r + j] = v / ljj;
    }
  }
  // Linv (lower) by forward substitution, then Rinv = Linv^T
  std::vector<double> Linv((size_t)r * r, 0.0);
  for (int c = 0; c < r; ++c) {
    for (int i = c; i < r; ++i) {
      double v = (i == c) ? 1.0 : 0.0;
      for (int k = c; k < i; ++k) v -= L[(size_t)i * r + k] * Linv[(size_t)k * r + c];
      Linv[(size_t)i * r + c] = v / L[(size_t)i * r + i];
    }
  }
  Rinv.assign((size_t)r * r, 0.0);
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < r; ++j) Rinv[(size_t)i * r + j] = Linv[(size_t)j * r + i];
  return 0;
}

// X (rows x r, row-major) <- orthonormal columns by CholeskyQR2; the Gram
// matrix is all-reduced across ranks when `sharded`.
static int cholqr2(ksvd_ctx* c, double* X, int64_t rows, int r, bool sharded) {
  cudaStream_t s = c->stream;
  const int64_t splits = std::max<int64_t>(1, std::min<int64_t>(256, cdiv(rows, 4096)));
  const int64_t rps = cdiv(std::max<int64_t>(rows, 1), splits);
  double *part = nullptr, *G = nullptr, *Rd = nullptr, *Y = nullptr;
  CK(cudaMallocAsync(&part, sizeof(double) * splits * r * r, s));
  CK(cudaMallocAsync(&G, sizeof(double) * r * r, s));
  CK(cudaMallocAsync(&Rd, sizeof(double) * r * r, s));
  CK(cudaMallocAsync(&Y, sizeof(double) * std::max<int64_t>(rows, 1) * r, s));
  std::vector<double> Gh((size_t)r * r), Rinv;
  for (int pass = 0; pass < 2; ++pass) {
    if (rows > 0) {
      const dim3 g((unsigned)cdiv(r, kGramT), (unsigned)cdiv(r, kGramT), (unsigned)splits);
      TRY(launch(c, KC_OTHER, k_gram_part, g, dim3(kThreads), 0, (const double*)X, rows, r,
                 rps, part));
      TRY(launch(c, KC_OTHER, k_gram_reduce, dim3((unsigned)cdiv((int64_t)r * r, kThreads)),
                 dim3(kThreads), 0, (const double*)part, (int)splits, r, G));
    } else {
      CK(cudaMemsetAsync(G, 0, sizeof(double) * r * r, s));
    }
    if (sharded) TRY(allreduce(c, G, (size_t)r * r));
    CK(cudaMemcpyAsync(Gh.data(), G, sizeof(double) * r * r, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    TRY(chol_rinv(r, Gh, Rinv));
    CK(cudaMemcpyAsync(Rd, Rinv.data(), sizeof(double) * r * r, cudaMemcpyHostToDevice, s));
    if (rows > 0) {
      const dim3 g((unsigned)cdiv(r, kGT), (unsigned)cdiv(rows, kGT));
      TRY(launch(c, KC_OTHER, k_gen_gemm<false, 0>, g, dim3(kThreads), 0, rows, (int64_t)r, r,
                 (const double*)X, (int64_t)r, (const double*)Rd, (int64_t)r, (void*)Y,
                 (int64_t)r, 0.0, (uint64_t)0, (int64_t)0, (int64_t)0));
      CK(cudaMemcpyAsync(X, Y, sizeof(double) * rows * r, cudaMemcpyDeviceToDevice, s));
    }
  }
  for (void* p : {(void*)part, (void*)G, (void*)Rd, (void*)Y}) CK(cudaFreeAsync(p, s));
  CK(cudaStreamSynchronize(s));
  return 0;
}

static int generate_into(ksvd_mat* M, const ksvd_gen_spec* sp) {
  ksvd_ctx* c = M->ctx;
  cudaStream_t s = c->stream;
  const int r = sp->rank;
  std::vector<double> sv(r);
  for (int i = 1; i <= r; ++i) {
    switch (sp->spectrum) {
      case KSVD_SPEC_HARMONIC: sv[i - 1] = sp->s0 / i; break;
      case KSVD_SPEC_EXP: sv[i - 1] = sp->s0 * std::exp(-(double)i / sp->p); break;
      default:
        sv[i - 1] = r > 1 ? sp->s0 * std::pow(10.0, -sp->p * (double)(i - 1) / (double)(r - 1))
                          : sp->s0;
    }
  }
  const int64_t ml = M->mloc, n = M->n;
  CK(cudaMalloc(&M->gen_ps, sizeof(double) * std::max<int64_t>(ml, 1) * r));
  CK(cudaMalloc(&M->gen_q, sizeof(double) * n * r));
  M->gen_r = r;
  const unsigned gg = (unsigned)std::min<int64_t>(c->sms * 8, 65535);
  if (ml > 0)
    TRY(launch(c, KC_OTHER, k_gen_gauss, dim3(gg), dim3(kThreads), 0, M->gen_ps, ml, r,
               (uint64_t)sp->seed, (uint32_t)KSVD_GEN_TAG_LEFT, M->row0));
  TRY(launch(c, KC_OTHER, k_gen_gauss, dim3(gg), dim3(kThreads), 0, M->gen_q, n, r,
             (uint64_t)sp->seed, (uint32_t)KSVD_GEN_TAG_RIGHT, (int64_t)0));
  TRY(cholqr2(c, M->gen_ps, ml, r, true));
  TRY(cholqr2(c, M->gen_q, n, r, false));
  double* sd = nullptr;
  CK(cudaMallocAsync(&sd, sizeof(double) * r, s));
  CK(cudaMemcpyAsync(sd, sv.data(), sizeof(double) * r, cudaMemcpyHostToDevice, s));
  if (ml > 0)
    TRY(launch(c, KC_OTHER, k_scale_cols, dim3(gg), dim3(kThreads), 0, M->gen_ps, ml, r,
               (const double*)sd));
  CK(cudaFreeAsync(sd, s));
  const size_t es = esize(M->dtype);
  if (ml > 0) {
    CK(cudaMemsetAsync(M->A, 0, (size_t)ml * M->lda * es, s));
    // rows in slabs of 65535 CTA rows (grid.y limit)
    const int64_t slab = (int64_t)65535 * kGT;
    for (int64_t i0 = 0; i0 < ml; i0 += slab) {
      const int64_t rows = std::min(slab, ml - i0);
      const dim3 g((unsigned)cdiv(n, kGT), (unsigned)cdiv(rows, kGT));
      void* dst = (char*)M->A + (size_t)i0 * M->lda * es;
      if (M->dtype == KSVD_F32)
        TRY(launch(c, KC_OTHER, k_gen_gemm<true, 2>, g, dim3(kThreads), 0, rows, n, r,
                   (const double*)(M->gen_ps + i0 * r), (int64_t)r, (const double*)M->gen_q,
                   (int64_t)r, dst, M->lda, sp->noise, (uint64_t)sp->seed, M->row0 + i0, n));
      else
        TRY(launch(c, KC_OTHER, k_gen_gemm<true, 1>, g, dim3(kThreads), 0, rows, n, r,
                   (const double*)(M->gen_ps + i0 * r), (int64_t)r, (const double*)M->gen_q,
                   (int64_t)r, dst, M->lda, sp->noise, (uint64_t)sp->seed, M->row0 + i0, n));
    }
  }
  CK(cudaStreamSynchronize(s));
  return 0;
}


// ---------------------------------------------------------------------------
// KLRM snapshots (reference matrixio.py:15-46)
struct KlrmHeader {
  char magic[4];
  uint32_t version;
  uint64_t rows, cols;
};
static_assert(sizeof(KlrmHeader) == 24, "KLRM header is <4sIQQ");

// Staging chunk: 64 MB for file reads and device->host copies; 16 MB for
// host->device uploads of pageable memory, where the first chunk's copy is
// not overlapped and a smaller chunk keeps the copy engine fed (measured on
// the B200 box, tools/r02_upload_chunks.sh: 0.8 GB 34.7 -> 46.6 GB/s, 8 GB
// 27.6-37 -> 44-49 GB/s; downloads stay faster with 64 MB).
// KSVD_IO_CHUNK_BYTES overrides both.
static int64_t io_chunk_bytes(bool upload = false) {
  static const long long env = [] {
    const char* e = getenv("KSVD_IO_CHUNK_BYTES");
    return e ? atoll(e) : 0ll;
  }();
  const long long b = env > 0 ? env : (upload ? (16ll << 20) : (64ll << 20));
  return (int64_t)std::max(4096ll, b);
}

static bool pread_all(int fd, void* buf, size_t bytes, off_t off) {
  char* p = static_cast<char*>(buf);
  while (bytes) {
    const ssize_t r = pread(fd, p, bytes, off);
    if (r <= 0) return false;
    p += r;
    bytes -= (size_t)r;
    off += r;
  }
  return true;
}
// Page-cache and pageable-memory copies are bound by one core's memcpy
// (~6 GB/s); split each chunk across io threads (KSVD_IO_THREADS, default
// min(8, cores): 37-44 GB/s uploads, 16 threads measured no faster) of a persistent pool -- spawning the threads per chunk
// cost more than the copy for small transfers.
static int io_threads() {
  static const int v = [] {
    const char* e = getenv("KSVD_IO_THREADS");
    const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    return std::max(1, e ? atoi(e) : std::min(8, hw));
  }();
  return v;
}

class IoPool {
 public:
  explicit IoPool(int n) {
    for (int t = 0; t < n; ++t) th_.emplace_back([this, t] { work(t); });
  }
  ~IoPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& x : th_) x.join();
  }
  // run job(t) for t in [0, n) on the pool (n <= size), caller waits
  template <class J>
  void run(int n, J&& job) {
    std::lock_guard<std::mutex> serial(run_mu_);  // one job at a time
    std::unique_lock<std::mutex> lk(mu_);
    job_ = [&job](int t) { job(t); };
    njob_ = n;
    pending_ = n;
    ++gen_;
    cv_.notify_all();
    done_cv_.wait(lk, [this] { return pending_ == 0; });
    job_ = nullptr;
  }
  int size() const { return (int)th_.size(); }

 private:
  void work(int t) {
    unsigned long long seen = 0;
    for (;;) {
      std::function<void(int)> job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        if (t >= njob_) continue;
        job = job_;
      }
      job(t);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_, run_mu_;
  std::condition_variable cv_, done_cv_;
  std::function<void(int)> job_;
  int njob_ = 0, pending_ = 0;
  unsigned long long gen_ = 0;
  bool stop_ = false;
};

static IoPool& io_pool() {
  static IoPool pool(io_threads());
  return pool;
}

template <class F>
static bool io_parallel(size_t bytes, F&& part) {
  const size_t grain = 1 << 20;
  const int T = (int)std::min<size_t>((size_t)io_threads(), (bytes + grain - 1) / grain);
  if (T <= 1) return part((size_t)0, bytes);
  const size_t step = ((bytes + T - 1) / T + 4095) & ~(size_t)4095;
  std::vector<char> ok(T, 0);
  io_pool().run(T, [&](int t) {
    const size_t lo = std::min(bytes, (size_t)t * step), hi = std::min(bytes, lo + step);
    ok[t] = part(lo, hi - lo) ? 1 : 0;
  });
  for (char o : ok)
    if (!o) return false;
  return true;
}
static bool pwrite_all(int fd, const void* buf, size_t bytes, off_t off) {
  const char* p = static_cast<const char*>(buf);
  while (bytes) {
    const ssize_t r = pwrite(fd, p, bytes, off);
    if (r <= 0) return false;
    p += r;
    bytes -= (size_t)r;
    off += r;
  }
  return true;
}

// Pinned double buffer + device staging for chunked transfers.
struct IoBuffers {
  void* host[2] = {nullptr, nullptr};
  double* dev = nullptr;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  ~IoBuffers() {
    for (int b = 0; b < 2; ++b) {
      if (host[b]) cudaFreeHost(host[b]);
      if (ev[b]) cudaEventDestroy(ev[b]);
    }
    if (dev) cudaFree(dev);
  }
};

static int klrm_read_into(ksvd_mat* M, int fd) {
  ksvd_ctx* c = M->ctx;
  cudaStream_t s = c->stream;
  const int64_t n = M->n, mloc = M->mloc;
  if (mloc == 0) return 0;
  const int64_t rowb = n * 8;
  const int64_t rpc = std::max<int64_t>(1, io_chunk_bytes() / rowb);  // rows per chunk
  const size_t cbytes = (size_t)rpc * rowb;
  IoBuffers io;
  for (int b = 0; b < 2; ++b) {
    CK(cudaHostAlloc(&io.host[b], cbytes, cudaHostAllocDefault));
    CK(cudaEventCreateWithFlags(&io.ev[b], cudaEventDisableTiming));
  }
  if (M->dtype == KSVD_F32) CK(cudaMalloc((void**)&io.dev, cbytes));
  const size_t es = esize(M->dtype);
  int k = 0;
  for (int64_t r = 0; r < mloc; r += rpc, ++k) {
    const int b = k & 1;
    const int64_t nr = std::min(rpc, mloc - r);
    if (k >= 2) CK(cudaEventSynchronize(io.ev[b]));  // buffer b's previous copy is done
    const off_t off = (off_t)sizeof(KlrmHeader) + (off_t)(M->row0 + r) * rowb;
    char* hb = static_cast<char*>(io.host[b]);
    if (!io_parallel((size_t)nr * rowb, [&](size_t lo, size_t len) {
          return pread_all(fd, hb + lo, len, off + (off_t)lo);
        }))
      return set_err(KSVD_ECONFIG, "KLRM: short read at row %lld", (long long)(M->row0 + r));
    if (M->dtype == KSVD_F64) {
      CK(cudaMemcpy2DAsync((char*)M->A + (size_t)r * M->lda * es, (size_t)M->lda * es,
                           io.host[b], (size_t)rowb, (size_t)rowb, (size_t)nr,
                           cudaMemcpyHostToDevice, s));
    } else {
      CK(cudaMemcpyAsync(io.dev, io.host[b], (size_t)nr * rowb, cudaMemcpyHostToDevice, s));
      TRY(launch(c, KC_OTHER, k_f64_to_f32_rows, dim3((unsigned)std::min<int64_t>(
                                                            cdiv(nr * n, kThreads), 65535)),
                 dim3(kThreads), 0, (const double*)io.dev, nr, n,
                 (float*)M->A + (size_t)r * M->lda, M->lda));
    }
    CK(cudaEventRecord(io.ev[b], s));
  }
  CK(cudaStreamSynchronize(s));
  return 0;
}

static int klrm_write_from(ksvd_mat* M, int fd) {
  ksvd_ctx* c = M->ctx;
  cudaStream_t s = c->stream;
  const int64_t n = M->n, mloc = M->mloc;
  if (mloc == 0) return 0;
  const int64_t rowb = n * 8;
  const int64_t rpc = std::max<int64_t>(1, io_chunk_bytes() / rowb);
  const size_t cbytes = (size_t)rpc * rowb;
  IoBuffers io;
  CK(cudaHostAlloc(&io.host[0], cbytes, cudaHostAllocDefault));
  if (M->dtype == KSVD_F32) CK(cudaMalloc((void**)&io.dev, cbytes));
  const size_t es = esize(M->dtype);
  for (int64_t r = 0; r < mloc; r += rpc) {
    const int64_t nr = std::min(rpc, mloc - r);
    if (M->dtype == KSVD_F64) {
      CK(cudaMemcpy2DAsync(io.host[0], (size_t)rowb, (char*)M->A + (size_t)r * M->lda * es,
                           (size_t)M->lda * es, (size_t)rowb, (size_t)nr,
                           cudaMemcpyDeviceToHost, s));
    } else {
      TRY(launch(c, KC_OTHER, k_f32_to_f64_rows, dim3((unsigned)std::min<int64_t>(
                                                            cdiv(nr * n, kThreads), 65535)),
                 dim3(kThreads), 0, (const float*)M->A + (size_t)r * M->lda, M->lda, nr, n,
                 io.dev));
      CK(cudaMemcpyAsync(io.host[0], io.dev, (size_t)nr * rowb, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    const off_t off = (off_t)sizeof(KlrmHeader) + (off_t)(M->row0 + r) * rowb;
    const char* hb = static_cast<const char*>(io.host[0]);
    if (!io_parallel((size_t)nr * rowb, [&](size_t lo, size_t len) {
          return pwrite_all(fd, hb + lo, len, off + (off_t)lo);
        }))
      return set_err(KSVD_ERUNTIME, "KLRM: write failed at row %lld", (long long)(M->row0 + r));
  }
  return 0;
}

// Small matrices: the whole loop as one cooperative kernel with A resident
// in shared memory (resident.cuh).  Eligible on one rank when every CTA's
// row block of A plus its slices of the bases fit its shared memory.
struct ResidentPlan {
  int G = 0, R = 0, C = 0;
  size_t smem = 0;
};

static bool resident_plan(ksvd_run* Rn, ResidentPlan* pl) {
  static const bool off = [] {
    const char* e = getenv("KSVD_RESIDENT");
    return e && strcmp(e, "0") == 0;
  }();
  ksvd_mat* M = Rn->M;
  ksvd_ctx* c = M->ctx;
  if (off || c->comm || M->fac || M->mloc != M->m) return false;
  const int64_t G0 = std::min<int64_t>(c->sms, M->m);
  const int64_t R = cdiv(M->m, G0);
  const int64_t G = cdiv(M->m, R);
  const int64_t C = cdiv(M->n, G);
  const int64_t kq = Rn->k_max + 1;
  // the layout of k_gk_resident's shared memory (resident.cuh)
  size_t words = ((size_t)kq * R + (size_t)Rn->k_max * C + R + C + kq + 2 + 1) & ~(size_t)1;
  words += (size_t)(M->n + 1) & ~(size_t)1;
  words += (((size_t)(kq + 1) * G + 1) & ~(size_t)1) + 2;
  const size_t smem = sizeof(double) * words + (size_t)R * M->n * esize(M->dtype);
  if (smem > kResidentSmemMax) return false;
  pl->G = (int)G;
  pl->R = (int)R;
  pl->C = (int)C;
  pl->smem = smem;
  return true;
}

template <typename TA>
static int resident_attr(int device) {
  return smem_attr((const void*)k_gk_resident<TA>, device, (int)kResidentSmemMax);
}

// q1_local: the start vector (fresh run, l = 0), or nullptr to resume after
// a restart with Q[:, :l+1] and P[:, :l] already in place
static int run_resident(ksvd_run* Rn, const ResidentPlan& pl, const double* q1_local,
                        int l = 0) {
  ksvd_mat* M = Rn->M;
  ksvd_ctx* c = M->ctx;
  cudaStream_t s = c->stream;
  TRY(grow_bases(Rn, Rn->k_max));
  if (q1_local)
    CK(cudaMemcpyAsync(Rn->Q, q1_local, sizeof(double) * M->mloc, cudaMemcpyHostToDevice, s));
  ResArgs a{};
  a.l = l;
  a.A = M->A;
  a.lda = M->lda;
  a.m = M->m;
  a.n = M->n;
  a.k_max = Rn->k_max;
  a.passes = Rn->reorth;
  a.eps = Rn->eps;
  a.R = pl.R;
  a.C = pl.C;
  a.kq = Rn->k_max + 1;
  a.Q = Rn->Q;
  a.P = Rn->P;
  a.ldq = Rn->ldq;
  a.ldp = Rn->ldp;
  a.alpha = Rn->alpha;
  a.beta = Rn->beta;
  a.w_out = Rn->w;
  a.st = Rn->st;
  a.tdbg = c->tdbg;
  // paired step (KSVD_RES_PAIR=0: the serialised 6-round step)
  static const bool res_pair_off = [] {
    const char* e = getenv("KSVD_RES_PAIR");
    return e && strcmp(e, "0") == 0;
  }();
  a.paired = (!res_pair_off && Rn->reorth == 2) ? 1 : 0;
  const size_t part_elems = 4 * (((size_t)(a.kq + 1) * pl.G + 1) & ~(size_t)1) + 2;
  const size_t z_elems = (size_t)pl.G * M->n;
  double* buf = nullptr;
  CK(cudaMallocAsync(&buf, sizeof(double) * (M->n_pad + part_elems + z_elems), s));
  a.pvec = buf;
  a.part = buf + M->n_pad;
  a.zpart = a.part + part_elems;
  void* args[] = {&a};
  const void* kern;
  if (M->dtype == KSVD_F32) {
    TRY(resident_attr<float>(c->device));
    kern = (const void*)k_gk_resident<float>;
  } else {
    TRY(resident_attr<double>(c->device));
    kern = (const void*)k_gk_resident<double>;
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->profiling) {
    TRY(get_event(c, &e0));
    TRY(get_event(c, &e1));
    CK(cudaEventRecord(e0, s));
  }
  const cudaError_t e = cudaLaunchCooperativeKernel(kern, dim3((unsigned)pl.G), dim3(kThreads),
                                                     args, pl.smem, s);
  cudaFreeAsync(buf, s);
  if (e != cudaSuccess)
    return set_err(KSVD_ERUNTIME, "resident GK launch: %s", cudaGetErrorString(e));
  if (c->profiling) {
    CK(cudaEventRecord(e1, s));
    c->pending.push_back({e0, e1, KC_RESIDENT});
  }
  c->launches++;
  if (c->tdbg) {
    unsigned long long t[8];
    CK(cudaMemcpyAsync(t, c->tdbg, sizeof t, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    fprintf(stderr, "[ksvd] resident phases (us, CTA 0, cumulative): load %.1f gemv_n %.1f "
            "cgs_left %.1f gemv_t %.1f cgs_right %.1f publish %.1f\n", t[0] * 1e-3, t[1] * 1e-3,
            t[2] * 1e-3, t[3] * 1e-3, t[4] * 1e-3, t[5] * 1e-3);
    CK(cudaMemsetAsync(c->tdbg, 0, sizeof t, s));
  }
  return read_state(Rn);
}

// ---------------------------------------------------------------------------
// C ABI
extern "C" {

const char* ksvd_last_error(void) { return g_err.c_str(); }
int ksvd_version(void) { return 1; }

int ksvd_device_count(int* count) {
  CK(cudaGetDeviceCount(count));
  return 0;
}

int ksvd_nccl_unique_id(char* uid) {
  ncclUniqueId id;
  NK(ncclGetUniqueId(&id));
  static_assert(sizeof(id) == KSVD_NCCL_UID_BYTES, "ncclUniqueId size");
  memcpy(uid, &id, sizeof id);
  return 0;
}

// Do all c->sms CTAs of a one-CTA-per-SM kernel become resident at once?
// The grid-synchronised kernels (k_cgs2_tile2, k_cgs_tile_phase) rely on it
// for their regular launches; an SM-limited MPS client or green context
// breaks it, and the context then launches them cooperatively (the driver
// checks residency and fails the launch cleanly instead).  KSVD_FORCE_COOP=1
// forces the cooperative launches (tests).
static int residency_probe(ksvd_ctx* c) {
  if (getenv("KSVD_FORCE_COOP")) {
    c->coop_cgs = true;
    return 0;
  }
  TRY(smem_attr((const void*)k_residency_probe, c->device, (int)kTileSmemMax));
  unsigned* cnt = nullptr;
  CK(cudaMalloc(&cnt, 16));
  CK(cudaMemsetAsync(cnt, 0, 16, c->stream));
  k_residency_probe<<<c->sms, kThreads, kTileSmemMax, c->stream>>>(
      cnt, reinterpret_cast<int*>(cnt + 2), (unsigned)c->sms);
  CK(cudaGetLastError());
  int failed = 0;
  CK(cudaMemcpyAsync(&failed, cnt + 2, sizeof failed, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaFree(cnt));
  c->coop_cgs = failed != 0;
  return 0;
}

int ksvd_ctx_create(int device, int rank, int nranks, const char* uid, ksvd_ctx** out) {
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return set_err(KSVD_ECONFIG, "bad rank %d / nranks %d", rank, nranks);
  if (nranks > 1 && !uid) return set_err(KSVD_ECONFIG, "nranks > 1 needs a NCCL unique id");
  CK(cudaSetDevice(device));
  auto* c = new ksvd_ctx();
  c->device = device;
  c->rank = rank;
  c->nranks = nranks;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  c->sms = prop.multiProcessorCount;
  CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  TRY(residency_probe(c));
  for (auto& e : c->marks) CK(cudaEventCreate(&e));
  for (auto& e : c->ring_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(cudaHostAlloc((void**)&c->hprog, sizeof(HostProg), cudaHostAllocMapped));
  if (getenv("KSVD_PHASE_TIMES")) {
    CK(cudaMalloc((void**)&c->tdbg, 128));
    CK(cudaMemset(c->tdbg, 0, 128));
  }
  CK(cudaHostGetDevicePointer((void**)&c->dprog, c->hprog, 0));
  {
    // keep freed pool memory mapped: per-call allocations are then cheap and
    // synchronisation points never trigger unmapping
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  }
  if (nranks > 1) {
    ncclUniqueId id;
    memcpy(&id, uid, sizeof id);
    NK(ncclCommInitRank(&c->comm, nranks, id, rank));
  } else if (getenv("KSVD_FORCE_NCCL") || getenv("KSVD_FORCE_PX")) {
    // test hook: a 1-rank communicator exercises the multi-rank code path
    // (all-reduces between the kernels) on a single GPU
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    NK(ncclCommInitRank(&c->comm, 1, id, 0));
    if (getenv("KSVD_FORCE_PX")) {  // ... and the peer exchange over a 1-rank group
      unsigned char h[KSVD_PX_HANDLE_BYTES];
      TRY(ksvd_px_export(c, 1 << 17, h));
      TRY(ksvd_px_open(c, h));
    }
  }
  *out = c;
  return 0;
}

int ksvd_ctx_destroy(ksvd_ctx* c) {
  if (!c) return 0;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (int r = 0; r < kPxMaxRanks; ++r)
    if (c->px_mapped[r]) cudaIpcCloseMemHandle(c->px_mapped[r]);
  if (c->px_local) cudaFree(c->px_local);
  if (c->px_err) cudaFree(c->px_err);
  if (c->comm) ncclCommDestroy(c->comm);
  for (auto& p : c->pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : c->pool) cudaEventDestroy(e);
  for (auto e : c->marks) cudaEventDestroy(e);
  for (auto e : c->ring_ev) cudaEventDestroy(e);
  if (c->hprog) cudaFreeHost(c->hprog);
  for (int b = 0; b < 2; ++b) {
    if (c->stage[b]) cudaFreeHost(c->stage[b]);
    if (c->stage_ev[b]) cudaEventDestroy(c->stage_ev[b]);
  }
  cudaStreamDestroy(c->stream);
  delete c;
  return 0;
}

int ksvd_px_export(ksvd_ctx* c, int64_t slot, unsigned char* handle) {
  if (!c->comm) return set_err(KSVD_ECONFIG, "peer exchange needs a multi-rank context");
  if (c->nranks > kPxMaxRanks)
    return set_err(KSVD_ECONFIG, "peer exchange supports up to %d ranks", kPxMaxRanks);
  if (slot < 1 || c->px_local) return set_err(KSVD_ECONFIG, "peer exchange: slot %lld",
                                              (long long)slot);
  CK(cudaSetDevice(c->device));
  const size_t recv = sizeof(double) * 2 * (size_t)c->nranks * slot;
  const size_t bytes = recv + sizeof(unsigned long long) * kPxCntStride * c->nranks;
  CK(cudaMalloc(&c->px_local, bytes));  // IPC needs a plain cudaMalloc allocation
  CK(cudaMemset(c->px_local, 0, bytes));
  CK(cudaMalloc((void**)&c->px_err, sizeof(int)));
  CK(cudaMemset(c->px_err, 0, sizeof(int)));
  c->px_slot = slot;
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, c->px_local));
  static_assert(sizeof(h) == KSVD_PX_HANDLE_BYTES, "IPC handle size");
  memcpy(handle, &h, sizeof h);
  return 0;
}

// Collective in two agreement rounds over NCCL, so a rank that cannot map a
// peer (no P2P path, devices hidden by CUDA_VISIBLE_DEVICES, ...) never
// leaves the others spinning: (1) every rank maps the peers and the ranks
// agree that all mappings succeeded; (2) only then the exchange runs a
// self-test against ncclAllReduce and is enabled iff it matched everywhere.
// Any failure leaves NCCL in charge and is not an error.
static int px_agree(ksvd_ctx* c, double* dev, bool mine, bool* all) {
  double v = mine ? 1.0 : 0.0;
  CK(cudaMemcpy(dev, &v, sizeof v, cudaMemcpyHostToDevice));
  NK(ncclAllReduce(dev, dev, 1, ncclDouble, ncclSum, c->comm, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaMemcpy(&v, dev, sizeof v, cudaMemcpyDeviceToHost));
  *all = v == (double)c->nranks;
  return 0;
}

int ksvd_px_open(ksvd_ctx* c, const unsigned char* handles) {
  if (!c->px_local) return set_err(KSVD_ECONFIG, "ksvd_px_export first");
  CK(cudaSetDevice(c->device));
  const size_t recv = sizeof(double) * 2 * (size_t)c->nranks * c->px_slot;
  bool mapped = true;
  for (int r = 0; r < c->nranks && mapped; ++r) {
    char* base;
    if (r == c->rank) {
      base = static_cast<char*>(c->px_local);
    } else {
      cudaIpcMemHandle_t h;
      memcpy(&h, handles + (size_t)r * KSVD_PX_HANDLE_BYTES, sizeof h);
      void* p = nullptr;
      if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();  // clear; reported through the agreement below
        mapped = false;
        break;
      }
      c->px_mapped[r] = p;
      base = static_cast<char*>(p);
    }
    c->px_recv[r] = reinterpret_cast<double*>(base);
    c->px_cnt[r] = reinterpret_cast<unsigned long long*>(base + recv);
  }
  const int64_t L = std::min<int64_t>(c->px_slot, 4099);
  double* v = nullptr;
  CK(cudaMalloc(&v, sizeof(double) * (2 * L + 1)));
  bool all = false;
  int rc = px_agree(c, v + 2 * L, mapped, &all);
  if (!rc && all) {
    // self-test: exact agreement is expected (small integers and quarters)
    std::vector<double> h0(L), h1(L);
    for (int64_t i = 0; i < L; ++i) h0[i] = (double)((c->rank + 1) * (i % 97) + 0.25 * i);
    CK(cudaMemcpy(v, h0.data(), sizeof(double) * L, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(v + L, h0.data(), sizeof(double) * L, cudaMemcpyHostToDevice));
    rc = px_allreduce(c, v, (size_t)L);
    int err = 0;
    if (!rc) {
      ncclResult_t nr = ncclAllReduce(v + L, v + L, L, ncclDouble, ncclSum, c->comm, c->stream);
      if (nr != ncclSuccess) rc = set_err(KSVD_ERUNTIME, "nccl: %s", ncclGetErrorString(nr));
    }
    if (!rc) {
      CK(cudaStreamSynchronize(c->stream));
      CK(cudaMemcpy(h0.data(), v, sizeof(double) * L, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(h1.data(), v + L, sizeof(double) * L, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(&err, c->px_err, sizeof(int), cudaMemcpyDeviceToHost));
    }
    if (!rc) rc = px_agree(c, v + 2 * L, !err && h0 == h1, &all);
  }
  cudaFree(v);
  c->px = !rc && all;
  if (!c->px)
    fprintf(stderr, "[ksvd] peer exchange unavailable on some rank (mapping or self-test): "
            "using NCCL\n");
  return rc;
}

int ksvd_px_enabled(ksvd_ctx* c, int* on) {
  *on = c->px ? 1 : 0;
  return 0;
}

int ksvd_ctx_sync(ksvd_ctx* c) {
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

int ksvd_ctx_release_pool(ksvd_ctx* c) {
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  cudaMemPool_t pool;
  CK(cudaDeviceGetDefaultMemPool(&pool, c->device));
  CK(cudaMemPoolTrimTo(pool, 0));
  return 0;
}

int ksvd_ctx_set_profiling(ksvd_ctx* c, int on) {
  TRY(collect_profile(c));
  c->profiling = on != 0;
  return 0;
}

int ksvd_ctx_kernel_stats(ksvd_ctx* c, int cls, int64_t* launches, double* ms) {
  if (cls < 0 || cls >= KC_NUM) return set_err(KSVD_ECONFIG, "kernel class %d", cls);
  CK(cudaSetDevice(c->device));
  TRY(collect_profile(c));
  *launches = c->prof_n[cls];
  *ms = c->prof_ms[cls];
  return 0;
}

int ksvd_ctx_reset_stats(ksvd_ctx* c) {
  CK(cudaSetDevice(c->device));
  TRY(collect_profile(c));
  for (int i = 0; i < KC_NUM; ++i) {
    c->prof_ms[i] = 0;
    c->prof_n[i] = 0;
  }
  c->launches = 0;
  return 0;
}

int ksvd_ctx_launch_count(ksvd_ctx* c, int64_t* launches) {
  *launches = c->launches;
  return 0;
}

int ksvd_ctx_mark(ksvd_ctx* c, int slot) {
  if (slot < 0 || slot >= 8) return set_err(KSVD_ECONFIG, "mark slot %d", slot);
  CK(cudaSetDevice(c->device));
  CK(cudaEventRecord(c->marks[slot], c->stream));
  return 0;
}

int ksvd_ctx_elapsed(ksvd_ctx* c, int s0, int s1, float* ms) {
  if (s0 < 0 || s0 >= 8 || s1 < 0 || s1 >= 8) return set_err(KSVD_ECONFIG, "mark slot");
  CK(cudaSetDevice(c->device));
  CK(cudaEventSynchronize(c->marks[s1]));
  CK(cudaEventElapsedTime(ms, c->marks[s0], c->marks[s1]));
  return 0;
}

// ---------------------------------------------------------------------------
// Host <-> device matrix transfers.  A pinned source/destination is one DMA;
// a pageable one (a plain numpy array) would go through the driver's own
// small bounce buffer at a fraction of the link rate, so it is staged here
// through a ring of two pinned chunks: io threads copy rows between the user
// buffer and chunk b while the DMA engine moves chunk b^1.
static bool host_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

static int ensure_stage(ksvd_ctx* c, size_t bytes) {
  if (c->stage_bytes >= bytes) return 0;
  CK(cudaStreamSynchronize(c->stream));
  for (int b = 0; b < 2; ++b) {
    if (c->stage[b]) CK(cudaFreeHost(c->stage[b]));
    c->stage[b] = nullptr;
    CK(cudaHostAlloc(&c->stage[b], bytes, cudaHostAllocDefault));
    if (!c->stage_ev[b]) CK(cudaEventCreateWithFlags(&c->stage_ev[b], cudaEventDisableTiming));
  }
  c->stage_bytes = bytes;
  return 0;
}

// bytes [lo, lo + len) of `rows` packed rows of `width` bytes, between the
// packed chunk `pk` and the strided user rows `u` (pitch `up`)
static void copy_packed(char* pk, char* u, size_t up, size_t width, size_t lo, size_t len,
                        bool to_packed) {
  while (len) {
    const size_t r = lo / width, off = lo % width, n = std::min(len, width - off);
    char* a = pk + lo;
    char* b = u + r * up + off;
    if (to_packed) memcpy(a, b, n);
    else memcpy(b, a, n);
    lo += n;
    len -= n;
  }
}

static int staged_copy(ksvd_ctx* c, void* dev, size_t dpitch, void* host, size_t hpitch,
                       size_t width, int64_t rows, bool to_device) {
  if (rows <= 0) return 0;
  cudaStream_t s = c->stream;
  // small transfers (< 4 MB) go direct: the driver's own staging is cheap
  // there, and the first staged call would allocate the pinned ring
  if (width * (size_t)rows < ((size_t)4 << 20) || host_pinned(host)) {
    CK(cudaMemcpy2DAsync(to_device ? dev : host, to_device ? dpitch : hpitch,
                         to_device ? host : dev, to_device ? hpitch : dpitch, width,
                         (size_t)rows, to_device ? cudaMemcpyHostToDevice
                                                 : cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return 0;
  }
  // uploads of a few chunks' worth: at least 8 chunks (>= 2 MB) so that the
  // copy engine starts early -- 16 MB (config 1) in ~1.0 instead of ~1.6 ms
  size_t cb = (size_t)io_chunk_bytes(to_device);
  if (to_device && !getenv("KSVD_IO_CHUNK_BYTES"))
    cb = std::min(cb, std::max<size_t>((size_t)2 << 20, (width * (size_t)rows + 7) / 8));
  const size_t chunk = std::max<size_t>(cb, width);
  const int64_t rpc = (int64_t)(chunk / width);
  TRY(ensure_stage(c, (size_t)rpc * width));
  char* d = static_cast<char*>(dev);
  char* h = static_cast<char*>(host);
  int64_t pend_r = -1, pend_n = 0;  // D2H: chunk waiting to be copied out
  int pend_b = 0;
  auto drain = [&]() -> bool {
    if (pend_r < 0) return true;
    if (cudaEventSynchronize(c->stage_ev[pend_b]) != cudaSuccess) return false;
    char* pk = static_cast<char*>(c->stage[pend_b]);
    char* u = h + (size_t)pend_r * hpitch;
    io_parallel((size_t)pend_n * width, [&](size_t lo, size_t len) {
      copy_packed(pk, u, hpitch, width, lo, len, false);
      return true;
    });
    pend_r = -1;
    return true;
  };
  static const bool dbg = getenv("KSVD_DEBUG_IO") != nullptr;
  using clk = std::chrono::steady_clock;
  double t_wait = 0, t_copy = 0;
  const auto t_start = clk::now();
  int k = 0;
  for (int64_t r = 0; r < rows; r += rpc, ++k) {
    const int b = k & 1;
    const int64_t nr = std::min(rpc, rows - r);
    char* pk = static_cast<char*>(c->stage[b]);
    if (to_device) {
      auto t0 = clk::now();
      if (k >= 2) CK(cudaEventSynchronize(c->stage_ev[b]));  // chunk b's DMA is done
      auto t1 = clk::now();
      char* u = h + (size_t)r * hpitch;
      io_parallel((size_t)nr * width, [&](size_t lo, size_t len) {
        copy_packed(pk, u, hpitch, width, lo, len, true);
        return true;
      });
      t_wait += std::chrono::duration<double, std::milli>(t1 - t0).count();
      t_copy += std::chrono::duration<double, std::milli>(clk::now() - t1).count();
      CK(cudaMemcpy2DAsync(d + (size_t)r * dpitch, dpitch, pk, width, width, (size_t)nr,
                           cudaMemcpyHostToDevice, s));
      CK(cudaEventRecord(c->stage_ev[b], s));
    } else {
      CK(cudaMemcpy2DAsync(pk, width, d + (size_t)r * dpitch, dpitch, width, (size_t)nr,
                           cudaMemcpyDeviceToHost, s));
      CK(cudaEventRecord(c->stage_ev[b], s));
      if (!drain()) return set_err(KSVD_ERUNTIME, "staged download failed");
      pend_r = r;
      pend_n = nr;
      pend_b = b;
    }
  }
  if (!drain()) return set_err(KSVD_ERUNTIME, "staged download failed");
  CK(cudaStreamSynchronize(s));
  if (dbg && to_device)
    fprintf(stderr, "[ksvd] staged upload %.1f MB in %d chunks: %.2f ms (host copies %.2f ms, "
            "DMA waits %.2f ms)\n", (double)width * rows / 1e6, k,
            std::chrono::duration<double, std::milli>(clk::now() - t_start).count(), t_copy,
            t_wait);
  return 0;
}

static int matrix_new(ksvd_ctx* c, const void* rows, int64_t m, int64_t n, int64_t row0,
                      int64_t mloc, int64_t src_ld, int dtype, cudaMemcpyKind kind,
                      ksvd_mat** out) {
  if (m < 1 || n < 1)
    return set_err(KSVD_ECONFIG, "expected a non-empty 2-d matrix, got %lldx%lld",
                   (long long)m, (long long)n);
  if (dtype != KSVD_F64 && dtype != KSVD_F32) return set_err(KSVD_ECONFIG, "dtype %d", dtype);
  if (row0 < 0 || mloc < 0 || row0 + mloc > m)
    return set_err(KSVD_ECONFIG, "row shard [%lld, %lld) outside %lld rows",
                   (long long)row0, (long long)(row0 + mloc), (long long)m);
  if (src_ld < n) return set_err(KSVD_ECONFIG, "src_ld %lld < n %lld", (long long)src_ld,
                                 (long long)n);
  CK(cudaSetDevice(c->device));
  auto* M = new ksvd_mat();
  M->ctx = c;
  M->m = m;
  M->n = n;
  M->row0 = row0;
  M->mloc = mloc;
  M->dtype = dtype;
  const int64_t es = (int64_t)esize(dtype);
  M->lda = lda_for(n, es);
  M->n_pad = rup(n, 64);
  M->m_pad = rup(std::max<int64_t>(mloc, 1), 64);
  int rc = alloc_matrix_buffers(M);
  if (rc) {
    free_matrix(M);
    return rc;
  }
  if (mloc > 0 && rows == nullptr && M->lda > n) {  // streamed in later: zero the padding
    cudaError_t e = cudaMemsetAsync(M->A, 0, (size_t)mloc * M->lda * es, c->stream);
    if (e != cudaSuccess) {
      free_matrix(M);
      return set_err(KSVD_ERUNTIME, "memset: %s", cudaGetErrorString(e));
    }
  }
  if (mloc > 0 && rows != nullptr) {
    if (M->lda > n) {
      cudaError_t e = cudaMemsetAsync(M->A, 0, (size_t)mloc * M->lda * es, c->stream);
      if (e != cudaSuccess) {
        free_matrix(M);
        return set_err(KSVD_ERUNTIME, "memset: %s", cudaGetErrorString(e));
      }
    }
    if (kind == cudaMemcpyHostToDevice) {
      rc = staged_copy(c, M->A, (size_t)M->lda * es, const_cast<void*>(rows),
                       (size_t)src_ld * es, (size_t)n * es, mloc, true);
      if (rc) {
        free_matrix(M);
        return rc;
      }
    } else {
      cudaError_t e =
          (src_ld == n && M->lda == n)  // contiguous on both sides: one linear copy
              ? cudaMemcpyAsync(M->A, rows, (size_t)mloc * n * es, kind, c->stream)
              : cudaMemcpy2DAsync(M->A, (size_t)M->lda * es, rows, (size_t)src_ld * es,
                                  (size_t)n * es, (size_t)mloc, kind, c->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
      if (e != cudaSuccess) {
        free_matrix(M);
        return set_err(KSVD_ERUNTIME, "matrix upload: %s", cudaGetErrorString(e));
      }
    }
  }
  *out = M;
  return 0;
}

int ksvd_matrix_from_host(ksvd_ctx* c, const void* rows, int64_t m, int64_t n, int64_t row0,
                          int64_t mloc, int64_t src_ld, int dtype, ksvd_mat** out) {
  if (mloc > 0 && !rows) return set_err(KSVD_ECONFIG, "null row pointer");
  return matrix_new(c, rows, m, n, row0, mloc, src_ld, dtype, cudaMemcpyHostToDevice, out);
}

int ksvd_matrix_from_device(ksvd_ctx* c, const void* rows, int64_t m, int64_t n,
                            int64_t row0, int64_t mloc, int64_t src_ld, int dtype,
                            ksvd_mat** out) {
  if (mloc > 0 && !rows) return set_err(KSVD_ECONFIG, "null row pointer");
  return matrix_new(c, rows, m, n, row0, mloc, src_ld, dtype, cudaMemcpyDeviceToDevice, out);
}

int ksvd_matrix_generate(ksvd_ctx* c, const ksvd_gen_spec* sp, ksvd_mat** out) {
  if (!sp || sp->m < 1 || sp->n < 1 || sp->rank < 1 || sp->rank > std::min(sp->m, sp->n))
    return set_err(KSVD_ECONFIG, "generator: need m, n >= 1 and 1 <= rank <= min(m, n)");
  if (sp->dtype != KSVD_F64 && sp->dtype != KSVD_F32)
    return set_err(KSVD_ECONFIG, "generator: dtype %d", sp->dtype);
  if (sp->spectrum < 0 || sp->spectrum > 2)
    return set_err(KSVD_ECONFIG, "generator: spectrum %d", sp->spectrum);
  CK(cudaSetDevice(c->device));
  const int64_t base = sp->m / c->nranks, extra = sp->m % c->nranks;
  const int64_t row0 = c->rank * base + std::min<int64_t>(c->rank, extra);
  const int64_t mloc = base + (c->rank < extra ? 1 : 0);
  auto* M = new ksvd_mat();
  M->ctx = c;
  M->m = sp->m;
  M->n = sp->n;
  M->row0 = row0;
  M->mloc = mloc;
  M->dtype = sp->dtype;
  const int64_t es = (int64_t)esize(sp->dtype);
  M->lda = lda_for(sp->n, es);
  M->n_pad = rup(sp->n, 64);
  M->m_pad = rup(std::max<int64_t>(mloc, 1), 64);
  int rc = alloc_matrix_buffers(M);
  if (!rc) rc = generate_into(M, sp);
  if (rc) {
    free_matrix(M);
    return rc;
  }
  *out = M;
  return 0;
}

int ksvd_matrix_gen_factors(ksvd_mat* M, double* Ps_local, double* Q, int* r) {
  ksvd_ctx* c = M->ctx;
  CK(cudaSetDevice(c->device));
  if (r) *r = M->gen_r;
  if (!M->gen_r) return set_err(KSVD_ECONFIG, "matrix was not generated on the device");
  if (Ps_local && M->mloc > 0)
    CK(cudaMemcpyAsync(Ps_local, M->gen_ps, sizeof(double) * M->mloc * M->gen_r,
                       cudaMemcpyDeviceToHost, c->stream));
  if (Q)
    CK(cudaMemcpyAsync(Q, M->gen_q, sizeof(double) * M->n * M->gen_r, cudaMemcpyDeviceToHost,
                       c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

int ksvd_matrix_from_klrm(ksvd_ctx* c, const char* path, int dtype, ksvd_mat** out) {
  if (dtype != KSVD_F64 && dtype != KSVD_F32) return set_err(KSVD_ECONFIG, "dtype %d", dtype);
  const int fd = open(path, O_RDONLY);
  if (fd < 0) return set_err(KSVD_ECONFIG, "%s: cannot open", path);
  struct FdGuard {
    int fd;
    ~FdGuard() { close(fd); }
  } guard{fd};
  KlrmHeader h{};
  if (!pread_all(fd, &h, sizeof h, 0)) return set_err(KSVD_ECONFIG, "%s: truncated header", path);
  if (memcmp(h.magic, "KLRM", 4) != 0)
    return set_err(KSVD_ECONFIG, "%s: bad magic %.4s, expected KLRM", path, h.magic);
  if (h.version != 1)
    return set_err(KSVD_ECONFIG, "%s: unsupported format version %u", path, h.version);
  const off_t size = lseek(fd, 0, SEEK_END);
  const unsigned long long want = (unsigned long long)h.rows * h.cols * 8ull;
  const unsigned long long have =
      size > (off_t)sizeof h ? (unsigned long long)(size - (off_t)sizeof h) : 0ull;
  if (have < want)
    return set_err(KSVD_ECONFIG, "%s: payload holds %llu bytes, header promises %llu", path,
                   have, want);
  const int64_t m = (int64_t)h.rows, n = (int64_t)h.cols;
  const int64_t base = m / c->nranks, extra = m % c->nranks;
  const int64_t row0 = c->rank * base + std::min<int64_t>(c->rank, extra);
  const int64_t mloc = base + (c->rank < extra ? 1 : 0);
  ksvd_mat* M = nullptr;
  TRY(matrix_new(c, nullptr, m, n, row0, mloc, n, dtype, cudaMemcpyHostToDevice, &M));
  const int rc = klrm_read_into(M, fd);
  if (rc) {
    free_matrix(M);
    return rc;
  }
  *out = M;
  return 0;
}

int ksvd_matrix_to_klrm(ksvd_mat* M, const char* path) {
  if (M->fac) return set_err(KSVD_ECONFIG, "factored operator has no dense rows");
  ksvd_ctx* c = M->ctx;
  CK(cudaSetDevice(c->device));
  const int fd = open(path, O_WRONLY | O_CREAT, 0644);
  if (fd < 0) return set_err(KSVD_ERUNTIME, "%s: cannot open for writing", path);
  struct FdGuard {
    int fd;
    ~FdGuard() { close(fd); }
  } guard{fd};
  if (c->rank == 0) {
    KlrmHeader h{};
    memcpy(h.magic, "KLRM", 4);
    h.version = 1;
    h.rows = (uint64_t)M->m;
    h.cols = (uint64_t)M->n;
    const off_t total = (off_t)sizeof h + (off_t)M->m * M->n * 8;
    if (ftruncate(fd, total) != 0 || !pwrite_all(fd, &h, sizeof h, 0))
      return set_err(KSVD_ERUNTIME, "%s: cannot write the header", path);
  }
  return klrm_write_from(M, fd);
}

int ksvd_matrix_from_factors(ksvd_ctx* c, const double* left_rows, const double* core,
                             const double* right, int64_t m, int64_t n, int64_t s1, int64_t s2,
                             int64_t row0, int64_t mloc, ksvd_mat** out) {
  if (m < 1 || n < 1 || s1 < 1 || s2 < 1)
    return set_err(KSVD_ECONFIG, "factored operator: %lldx%lld with core %lldx%lld",
                   (long long)m, (long long)n, (long long)s1, (long long)s2);
  if (row0 < 0 || mloc < 0 || row0 + mloc > m)
    return set_err(KSVD_ECONFIG, "row shard [%lld, %lld) outside %lld rows", (long long)row0,
                   (long long)(row0 + mloc), (long long)m);
  if ((mloc > 0 && !left_rows) || !core || !right)
    return set_err(KSVD_ECONFIG, "null factor pointer");
  CK(cudaSetDevice(c->device));
  auto* M = new ksvd_mat();
  M->ctx = c;
  M->m = m;
  M->n = n;
  M->row0 = row0;
  M->mloc = mloc;
  M->dtype = KSVD_F64;
  M->n_pad = rup(n, 64);
  M->m_pad = rup(std::max<int64_t>(mloc, 1), 64);
  M->fac = new ksvd_mat::Factored();
  M->fac->s1 = s1;
  M->fac->s2 = s2;
  auto fail = [&](int rc) {
    free_matrix(M);
    return rc;
  };
  int rc = matrix_new(c, left_rows, std::max<int64_t>(mloc, 1), s1, 0, mloc, s1, KSVD_F64,
                      cudaMemcpyHostToDevice, &M->fac->L);
  if (!rc)
    rc = matrix_new(c, right, n, s2, 0, n, s2, KSVD_F64, cudaMemcpyHostToDevice, &M->fac->R);
  if (rc) return fail(rc);
  cudaStream_t st = c->stream;
  const size_t vec = sizeof(double) * std::max(M->n_pad, M->m_pad);
  const size_t sv = sizeof(double) * rup(std::max(s1, s2), 64);
  cudaError_t e = cudaSuccess;
  auto ok = [&](cudaError_t x) {
    if (e == cudaSuccess) e = x;
  };
  ok(cudaMallocAsync((void**)&M->fac->C, sizeof(double) * s1 * s2, st));
  ok(cudaMallocAsync((void**)&M->fac->t1, sv, st));
  ok(cudaMallocAsync((void**)&M->fac->t2, sv, st));
  ok(cudaMallocAsync((void**)&M->dx, vec, st));
  ok(cudaMallocAsync((void**)&M->dy, vec, st));
  ok(cudaMallocAsync((void**)&M->st0, sizeof(DevState), st));
  if (e == cudaSuccess) {
    ok(cudaMemcpyAsync(M->fac->C, core, sizeof(double) * s1 * s2, cudaMemcpyHostToDevice, st));
    ok(cudaMemsetAsync(M->fac->t1, 0, sv, st));
    ok(cudaMemsetAsync(M->fac->t2, 0, sv, st));
    ok(cudaMemsetAsync(M->dx, 0, vec, st));
    ok(cudaMemsetAsync(M->dy, 0, vec, st));
    ok(cudaMemsetAsync(M->st0, 0, sizeof(DevState), st));
    ok(cudaStreamSynchronize(st));
  }
  if (e != cudaSuccess)
    return fail(set_err(KSVD_ERUNTIME, "factored operator: %s", cudaGetErrorString(e)));
  *out = M;
  return 0;
}

int ksvd_dense_svd_dev(ksvd_ctx* c, int k, const double* T, double* U, double* s, double* V) {
  if (k <= 0) return set_err(KSVD_ECONFIG, "empty matrix");
  const int kk = (k + 1) & ~1;
  const size_t smem = sizeof(double) * (2 * (size_t)kk * k + kk);
  if (smem > kResidentSmemMax) return ksvd_dense_svd(k, T, U, s, V);  // host Jacobi
  CK(cudaSetDevice(c->device));
  TRY(smem_attr((const void*)k_dense_svd_cta, c->device, (int)kResidentSmemMax));
  cudaStream_t st = c->stream;
  const size_t kk2 = (size_t)k * k;
  double* buf = nullptr;
  CK(cudaMallocAsync(&buf, sizeof(double) * (3 * kk2 + k) + sizeof(int) * 2, st));
  double *Td = buf, *Ud = buf + kk2, *Vd = buf + 2 * kk2, *sd = buf + 3 * kk2;
  int* info = reinterpret_cast<int*>(sd + k);
  CK(cudaMemcpyAsync(Td, T, sizeof(double) * kk2, cudaMemcpyHostToDevice, st));
  int rc = launch(c, KC_OTHER, k_dense_svd_cta, dim3(1), dim3(kSvdThreads), smem, k,
                  (const double*)Td, Ud, sd, Vd, info);
  int sweeps = 0;
  if (!rc) {
    CK(cudaMemcpyAsync(U, Ud, sizeof(double) * kk2, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(V, Vd, sizeof(double) * kk2, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(s, sd, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&sweeps, info, sizeof(int), cudaMemcpyDeviceToHost, st));
  }
  cudaFreeAsync(buf, st);
  CK(cudaStreamSynchronize(st));
  if (!rc && sweeps >= 80) rc = set_err(KSVD_ENUMERIC, "Jacobi SVD did not converge");
  return rc;
}

int ksvd_matrix_free(ksvd_mat* M) { return free_matrix(M); }

int ksvd_matrix_shape(ksvd_mat* M, int64_t* m, int64_t* n, int64_t* row0, int64_t* mloc,
                      int* dtype, int64_t* ld) {
  if (m) *m = M->m;
  if (n) *n = M->n;
  if (row0) *row0 = M->row0;
  if (mloc) *mloc = M->mloc;
  if (dtype) *dtype = M->dtype;
  if (ld) *ld = M->lda;
  return 0;
}

int ksvd_matrix_to_host(ksvd_mat* M, void* rows) {
  if (M->fac) return set_err(KSVD_ECONFIG, "factored operator has no dense rows");
  ksvd_ctx* c = M->ctx;
  CK(cudaSetDevice(c->device));
  if (M->mloc == 0) return 0;
  const size_t es = esize(M->dtype);
  return staged_copy(c, M->A, (size_t)M->lda * es, rows, (size_t)M->n * es, (size_t)M->n * es,
                     M->mloc, false);
}

static int reset_state(ksvd_ctx* c, DevState* st) {
  CK(cudaMemsetAsync(st, 0, sizeof(DevState), c->stream));
  return 0;
}

int ksvd_matvec(ksvd_mat* M, const double* x, double* y) {
  ksvd_ctx* c = M->ctx;
  CK(cudaSetDevice(c->device));
  TRY(reset_state(c, M->st0));
  CK(cudaMemcpyAsync(M->dx, x, sizeof(double) * M->n, cudaMemcpyHostToDevice, c->stream));
  TRY(enqueue_gemv_n(M, M->dx, nullptr, nullptr, nullptr, nullptr, M->dy, M->st0, 0));
  if (M->mloc > 0)
    CK(cudaMemcpyAsync(y, M->dy, sizeof(double) * M->mloc, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

int ksvd_rmatvec(ksvd_mat* M, const double* y, double* z) {
  ksvd_ctx* c = M->ctx;
  CK(cudaSetDevice(c->device));
  TRY(reset_state(c, M->st0));
  if (M->mloc > 0)
    CK(cudaMemcpyAsync(M->dx, y, sizeof(double) * M->mloc, cudaMemcpyHostToDevice, c->stream));
  TRY(enqueue_gemv_t(M, M->dx, nullptr, nullptr, nullptr, nullptr, M->dy, M->st0, 0, false));
  CK(cudaMemcpyAsync(z, M->dy, sizeof(double) * M->n, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

int ksvd_matmat(ksvd_mat* M, const double* X, int k, double* Y) {
  ksvd_ctx* c = M->ctx;
  CK(cudaSetDevice(c->device));
  if (k <= 0) return k == 0 ? 0 : set_err(KSVD_ECONFIG, "k = %d", k);
  double *dX = nullptr, *dY = nullptr;
  // X columns at a 512-byte pitch (16-byte aligned cp.async sources)
  CK(cudaMallocAsync(&dX, sizeof(double) * M->n_pad * k, c->stream));
  CK(cudaMallocAsync(&dY, sizeof(double) * std::max<int64_t>(M->mloc, 1) * k, c->stream));
  CK(cudaMemcpy2DAsync(dX, sizeof(double) * M->n_pad, X, sizeof(double) * M->n,
                       sizeof(double) * M->n, k, cudaMemcpyHostToDevice, c->stream));
  int rc = multi_rhs(M, dX, M->n_pad, k, nullptr, dY, M->mloc);
  if (!rc && M->mloc > 0) {
    cudaError_t e = cudaMemcpyAsync(Y, dY, sizeof(double) * M->mloc * k,
                                    cudaMemcpyDeviceToHost, c->stream);
    if (e != cudaSuccess) rc = set_err(KSVD_ERUNTIME, "matmat D2H: %s", cudaGetErrorString(e));
  }
  cudaFreeAsync(dX, c->stream);
  cudaFreeAsync(dY, c->stream);
  CK(cudaStreamSynchronize(c->stream));
  return rc;
}

int ksvd_gk_run(ksvd_mat* M, int k_max, double eps, int reorth, const double* q1_local,
                ksvd_run** out) {
  ksvd_ctx* c = M->ctx;
  if (k_max < 1 || k_max > std::min(M->m, M->n))
    return set_err(KSVD_ECONFIG, "k_max must be in [1, min(m,n)] = [1, %lld], got %d",
                   (long long)std::min(M->m, M->n), k_max);
  if (!(eps > 0)) return set_err(KSVD_ECONFIG, "eps must be > 0, got %g", eps);
  if (reorth != 1 && reorth != 2)
    return set_err(KSVD_ECONFIG, "reorth_passes must be 1 or 2, got %d", reorth);
  CK(cudaSetDevice(c->device));
  auto* R = new ksvd_run();
  R->M = M;
  R->k_max = k_max;
  R->eps = eps;
  R->reorth = reorth;
  R->ldq = M->m_pad;
  R->ldp = M->n_pad;
  auto fail = [&](int rc) {
    free_run(R);
    return rc;
  };
  cudaError_t e = cudaSuccess;
#define RUN_CK(x)                                                             \
  do {                                                                        \
    e = (x);                                                                  \
    if (e != cudaSuccess)                                                     \
      return fail(set_err(KSVD_ERUNTIME, "%s: %s", #x, cudaGetErrorString(e))); \
  } while (0)
  cudaStream_t st_ = c->stream;
  RUN_CK(cudaMallocAsync(&R->w, sizeof(double) * R->ldq, st_));
  RUN_CK(cudaMallocAsync(&R->z, sizeof(double) * R->ldp, st_));
  RUN_CK(cudaMemsetAsync(R->w, 0, sizeof(double) * R->ldq, c->stream));
  RUN_CK(cudaMemsetAsync(R->z, 0, sizeof(double) * R->ldp, c->stream));
  RUN_CK(cudaMallocAsync(&R->alpha, sizeof(double) * (k_max + 2), st_));
  RUN_CK(cudaMallocAsync(&R->beta, sizeof(double) * (k_max + 3), st_));
  RUN_CK(cudaMemsetAsync(R->alpha, 0, sizeof(double) * (k_max + 2), c->stream));
  RUN_CK(cudaMemsetAsync(R->beta, 0, sizeof(double) * (k_max + 3), c->stream));
  RUN_CK(cudaMallocAsync(&R->slot, sizeof(double) * 8, st_));
  RUN_CK(cudaMallocAsync((void**)&R->st, sizeof(DevState), st_));
  RUN_CK(cudaMallocAsync((void**)&R->st_aux, sizeof(DevState), st_));
  RUN_CK(cudaMemsetAsync(R->st, 0, sizeof(DevState), c->stream));
  RUN_CK(cudaMemsetAsync(R->st_aux, 0, sizeof(DevState), c->stream));
  c->hprog->prog = -1;
  c->hprog->halt_step = INT_MAX;
  c->hprog->status = 0;
#undef RUN_CK
  ResidentPlan pl;
  int rc = resident_plan(R, &pl) ? run_resident(R, pl, q1_local) : run_loop(R, q1_local);
  if (rc) return fail(rc);
  *out = R;
  return 0;
}

int ksvd_run_info(ksvd_run* R, int* k_prime, int* flags, double* alphas, double* betas) {
  ksvd_ctx* c = R->M->ctx;
  CK(cudaSetDevice(c->device));
  if (k_prime) *k_prime = R->kprime;
  if (flags) *flags = R->flags;
  const int kp = R->kprime;
  // + alpha_{k'+1} after an alpha breakdown (its residual, see the header)
  const int na = kp + ((R->flags & KSVD_RUN_ALPHA_BREAK) && kp < R->k_max ? 1 : 0);
  if (alphas && na > 0)
    CK(cudaMemcpyAsync(alphas, R->alpha + 1, sizeof(double) * na, cudaMemcpyDeviceToHost,
                       c->stream));
  // betas[1..k'] = beta_2..beta_{k'+1}
  if (betas && kp > 0 && !(R->flags & KSVD_RUN_DEGENERATE))
    CK(cudaMemcpyAsync(betas + 1, R->beta + 2, sizeof(double) * kp, cudaMemcpyDeviceToHost,
                       c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

int ksvd_run_extend(ksvd_run* R, const double* v_local, double nrm, int* accepted) {
  ksvd_mat* M = R->M;
  ksvd_ctx* c = M->ctx;
  CK(cudaSetDevice(c->device));
  const int kp = R->kprime;
  if (kp >= M->m) return set_err(KSVD_ECONFIG, "left space exhausted (k' = m)");
  TRY(grow_bases(R, std::min(kp, R->k_max)));
  TRY(reset_state(c, R->st_aux));
  if (v_local && M->mloc > 0)
    CK(cudaMemcpyAsync(R->w, v_local, sizeof(double) * M->mloc, cudaMemcpyHostToDevice,
                       c->stream));
  const unsigned g = (unsigned)cdiv(std::max<int64_t>(M->mloc, 1), kThreads);
  TRY(launch(c, KC_OTHER, k_scale_val, dim3(g), dim3(kThreads), 0, (const double*)R->w, nrm,
             R->w, M->mloc, (const DevState*)R->st_aux));
  // v = orthogonalize(v, Q[:, :k'], passes=2); nrm2 = ||v||  (bidiag.py:102-103)
  TRY(cgs(c, &R->left, R->Q, R->ldq, kp, R->w, M->mloc, 2, true, 0.5, R->slot,
          R->st_aux, kp, ST_CUT));
  DevState h{};
  CK(cudaMemcpyAsync(&h, R->st_aux, sizeof h, cudaMemcpyDeviceToHost, c->stream));
  double nrm2 = 0;
  CK(cudaMemcpyAsync(&nrm2, R->slot, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (h.status == ST_NONFINITE)
    return set_err(KSVD_ENUMERIC, "non-finite values in the terminal column");
  // accepted iff nrm2 > 0.5 (strict): the CUT test above fires for < 0.5
  *accepted = (h.status == ST_RUNNING && nrm2 > 0.5) ? 1 : 0;
  if (*accepted) {
    TRY(reset_state(c, R->st_aux));
    TRY(launch(c, KC_OTHER, k_scale, dim3(g), dim3(kThreads), 0, (const double*)R->w,
               (const double*)R->slot, Qcol(R, kp), M->mloc, (const DevState*)R->st_aux));
    CK(cudaStreamSynchronize(c->stream));
  }
  return 0;
}

int ksvd_run_bases(ksvd_run* R, double* Q, int q_cols, double* P, int p_cols) {
  ksvd_mat* M = R->M;
  ksvd_ctx* c = M->ctx;
  CK(cudaSetDevice(c->device));
  if (q_cols < 0 || q_cols > R->cap + 1 || p_cols < 0 || p_cols > R->cap)
    return set_err(KSVD_ECONFIG, "bases: %d/%d columns requested, %d allocated", q_cols,
                   p_cols, R->cap);
  if (Q && q_cols > 0 && M->mloc > 0)
    TRY(staged_copy(c, R->Q, sizeof(double) * R->ldq, Q, sizeof(double) * M->mloc,
                      sizeof(double) * M->mloc, q_cols, false));
  if (P && p_cols > 0)
    TRY(staged_copy(c, R->P, sizeof(double) * R->ldp, P, sizeof(double) * M->n,
                      sizeof(double) * M->n, p_cols, false));
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

int ksvd_ritz(ksvd_run* R, const double* G, const double* sigma, int take, int ortho,
              double* U, double* V, int* n_good) {
  ksvd_mat* M = R->M;
  ksvd_ctx* c = M->ctx;
  CK(cudaSetDevice(c->device));
  const int kp = R->kprime;
  if (take < 0 || take > kp) return set_err(KSVD_ECONFIG, "take %d outside [0, k'=%d]", take, kp);
  *n_good = 0;
  if (take == 0) return 0;
  const int64_t ldu = M->m_pad, ldv = M->n_pad;
  for (double* p : {R->G, R->V, R->U, R->sig})
    if (p) cudaFreeAsync(p, c->stream);
  R->G = R->V = R->U = R->sig = nullptr;
  CK(cudaMallocAsync(&R->G, sizeof(double) * kp * take, c->stream));
  CK(cudaMallocAsync(&R->V, sizeof(double) * ldv * take, c->stream));
  CK(cudaMallocAsync(&R->U, sizeof(double) * ldu * take, c->stream));
  CK(cudaMallocAsync(&R->sig, sizeof(double) * take, c->stream));
  CK(cudaMemsetAsync(R->V, 0, sizeof(double) * ldv * take, c->stream));
  CK(cudaMemsetAsync(R->U, 0, sizeof(double) * ldu * take, c->stream));
  CK(cudaMemcpyAsync(R->G, G, sizeof(double) * kp * take, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(R->sig, sigma, sizeof(double) * take, cudaMemcpyHostToDevice, c->stream));
  // V = P[:, :k'] G  (fsvd.py:191)
  TRY(basis_combine(c, R->P, R->ldp, M->n, kp, R->G, take, R->V, ldv));
  // U[:, t] = A V[:, t] / sigma_t, one pass over A (fsvd.py:192-194)
  TRY(multi_rhs(M, R->V, ldv, take, R->sig, R->U, ldu));
  int good = take;
  const int ldm = (int)rup(std::max<int64_t>(M->mloc, 1), 2);
  const size_t uf_smem = sizeof(double) * ((size_t)take * ldm + take);
  if (ortho && c->comm == nullptr && uf_smem <= kResidentSmemMax) {
    // the same filter in one single-CTA launch (U fits shared memory)
    TRY(reset_state(c, R->st_aux));
    TRY(smem_attr((const void*)k_ufilter_small, c->device, (int)kResidentSmemMax));
    TRY(launch(c, KC_OTHER, k_ufilter_small, dim3(1), dim3(kUfThreads), uf_smem, R->U, ldu,
               (int)M->mloc, take, ldm, 1e-2, R->st_aux));
    DevState h{};
    CK(cudaMemcpyAsync(&h, R->st_aux, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (h.status == ST_NONFINITE) return set_err(KSVD_ENUMERIC, "non-finite Ritz vectors");
    if (h.status == ST_CUT) good = h.kprime;
  } else if (ortho) {
    // CGS2 column filter, cut at the first residual < 1e-2 (fsvd.py:145-155)
    TRY(reset_state(c, R->st_aux));
    const unsigned g = (unsigned)cdiv(std::max<int64_t>(M->mloc, 1), kThreads);
    for (int t = 0; t < take; ++t) {
      double* ut = R->U + (int64_t)t * ldu;
      TRY(cgs(c, &R->left, R->U, ldu, t, ut, M->mloc, 2, true, 1e-2, R->slot + (t % 8),
              R->st_aux, t, ST_CUT));
      TRY(launch(c, KC_OTHER, k_scale, dim3(g), dim3(kThreads), 0, (const double*)ut,
                 (const double*)(R->slot + (t % 8)), ut, M->mloc, (const DevState*)R->st_aux));
    }
    DevState h{};
    CK(cudaMemcpyAsync(&h, R->st_aux, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (h.status == ST_NONFINITE) return set_err(KSVD_ENUMERIC, "non-finite Ritz vectors");
    if (h.status == ST_CUT) good = h.kprime;
  }
  // fix_signs (linops.py:271-282)
  if (good > 0)
    TRY(launch(c, KC_OTHER, k_fix_signs, dim3(good), dim3(kThreads), 0, R->V, ldv, M->n, R->U,
               ldu, M->mloc));
  if (good > 0) {
    if (M->mloc > 0)
      TRY(staged_copy(c, R->U, sizeof(double) * ldu, U, sizeof(double) * M->mloc,
                      sizeof(double) * M->mloc, good, false));
    TRY(staged_copy(c, R->V, sizeof(double) * ldv, V, sizeof(double) * M->n,
                      sizeof(double) * M->n, good, false));
  }
  CK(cudaStreamSynchronize(c->stream));
  *n_good = good;
  return 0;
}

int ksvd_run_restart(ksvd_run* R, int l, const double* X, const double* Y, int k_new) {
  ksvd_mat* M = R->M;
  ksvd_ctx* c = M->ctx;
  CK(cudaSetDevice(c->device));
  const int k = R->kprime;
  if (R->status != ST_RUNNING || k != R->k_max)
    return set_err(KSVD_ECONFIG, "restart needs a run that completed its %d steps", R->k_max);
  if (l < 0 || l >= k) return set_err(KSVD_ECONFIG, "restart keeps l=%d of k=%d", l, k);
  if (k_new <= l || k_new > std::min(M->m, M->n))
    return set_err(KSVD_ECONFIG, "restart size %d outside (%d, %lld]", k_new, l,
                   (long long)std::min(M->m, M->n));
  if (l > 0 && (!X || !Y)) return set_err(KSVD_ECONFIG, "null restart combination");
  cudaStream_t s = c->stream;
  double *Xd = nullptr, *Yd = nullptr, *Qt = nullptr, *Pt = nullptr;
  auto release = [&] {
    for (double* p : {Xd, Yd, Qt, Pt})
      if (p) cudaFreeAsync(p, s);
  };
  const size_t nl = (size_t)std::max(l, 1);
  cudaError_t e = cudaSuccess;
  auto ok = [&](cudaError_t x) {
    if (e == cudaSuccess) e = x;
  };
  ok(cudaMallocAsync(&Xd, sizeof(double) * k * nl, s));
  ok(cudaMallocAsync(&Yd, sizeof(double) * k * nl, s));
  ok(cudaMallocAsync(&Qt, sizeof(double) * R->ldq * (l + 1), s));
  ok(cudaMallocAsync(&Pt, sizeof(double) * R->ldp * nl, s));
  if (e == cudaSuccess && l > 0) {
    ok(cudaMemcpyAsync(Xd, X, sizeof(double) * k * l, cudaMemcpyHostToDevice, s));
    ok(cudaMemcpyAsync(Yd, Y, sizeof(double) * k * l, cudaMemcpyHostToDevice, s));
  }
  if (e != cudaSuccess) {
    release();
    return set_err(KSVD_ERUNTIME, "restart: %s", cudaGetErrorString(e));
  }
  int rc = 0;
  // Ritz combinations of the current bases, then q_{k+1} as column l
  if (l > 0) {
    rc = basis_combine(c, R->Q, R->ldq, M->mloc, k, Xd, l, Qt, R->ldq);
    if (!rc) rc = basis_combine(c, R->P, R->ldp, M->n, k, Yd, l, Pt, R->ldp);
  }
  if (!rc) {
    ok(cudaMemcpyAsync(Qt + (size_t)l * R->ldq, R->Q + (size_t)k * R->ldq,
                       sizeof(double) * R->ldq, cudaMemcpyDeviceToDevice, s));
    ok(cudaMemcpyAsync(R->Q, Qt, sizeof(double) * R->ldq * (l + 1), cudaMemcpyDeviceToDevice, s));
    if (l > 0)
      ok(cudaMemcpyAsync(R->P, Pt, sizeof(double) * R->ldp * l, cudaMemcpyDeviceToDevice, s));
    if (e != cudaSuccess) rc = set_err(KSVD_ERUNTIME, "restart: %s", cudaGetErrorString(e));
  }
  release();
  if (rc) return rc;
  // room for k_new steps: scalars are re-allocated, bases grow on demand
  if (k_new > R->k_max) {
    for (double* p : {R->alpha, R->beta}) CK(cudaFreeAsync(p, s));
    CK(cudaMallocAsync(&R->alpha, sizeof(double) * (k_new + 2), s));
    CK(cudaMallocAsync(&R->beta, sizeof(double) * (k_new + 3), s));
  }
  R->k_max = k_new;
  CK(cudaMemsetAsync(R->alpha, 0, sizeof(double) * (k_new + 2), s));
  CK(cudaMemsetAsync(R->beta, 0, sizeof(double) * (k_new + 3), s));
  CK(cudaMemsetAsync(R->st, 0, sizeof(DevState), s));
  c->hprog->prog = -1;
  c->hprog->halt_step = INT_MAX;
  c->hprog->status = 0;
  ResidentPlan pl;
  if (resident_plan(R, &pl)) return run_resident(R, pl, nullptr, l);
  // z = A^T q_{l+1}; CGS2 against the l kept right Ritz vectors (the spike);
  // alpha_{l+1} < eps: the kept space is invariant (k' = l)
  TRY(enqueue_gemv_t(M, R->Q + (size_t)l * R->ldq, nullptr, nullptr, nullptr, nullptr, R->z,
                     R->st, l, true));
  TRY(cgs(c, &R->right, R->P, R->ldp, l, R->z, M->n, l > 0 ? R->reorth : 0, false, R->eps,
          R->alpha + l + 1, R->st, l, l > 0 ? ST_ALPHA_BREAK : ST_DEGENERATE, c->dprog, 1));
  return run_steps(R, l + 1);
}

int ksvd_run_ritz_bases(ksvd_run* R, const double* X, int kq, const double* Y, int kp, int take,
                        double* U, double* V) {
  ksvd_mat* M = R->M;
  ksvd_ctx* c = M->ctx;
  CK(cudaSetDevice(c->device));
  if (take <= 0) return take == 0 ? 0 : set_err(KSVD_ECONFIG, "take %d", take);
  if (kq < 1 || kq > R->cap + 1 || kp < 1 || kp > R->cap)
    return set_err(KSVD_ECONFIG, "basis columns kq=%d kp=%d outside the run", kq, kp);
  cudaStream_t s = c->stream;
  const int64_t ldu = M->m_pad, ldv = M->n_pad;
  for (double* p : {R->G, R->V, R->U, R->sig})
    if (p) cudaFreeAsync(p, s);
  R->G = R->V = R->U = R->sig = nullptr;
  CK(cudaMallocAsync(&R->G, sizeof(double) * ((size_t)kq + kp) * take, s));
  CK(cudaMallocAsync(&R->V, sizeof(double) * ldv * take, s));
  CK(cudaMallocAsync(&R->U, sizeof(double) * ldu * take, s));
  CK(cudaMemsetAsync(R->U, 0, sizeof(double) * ldu * take, s));
  double* Xd = R->G;
  double* Yd = R->G + (size_t)kq * take;
  CK(cudaMemcpyAsync(Xd, X, sizeof(double) * kq * take, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(Yd, Y, sizeof(double) * kp * take, cudaMemcpyHostToDevice, s));
  TRY(basis_combine(c, R->Q, R->ldq, M->mloc, kq, Xd, take, R->U, ldu));
  TRY(basis_combine(c, R->P, R->ldp, M->n, kp, Yd, take, R->V, ldv));
  TRY(launch(c, KC_OTHER, k_fix_signs, dim3(take), dim3(kThreads), 0, R->V, ldv, M->n, R->U,
             ldu, M->mloc));
  if (M->mloc > 0)
    TRY(staged_copy(c, R->U, sizeof(double) * ldu, U, sizeof(double) * M->mloc,
                      sizeof(double) * M->mloc, take, false));
  TRY(staged_copy(c, R->V, sizeof(double) * ldv, V, sizeof(double) * M->n,
                      sizeof(double) * M->n, take, false));
  CK(cudaStreamSynchronize(s));
  return 0;
}

int ksvd_run_free(ksvd_run* R) {
  free_run(R);
  return 0;
}

}  // extern "C"
