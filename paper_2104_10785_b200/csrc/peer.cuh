// peer.cuh -- all-reduce of the GK step's small vectors over NVLink peer
// memory (included by ksvd.cu).
//
// Every rank owns a receive area in its HBM, exported with CUDA IPC and
// mapped by every peer: 2 parities x N sender slots x `slot` doubles, plus
// one arrival counter per sender (128-byte apart).  k_px_allreduce pushes
// this rank's vector straight into its slot on every peer (NVLink stores),
// bumps each peer's counter for this rank once per CTA, waits until every
// sender's cumulative counter reaches the host-tracked total, and sums the N
// slots in rank
// order -- the same bits on every rank, no NCCL launch, one kernel.  The
// parity (seq & 1) double-buffers the slots: a rank can only run ahead by
// one collective, since collective s+1 needs every peer's push for s+1.
// Counters are cumulative (never reset).  A bounded spin turns a missing
// peer into an error flag instead of a hang.
#pragma once

namespace ksvd {

constexpr int kPxMaxRanks = 8;
constexpr int kPxCntStride = 16;  // counters 128 bytes apart

struct PxArgs {
  double* buf;
  int64_t L;
  double* recv[kPxMaxRanks];              // rank r's receive area (mapped)
  unsigned long long* cnt[kPxMaxRanks];   // rank r's counters (mapped)
  const double* my_recv;
  const unsigned long long* my_cnt;
  int rank, N;
  unsigned long long seq;
  unsigned long long want;  // cumulative arrivals expected from every sender
  int64_t slot;
  int* err;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(kThreads) k_px_allreduce(PxArgs a) {
  const int par = (int)(a.seq & 1);
  const int64_t chunk = (a.L + gridDim.x - 1) / gridDim.x;
  const int64_t e0 = (int64_t)blockIdx.x * chunk;
  const int64_t e1 = min(a.L, e0 + chunk);
  // push: my elements into my slot on every rank (self included)
  for (int r = 0; r < a.N; ++r) {
    double* dst = a.recv[r] + ((int64_t)par * a.N + a.rank) * a.slot;
    for (int64_t e = e0 + threadIdx.x; e < e1; e += kThreads) dst[e] = a.buf[e];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x < a.N)
    atomicAdd_system(a.cnt[threadIdx.x] + (int64_t)a.rank * kPxCntStride, 1ull);
  // wait for every sender's CTAs (cumulative count: every rank issues the
  // same collectives with the same grid sizes)
  if (threadIdx.x < a.N) {
    const unsigned long long want = a.want;
    const unsigned long long* c = a.my_cnt + (int64_t)threadIdx.x * kPxCntStride;
    long long spins = 0;
    while (ld_acquire_sys(c) < want) {
      // ~a minute: a peer never arrived (a legitimately late peer -- host
      // work between calls -- is far inside this); once flagged, later
      // calls do not wait
      if (*reinterpret_cast<volatile int*>(a.err) || ++spins > (1ll << 30)) {
        atomicExch(a.err, 1);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  __threadfence_system();
  for (int64_t e = e0 + threadIdx.x; e < e1; e += kThreads) {
    double v = 0.0;
    for (int s = 0; s < a.N; ++s) v += __ldcg(a.my_recv + ((int64_t)par * a.N + s) * a.slot + e);
    a.buf[e] = v;
  }
}

// The multi-rank A^T q epilogue as ONE kernel: the split partial sums of
// k_gemv_t2 reduced for this CTA's columns (fixed order), pushed straight
// into every peer's slot, the cross-rank sum in rank order, then
// z -= beta p and the non-finite check (k_gemv_t_finalize + all-reduce +
// k_axpy_check fused).  Never skips on a halted run: every rank pushes and
// counts in every call, so the cumulative counters stay in step.
__global__ void __launch_bounds__(kThreads)
k_gemv_t_fin_px(PxArgs a, const double* __restrict__ part, int64_t ldz, int nsplit, int64_t n,
                const double* __restrict__ beta, const double* __restrict__ pprev,
                DevState* st, int step, int check) {
  const int par = (int)(a.seq & 1);
  const int64_t chunk = (a.L + gridDim.x - 1) / gridDim.x;
  const int64_t e0 = (int64_t)blockIdx.x * chunk;
  const int64_t e1 = min(a.L, e0 + chunk);
  for (int64_t e = e0 + threadIdx.x; e < e1; e += kThreads) {
    double v = 0.0;
    if (e < n)
      for (int k = 0; k < nsplit; ++k) v += part[(int64_t)k * ldz + e];
    for (int r = 0; r < a.N; ++r) a.recv[r][((int64_t)par * a.N + a.rank) * a.slot + e] = v;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x < a.N)
    atomicAdd_system(a.cnt[threadIdx.x] + (int64_t)a.rank * kPxCntStride, 1ull);
  if (threadIdx.x < a.N) {
    const unsigned long long* c = a.my_cnt + (int64_t)threadIdx.x * kPxCntStride;
    long long spins = 0;
    while (ld_acquire_sys(c) < a.want) {
      if (*reinterpret_cast<volatile int*>(a.err) || ++spins > (1ll << 30)) {
        atomicExch(a.err, 1);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  __threadfence_system();
  for (int64_t e = e0 + threadIdx.x; e < e1; e += kThreads) {
    double v = 0.0;
    for (int s = 0; s < a.N; ++s) v += __ldcg(a.my_recv + ((int64_t)par * a.N + s) * a.slot + e);
    if (e < n && pprev) v = v - (*beta) * pprev[e];
    a.buf[e] = e < n ? v : 0.0;
    if (check && e < n) flag_nonfinite(st, v, step);
  }
}

}  // namespace ksvd
