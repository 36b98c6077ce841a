// exec.cu -- FAST stage execution over NVLink 5 / NVSwitch (sm_100a).
//
// One process per GPU.  Every rank owns ONE symmetric allocation exported
// with CUDA IPC and mapped by every peer:
//
//   [0, 4 KiB)          flags: u64 counters (see CTR_*), peers add to them
//   [4 KiB, +2*G*G*8)   demand matrix, double-buffered by call parity
//   recv region         alltoallv result (source-major segments)
//   staging region      balanced-in bytes and proxy-held redistribution bytes
//
// Kernels (all stream-ordered on the caller's stream, no host round trip):
//   gather_demand_kernel  P2P all-gather of the per-rank demand rows
//   plan_kernel           plan_compile_par (plan_par.cuh), one CTA
//   exec_kernel           persistent, `blocks` CTAs per rank: entry barrier,
//                         then the rank's ops in phase order, chunked, each
//                         chunk a 16-byte-vectorised copy into peer HBM
//                         followed by a release-add on the consumer's counter;
//                         consumers acquire before reading staging.
//
// Deadlock freedom: ops are emitted in phase order (balance < direct <
// from-staging < redistribution) and every wait targets an earlier phase, so
// with all CTAs of all ranks co-resident (grid <= SM count) every wait is
// eventually satisfied.  Every wait is bounded by a timeout that records
// status 3 instead of hanging the device.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "fastb200.h"
#include "launch.cuh"
#include "plan_par.cuh"
#include "synth_dev.cuh"

namespace {

constexpr int64_t kCtrBytes = 4096;                                // counters
constexpr int64_t kFlagBytes = kCtrBytes + (int64_t)FAST_MAX_SLOTS * 8;  // + slot flags
constexpr int CTR_ARRIVE = 0;   // entry barrier, monotonic (+1 per peer/call)
constexpr int CTR_GO = 1;       // local: barrier passed for epoch
constexpr int CTR_RECV = 3;     // chunks landed in my recv
constexpr int CTR_GATHER = 4;   // demand rows landed (monotonic)
constexpr int CTR_STATUS = 5;   // local error word
constexpr int CTR_WORK_P = 6;   // local: next producer chunk (reset per call)
constexpr int CTR_WORK_F = 7;   // local: next forwarder chunk (reset per call)
constexpr int CTR_EPOCH = 9;    // local: epoch of the current call (device-side
                                // source of truth, so calls can be graph-captured)
constexpr int kMaxStages = 256;
#ifndef FAST_EXEC_THREADS
#define FAST_EXEC_THREADS 512
#endif
constexpr int kExecThreads = FAST_EXEC_THREADS;
constexpr long long kSpinLimitNs = 20LL * 1000 * 1000 * 1000;  // 20 s

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Protocol fuzzing (-DFAST_EXEC_FUZZ, test builds only): a pseudo-random
// 0..4 us sleep before every signal and every wait, so the flag protocol is
// exercised under arbitrary interleavings of producers and consumers.
#ifdef FAST_EXEC_FUZZ
__device__ __forceinline__ void fuzz_delay() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  uint32_t h = (uint32_t)(t ^ (t >> 17)) * 0x9E3779B1u ^ (blockIdx.x * 0x85EBCA6Bu) ^
               (threadIdx.x * 0xC2B2AE35u) ^ (blockIdx.y * 0x27D4EB2Fu);
  h ^= h >> 15;
  if (h & 1) __nanosleep(h % 4096);
}
#define FAST_FUZZ() fuzz_delay()
#else
#define FAST_FUZZ()
#endif

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  FAST_FUZZ();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_release_sys_add(uint64_t* p, uint64_t v) {
  FAST_FUZZ();
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spin until *p >= target (acquire).  false on timeout.  Polling backs off
// exponentially (to 512 ns) so that many waiting CTAs do not flood one L2
// line while the CTA they wait for is working.
__device__ bool wait_geq(const uint64_t* p, uint64_t target, bool sys) {
  FAST_FUZZ();
  const uint64_t t0 = globaltimer();
  unsigned sleep_ns = 32;
  int spins = 0;
  for (;;) {
    const uint64_t v = sys ? ld_acquire_sys(p) : ld_acquire_gpu(p);
    if (v >= target) return true;
    if (++spins > 8) {
      __nanosleep(sleep_ns);
      sleep_ns = sleep_ns < 512 ? sleep_ns * 2 : 512;
      if ((int64_t)(globaltimer() - t0) > kSpinLimitNs) return false;
    }
  }
}

#ifndef FAST_COPY_UNROLL
#define FAST_COPY_UNROLL 4  // 16-byte vectors in flight per thread per copy loop
#endif
constexpr int kMaxRanks = 16;       // one NVSwitch node
constexpr int kTimelineStride = FAST_TIMELINE_STRIDE;
static_assert(FAST_TIMELINE_STRIDE == FAST_TL_STAGE0 + 4 * kMaxStages, "timeline layout");

struct ExecArgs {
  uint8_t* const* peers;  // [world] base of every rank's symmetric block
  const fast_op* ops;
  const int32_t* n_ops;
  const int32_t* plan_status;
  const uint8_t* sends[kMaxRanks];  // indexed by blockIdx.y (local rank slot)
  const uint8_t* send;
  int64_t recv_off, staging_off;  // region offsets inside a symmetric block
  int64_t chunk;
  int64_t epoch;
  int64_t* timeline;
  int rank, world;
  int skip_barrier;  // caller already synchronised the ranks for this epoch
  // fused pack -> send (fast_comm_set_send_rows): when row_src is set, SEND
  // offsets are virtual; virtual row r is row row_src[r] of rows_base
  const uint8_t* rows_base;
  const int32_t* row_src;
  uint32_t row_vec, row_magic;  // row_bytes / 16; udiv magic for it
  int row_l;                    // ceil(log2(row_vec))
  const uint8_t* rows_bases[kMaxRanks];  // group mode: per local rank slot
  const int32_t* row_srcs[kMaxRanks];
  int64_t send_cap;  // bytes readable from the send side (-1: unchecked)
  int64_t recv_cap, staging_cap;  // region sizes of every rank's block
};

__device__ __forceinline__ uint64_t* ctr(uint8_t* base, int idx) {
  return reinterpret_cast<uint64_t*>(base) + idx;
}
__device__ __forceinline__ uint64_t* slot_flag(uint8_t* base, int64_t slot) {
  return reinterpret_cast<uint64_t*>(base + kCtrBytes) + slot;
}

// ---- CTA-wide byte copy, 16-byte vectorised on the destination ------------
__device__ __forceinline__ uint4 ld16(const uint8_t* p, bool nc) {
  uint4 v;
  if (nc) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  } else {
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  }
  return v;
}
__device__ __forceinline__ void st16(uint8_t* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

// Extract 16 bytes starting `sh` (1..15) bytes into the 32-byte window a:b.
__device__ __forceinline__ uint4 shift_window(const uint4 a, const uint4 b, int sh) {
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  const int ws = sh >> 2, bs = (sh & 3) * 8;
  uint32_t o[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (ws == c) { lo = w[c + j]; hi = w[c + j + 1]; }
    o[j] = __funnelshift_r(lo, hi, bs);
  }
  return make_uint4(o[0], o[1], o[2], o[3]);
}

__device__ void cta_copy(uint8_t* dst, const uint8_t* src, int64_t len, bool nc) {
  const int tid = threadIdx.x, nt = blockDim.x;
  int64_t head = (16 - ((uintptr_t)dst & 15)) & 15;
  if (head > len) head = len;
  if (tid < head) dst[tid] = src[tid];
  dst += head;
  src += head;
  len -= head;
  const int64_t nw = len >> 4;
  const int sh = (int)((uintptr_t)src & 15);
  constexpr int U = FAST_COPY_UNROLL;
  if (sh == 0) {
    int64_t wi = tid;
    for (; wi + (U - 1) * nt < nw; wi += U * nt) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld16(src + (wi + u * nt) * 16, nc);
#pragma unroll
      for (int u = 0; u < U; ++u) st16(dst + (wi + u * nt) * 16, v[u]);
    }
    for (; wi < nw; wi += nt) st16(dst + wi * 16, ld16(src + wi * 16, nc));
  } else {
    const uint8_t* sa = src - sh;  // 16-byte aligned
    int64_t wi = tid;
    for (; wi + (U - 1) * nt < nw; wi += U * nt) {
      uint4 a[U], b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a[u] = ld16(sa + (wi + u * nt) * 16, nc);
        b[u] = ld16(sa + (wi + u * nt) * 16 + 16, nc);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) st16(dst + (wi + u * nt) * 16, shift_window(a[u], b[u], sh));
    }
    for (; wi < nw; wi += nt)
      st16(dst + wi * 16, shift_window(ld16(sa + wi * 16, nc), ld16(sa + wi * 16 + 16, nc), sh));
  }
  const int64_t tail = len - nw * 16;
  if (tid < tail) dst[nw * 16 + tid] = src[nw * 16 + tid];
}

// ---- row-mapped source (fused MoE pack -> lane send) ------------------------
// Virtual send word vw (16 B) lies in virtual row q = vw / row_vec, which is
// token row row_src[q]; the division is Granlund-Montgomery (exact for every
// u32 vw), so the per-word cost is one umulhi and an L1-resident index load.
__device__ __forceinline__ const uint8_t* vword(const ExecArgs& a, uint32_t vw) {
  uint32_t q = vw;
  if (a.row_vec > 1) {
    const uint32_t t = __umulhi(vw, a.row_magic);
    q = (t + ((vw - t) >> 1)) >> (a.row_l - 1);
  }
  const uint32_t r = vw - q * a.row_vec;
  return a.rows_base + ((int64_t)__ldg(a.row_src + q) * a.row_vec + r) * 16;
}

// cta_copy with the source bytes [vsrc, vsrc + len) of the virtual send buffer
__device__ void cta_copy_rows(uint8_t* dst, int64_t vsrc, int64_t len, const ExecArgs& a) {
  const int tid = threadIdx.x, nt = blockDim.x;
  int64_t head = (16 - ((uintptr_t)dst & 15)) & 15;
  if (head > len) head = len;
  if (tid < head) dst[tid] = vword(a, (uint32_t)((vsrc + tid) >> 4))[(vsrc + tid) & 15];
  dst += head;
  vsrc += head;
  len -= head;
  const int64_t nw = len >> 4;
  const int sh = (int)(vsrc & 15);
  const uint32_t w0 = (uint32_t)(vsrc >> 4);
  constexpr int U = FAST_COPY_UNROLL;
  if (sh == 0) {
    int64_t wi = tid;
    for (; wi + (U - 1) * nt < nw; wi += U * nt) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld16(vword(a, w0 + (uint32_t)(wi + u * nt)), true);
#pragma unroll
      for (int u = 0; u < U; ++u) st16(dst + (wi + u * nt) * 16, v[u]);
    }
    for (; wi < nw; wi += nt) st16(dst + wi * 16, ld16(vword(a, w0 + (uint32_t)wi), true));
  } else {
    int64_t wi = tid;
    for (; wi + (U - 1) * nt < nw; wi += U * nt) {
      uint4 x[U], y[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        x[u] = ld16(vword(a, w0 + (uint32_t)(wi + u * nt)), true);
        y[u] = ld16(vword(a, w0 + (uint32_t)(wi + u * nt) + 1), true);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) st16(dst + (wi + u * nt) * 16, shift_window(x[u], y[u], sh));
    }
    for (; wi < nw; wi += nt)
      st16(dst + wi * 16, shift_window(ld16(vword(a, w0 + (uint32_t)wi), true),
                                       ld16(vword(a, w0 + (uint32_t)wi + 1), true), sh));
  }
  const int64_t tail = len - nw * 16;
  if (tid < tail) {
    const int64_t v = vsrc + nw * 16 + tid;
    dst[nw * 16 + tid] = vword(a, (uint32_t)(v >> 4))[v & 15];
  }
}

// ---- kernels ----------------------------------------------------------------

// P2P all-gather of this rank's demand row (one warp): row[rank] (own
// segment, kept local) goes to the self-size vector, D keeps a zero
// diagonal (DemandMatrix invariant, model.py:97-98).  Returns false on timeout.
__device__ bool gather_rows(uint8_t* const* peers, const int64_t* row, int64_t epoch, int rank,
                            int world, int64_t demand_off) {
  const int G = world;
  const int par = (int)(epoch & 1);
  const int lane = threadIdx.x & 31;
  for (int r = lane; r < world; r += 32) {
    int64_t* dm = reinterpret_cast<int64_t*>(peers[r] + demand_off) + (int64_t)par * (G * G + G);
    for (int h = 0; h < G; ++h) dm[(int64_t)rank * G + h] = h == rank ? 0 : row[h];
    dm[(int64_t)G * G + rank] = row[rank];
  }
  __syncwarp();
  bool ok = true;
  if (lane == 0) {
    __threadfence_system();
    for (int r = 0; r < world; ++r) red_release_sys_add(ctr(peers[r], CTR_GATHER), 1);
    ok = wait_geq(ctr(peers[rank], CTR_GATHER), (uint64_t)epoch * world, true);
  }
  const bool all_ok = __shfl_sync(0xffffffffu, ok ? 1 : 0, 0) != 0;
  // lane 0's acquire covers the peers' rows; __syncwarp orders the other
  // lanes' later reads of them after it (a shuffle alone orders no memory)
  __syncwarp();
  return all_ok;
}

// epoch_in > 0: use it; 0: this call's epoch is the device counter + 1.
// After the gather the matrix (+ self sizes) is copied into the fixed third
// slot, so later kernels of the call take call-invariant pointers.
__global__ void bump_epoch_kernel(uint8_t* me) {
  volatile uint64_t* ep = reinterpret_cast<volatile uint64_t*>(me) + CTR_EPOCH;
  *ep = *ep + 1;
}

__global__ void gather_demand_kernel(uint8_t* const* peers, const int64_t* row,
                                     int64_t epoch_in, int rank, int world,
                                     int64_t demand_off, int32_t* zero_status) {
  __shared__ int64_t s_epoch;
  pdl_trigger();  // the synthesis kernels may launch; they wait for this grid
  if (threadIdx.x >= 32) return;
  if (zero_status && threadIdx.x == 0) *zero_status = FAST_OK;  // the call's synthesis status
  uint8_t* me = peers[rank];
  if (threadIdx.x == 0) {
    volatile uint64_t* ep = reinterpret_cast<volatile uint64_t*>(me) + CTR_EPOCH;
    const int64_t e = epoch_in > 0 ? epoch_in : (int64_t)*ep + 1;
    *ep = (uint64_t)e;
    s_epoch = e;
  }
  __syncwarp();
  const int64_t e = s_epoch;
  const bool ok = gather_rows(peers, row, e, rank, world, demand_off);
  if (!ok && threadIdx.x == 0)
    atomicExch(reinterpret_cast<unsigned long long*>(ctr(me, CTR_STATUS)), 3ull);
  const int64_t slot = (int64_t)world * world + world;
  const int64_t* src = reinterpret_cast<const int64_t*>(me + demand_off) + (e & 1) * slot;
  int64_t* dst = reinterpret_cast<int64_t*>(me + demand_off) + 2 * slot;
  for (int64_t i = threadIdx.x; i < slot; i += 32) dst[i] = src[i];
}

__device__ __forceinline__ int64_t nchunks(int64_t len, int64_t chunk) {
  return (len + chunk - 1) / chunk;
}

// Raw CTA copy of `bytes` split over the grid (NVLink characterisation:
// dst or src may be a peer mapping).  nc: read the source through the
// non-coherent path.
__global__ void __launch_bounds__(kExecThreads) raw_copy_kernel(uint8_t* dst, const uint8_t* src,
                                                                int64_t bytes, int64_t chunk,
                                                                int nc) {
  const int64_t nch = (bytes + chunk - 1) / chunk;
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const int64_t off = c * chunk;
    const int64_t len = bytes - off < chunk ? bytes - off : chunk;
    cta_copy(dst + off, src + off, len, nc != 0);
  }
}

// Device plan kernel: takes n_stages / synthesis status from device memory.
// The plan is a sequential walk (one thread), so every input it touches and
// its workspace are first staged into shared memory by the whole CTA when
// they fit (`smem_ok`); otherwise it runs on the global copies.
constexpr int kPlanThreads = 256;
constexpr size_t kPlanSmemMax = 160 * 1024;

__host__ __device__ inline int plan_stage_cap(int n) { return n * n - 2 * n + 2; }

__host__ __device__ inline size_t plan_smem_bytes(int n, int m) {
  const int64_t G = (int64_t)n * m, K = plan_stage_cap(n);
  size_t b = (size_t)fastplan::par_ws_bytes(n, m, (int)K) + 16;
  b += (size_t)(G * G + G) * 8;        // D + self sizes
  b += (size_t)K * 4 + 16;             // order
  b += (size_t)K * n + 16;             // perm
  b += (size_t)K * n * 8 + 16;         // stage bytes
  return (b + 127) & ~(size_t)127;
}

// Stage the plan inputs + workspace in `psm` (whole CTA) when they fit
// (`smem_ok`), else run on the global copies and the global workspace; the
// whole CTA then builds the plan (plan_par.cuh).  Caller guarantees the
// synthesis status is OK.
// SMEM is a template parameter (not a runtime flag) so that, with the build
// fully inlined, every staged pointer keeps the shared address space and the
// plan runs on LDS/STS rather than generic loads.
template <bool SMEM>
__device__ __forceinline__ void plan_cta(fastplan::PlanIn in, fastplan::PlanOut out, char* psm) {
  void* ws = out.ws;
  if constexpr (SMEM) {
    const int n = in.n, G = in.n * in.m, K = in.K;
    char* p = psm;
    ws = p; p += ((size_t)fastplan::par_ws_bytes(in.n, in.m, K) + 16 + 15) & ~(size_t)15;
    int64_t* D = (int64_t*)p; p += (size_t)G * G * 8;
    int64_t* ss = (int64_t*)p; p += (size_t)G * 8;
    int32_t* ord = (int32_t*)p; p += ((size_t)K * 4 + 16 + 15) & ~(size_t)15;
    int64_t* sb = (int64_t*)p; p += (size_t)K * n * 8 + 16;
    uint8_t* pm = (uint8_t*)p;
    for (int i = threadIdx.x; i < G * G; i += blockDim.x) D[i] = in.D[i];
    for (int i = threadIdx.x; i < G; i += blockDim.x) ss[i] = in.send_self ? in.send_self[i] : 0;
    for (int i = threadIdx.x; i < in.n_stages; i += blockDim.x) ord[i] = in.order[i];
    // only the kept stages' rows are read by the plan
    for (int i = threadIdx.x; i < in.n_stages * n; i += blockDim.x) {
      const int k = in.order[i / n], u = i % n;
      sb[(int64_t)k * n + u] = in.sbytes[(int64_t)k * n + u];
      pm[(int64_t)k * n + u] = in.perm[(int64_t)k * n + u];
    }
    __syncthreads();
    in.D = D;
    in.send_self = in.send_self ? ss : nullptr;
    in.order = ord;
    in.sbytes = sb;
    in.perm = pm;
  }
  fastplan::plan_compile_par(in, out, ws);
}

__global__ void __launch_bounds__(kPlanThreads)
    fast_plan_kernel_dev(fastplan::PlanIn in, fastplan::PlanOut out, const int32_t* n_stages,
                         const int32_t* sched_status, int smem_ok) {
  extern __shared__ __align__(16) char psm[];
  pdl_trigger();
  pdl_wait();  // the schedule comes from the previous kernel of the chain
  PLAN_STAMP(9);
  if (*sched_status != FAST_OK) {
    if (threadIdx.x == 0) {
      *out.n_ops = 0;
      *out.status = *sched_status;
    }
    return;
  }
  PLAN_STAMP(0);
  in.n_stages = *n_stages;
  if (smem_ok) plan_cta<true>(in, out, psm);
  else plan_cta<false>(in, out, psm);
}

// ---- fused single-launch path (n <= 6): everything before the exec loop ----
constexpr int kFusedMaxN = 6;  // stage capacity <= 32: the decompose warp sorts

struct FusedArgs {
  const int64_t* counts;     // this rank's demand row (device)
  int n, m;
  int64_t demand_off;
  fast_sched_bufs sched;     // B = 1
  fastplan::PlanIn pin;      // shape / capacities (pointers filled in)
  fastplan::PlanOut pout;
};

__host__ __device__ inline size_t fused_smem_bytes(int n, int m) {
  const size_t tiles = (size_t)n * n * (m * m + 1) * 8;
  return ((tiles + 127) & ~(size_t)127) + ((dec_smem_bytes_t<1>(n) + 127) & ~(size_t)127) +
         plan_smem_bytes(n, m);
}

// CTA 0 of the fused exec kernel: gather -> balance -> decompose/strip/sort
// -> plan, all on this device, before the entry barrier opens the exec loop.
__device__ bool fused_prologue(const FusedArgs& f, uint8_t* const* peers, int rank, int world,
                               int64_t epoch, char* sm, int64_t* tl) {
  __shared__ int s_ok;
  const int tid = threadIdx.x;
  if (tid == 0) s_ok = 1;
  if (tl && tid == 0) tl[5] = (int64_t)globaltimer();
  __syncthreads();
  if (tid < 32 && !gather_rows(peers, f.counts, epoch, rank, world, f.demand_off) && tid == 0)
    s_ok = 0;
  const int n = f.n, m = f.m, G = n * m;
  const int64_t* D = reinterpret_cast<const int64_t*>(peers[rank] + f.demand_off) +
                     (epoch & 1) * ((int64_t)G * G + G);
  __syncthreads();
  {  // the fixed slot always holds the latest gathered matrix (+ self sizes)
    int64_t* fixed = reinterpret_cast<int64_t*>(peers[rank] + f.demand_off) +
                     2 * ((int64_t)G * G + G);
    for (int i = tid; i < G * G + G; i += blockDim.x) fixed[i] = D[i];
  }
  if (tid == 0) *f.sched.status = FAST_OK;
  if (tl && tid == 0) tl[6] = (int64_t)globaltimer();
  __syncthreads();
  if (!s_ok) {
    // the other CTAs read the plan after GO: never leave them the previous
    // call's op list
    if (tid == 0) {
      *f.pout.n_ops = 0;
      *f.pout.status = FAST_EINVARIANT;
      __threadfence();
    }
    __syncthreads();
    return false;
  }
  // build_balance_plan + reduce_to_server_level, one thread per tile
  const int TS = m * m + 1;
  const int slots = m > 1 ? m - 1 : 1;
  for (int t = tid; t < n * n; t += blockDim.x) {
    const int i = t / n, j = t % n;
    int64_t* tl = reinterpret_cast<int64_t*>(sm) + (int64_t)t * TS;
    bool bad = false;
    int64_t sum = 0;
    for (int p = 0; p < m; ++p)
      for (int q = 0; q < m; ++q) {
        const int64_t v = D[(int64_t)(i * m + p) * G + j * m + q];
        tl[p * m + q] = v;
        if (v < 0) { bad = true; continue; }
        if (i == j && p == q && v != 0) bad = true;
        sum = sat_add(sum, v);
      }
    f.sched.server[i * n + j] = sum;
    if (bad || sum >= kMaxSafeTotal) {  // past the 2^62 guard: model.py:26
      raise_status(f.sched.status, FAST_EVALIDATION);
    } else if (i != j) {
      const int tidx = i * (n - 1) + (j < i ? j : j - 1);
      int nm = balance_tile<0>(tl, m, f.sched.moves + (int64_t)tidx * slots, slots);
      if (nm < 0) { raise_status(f.sched.status, FAST_EINVARIANT); nm = 0; }
      f.sched.move_count[tidx] = nm;
    }
    for (int p = 0; p < m; ++p)
      for (int q = 0; q < m; ++q)
        f.sched.balanced[(int64_t)(i * m + p) * G + j * m + q] = tl[p * m + q];
  }
  __threadfence_block();
  __syncthreads();
  if (tl && tid == 0) tl[7] = (int64_t)globaltimer();
  char* dsm = sm + (((size_t)n * n * TS * 8 + 127) & ~(size_t)127);
  if (tid < 32)
    decompose_one<1>(dsm, f.sched.server, 0, n, FAST_DEC_SERVER, 1, f.sched, tid);
  __threadfence_block();
  __syncthreads();
  if (tl && tid == 0) tl[12] = (int64_t)globaltimer();
  const int st = *f.sched.status;
  fastplan::PlanOut out = f.pout;
  if (st != FAST_OK) {
    if (tid == 0) {
      *out.n_ops = 0;
      *out.status = st;
    }
    return true;  // the exec loop sees plan status != OK and moves nothing
  }
  fastplan::PlanIn in = f.pin;
  in.D = D;
  in.send_self = D + (int64_t)G * G;
  in.n_stages = *f.sched.n_stages;
  in.order = f.sched.stage_order;
  in.perm = f.sched.stage_perm;
  in.sbytes = f.sched.stage_bytes;
  char* psm = dsm + ((dec_smem_bytes_t<1>(n) + 127) & ~(size_t)127);
  plan_cta<true>(in, out, psm);
  __threadfence();
  __syncthreads();
  return true;
}

// grid (blocks, ranks_in_launch): blockIdx.y selects the rank this CTA acts
// for -- 1 in the multi-process mode, all `world` ranks in the one-GPU group
// mode (cooperative launch, so every rank's CTAs are co-resident).
template <bool FUSED>
__global__ void __launch_bounds__(kExecThreads) exec_kernel(ExecArgs a, FusedArgs f) {
  __shared__ unsigned long long s_red[3];  // recv chunks expected, producer / redist bytes
  __shared__ int s_fail;
  extern __shared__ __align__(16) char fsm[];
  pdl_wait();  // the plan comes from the previous kernel of the chain
  a.rank += blockIdx.y;
  a.send = a.sends[blockIdx.y];
  if (a.row_srcs[blockIdx.y]) {
    a.rows_base = a.rows_bases[blockIdx.y];
    a.row_src = a.row_srcs[blockIdx.y];
  }
  if (a.timeline) a.timeline += (int64_t)blockIdx.y * kTimelineStride;
  uint8_t* me = a.peers[a.rank];
  uint64_t* status = ctr(me, CTR_STATUS);
  const int tid = threadIdx.x;
  const uint64_t epoch =
      a.epoch > 0 ? (uint64_t)a.epoch : *reinterpret_cast<volatile uint64_t*>(ctr(me, CTR_EPOCH));
  if (tid == 0) s_fail = 0;
  // fused path: CTA 0 gathers D, synthesises the schedule and compiles the
  // plan before the barrier; the other CTAs wait for GO as usual
  if (FUSED && blockIdx.x == 0) {
    if (!fused_prologue(f, a.peers, a.rank, a.world, (int64_t)epoch, fsm, a.timeline) && tid == 0)
      s_fail = 1;
    __syncthreads();
  }

  // measured timeline: open every window (start = max, end = 0) before the
  // barrier releases the other CTAs
  if (a.timeline && blockIdx.x == 0) {
    uint64_t* t = reinterpret_cast<uint64_t*>(a.timeline);
    for (int i = FAST_TL_BALANCE + tid; i < kTimelineStride; i += blockDim.x)
      if (i < 12 || i >= FAST_TL_STAGE0) t[i] = ((i & 1) == 0) ? ~0ull : 0ull;
    __syncthreads();
  }
  // ---- entry barrier (CTA 0): reset the recv counter, arrive everywhere ---
  if (blockIdx.x == 0 && tid == 0) {
    if (a.timeline) a.timeline[0] = (int64_t)globaltimer();
    // RECV is zero here: every exec leaves it zeroed at exit, and a peer can
    // only signal epoch e after this rank published its demand row for e
    reinterpret_cast<volatile uint64_t*>(me)[CTR_WORK_P] = 0;
    reinterpret_cast<volatile uint64_t*>(me)[CTR_WORK_F] = 0;
    __threadfence_system();
    for (int r = 0; r < a.world; ++r)
      if (r != a.rank) red_release_sys_add(ctr(a.peers[r], CTR_ARRIVE), 1);
    // fast_alltoallv: the demand all-gather of this epoch already proved that
    // every peer entered it (hence finished the previous one); no wait needed
    if (!a.skip_barrier && !wait_geq(ctr(me, CTR_ARRIVE), epoch * (a.world - 1), true))
      s_fail = 1;
    st_release_gpu(ctr(me, CTR_GO), epoch);
    if (a.timeline) a.timeline[1] = (int64_t)globaltimer();
  } else if (tid == 0) {
    if (!wait_geq(ctr(me, CTR_GO), epoch, false)) s_fail = 1;
  }
  if (tid < 3) s_red[tid] = 0ull;
  __syncthreads();
  const int nops = (*a.plan_status == FAST_OK) ? *a.n_ops : 0;
  // bounds of every op this rank executes (defence in depth: the plan
  // compile already sizes everything): the send side against the caller's
  // send buffer, the destination / staging ranges against the regions, the
  // flag slots against the slot table.  Any violation: nothing is copied.
  {
    bool over = false;
    for (int i = tid; i < nops; i += blockDim.x) {
      const fast_op o = a.ops[i];
      if (o.exec_rank != a.rank) continue;
      const int64_t dcap = o.dst_buf == FAST_BUF_RECV ? a.recv_cap : a.staging_cap;
      over |= o.len < 0 || o.src_off < 0 || o.dst_off < 0 || o.dst_off + o.len > dcap;
      over |= o.dst_rank < 0 || o.dst_rank >= a.world;
      if (o.src_buf == FAST_BUF_SEND) over |= a.send_cap >= 0 && o.src_off + o.len > a.send_cap;
      else over |= o.src_off + o.len > a.staging_cap;
      if (o.sig_slot >= 0) over |= o.sig_slot + nchunks(o.len, a.chunk) > FAST_MAX_SLOTS;
      if (o.wait_slot >= 0)
        over |= o.wait_slot + (o.wait_off + o.len + a.chunk - 1) / a.chunk > FAST_MAX_SLOTS;
    }
    if (__syncthreads_or(over)) {
      if (tid == 0) s_fail = 2;  // validation: nothing is copied
      __syncthreads();
    }
  }
  {
    unsigned long long rc = 0, pb = 0, rb = 0;
    for (int i = tid; i < nops; i += blockDim.x) {
      const fast_op o = a.ops[i];
      if (o.dst_rank == a.rank && o.dst_buf == FAST_BUF_RECV) rc += nchunks(o.len, a.chunk);
      if (o.exec_rank == a.rank) {
        if (o.phase == FAST_PH_REDIST) rb += o.len;
        else pb += o.len;
      }
    }
    if (rc) atomicAdd(&s_red[0], rc);
    if (pb) atomicAdd(&s_red[1], pb);
    if (rb) atomicAdd(&s_red[2], rb);
  }
  __syncthreads();
  // CTA pools: producers (balance, intra, stage sends) and forwarders
  // (redistribution), sized by bytes; producers never wait on forwarders.
  const int NB = gridDim.x;
  int R = 0;
  if (s_red[2] > 0 && NB > 1) {
    R = (int)((double)NB * (double)s_red[2] / (double)(s_red[1] + s_red[2]) + 0.5);
    R = R < 1 ? 1 : (R > NB - 1 ? NB - 1 : R);
  }
  const bool fwd = (int)blockIdx.x >= NB - R;

  // Dynamic chunk scheduling: each pool hands out its chunks in op-list
  // (phase) order through a local atomic counter, so every chunk a CTA waits
  // on was handed out earlier -- the same deadlock argument as a static
  // deal -- while fast CTAs absorb the tail.
  __shared__ long long s_item;
  unsigned long long* wctr =
      reinterpret_cast<unsigned long long*>(ctr(me, fwd ? CTR_WORK_F : CTR_WORK_P));
  int i = 0;          // op cursor (monotone: grabbed items only increase)
  int64_t base = 0;   // first item index of op i within this pool
  for (;;) {
    if (tid == 0) s_item = s_fail ? -1 : (long long)atomicAdd(wctr, 1ull);
    __syncthreads();
    const long long it = s_item;
    __syncthreads();
    if (it < 0) break;
    // advance to the op holding item `it`
    int64_t nc = 0;
    bool found = false;
    for (; i < nops; ++i) {
      const fast_op& q = a.ops[i];
      if (q.exec_rank != a.rank) continue;
      if (R > 0 && ((q.phase == FAST_PH_REDIST) != fwd)) continue;
      nc = nchunks(q.len, a.chunk);
      if (it < base + nc) { found = true; break; }
      base += nc;
    }
    if (!found) break;
    const fast_op o = a.ops[i];
    const int64_t c = it - base;
    const uint8_t* src = (o.src_buf == FAST_BUF_SEND ? a.send : me + a.staging_off) + o.src_off;
    uint8_t* peer = a.peers[o.dst_rank];
    uint8_t* dst = peer + (o.dst_buf == FAST_BUF_RECV ? a.recv_off : a.staging_off) + o.dst_off;
    const int64_t off = c * a.chunk;
    const int64_t len = o.len - off < a.chunk ? o.len - off : a.chunk;
    if (o.wait_slot >= 0) {  // producer chunks covering this chunk's source bytes
      if (tid == 0) {
        const int64_t p0 = (o.wait_off + off) / a.chunk;
        const int64_t p1 = (o.wait_off + off + len - 1) / a.chunk;
        for (int64_t q = p0; q <= p1 && !s_fail; ++q)
          if (!wait_geq(slot_flag(me, o.wait_slot + q), epoch, true)) s_fail = 1;
      }
      __syncthreads();
      if (s_fail) break;
    }
    uint64_t t_chunk = 0;
    if (a.timeline && tid == 0) t_chunk = globaltimer();
    if (o.src_buf == FAST_BUF_SEND && a.row_src)
      cta_copy_rows(dst + off, o.src_off + off, len, a);
    else
      cta_copy(dst + off, src + off, len, o.src_buf == FAST_BUF_SEND);
    __syncthreads();
    if (tid == 0) {
      __threadfence_system();
      if (o.sig_slot >= 0) st_release_sys(slot_flag(peer, o.sig_slot + c), epoch);
      else red_release_sys_add(ctr(peer, CTR_RECV), 1);
      if (a.timeline) {  // (first start, last end) of this chunk's phase window
        int w;
        if (o.phase == FAST_PH_BALANCE) w = FAST_TL_BALANCE;
        else if (o.stage == FAST_STAGE_INTRA) w = FAST_TL_INTRA;
        else w = FAST_TL_STAGE0 + 4 * o.stage + (o.phase == FAST_PH_REDIST ? 2 : 0);
        unsigned long long* t = reinterpret_cast<unsigned long long*>(a.timeline) + w;
        atomicMin(t, (unsigned long long)t_chunk);
        atomicMax(t + 1, (unsigned long long)globaltimer());
      }
    }
  }
  __syncthreads();
  if (blockIdx.x == 0 && tid == 0) {
    if (a.timeline) a.timeline[3] = (int64_t)globaltimer();
    if (!s_fail && !wait_geq(ctr(me, CTR_RECV), (uint64_t)s_red[0], true)) s_fail = 1;
    reinterpret_cast<volatile uint64_t*>(me)[CTR_RECV] = 0;  // ready for the next epoch
    if (a.timeline) a.timeline[4] = (int64_t)globaltimer();
  }
  __syncthreads();
  // status word: 3 = a wait timed out (protocol), 2 = the counts overrun the
  // send buffer.  Either leaves the communicator's counters out of step with
  // its peers: it must be recreated (FastComm.check raises).
  if (tid == 0 && s_fail)
    atomicMax(reinterpret_cast<unsigned long long*>(status), s_fail == 2 ? 2ull : 3ull);
}

}  // namespace

struct fast_comm {
  int rank, world, gmax;
  int64_t recv_bytes, staging_bytes;
  int64_t demand_off, recv_off, staging_off, total;
  uint8_t* base;             // own symmetric allocation
  uint8_t** peers_host;      // [world]
  uint8_t** peers_dev;       // [world] device copy
  cudaIpcMemHandle_t handle;
  int opened;
  int64_t epoch;  // calls issued through fast_alltoallv
  int no_fuse;    // 1: always use the multi-launch path
  // fast_comm_set_send_rows state (row_src == nullptr: plain send buffer)
  const uint8_t* rows_base;
  const int32_t* row_src;
  uint32_t row_vec, row_magic;
  int row_l;
  int64_t send_cap;  // fast_comm_set_send_capacity (-1: unchecked)
  int no_pdl;        // 1: plain launches on the alltoallv chain
  int copy_self;     // 1: the exec also copies each rank's own segment
};

static void set_rowmap(ExecArgs& a, const fast_comm* c) {
  a.rows_base = c->rows_base;
  a.row_src = c->row_src;
  a.row_vec = c->row_vec;
  a.row_magic = c->row_magic;
  a.row_l = c->row_l;
}

extern "C" {

size_t fast_plan_workspace_bytes(int n, int m) {
  const int64_t seq = fastplan::plan_ws_bytes(n, m);
  const int64_t par = fastplan::par_ws_bytes(n, m, plan_stage_cap(n));
  return (size_t)(seq > par ? seq : par);
}

int64_t fast_plan_op_capacity(int n, int m) {
  return fastplan::plan_op_capacity(n, m, n * n - 2 * n + 2);
}

static int plan_compile_launch(const int64_t* D, const int64_t* send_self, int n, int m,
                               const fast_sched_bufs* sched, int64_t recv_capacity,
                               int64_t staging_capacity, int64_t chunk_bytes,
                               const fast_plan* plan, void* stream, bool pdl,
                               int copy_self = 0);

int fast_plan_compile(const int64_t* D, const int64_t* send_self, int n, int m,
                      const fast_sched_bufs* sched, int64_t recv_capacity,
                      int64_t staging_capacity, int64_t chunk_bytes, const fast_plan* plan,
                      void* stream) {
  return plan_compile_launch(D, send_self, n, m, sched, recv_capacity, staging_capacity,
                             chunk_bytes, plan, stream, false, 0);
}

int fast_plan_compile_ex(const int64_t* D, const int64_t* send_self, int n, int m,
                         const fast_sched_bufs* sched, int64_t recv_capacity,
                         int64_t staging_capacity, int64_t chunk_bytes, const fast_plan* plan,
                         int flags, void* stream) {
  if (flags & ~FAST_PLAN_COPY_SELF) return FAST_EVALIDATION;
  return plan_compile_launch(D, send_self, n, m, sched, recv_capacity, staging_capacity,
                             chunk_bytes, plan, stream, false,
                             (flags & FAST_PLAN_COPY_SELF) ? 1 : 0);
}

}  // extern "C"

static int plan_compile_launch(const int64_t* D, const int64_t* send_self, int n, int m,
                               const fast_sched_bufs* sched, int64_t recv_capacity,
                               int64_t staging_capacity, int64_t chunk_bytes,
                               const fast_plan* plan, void* stream, bool pdl, int copy_self) {
  if (!sched || !plan || n < 2 || m < 1 || m > FAST_MAX_GPUS_PER_SERVER) return FAST_EVALIDATION;
  fastplan::PlanIn in;
  in.n = n;
  in.m = m;
  in.K = n * n - 2 * n + 2;
  in.D = D;
  in.send_self = send_self;
  in.n_stages = -1;  // read on the device
  in.order = sched->stage_order;
  in.perm = sched->stage_perm;
  in.sbytes = sched->stage_bytes;
  in.recv_cap = recv_capacity;
  in.staging_cap = staging_capacity;
  in.op_cap = plan->op_capacity;
  in.chunk = chunk_bytes & ~(int64_t)15;
  in.copy_self = copy_self;
  fastplan::PlanOut out;
  out.ops = plan->ops;
  out.n_ops = plan->n_ops;
  out.staging_used = plan->staging_used;
  out.status = plan->status;
  out.ws = plan->workspace;
  out.scratch = nullptr;
  const size_t smem = plan_smem_bytes(n, m);
  const int smem_ok = smem <= kPlanSmemMax;
  static size_t plan_attr = 0;  // largest dynamic smem already granted
  if (smem_ok && smem > plan_attr) {
    if (cudaFuncSetAttribute(fast_plan_kernel_dev, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return FAST_ECUDA;
    plan_attr = smem;
  }
  return launch_k(fast_plan_kernel_dev, dim3(1), dim3(kPlanThreads), smem_ok ? smem : 0,
                  (cudaStream_t)stream, pdl, in, out, (const int32_t*)sched->n_stages,
                  (const int32_t*)sched->status, smem_ok) == cudaSuccess
             ? FAST_OK
             : FAST_ECUDA;
}

extern "C" {

#ifdef FAST_PLAN_PROFILE
int fast_debug_plan_prof(long long* out16) {
  return cudaMemcpyFromSymbol(out16, fastplan::g_plan_prof, 16 * sizeof(long long)) == cudaSuccess
             ? 0 : FAST_ECUDA;
}
#endif

int fast_plan_compile_host(const int64_t* D, const int64_t* send_self, int n, int m,
                           int n_stages, const int32_t* order,
                           const uint8_t* perm, const int64_t* sbytes, int64_t recv_capacity,
                           int64_t staging_capacity, int64_t chunk_bytes, fast_op* ops,
                           int64_t op_capacity,
                           int32_t* n_ops, int64_t* staging_used, void* workspace) {
  if (n < 2 || m < 1 || m > FAST_MAX_GPUS_PER_SERVER || !D || !ops || !workspace)
    return FAST_EVALIDATION;
  fastplan::PlanIn in;
  in.n = n;
  in.m = m;
  in.K = n * n - 2 * n + 2;
  in.D = D;
  in.send_self = send_self;
  in.n_stages = n_stages;
  in.order = order;
  in.perm = perm;
  in.sbytes = sbytes;
  in.recv_cap = recv_capacity;
  in.staging_cap = staging_capacity;
  in.op_cap = op_capacity;
  in.chunk = chunk_bytes & ~(int64_t)15;
  in.copy_self = 0;
  int32_t status = 0;
  fastplan::PlanOut out;
  out.ops = ops;
  out.n_ops = n_ops;
  out.staging_used = staging_used;
  out.status = &status;
  out.ws = workspace;
  out.scratch = nullptr;
  fastplan::plan_compile(in, out);
  return status;
}

int fast_comm_create(int rank, int world, int max_gpus_per_row, int64_t recv_bytes,
                     int64_t staging_bytes, fast_comm** out) {
  (void)max_gpus_per_row;
  if (!out || world < 1 || rank < 0 || rank >= world || recv_bytes < 0 || staging_bytes < 0)
    return FAST_EVALIDATION;
  fast_comm* c = (fast_comm*)calloc(1, sizeof(fast_comm));
  if (!c) return FAST_ECUDA;
  c->send_cap = -1;
  c->rank = rank;
  c->world = world;
  c->recv_bytes = recv_bytes;
  c->staging_bytes = staging_bytes;
  c->demand_off = kFlagBytes;  // counters + per-chunk slot flags
  c->recv_off = fastplan::align16(c->demand_off + 3 * ((int64_t)world * world + world) * 8 + 256);
  c->recv_off = (c->recv_off + 4095) & ~(int64_t)4095;
  c->staging_off = (c->recv_off + recv_bytes + 64 + 4095) & ~(int64_t)4095;
  c->total = (c->staging_off + staging_bytes + 64 + 4095) & ~(int64_t)4095;
  if (cudaMalloc(&c->base, (size_t)c->total) != cudaSuccess) { free(c); return FAST_ECUDA; }
  if (cudaMemset(c->base, 0, (size_t)c->recv_off) != cudaSuccess ||
      cudaIpcGetMemHandle(&c->handle, c->base) != cudaSuccess) {
    cudaFree(c->base);
    free(c);
    return FAST_ECUDA;
  }
  c->peers_host = (uint8_t**)calloc(world, sizeof(uint8_t*));
  c->peers_host[rank] = c->base;
  c->no_fuse = 1;  // the fused single launch is opt-in (fast_comm_set_fused)
  if (cudaMalloc(&c->peers_dev, sizeof(uint8_t*) * world) != cudaSuccess) {
    cudaFree(c->base);
    free(c->peers_host);
    free(c);
    return FAST_ECUDA;
  }
  cudaDeviceSynchronize();
  *out = c;
  return FAST_OK;
}

int fast_comm_ipc_handle(const fast_comm* c, void* handle64) {
  if (!c || !handle64) return FAST_EVALIDATION;
  memcpy(handle64, &c->handle, sizeof(cudaIpcMemHandle_t));
  return FAST_OK;
}

int fast_comm_open_peers(fast_comm* c, const void* handles) {
  if (!c || !handles) return FAST_EVALIDATION;
  const uint8_t* h = (const uint8_t*)handles;
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank) continue;
    cudaIpcMemHandle_t hd;
    memcpy(&hd, h + (size_t)r * 64, sizeof(hd));
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
      return FAST_ECUDA;
    c->peers_host[r] = (uint8_t*)p;
  }
  if (cudaMemcpy(c->peers_dev, c->peers_host, sizeof(uint8_t*) * c->world,
                 cudaMemcpyHostToDevice) != cudaSuccess)
    return FAST_ECUDA;
  c->opened = 1;
  return FAST_OK;
}

int fast_comm_destroy(fast_comm* c) {
  if (!c) return FAST_OK;
  cudaDeviceSynchronize();
  if (c->opened == 1)
    for (int r = 0; r < c->world; ++r)
      if (r != c->rank && c->peers_host[r]) cudaIpcCloseMemHandle(c->peers_host[r]);
  cudaFree(c->peers_dev);
  cudaFree(c->base);
  free(c->peers_host);
  free(c);
  return FAST_OK;
}

void* fast_comm_recv_ptr(const fast_comm* c) { return c ? c->base + c->recv_off : nullptr; }
void* fast_comm_staging_ptr(const fast_comm* c) { return c ? c->base + c->staging_off : nullptr; }
int64_t* fast_comm_demand_ptr(const fast_comm* c, int64_t epoch) {
  if (!c) return nullptr;
  // epoch > 0: that call's double-buffered slot; epoch <= 0: the fixed slot
  // holding the most recently gathered matrix
  const int64_t slot = epoch > 0 ? (epoch & 1) : 2;
  return reinterpret_cast<int64_t*>(c->base + c->demand_off) +
         slot * ((int64_t)c->world * c->world + c->world);
}
int64_t fast_comm_recv_capacity(const fast_comm* c) { return c ? c->recv_bytes : 0; }
int64_t fast_comm_staging_capacity(const fast_comm* c) { return c ? c->staging_bytes : 0; }

int fast_gather_demand(fast_comm* c, const int64_t* row, int64_t epoch, void* stream) {
  if (!c || !c->opened || !row || epoch < 1) return FAST_EVALIDATION;
  gather_demand_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(c->peers_dev, row, epoch, c->rank,
                                                           c->world, c->demand_off, nullptr);
  return cudaGetLastError() == cudaSuccess ? FAST_OK : FAST_ECUDA;
}

// Every CTA of every rank must be resident at once (CTAs wait on flags that
// other ranks' CTAs raise), so the grid may not exceed one wave.
static int max_resident_blocks() {
  static int cached = -1;  // one device per process (one rank per GPU)
  if (cached >= 0) return cached;
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, exec_kernel<false>, kExecThreads, 0) !=
          cudaSuccess)
    return 0;
  cached = sms * per_sm;
  return cached;
}

static int exec_launch(fast_comm* c, const fast_plan* plan, const void* send, int64_t epoch,
                       int blocks, int64_t chunk_bytes, int64_t* timeline_ns, void* stream,
                       int skip_barrier, bool pdl = false);

int fast_exec(fast_comm* c, const fast_plan* plan, const void* send, int64_t epoch, int blocks,
              int64_t chunk_bytes, int64_t* timeline_ns, void* stream) {
  return exec_launch(c, plan, send, epoch, blocks, chunk_bytes, timeline_ns, stream, 0);
}

static int exec_launch(fast_comm* c, const fast_plan* plan, const void* send, int64_t epoch,
                       int blocks, int64_t chunk_bytes, int64_t* timeline_ns, void* stream,
                       int skip_barrier, bool pdl) {
  // epoch 0: the kernel reads this call's epoch from the device counter
  if (!c || !c->opened || !plan || epoch < 0 || blocks < 1 || chunk_bytes < 16)
    return FAST_EVALIDATION;
  if (blocks > max_resident_blocks()) return FAST_EVALIDATION;
  ExecArgs a;
  memset(&a, 0, sizeof(a));
  a.peers = c->peers_dev;
  a.ops = plan->ops;
  a.n_ops = plan->n_ops;
  a.plan_status = plan->status;
  a.sends[0] = (const uint8_t*)send;
  a.recv_off = c->recv_off;
  a.staging_off = c->staging_off;
  a.chunk = chunk_bytes & ~(int64_t)15;
  a.epoch = epoch;
  a.timeline = timeline_ns;
  a.rank = c->rank;
  a.world = c->world;
  a.skip_barrier = skip_barrier;
  set_rowmap(a, c);
  a.send_cap = c->send_cap;
  a.recv_cap = c->recv_bytes;
  a.staging_cap = c->staging_bytes;
  FusedArgs f;
  memset(&f, 0, sizeof(f));
  return launch_k(exec_kernel<false>, dim3(blocks), dim3(kExecThreads), 0, (cudaStream_t)stream,
                  pdl, a, f) == cudaSuccess
             ? FAST_OK
             : FAST_ECUDA;
}

int fast_comm_create_group(int world, int64_t recv_bytes, int64_t staging_bytes,
                           fast_comm** comms) {
  if (!comms || world < 1 || world > kMaxRanks) return FAST_EVALIDATION;
  for (int r = 0; r < world; ++r) {
    int rc = fast_comm_create(r, world, 0, recv_bytes, staging_bytes, &comms[r]);
    if (rc != FAST_OK) {
      for (int q = 0; q < r; ++q) fast_comm_destroy(comms[q]);
      return rc;
    }
  }
  for (int r = 0; r < world; ++r) {
    for (int q = 0; q < world; ++q) comms[r]->peers_host[q] = comms[q]->base;
    if (cudaMemcpy(comms[r]->peers_dev, comms[r]->peers_host, sizeof(uint8_t*) * world,
                   cudaMemcpyHostToDevice) != cudaSuccess)
      return FAST_ECUDA;
    comms[r]->opened = 2;  // group member: peers are local allocations
  }
  return FAST_OK;
}

int fast_exec_group(fast_comm* const* comms, int world, const fast_plan* plan,
                    const void* const* sends, int64_t epoch, int blocks,
                    int64_t chunk_bytes, int64_t* timeline_ns, void* stream) {
  if (!comms || world < 1 || world > kMaxRanks || !plan || epoch < 1 || blocks < 1 ||
      chunk_bytes < 16)
    return FAST_EVALIDATION;
  if (blocks * world > max_resident_blocks()) return FAST_EVALIDATION;
  ExecArgs a;
  memset(&a, 0, sizeof(a));
  a.peers = comms[0]->peers_dev;
  a.ops = plan->ops;
  a.n_ops = plan->n_ops;
  a.plan_status = plan->status;
  for (int r = 0; r < world; ++r) {
    a.sends[r] = (const uint8_t*)sends[r];
    if (!comms[r]->row_src) continue;
    if (a.row_vec && a.row_vec != comms[r]->row_vec) return FAST_EVALIDATION;
    a.rows_bases[r] = comms[r]->rows_base;
    a.row_srcs[r] = comms[r]->row_src;
    a.row_vec = comms[r]->row_vec;
    a.row_magic = comms[r]->row_magic;
    a.row_l = comms[r]->row_l;
  }
  a.recv_off = comms[0]->recv_off;
  a.staging_off = comms[0]->staging_off;
  a.chunk = chunk_bytes & ~(int64_t)15;
  a.epoch = epoch;
  a.timeline = timeline_ns;
  a.rank = 0;
  a.world = world;
  a.send_cap = -1;
  a.recv_cap = comms[0]->recv_bytes;
  a.staging_cap = comms[0]->staging_bytes;
  FusedArgs f;
  memset(&f, 0, sizeof(f));
  void* args[] = {&a, &f};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)exec_kernel<false>, dim3(blocks, world),
                                              dim3(kExecThreads), args, 0,
                                              (cudaStream_t)stream);
  return e == cudaSuccess ? FAST_OK : FAST_ECUDA;
}

void* fast_comm_peer_ptr(const fast_comm* c, int rank) {
  if (!c || rank < 0 || rank >= c->world || !c->opened) return nullptr;
  return c->peers_host[rank];
}

int fast_debug_copy(void* dst, const void* src, int64_t bytes, int blocks, int64_t chunk,
                    int nc, void* stream) {
  if (!dst || !src || bytes < 0 || blocks < 1 || chunk < 16) return FAST_EVALIDATION;
  raw_copy_kernel<<<blocks, kExecThreads, 0, (cudaStream_t)stream>>>(
      (uint8_t*)dst, (const uint8_t*)src, bytes, chunk & ~(int64_t)15, nc);
  return cudaGetLastError() == cudaSuccess ? FAST_OK : FAST_ECUDA;
}

int fast_debug_memcpy(void* dst, const void* src, int64_t bytes, void* stream) {
  if (!dst || !src || bytes < 0) return FAST_EVALIDATION;
  return cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice,
                         (cudaStream_t)stream) == cudaSuccess
             ? FAST_OK
             : FAST_ECUDA;
}

// Single-launch fused path (n <= 6): gather, synthesis and plan run in CTA 0
// of the exec kernel itself.
static int launch_fused(fast_comm* c, const void* send, const int64_t* counts, int n, int m,
                        const fast_sched_bufs* sched, const fast_plan* plan, int blocks,
                        int64_t chunk_bytes, int64_t* timeline_ns, cudaStream_t stream) {
  const size_t smem = fused_smem_bytes(n, m);
  static size_t fused_attr = 0;
  static int fused_resident = 0;
  if (smem > fused_attr) {
    if (cudaFuncSetAttribute(exec_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return FAST_ECUDA;
    int dev = 0, sms = 0, per_sm = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, exec_kernel<true>, kExecThreads,
                                                      smem) != cudaSuccess)
      return FAST_ECUDA;
    fused_attr = smem;
    fused_resident = sms * per_sm;
  }
  if (blocks > fused_resident) return FAST_EVALIDATION;
  // device-side epoch (graph-capturable): bump it, the kernel reads it
  bump_epoch_kernel<<<1, 1, 0, stream>>>(c->base);
  c->epoch += 1;
  ExecArgs a;
  memset(&a, 0, sizeof(a));
  a.peers = c->peers_dev;
  a.ops = plan->ops;
  a.n_ops = plan->n_ops;
  a.plan_status = plan->status;
  a.sends[0] = (const uint8_t*)send;
  a.recv_off = c->recv_off;
  a.staging_off = c->staging_off;
  a.chunk = chunk_bytes & ~(int64_t)15;
  a.epoch = 0;
  a.timeline = timeline_ns;
  a.rank = c->rank;
  a.world = c->world;
  a.skip_barrier = 1;  // the in-kernel demand all-gather synchronises the ranks
  set_rowmap(a, c);
  a.send_cap = c->send_cap;
  a.recv_cap = c->recv_bytes;
  a.staging_cap = c->staging_bytes;
  FusedArgs f;
  memset(&f, 0, sizeof(f));
  f.counts = counts;
  f.n = n;
  f.m = m;
  f.demand_off = c->demand_off;
  f.sched = *sched;
  f.pin.n = n;
  f.pin.m = m;
  f.pin.K = n * n - 2 * n + 2;
  f.pin.recv_cap = c->recv_bytes;
  f.pin.staging_cap = c->staging_bytes;
  f.pin.op_cap = plan->op_capacity;
  f.pin.chunk = a.chunk;
  f.pin.copy_self = c->copy_self;
  f.pout.ops = plan->ops;
  f.pout.n_ops = plan->n_ops;
  f.pout.staging_used = plan->staging_used;
  f.pout.status = plan->status;
  f.pout.ws = plan->workspace;
  f.pout.scratch = nullptr;
  exec_kernel<true><<<blocks, kExecThreads, smem, stream>>>(a, f);
  return cudaGetLastError() == cudaSuccess ? FAST_OK : FAST_ECUDA;
}

int fast_comm_set_fused(fast_comm* c, int enable) {
  if (!c) return FAST_EVALIDATION;
  c->no_fuse = enable ? 0 : 1;
  return FAST_OK;
}

int fast_alltoallv(fast_comm* c, const void* send, const int64_t* counts, int n, int m,
                   const fast_sched_bufs* sched, const fast_plan* plan, int blocks,
                   int64_t chunk_bytes, int64_t* timeline_ns, void* stream) {
  if (!c || !c->opened || !send || !counts || !sched || !plan) return FAST_EVALIDATION;
  if ((int64_t)n * m != c->world || n < 2 || m > FAST_MAX_GPUS_PER_SERVER || chunk_bytes < 16)
    return FAST_EVALIDATION;
  if (!c->no_fuse && n <= kFusedMaxN && fused_smem_bytes(n, m) <= 200 * 1024)
    return launch_fused(c, send, counts, n, m, sched, plan, blocks, chunk_bytes, timeline_ns,
                        (cudaStream_t)stream);
  // device-side epoch (gather_demand_kernel bumps it): every argument below
  // is call-invariant, so the whole call can be captured in a CUDA graph
  // the gather also zeroes the call's synthesis status, so no memset node
  // breaks the programmatic (PDL) chain gather -> synthesis -> plan -> exec
  gather_demand_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(c->peers_dev, counts, 0, c->rank,
                                                           c->world, c->demand_off,
                                                           sched->status);
  if (cudaGetLastError() != cudaSuccess) return FAST_ECUDA;
  c->epoch += 1;
  int rc;
  const bool pdl = !c->no_pdl;
  int64_t* D = fast_comm_demand_ptr(c, 0);
  rc = fast_synth_batch_chain(D, 1, n, m, sched, (cudaStream_t)stream, pdl);
  if (rc != FAST_OK) return rc;
  rc = plan_compile_launch(D, D + (int64_t)c->world * c->world, n, m, sched, c->recv_bytes,
                           c->staging_bytes, chunk_bytes, plan, stream, pdl, c->copy_self);
  if (rc != FAST_OK) return rc;
  return exec_launch(c, plan, send, 0, blocks, chunk_bytes, timeline_ns, stream, 1, pdl);
}

int fast_comm_set_copy_self(fast_comm* c, int enable) {
  if (!c) return FAST_EVALIDATION;
  c->copy_self = enable ? 1 : 0;
  return FAST_OK;
}

int fast_comm_set_pdl(fast_comm* c, int enable) {
  if (!c) return FAST_EVALIDATION;
  c->no_pdl = enable ? 0 : 1;
  return FAST_OK;
}

int fast_comm_set_send_capacity(fast_comm* c, int64_t bytes) {
  if (!c) return FAST_EVALIDATION;
  c->send_cap = bytes < 0 ? -1 : bytes;
  return FAST_OK;
}

int fast_comm_set_send_rows(fast_comm* c, const void* rows_base, const int32_t* row_src,
                            int64_t row_bytes, int64_t n_rows) {
  if (!c) return FAST_EVALIDATION;
  if (!row_src) {
    c->rows_base = nullptr;
    c->row_src = nullptr;
    return FAST_OK;
  }
  if (!rows_base || row_bytes < 16 || (row_bytes & 15) || ((uintptr_t)rows_base & 15) ||
      n_rows < 0 || row_bytes / 16 > 0xffffffffll ||
      (n_rows * (row_bytes / 16)) >= ((int64_t)1 << 32))
    return FAST_EVALIDATION;
  const uint32_t d = (uint32_t)(row_bytes / 16);
  int l = 0;
  while (((uint64_t)1 << l) < d) ++l;
  c->rows_base = (const uint8_t*)rows_base;
  c->row_src = row_src;
  c->row_vec = d;
  c->row_l = l;
  c->row_magic = d > 1 ? (uint32_t)((((uint64_t)1 << 32) * (((uint64_t)1 << l) - d)) / d + 1) : 0;
  return FAST_OK;
}

int64_t fast_comm_epoch(const fast_comm* c) { return c ? c->epoch : -1; }

int fast_comm_set_epoch(fast_comm* c, int64_t epoch) {
  if (!c || epoch < 0) return FAST_EVALIDATION;
  c->epoch = epoch;
  return FAST_OK;
}

int fast_comm_status(const fast_comm* c, int32_t* status_host) {
  if (!c || !status_host) return FAST_EVALIDATION;
  uint64_t v = 0;
  if (cudaMemcpy(&v, c->base + CTR_STATUS * 8, 8, cudaMemcpyDeviceToHost) != cudaSuccess)
    return FAST_ECUDA;
  *status_host = (int32_t)v;
  return FAST_OK;
}

}  // extern "C"

