// synth.cu -- batched FAST schedule synthesis on B200 (sm_100a).
//
// Three stream-ordered kernels replace tiersched.synthesize_fast
// (pipeline.py:52-59) for a whole batch of demand matrices:
//
//   balance_reg_kernel / balance_kernel
//                    build_balance_plan + reduce_to_server_level
//                    (balance.py:77-174, model.py:169-178).  One CTA per
//                    (server row i, block of J destination servers); the
//                    m rows x J*m columns strip is staged into shared memory
//                    with coalesced loads (even m <= 16: every row load of a
//                    thread in flight at once, tile row sums reduced by the
//                    loading threads), one thread balances one m x m cross
//                    tile in place, the strip is written back coalesced.
//                    HBM-bound: 8*G^2 B read + 8*G^2 B written.
//   decompose_kernel embed_doubly_stochastic + decompose + strip_auxiliary
//                    (birkhoff.py:75-252).  One warp per matrix.  Support of
//                    the work matrix is a bitset in shared memory; the Kuhn
//                    DFS (birkhoff.py:172-180) runs on lane 0 as an explicit
//                    stack over the bitset (first-set-bit = the reference's
//                    in-order column scan); min/subtract/strip/free run on
//                    all lanes.  Latency-bound (a dependent chain of up to
//                    n^2-2n+2 peels), so many matrices are resident per SM.
//   sort_kernel      sort_stages_ascending (birkhoff.py:255-266): bitonic
//                    sort of (weight, src0|dst0|raw index) keys in shared
//                    memory, one CTA per matrix; the raw index in the key
//                    makes it equal to Python's stable sort.
#include <cuda_runtime.h>
#include <stdint.h>

#include "fastb200.h"
#include "launch.cuh"

namespace {

#ifndef FAST_BAL_THREADS
#define FAST_BAL_THREADS 128
#endif
#ifndef FAST_BAL_STRIP_KB
#define FAST_BAL_STRIP_KB 16
#endif
constexpr int kBalThreads = FAST_BAL_THREADS;
#ifndef FAST_DEC_WARPS
#define FAST_DEC_WARPS 1
#endif
constexpr int kDecWarps = FAST_DEC_WARPS;  // matrices per CTA in decompose_kernel

// Optional section timers (debug builds with -DFAST_DEC_PROFILE only).
#ifdef FAST_DEC_PROFILE
__device__ unsigned long long g_dec_prof[8];
#define DPROF_T(var) const long long var = clock64()
#define DPROF_ADD(slot, val) \
  if ((threadIdx.x & 31) == 0) atomicAdd(&g_dec_prof[slot], (unsigned long long)(val))
#else
#define DPROF_T(var)
#define DPROF_ADD(slot, val)
#endif

}  // namespace

#include "synth_dev.cuh"

namespace {

// grid (n, ceil(n/J), B), block kBalThreads, dyn smem J*(m*m+1)*8.
// Stage-in/out walk the strip row by row (no integer division by a runtime
// value); even m moves 16-byte pairs (rows of a G x G int64 matrix with G
// even are 16-byte aligned), odd m single words.
template <int M>
__device__ __forceinline__ void strip_rows(int64_t* __restrict__ sm,
                                           const int64_t* __restrict__ g_in,
                                           int64_t* __restrict__ g_out,
                                           const int m_rt, const int64_t G,
                                           const int Jc, const bool load) {
  const int m = M ? M : m_rt;
  const int TS = m * m + 1;
  const int cols = Jc * m;
  if ((M ? (M % 2 == 0) : (m % 2 == 0))) {
    const int pairs = cols >> 1;
    for (int r = 0; r < m; ++r) {
      const int64_t rowoff = (int64_t)r * G;
      for (int e = threadIdx.x; e < pairs; e += blockDim.x) {
        const int col = 2 * e;
        const int jj = col / m, c = col - jj * m;
        int64_t* sp = sm + jj * TS + r * m + c;
        if (load) {
          const longlong2 x = __ldcs(reinterpret_cast<const longlong2*>(g_in + rowoff + col));
          sp[0] = x.x;
          sp[1] = x.y;
        } else {
          longlong2 x;
          x.x = sp[0];
          x.y = sp[1];
          __stcs(reinterpret_cast<longlong2*>(g_out + rowoff + col), x);
        }
      }
    }
  } else {
    for (int r = 0; r < m; ++r) {
      const int64_t rowoff = (int64_t)r * G;
      for (int col = threadIdx.x; col < cols; col += blockDim.x) {
        const int jj = col / m, c = col - jj * m;
        int64_t* sp = sm + jj * TS + r * m + c;
        if (load) *sp = __ldcs(g_in + rowoff + col);
        else __stcs(g_out + rowoff + col, *sp);
      }
    }
  }
}

template <int M>
__global__ void __launch_bounds__(kBalThreads)
    balance_kernel(const int64_t* __restrict__ D, const int n, const int m_rt,
                   const int J, fast_sched_bufs out) {
  extern __shared__ int64_t sm[];
  pdl_trigger();
  pdl_wait();  // D comes from the previous kernel of an alltoallv chain
  const int m = M ? M : m_rt;
  const int b = blockIdx.z, i = blockIdx.x, j0 = blockIdx.y * J;
  const int Jc = min(J, n - j0);
  const int64_t G = (int64_t)n * m;
  const int TS = m * m + 1;  // +1 word of padding per tile (bank spread)
  const int64_t* Db = D + (int64_t)b * G * G + (int64_t)i * m * G + j0 * m;
  int64_t* Bb = out.balanced + (int64_t)b * G * G + (int64_t)i * m * G + j0 * m;

  strip_rows<M>(sm, Db, nullptr, m, G, Jc, true);
  __syncthreads();

  if (threadIdx.x < Jc) {
    const int jj = threadIdx.x, j = j0 + jj;
    int64_t* t = sm + jj * TS;
    int32_t* st = out.status + b;
    constexpr int MM = M ? M : 1;
    int64_t rs[MM];  // plain row sums (M > 0 only), reused by balance_tile
    bool bad = false;
    int64_t s = 0, tp = 0;  // saturating / plain tile totals
#pragma unroll
    for (int p = 0; p < MM; ++p) rs[p] = 0;
    for (int p = 0; p < m; ++p) {
      int64_t r = 0;
      for (int q = 0; q < m; ++q) {
        const int64_t v = t[p * m + q];
        r += v;
        if (v < 0) { bad = true; continue; }
        if (i == j && p == q && v != 0) bad = true;
        s = sat_add(s, v);
      }
      tp += r;
      if (M) {
#pragma unroll
        for (int pp = 0; pp < MM; ++pp)
          if (pp == p) rs[pp] = r;
      }
    }
    out.server[(int64_t)b * n * n + i * n + j] = s;
    // a tile at the 2^62 guard already puts the matrix total there: that is
    // the model's validation error (model.py:26), not a balancing failure
    if (bad || s >= kMaxSafeTotal) {
      raise_status(st, FAST_EVALIDATION);
    } else if (i != j) {
      const int T = n * (n - 1);
      const int slots = m > 1 ? m - 1 : 1;
      const int tidx = i * (n - 1) + (j < i ? j : j - 1);
      fast_move* mv = out.moves + ((int64_t)b * T + tidx) * slots;
      uint64_t mk = 0;
      int nm = balance_tile<M>(t, m, mv, slots, M ? rs : nullptr, &mk);
      if (out.tile_mask) out.tile_mask[(int64_t)b * T + tidx] = mk;
      if (nm < 0) {
        raise_status(st, FAST_EINVARIANT);
        nm = 0;
      }
      out.move_count[(int64_t)b * T + tidx] = nm;
    }
  }
  __syncthreads();
  strip_rows<M>(sm, nullptr, Bb, m, G, Jc, false);
}

__host__ __device__ constexpr int ceil_log2(int x) { return x <= 1 ? 0 : 1 + ceil_log2((x + 1) / 2); }

// ---------------------------------------------------------------------------
// balance_reg_kernel<M> (even M <= 16, the default for those): the same per-tile
// work as balance_kernel, with the strip staged through REGISTERS so each
// thread has all M of its 16-byte row loads in flight at once (the staged
// kernel issued one load per row and waited on it: 37 % of its stall samples
// sat on that wait, profiles/r2_synth_ncu_full_summary.txt), and with the
// per-tile prologue (row sums, the saturating server total, the validation
// of balance_kernel's loop) done by all threads at load time instead of by
// the one thread that balances the tile:
//   * thread e owns column pair 2*(e % (M/2)) of tile e / (M/2) in every row;
//   * the M/2 threads of a tile butterfly-reduce their row partial sums and
//     the OR of their cells (a tile whose cells are all < 2^(62 - 2 log2 M)
//     cannot reach the 2^62 guard, so its saturating total is the plain one;
//     any other tile -- negative, huge -- takes balance_kernel's exact loop);
// J = 128 / (M/2) tiles per CTA (32 at m = 8: one full warp balances them).
// Load side of one strip (thread e < kBalThreads of the CTA): its M row pairs
// are in x[]; stores them into the tile, reduces the tile's row sums and the
// OR of its cells over the PPR threads of the tile (consecutive lanes).
template <int M>
__device__ __forceinline__ void bal_stage_in(const longlong2 (&x)[M], int64_t* __restrict__ sm,
                                             int64_t* __restrict__ rsum,
                                             uint64_t* __restrict__ tflag, const int e) {
  constexpr int PPR = M / 2, TS = M * M + 1;
  const int jj = e / PPR, c = 2 * (e % PPR);
  int64_t* t = sm + jj * TS;
  int64_t part[M];
  uint64_t orv = 0;
#pragma unroll
  for (int r = 0; r < M; ++r) {
    t[r * M + c] = x[r].x;
    t[r * M + c + 1] = x[r].y;
    part[r] = x[r].x + x[r].y;
    orv |= (uint64_t)x[r].x | (uint64_t)x[r].y;
  }
  // a CTA edge tile (jj >= Jc) is skipped by all PPR lanes of its group together
  const unsigned grp = (PPR >= 32) ? 0xffffffffu
                                   : (((1u << PPR) - 1u) << ((e & 31) & ~(PPR - 1)));
#pragma unroll
  for (int off = 1; off < PPR; off <<= 1) {
#pragma unroll
    for (int r = 0; r < M; ++r) part[r] += __shfl_xor_sync(grp, part[r], off);
    orv |= __shfl_xor_sync(grp, orv, off);
  }
  const int q = e % PPR;
#pragma unroll
  for (int r = 0; r < M; ++r)
    if (r % PPR == q) rsum[jj * M + r] = part[r];
  if (q == 0) tflag[jj] = orv;
}

// Tile (i, j) of matrix b, staged at t with its row sums / cell OR: server
// total, validation, balance_senders, moves and mask (balance_kernel's
// per-tile work with the prologue already reduced).
template <int M>
__device__ __forceinline__ void bal_tile_work(int64_t* __restrict__ t,
                                              const int64_t* __restrict__ rsum_t,
                                              const uint64_t orv, const int b, const int i,
                                              const int j, const int n,
                                              const fast_sched_bufs& out) {
  constexpr int BITS = 62 - ceil_log2(M * M);  // M*M cells below 2^BITS sum below 2^62
  int32_t* st = out.status + b;
  int64_t rs[M];
  bool bad = false;
  int64_t s = 0, tp = 0;  // saturating / plain tile totals
#pragma unroll
  for (int p = 0; p < M; ++p) rs[p] = rsum_t[p];
  if ((orv >> BITS) == 0) {
#pragma unroll
    for (int p = 0; p < M; ++p) tp += rs[p];
    s = tp;
    if (i == j)  // intra tile: the diagonal must be empty
#pragma unroll
      for (int p = 0; p < M; ++p) bad |= t[p * M + p] != 0;
  } else {  // balance_kernel's exact loop (negative cells, the 2^62 guard)
#pragma unroll
    for (int p = 0; p < M; ++p) {
      for (int q = 0; q < M; ++q) {
        const int64_t v = t[p * M + q];
        if (v < 0) { bad = true; continue; }
        if (i == j && p == q && v != 0) bad = true;
        s = sat_add(s, v);
      }
      tp += rs[p];
    }
  }
  out.server[(int64_t)b * n * n + i * n + j] = s;
  // a tile at the 2^62 guard already puts the matrix total there: that is
  // the model's validation error (model.py:26), not a balancing failure
  if (bad || s >= kMaxSafeTotal) {
    raise_status(st, FAST_EVALIDATION);
  } else if (i != j) {
    const int T = n * (n - 1);
    constexpr int slots = M > 1 ? M - 1 : 1;
    const int tidx = i * (n - 1) + (j < i ? j : j - 1);
    fast_move* mv = out.moves + ((int64_t)b * T + tidx) * slots;
    uint64_t mk = 0;
#ifdef FAST_BAL_NOCOMPUTE  // timing experiment only: the memory phases alone
    int nm = 0;
    (void)mv;
#else
#ifndef FAST_BAL_NO32
    // tile total below 2^31 (no negative cells here): the greedy in 32 bits
    int nm = tp < ((int64_t)1 << 31) ? balance_tile<M, int32_t>(t, M, mv, slots, rs, &mk)
                                     : balance_tile<M>(t, M, mv, slots, rs, &mk);
#else
    int nm = balance_tile<M>(t, M, mv, slots, rs, &mk);
#endif
#endif
    if (out.tile_mask) out.tile_mask[(int64_t)b * T + tidx] = mk;
    if (nm < 0) {
      raise_status(st, FAST_EINVARIANT);
      nm = 0;
    }
    out.move_count[(int64_t)b * T + tidx] = nm;
  }
}

#ifndef FAST_BAL_MINB
#define FAST_BAL_MINB 8  // <= 64 registers: 8 CTAs of 128 threads per SM
#endif
template <int M>
__global__ void __launch_bounds__(kBalThreads, M >= 16 ? 1 : FAST_BAL_MINB)
    balance_reg_kernel(const int64_t* __restrict__ D, const int n,
                       fast_sched_bufs out) {
  static_assert(M % 2 == 0 && M <= 16, "even m <= 16");
  constexpr int PPR = M / 2;                // 16-B pairs per tile row
  constexpr int J = kBalThreads / PPR;      // tiles per CTA
  constexpr int TS = M * M + 1;             // +1 word of padding per tile
  extern __shared__ int64_t sm[];
  int64_t* rsum = sm + J * TS;                                  // [J][M]
  uint64_t* tflag = reinterpret_cast<uint64_t*>(rsum + J * M);  // [J]
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.z, i = blockIdx.x, j0 = blockIdx.y * J;
  const int Jc = min(J, n - j0);
  const int64_t G = (int64_t)n * M;
  const int64_t* Db = D + (int64_t)b * G * G + (int64_t)i * M * G + j0 * M;
  int64_t* Bb = out.balanced + (int64_t)b * G * G + (int64_t)i * M * G + j0 * M;

  const int e = threadIdx.x;
  if (e / PPR < Jc) {
    longlong2 x[M];
#pragma unroll
    for (int r = 0; r < M; ++r)
      x[r] = __ldcs(reinterpret_cast<const longlong2*>(Db + r * G + 2 * e));
    bal_stage_in<M>(x, sm, rsum, tflag, e);
  }
  __syncthreads();
  if (threadIdx.x < Jc) {
    const int jj = threadIdx.x;
    bal_tile_work<M>(sm + jj * TS, rsum + jj * M, tflag[jj], b, i, j0 + jj, n, out);
  }
  __syncthreads();
  strip_rows<M>(sm, nullptr, Bb, M, G, Jc, false);
}

#ifdef FAST_BAL_PIPE
// ---------------------------------------------------------------------------
// balance_pipe_kernel<M> (opt-in, -DFAST_BAL_PIPE; SLOWER, kept for the record): the
// register-staged kernel as a persistent, software-pipelined loop over
// strips.  kBalThreads load/store threads plus ceil(J/32) balancing warps
// per CTA; while the balancing warps work on strip k, the load threads
// already hold strip k+1's row loads in flight in registers, so the HBM
// stream no longer stops for the sequential greedy (the register-staged
// kernel spent 46 % of its stall samples at the barrier behind it and ran
// its memory phases alone in 2.77 ms against 3.67 ms with the greedy).
// Per strip: stage-in (the loaded registers -> tile, row sums) | barrier |
// issue strip k+1's loads, balance strip k | barrier | store strip k.  A
// load thread reads back in the store phase exactly the cells it staged in,
// so the next stage-in needs no extra barrier.
// Measured (n=128 x 8, B=1000, profiles/r2_balance_reg_ab.log): 4.98-5.70 ms
// for 3-6 CTAs per SM against 3.66 ms for balance_reg_kernel: one strip in
// flight per CTA and 4-6 CTAs per SM hold too few bytes in flight for HBM
// (the memory phases alone: 2.95 ms, vs 2.77 ms in the register-staged kernel).
template <int M>
constexpr int bal_pipe_threads() {
  return kBalThreads + ((kBalThreads / (M / 2) + 31) / 32) * 32;
}
#ifndef FAST_BAL_PIPE_MINB
#define FAST_BAL_PIPE_MINB 5
#endif
template <int M>
__global__ void __launch_bounds__(bal_pipe_threads<M>(), FAST_BAL_PIPE_MINB)
    balance_pipe_kernel(const int64_t* __restrict__ D, const int n, const int nstrips,
                        fast_sched_bufs out) {
  static_assert(M % 2 == 0 && M <= 8, "even m <= 8");
  constexpr int PPR = M / 2;
  constexpr int J = kBalThreads / PPR;
  constexpr int TS = M * M + 1;
  extern __shared__ int64_t sm[];
  int64_t* rsum = sm + J * TS;
  uint64_t* tflag = reinterpret_cast<uint64_t*>(rsum + J * M);
  pdl_trigger();
  pdl_wait();
  const int NJB = (n + J - 1) / J;
  const int64_t G = (int64_t)n * M;
  const int e = threadIdx.x;
  const bool loader = e < kBalThreads;
  // strip id -> (matrix b, server row i, first destination server j0)
  auto decode = [&](int sid, int& b, int& i, int& j0) {
    const int q = sid / NJB;
    j0 = (sid - q * NJB) * J;
    b = q / n;
    i = q - b * n;
  };
  auto rows_at = [&](int b, int i, int j0) -> int64_t {
    return (int64_t)b * G * G + (int64_t)i * M * G + j0 * M;
  };
  longlong2 x[M];
  int sid = blockIdx.x;
  if (loader && sid < nstrips) {
    int b, i, j0;
    decode(sid, b, i, j0);
    if (e / PPR < min(J, n - j0)) {
      const int64_t* Db = D + rows_at(b, i, j0);
#pragma unroll
      for (int r = 0; r < M; ++r)
        x[r] = __ldcs(reinterpret_cast<const longlong2*>(Db + r * G + 2 * e));
    }
  }
  for (; sid < nstrips; sid += gridDim.x) {
    int b, i, j0;
    decode(sid, b, i, j0);
    const int Jc = min(J, n - j0);
    const bool mine = loader && e / PPR < Jc;
    if (mine) bal_stage_in<M>(x, sm, rsum, tflag, e);
    __syncthreads();
    if (loader) {
      const int nsid = sid + gridDim.x;
      if (nsid < nstrips) {
        int nb, ni, nj0;
        decode(nsid, nb, ni, nj0);
        if (e / PPR < min(J, n - nj0)) {
          const int64_t* Db = D + rows_at(nb, ni, nj0);
#pragma unroll
          for (int r = 0; r < M; ++r)
            x[r] = __ldcs(reinterpret_cast<const longlong2*>(Db + r * G + 2 * e));
        }
      }
    } else {
      const int jj = e - kBalThreads;
      if (jj < Jc) bal_tile_work<M>(sm + jj * TS, rsum + jj * M, tflag[jj], b, i, j0 + jj, n, out);
    }
    __syncthreads();
    if (mine) {
      const int jj = e / PPR, c = 2 * (e % PPR);
      const int64_t* t = sm + jj * TS;
      int64_t* Bb = out.balanced + rows_at(b, i, j0);
#pragma unroll
      for (int r = 0; r < M; ++r) {
        longlong2 y;
        y.x = t[r * M + c];
        y.y = t[r * M + c + 1];
        __stcs(reinterpret_cast<longlong2*>(Bb + r * G + 2 * e), y);
      }
    }
  }
}
#endif  // FAST_BAL_PIPE

#ifdef FAST_BAL_TMA
// ---------------------------------------------------------------------------
// balance_tma_kernel (opt-in, -DFAST_BAL_TMA; slower, see launch_balance):
// the same per-tile work as balance_kernel, as a persistent pipeline fed by
// the TMA engine.  Each thread owns one m x m tile
// slot per buffer (tile-major, padded) and runs its own two-deep pipeline:
// the m tile rows of its NEXT tile are fetched with 1-D bulk copies
// (cp.async.bulk ... mbarrier::complete_tx) into the other buffer while it
// balances the current one, and the balanced rows go back with bulk stores
// (cp.async.bulk.global.shared::cta).  No CTA-wide barrier: every thread
// waits only on its own mbarrier, so the HBM stream never stalls behind the
// slowest greedy of a strip.  grid = resident CTAs, block = kTmaTiles.
constexpr int kTmaTiles = 64;  // tiles (threads) per CTA

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n\t}" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
      "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_load(void* smem, const void* gmem, unsigned bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem), "r"(bytes),
      "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void bulk_store(void* gmem, const void* smem, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem),
               "r"((uint32_t)__cvta_generic_to_shared(smem)), "r"(bytes) : "memory");
}

template <int M>
__global__ void __launch_bounds__(kTmaTiles)
    balance_tma_kernel(const int64_t* __restrict__ D, const int n, const int B,
                       fast_sched_bufs out) {
  constexpr int TS = M * M + 2;  // int64 per tile slot: 16-byte aligned, banks staggered
  extern __shared__ __align__(128) int64_t tsm[];
  __shared__ __align__(8) uint64_t bars[2][kTmaTiles];
  const int jj = threadIdx.x;
  const int64_t G = (int64_t)n * M;
  const int nj = (n + kTmaTiles - 1) / kTmaTiles;  // strips per server row
  const int64_t items = (int64_t)B * n * nj;
  mbar_init(&bars[0][jj], 1);
  mbar_init(&bars[1][jj], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int slots = M > 1 ? M - 1 : 1;
  const int T = n * (n - 1);

  // item -> (b, i, j) of this thread's tile; valid = j < n
  auto tile_of = [&](int64_t it, int& b, int& i, int& j) {
    b = (int)(it / ((int64_t)n * nj));
    const int64_t r = it - (int64_t)b * n * nj;
    i = (int)(r / nj);
    j = (int)(r - (int64_t)i * nj) * kTmaTiles + jj;
  };
  auto fetch = [&](int64_t it, int k) {
    int b, i, j;
    tile_of(it, b, i, j);
    if (j >= n) return;
    const int64_t* src = D + (int64_t)b * G * G + (int64_t)i * M * G + (int64_t)j * M;
    mbar_expect_tx(&bars[k][jj], M * M * 8);
    int64_t* sl = tsm + (int64_t)(k * kTmaTiles + jj) * TS;
#pragma unroll
    for (int p = 0; p < M; ++p) bulk_load(sl + p * M, src + p * G, M * 8, &bars[k][jj]);
  };

  int64_t it = blockIdx.x;
  if (it < items) fetch(it, 0);
  unsigned phase[2] = {0u, 0u};
  for (int k = 0; it < items; it += gridDim.x, k ^= 1) {
    const int64_t nxt = it + gridDim.x;
    if (nxt < items) {
      // the next tile goes into the other slot: its previous bulk store must
      // have finished reading it
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      fetch(nxt, k ^ 1);
    }
    int b, i, j;
    tile_of(it, b, i, j);
    if (j >= n) continue;
    mbar_wait(&bars[k][jj], phase[k]);
    phase[k] ^= 1u;
    int64_t* t = tsm + (int64_t)(k * kTmaTiles + jj) * TS;
    int32_t* st = out.status + b;
    int64_t rs[M];
    bool bad = false;
    int64_t s = 0, tp = 0;
#pragma unroll
    for (int p = 0; p < M; ++p) {
      int64_t r = 0;
#pragma unroll
      for (int q = 0; q < M; ++q) {
        const int64_t v = t[p * M + q];
        r += v;
        if (v < 0) { bad = true; continue; }
        if (i == j && p == q && v != 0) bad = true;
        s = sat_add(s, v);
      }
      rs[p] = r;
      tp += r;
    }
    out.server[(int64_t)b * n * n + i * n + j] = s;
    // a tile at the 2^62 guard already puts the matrix total there: that is
    // the model's validation error (model.py:26), not a balancing failure
    if (bad || s >= kMaxSafeTotal) {
      raise_status(st, FAST_EVALIDATION);
    } else if (i != j) {
      const int tidx = i * (n - 1) + (j < i ? j : j - 1);
      fast_move* mv = out.moves + ((int64_t)b * T + tidx) * slots;
      uint64_t mk = 0;
      int nm = balance_tile<M>(t, M, mv, slots, rs, &mk);
      if (out.tile_mask) out.tile_mask[(int64_t)b * T + tidx] = mk;
      if (nm < 0) {
        raise_status(st, FAST_EINVARIANT);
        nm = 0;
      }
      out.move_count[(int64_t)b * T + tidx] = nm;
    }
    // generic-proxy writes of the tile -> visible to the bulk (async) proxy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    int64_t* dst = out.balanced + (int64_t)b * G * G + (int64_t)i * M * G + (int64_t)j * M;
#pragma unroll
    for (int p = 0; p < M; ++p) bulk_store(dst + p * G, t + p * M, M * 8);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

#endif  // FAST_BAL_TMA

// One warp per matrix (decompose_one, synth_dev.cuh).
template <int NW, bool WB>
__global__ void __launch_bounds__(kDecWarps * 32)
    decompose_kernel(const int64_t* __restrict__ S_all, const int B,
                     const int n, const int mode, const int check_total,
                     fast_sched_bufs out) {
  extern __shared__ __align__(16) char dsm[];
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * kDecWarps + warp;
  if (b >= B) return;
  decompose_one<NW, WB>(dsm + warp * dec_smem_bytes_t<NW>(n), S_all, b, n, mode, check_total,
                        out, lane);
}

// ---------------------------------------------------------------------------
// synth_small_kernel: the whole synthesis of one small matrix in ONE CTA
// (n <= 6: stage capacity <= 32, so the decomposition warp also sorts) --
// per-call latency for single small matrices (BASELINE configs 1-4) and the
// alltoallv chain, where the balance / decompose launch pair (and the status
// memset) cost more than their work.  Same per-tile code as balance_kernel
// (validation, saturating server total, balance_senders, moves, mask), one
// thread per tile straight from global memory, then decompose_one on warp 0.
constexpr int kSmallThreads = 64;
constexpr int kSmallMaxN = 6;

__host__ __device__ inline size_t small_smem_bytes(int n, int m) {
  return (((size_t)n * n * (m * m + 1) * 8 + 127) & ~(size_t)127) + dec_smem_bytes_t<1>(n);
}

template <int M, bool WB>
__global__ void __launch_bounds__(kSmallThreads)
    synth_small_kernel(const int64_t* __restrict__ D, const int n, const int m_rt,
                       fast_sched_bufs out) {
  extern __shared__ __align__(16) char ssm[];
  pdl_trigger();
  pdl_wait();  // D comes from the previous kernel of an alltoallv chain
  const int m = M ? M : m_rt;
  const int b = blockIdx.x, tid = threadIdx.x;
  const int G = n * m, TS = m * m + 1, T = n * (n - 1), slots = m > 1 ? m - 1 : 1;
  const int64_t* Db = D + (int64_t)b * G * G;
  int64_t* tiles = reinterpret_cast<int64_t*>(ssm);
  int32_t* st = out.status + b;
  if (tid == 0) *st = FAST_OK;
  // coalesced stage-in of the whole matrix into tile-major shared memory
  for (int x = tid; x < G * G; x += blockDim.x) {
    const int r = x / G, c = x - r * G;
    const int i = r / m, p = r - i * m, j = c / m, q = c - j * m;
    tiles[(i * n + j) * TS + p * m + q] = __ldg(Db + x);
  }
  __syncthreads();
  for (int t = tid; t < n * n; t += blockDim.x) {
    const int i = t / n, j = t - i * n;
    int64_t* tl = tiles + (int64_t)t * TS;
    constexpr int MM = M ? M : 1;
    int64_t rs[MM];
    bool bad = false;
    int64_t s = 0;
#pragma unroll
    for (int p = 0; p < MM; ++p) rs[p] = 0;
    for (int p = 0; p < m; ++p) {
      int64_t r = 0;
      for (int q = 0; q < m; ++q) {
        const int64_t v = tl[p * m + q];
        r += v;
        if (v < 0) { bad = true; continue; }
        if (i == j && p == q && v != 0) bad = true;
        s = sat_add(s, v);
      }
      if (M) {
#pragma unroll
        for (int pp = 0; pp < MM; ++pp)
          if (pp == p) rs[pp] = r;
      }
    }
    out.server[(int64_t)b * n * n + t] = s;
    if (bad || s >= kMaxSafeTotal) {  // see balance_kernel
      raise_status(st, FAST_EVALIDATION);
    } else if (i != j) {
      const int tidx = i * (n - 1) + (j < i ? j : j - 1);
      uint64_t mk = 0;
      int nm = balance_tile<M>(tl, m, out.moves + ((int64_t)b * T + tidx) * slots, slots,
                               M ? rs : nullptr, &mk);
      if (out.tile_mask) out.tile_mask[(int64_t)b * T + tidx] = mk;
      if (nm < 0) {
        raise_status(st, FAST_EINVARIANT);
        nm = 0;
      }
      out.move_count[(int64_t)b * T + tidx] = nm;
    }
  }
  __syncthreads();  // balanced tiles, server totals and status are in place
  int64_t* Bb = out.balanced + (int64_t)b * G * G;
  for (int x = tid; x < G * G; x += blockDim.x) {
    const int r = x / G, c = x - r * G;
    const int i = r / m, p = r - i * m, j = c / m, q = c - j * m;
    Bb[x] = tiles[(i * n + j) * TS + p * m + q];
  }
  if (tid < 32)
    decompose_one<1, WB>(ssm + (small_smem_bytes(n, m) - dec_smem_bytes_t<1>(n)), out.server,
                         b, n, FAST_DEC_SERVER, 1, out, tid);
}

// ---------------------------------------------------------------------------
// sort_stages_ascending (birkhoff.py:255-266): sort of the kept stages by
// (weight, src0, dst0, raw index) -- the raw index makes it equal to
// Python's stable sort.  Bitonic network in the "flip" form (every merge
// ascending, the first step of each merge compares i with its mirror), which
// sorts any count by skipping partners past the end: no padding.
//
// Common case: weight < 2^36, so (weight, src0, dst0, idx) packs into ONE
// u64 (36 + 7 + 7 + 14 bits) and the keys live in shared memory: 8 bytes per
// stage (129 KiB at n = 128), small enough to co-reside with the latency-
// bound decomposition CTAs of concurrent batches.  Wider weights: the same
// network runs on the (weight, tie) pairs in the global workspace.
template <typename CMPX>
__device__ __forceinline__ void bitonic_flip(const int cnt, CMPX cmpx) {
  int P = 1;
  while (P < cnt) P <<= 1;
  for (int kk = 2; kk <= P; kk <<= 1) {
    const int half = kk >> 1;
    for (int x = threadIdx.x; x < P / 2; x += blockDim.x) {
      const int blk = x / half, o = x - blk * half;
      const int i = blk * kk + o, j = blk * kk + kk - 1 - o;
      if (j < cnt) cmpx(i, j);
    }
    __syncthreads();
    for (int h = half >> 1; h > 0; h >>= 1) {
      for (int x = threadIdx.x; x < P / 2; x += blockDim.x) {
        const int blk = x / h, o = x - blk * h;
        const int i = blk * 2 * h + o, j = i + h;
        if (j < cnt) cmpx(i, j);
      }
      __syncthreads();
    }
  }
}

constexpr int kSortThreads = 1024;
__global__ void __launch_bounds__(kSortThreads)
    sort_kernel(const int n, fast_sched_bufs out) {
  extern __shared__ __align__(16) unsigned long long sk[];
  __shared__ unsigned long long s_max;
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x;
  const int K = stage_cap(n);
  if (out.status[b] != FAST_OK) return;
  const int kept = out.n_stages[b];
  if (kept <= 0) return;
  uint64_t* work = (uint64_t*)((char*)out.workspace + (size_t)b * dec_ws_bytes_per_matrix(n));
  uint64_t* key_w = work + (size_t)n * n;
  uint32_t* key_t = (uint32_t*)(key_w + K);
  if (threadIdx.x == 0) s_max = 0;
  __syncthreads();
  unsigned long long mx = 0;
  for (int i = threadIdx.x; i < kept; i += blockDim.x) mx = key_w[i] > mx ? key_w[i] : mx;
  atomicMax(&s_max, mx);
  __syncthreads();
  int32_t* ord = out.stage_order + (int64_t)b * K;
  if (s_max < (1ull << 36)) {
    for (int i = threadIdx.x; i < kept; i += blockDim.x) {
      const uint32_t t = key_t[i];  // src0 << 24 | dst0 << 16 | raw index
      sk[i] = (key_w[i] << 28) | ((unsigned long long)((t >> 24) & 127) << 21) |
              ((unsigned long long)((t >> 16) & 127) << 14) | (t & 0x3fffu);
    }
    __syncthreads();
    bitonic_flip(kept, [&](int i, int j) {
      const unsigned long long a = sk[i], c = sk[j];
      if (a > c) { sk[i] = c; sk[j] = a; }
    });
    for (int i = threadIdx.x; i < kept; i += blockDim.x) ord[i] = (int32_t)(sk[i] & 0x3fffu);
  } else {
    volatile uint64_t* vw = key_w;
    volatile uint32_t* vt = key_t;
    bitonic_flip(kept, [&](int i, int j) {
      const uint64_t wa = vw[i], wb = vw[j];
      const uint32_t ta = vt[i], tb = vt[j];
      if (wa > wb || (wa == wb && ta > tb)) {
        vw[i] = wb; vw[j] = wa;
        vt[i] = tb; vt[j] = ta;
      }
    });
    for (int i = threadIdx.x; i < kept; i += blockDim.x) ord[i] = (int32_t)(vt[i] & 0xffffu);
  }
}

size_t sort_smem_bytes(int n) { return (size_t)stage_cap(n) * 8; }

// ---------------------------------------------------------------------------
// Compact result (fast_compact_batch): the changed cells of the balanced
// cross tiles, gathered per matrix in tile order then bit order.
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* sh_warp, int64_t& total) {
  // blockDim.x == kCompactThreads; sh_warp holds one slot per warp
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh_warp[warp] = x;
  __syncthreads();
  int64_t wbase = 0, tot = 0;
  for (int w = 0; w < nw; ++w) {
    const int64_t t = sh_warp[w];
    if (w < warp) wbase += t;
    tot += t;
  }
  __syncthreads();
  total = tot;
  return wbase + x - v;
}

constexpr int kCompactThreads = 512;

// Aux run-out table (fast_strip_rec) from the decomposition's raw stages,
// a post-pass that keeps the bookkeeping out of the peel loop.  One thread
// per source row u replays strip_auxiliary (birkhoff.py:225-252) for the
// row's auxiliary cells: they form one NW-corner staircase range
// [lo_u, hi_u] (consecutive rows share at most one column, so the ranges
// hold <= 2n-1 cells in all); the thread walks the raw stages in order
// (perm[k][u] for the n threads is one coalesced 128-byte row per stage) and
// charges the cell its row is matched to.  Record slot = the cell's position
// in the concatenated ranges.
constexpr int kStripThreads = FAST_MAX_SERVERS;
constexpr int kStripTile = 128;
__global__ void __launch_bounds__(kStripThreads)
    strip_table_kernel(const int n, const fast_sched_bufs out) {
  __shared__ int64_t shw[kStripThreads / 32];
  __shared__ int64_t left[2 * FAST_MAX_SERVERS + 2];
  __shared__ __align__(16) uint8_t tperm[kStripTile * FAST_MAX_SERVERS];
  __shared__ int64_t tw[kStripTile];
  const int b = blockIdx.x, u = threadIdx.x;
  const int K = stage_cap(n), slots = 2 * n + 2;
  fast_strip_rec* rec = out.strip + (int64_t)b * slots;
  const bool ok = out.status[b] == FAST_OK;
  const int64_t* aux = out.aux + (int64_t)b * n * n;
  int lo = 0, hi = -1;
  if (ok && u < n) {
    for (int v = 0; v < n; ++v) {
      if (aux[(int64_t)u * n + v] > 0) {
        if (hi < 0) lo = v;
        hi = v;
      }
    }
  }
  int64_t tot;
  const int off = (int)block_excl_scan(hi >= lo ? hi - lo + 1 : 0, shw, tot);
  for (int i = threadIdx.x; i < slots; i += blockDim.x) {
    fast_strip_rec r;
    r.real = 0;
    r.stage = -1;
    r.src = r.dst = 0;
    rec[i] = r;
  }
  const bool mine = hi >= lo && off + (hi - lo) < slots;  // always (staircase bound)
  int pending = 0;
  if (mine) {
    for (int v = lo; v <= hi; ++v) {
      const int64_t a = aux[(int64_t)u * n + v];
      left[off + v - lo] = a;
      pending += a > 0;
    }
  }
  __syncthreads();  // rec[] initialised before any thread writes a record
  const int nr = ok ? out.n_raw[b] : 0;
  // stage tiles: kStripTile raw stages' permutation rows and weights are
  // staged in shared memory with 16-byte loads, then each thread walks its
  // column of the tile (a shared-memory latency per stage, not a global one)
  const uint8_t* perm = out.stage_perm + (int64_t)b * K * n;
  const int64_t* wt = out.stage_weight + (int64_t)b * K;
  const int rowv = n >> 4;  // 16-byte words per permutation row (n % 16 == 0 path)
  for (int k0 = 0; k0 < nr && __syncthreads_or(pending > 0); k0 += kStripTile) {
    const int kt = nr - k0 < kStripTile ? nr - k0 : kStripTile;
    if ((n & 15) == 0) {
      const uint4* src = reinterpret_cast<const uint4*>(perm + (int64_t)k0 * n);
      for (int i = threadIdx.x; i < kt * rowv; i += blockDim.x)
        reinterpret_cast<uint4*>(tperm)[i] = src[i];
    } else {
      for (int i = threadIdx.x; i < kt * n; i += blockDim.x) tperm[i] = perm[(int64_t)k0 * n + i];
    }
    for (int i = threadIdx.x; i < kt; i += blockDim.x) tw[i] = wt[k0 + i];
    __syncthreads();
    if (pending > 0) {
      for (int k = 0; k < kt; ++k) {
        const int v = tperm[k * n + u];
        if (v < lo || v > hi) continue;
        const int64_t l = left[off + v - lo];
        if (l <= 0) continue;
        const int64_t w = tw[k];
        const int64_t ch = l < w ? l : w;
        left[off + v - lo] = l - ch;
        if (l == ch) {
          fast_strip_rec r;
          r.real = w - ch;
          r.stage = k0 + k;
          r.src = (int16_t)u;
          r.dst = (int16_t)v;
          rec[off + v - lo] = r;
          --pending;
        }
      }
    }
  }
}

__global__ void __launch_bounds__(kCompactThreads)
    compact_count_kernel(const fast_sched_bufs out, const int T, int64_t* __restrict__ cnt) {
  __shared__ int64_t shw[kCompactThreads / 32];
  const int b = blockIdx.x;
  int64_t c = 0;
  if (out.status[b] == FAST_OK)
    for (int t = threadIdx.x; t < T; t += blockDim.x)
      c += __popcll(out.tile_mask[(int64_t)b * T + t]);
  int64_t tot;
  block_excl_scan(c, shw, tot);
  if (threadIdx.x == 0) cnt[b] = tot;
}

__global__ void __launch_bounds__(kCompactThreads)
    compact_scan_kernel(const int64_t* __restrict__ cnt, const int B, int64_t* __restrict__ base) {
  __shared__ int64_t shw[kCompactThreads / 32];
  int64_t carry = 0;
  for (int b0 = 0; b0 < B; b0 += blockDim.x) {
    const int i = b0 + threadIdx.x;
    const int64_t v = i < B ? cnt[i] : 0;
    int64_t tot;
    const int64_t ex = block_excl_scan(v, shw, tot);
    if (i < B) base[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) base[B] = carry;
}

// one CTA per matrix; rounds of blockDim consecutive tiles (coalesced mask
// reads), a block scan places each tile's values
__global__ void __launch_bounds__(kCompactThreads)
    compact_pack_kernel(const fast_sched_bufs out, const int n, const int m,
                        const int64_t* __restrict__ base, int64_t* __restrict__ vals) {
  __shared__ int64_t shw[kCompactThreads / 32];
  const int b = blockIdx.x;
  if (out.status[b] != FAST_OK) return;
  const int T = n * (n - 1);
  const int64_t G = (int64_t)n * m;
  const uint64_t* mk = out.tile_mask + (int64_t)b * T;
  const int64_t* Bb = out.balanced + (int64_t)b * G * G;
  int64_t o = base[b];
  for (int t0 = 0; t0 < T; t0 += blockDim.x) {
    const int t = t0 + threadIdx.x;
    uint64_t x = t < T ? mk[t] : 0ull;
    int64_t tot;
    int64_t w = o + block_excl_scan(__popcll(x), shw, tot);
    if (x) {
      const int i = t / (n - 1), jj = t - i * (n - 1), j = jj < i ? jj : jj + 1;
      const int64_t* tile = Bb + (int64_t)i * m * G + (int64_t)j * m;
      while (x) {
        const int bit = __ffsll((long long)x) - 1;
        x &= x - 1;
        const int p = bit / m, q = bit - p * m;
        vals[w++] = tile[(int64_t)p * G + q];
      }
    }
    o += tot;
  }
}

int check(cudaError_t e) { return e == cudaSuccess ? FAST_OK : FAST_ECUDA; }

#ifdef FAST_BAL_TMA
template <int M>
int launch_balance_tma(const int64_t* D, int B, int n, const fast_sched_bufs* out,
                       cudaStream_t s) {
  const size_t smem = (size_t)2 * kTmaTiles * (M * M + 2) * 8;
  static int grid = 0;
  if (!grid) {
    if (cudaFuncSetAttribute(balance_tma_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return FAST_ECUDA;
    int dev = 0, sms = 0, per_sm = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, balance_tma_kernel<M>, kTmaTiles,
                                                      smem) != cudaSuccess)
      return FAST_ECUDA;
    grid = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int64_t items = (int64_t)B * n * ((n + kTmaTiles - 1) / kTmaTiles);
  const int g = items < grid ? (int)items : grid;
  balance_tma_kernel<M><<<g, kTmaTiles, smem, s>>>(D, n, B, *out);
  return check(cudaGetLastError());
}

#endif  // FAST_BAL_TMA

int launch_balance(const int64_t* D, int B, int n, int m,
                   const fast_sched_bufs* out, cudaStream_t s, bool pdl = false) {
  // even m moves 16-byte pairs of D / balanced: refuse misaligned views
  // loudly instead of faulting on the device
  if (m % 2 == 0 && (((uintptr_t)D | (uintptr_t)out->balanced) & 15)) return FAST_EVALIDATION;
#ifdef FAST_BAL_TMA
  // opt-in: the TMA-fed per-thread pipeline.  Measured 2.3x SLOWER than the
  // staged kernel below (13.0 vs 5.6 ms at n=128 x 8, B=1000;
  // profiles/r2_balance_tma_ab.log): one 64-byte bulk copy per tile row is
  // 262M TMA operations per batch, and the TMA issue rate, not HBM, bounds it.
  if (m == 8 && n >= kTmaTiles && (int64_t)B * n >= 2048)
    return launch_balance_tma<8>(D, B, n, out, s);
#endif
#if defined(FAST_BAL_PIPE) && !defined(FAST_BAL_STAGED)
  // opt-in: the persistent pipelined kernel (measured slower, see above)
  if (m == 2 || m == 4 || m == 8) {
    const int J = kBalThreads / (m / 2);
    const size_t smem = (size_t)J * ((m * m + 1) * 8 + m * 8 + 8);
    const int64_t strips64 = (int64_t)B * n * ((n + J - 1) / J);
    if (strips64 <= INT32_MAX) {
      const int strips = (int)strips64;
      static int per_sm[9] = {0}, sms = 0;
      cudaError_t e = cudaSuccess;
      if (!sms) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
          return FAST_ECUDA;
      }
#define FAST_BAL_PIPE_CASE(MV)                                                              \
  case MV: {                                                                           \
    if (!per_sm[MV] && cudaOccupancyMaxActiveBlocksPerMultiprocessor(                  \
                           &per_sm[MV], balance_pipe_kernel<MV>,                       \
                           bal_pipe_threads<MV>(), smem) != cudaSuccess)                \
      return FAST_ECUDA;                                                               \
    const int g = min(strips, sms * max(per_sm[MV], 1));                               \
    e = launch_k(balance_pipe_kernel<MV>, dim3(g), dim3(bal_pipe_threads<MV>()), smem, \
                 s, pdl, D, n, strips, *out);                                          \
    break;                                                                             \
  }
      switch (m) {
        FAST_BAL_PIPE_CASE(2)
        FAST_BAL_PIPE_CASE(4)
        FAST_BAL_PIPE_CASE(8)
      }
#undef FAST_BAL_PIPE_CASE
      if (e != cudaSuccess) return FAST_ECUDA;
      return check(cudaGetLastError());
    }
  }
#endif
#ifndef FAST_BAL_STAGED
  // even m <= 16: the register-staged kernel (all row loads of a thread in
  // flight, tile prologue at load time); -DFAST_BAL_STAGED for the A/B
  if (m == 2 || m == 4 || m == 8 || m == 16) {
    const int J = kBalThreads / (m / 2);
    const size_t smem = (size_t)J * ((m * m + 1) * 8 + m * 8 + 8);
    const dim3 grid(n, (n + J - 1) / J, B);
    cudaError_t e = cudaSuccess;
    switch (m) {
      case 2: e = launch_k(balance_reg_kernel<2>, grid, dim3(kBalThreads), smem, s, pdl, D, n, *out); break;
      case 4: e = launch_k(balance_reg_kernel<4>, grid, dim3(kBalThreads), smem, s, pdl, D, n, *out); break;
      case 8: e = launch_k(balance_reg_kernel<8>, grid, dim3(kBalThreads), smem, s, pdl, D, n, *out); break;
      default: e = launch_k(balance_reg_kernel<16>, grid, dim3(kBalThreads), smem, s, pdl, D, n, *out);
    }
    if (e != cudaSuccess) return FAST_ECUDA;
    return check(cudaGetLastError());
  }
#endif
  const size_t tile_bytes = (size_t)(m * m + 1) * 8;
  // ~32 KiB strips: several CTAs per SM overlap the per-tile sequential
  // balancing of one CTA with the HBM traffic of the others.
  int J = (int)((FAST_BAL_STRIP_KB * 1024) / tile_bytes);
  if (J > 64) J = 64;
  if (J > n) J = n;
  if (J < 1) J = 1;  // m >= 45: one 16+ KiB tile per CTA
  const size_t smem = (size_t)J * tile_bytes;
  dim3 grid(n, (n + J - 1) / J, B);
  cudaError_t e;
#define FAST_BAL_CASE(MV)                                                    \
  case MV:                                                                   \
    if (smem > 48 * 1024) {                                                  \
      e = cudaFuncSetAttribute(balance_kernel<MV>,                           \
                               cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                               (int)smem);                                   \
      if (e != cudaSuccess) return FAST_ECUDA;                               \
    }                                                                        \
    e = launch_k(balance_kernel<MV>, grid, dim3(kBalThreads), smem, s, pdl,   \
                 D, n, m, J, *out);                                          \
    if (e != cudaSuccess) return FAST_ECUDA;                                 \
    break;
  switch (m) {
    FAST_BAL_CASE(1)
    FAST_BAL_CASE(2)
    FAST_BAL_CASE(4)
    FAST_BAL_CASE(8)
    FAST_BAL_CASE(16)
    default:
      e = cudaFuncSetAttribute(balance_kernel<0>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem);
      if (smem > 48 * 1024 && e != cudaSuccess) return FAST_ECUDA;
      e = launch_k(balance_kernel<0>, grid, dim3(kBalThreads), smem, s, pdl, D, n, m, J, *out);
      if (e != cudaSuccess) return FAST_ECUDA;
  }
#undef FAST_BAL_CASE
  return check(cudaGetLastError());
}

template <int NW, bool WB>
int launch_decompose_wb(const int64_t* S, int B, int n, int mode, int check_total,
                        const fast_sched_bufs* out, cudaStream_t s, bool pdl) {
  const size_t smem = dec_smem_bytes_t<NW>(n) * kDecWarps;
  static size_t granted = 0;  // per template instance
  if (smem > 48 * 1024 && smem > granted) {
    if (cudaFuncSetAttribute(decompose_kernel<NW, WB>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return FAST_ECUDA;
    granted = smem;
  }
  const int grid = (B + kDecWarps - 1) / kDecWarps;
  return launch_k(decompose_kernel<NW, WB>, dim3(grid), dim3(kDecWarps * 32), smem, s, pdl, S, B,
                  n, mode, check_total, *out) == cudaSuccess
             ? FAST_OK
             : FAST_ECUDA;
}

template <int NW>
int launch_decompose_t(const int64_t* S, int B, int n, int mode, int check_total,
                       const fast_sched_bufs* out, cudaStream_t s, bool pdl) {
  return out->stage_bytes
             ? launch_decompose_wb<NW, true>(S, B, n, mode, check_total, out, s, pdl)
             : launch_decompose_wb<NW, false>(S, B, n, mode, check_total, out, s, pdl);
}

int launch_decompose(const int64_t* S, int B, int n, int mode, int check_total,
                     const fast_sched_bufs* out, cudaStream_t s,
                     cudaEvent_t after_decompose = nullptr, bool pdl = false) {
  int rc;
  switch ((n + 31) / 32) {
    case 1: rc = launch_decompose_t<1>(S, B, n, mode, check_total, out, s, pdl); break;
    case 2: rc = launch_decompose_t<2>(S, B, n, mode, check_total, out, s, pdl); break;
    case 3: rc = launch_decompose_t<3>(S, B, n, mode, check_total, out, s, pdl); break;
    default: rc = launch_decompose_t<4>(S, B, n, mode, check_total, out, s, pdl); break;
  }
  if (rc != FAST_OK) return rc;
  if (cudaGetLastError() != cudaSuccess) return FAST_ECUDA;
  if (after_decompose && cudaEventRecord(after_decompose, s) != cudaSuccess)
    return FAST_ECUDA;
  if (stage_cap(n) <= 32) return FAST_OK;  // sorted inside decompose_kernel
  const size_t ssmem = sort_smem_bytes(n);
  static size_t sort_granted = 0;
  if (ssmem > 48 * 1024 && ssmem > sort_granted) {
    if (cudaFuncSetAttribute(sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)ssmem) != cudaSuccess)
      return FAST_ECUDA;
    sort_granted = ssmem;
  }
  int threads = (stage_cap(n) / 2 + 31) & ~31;
  threads = threads < 32 ? 32 : (threads > kSortThreads ? kSortThreads : threads);
  return check(launch_k(sort_kernel, dim3(B), dim3(threads), ssmem, s, pdl, n, *out));
}

// One-launch synthesis for small n (synth_small_kernel).  Returns -1 (not
// an error code: the caller takes the batched kernels) when the shape does
// not fit; the even-m alignment contract is the same as launch_balance's.
int launch_synth_small(const int64_t* D, int B, int n, int m, const fast_sched_bufs* out,
                       cudaStream_t s, bool pdl) {
  const size_t smem = small_smem_bytes(n, m);
#ifdef FAST_NO_SMALL  // A/B: always the batched kernels
  return -1;
#endif
  if (n > kSmallMaxN || smem > 48 * 1024) return -1;
  if (m % 2 == 0 && (((uintptr_t)D | (uintptr_t)out->balanced) & 15)) return FAST_EVALIDATION;
  const bool wb = out->stage_bytes != nullptr;
  cudaError_t e;
#define FAST_SMALL(MV)                                                                  \
  e = wb ? launch_k(synth_small_kernel<MV, true>, dim3(B), dim3(kSmallThreads), smem, s, \
                    pdl, D, n, m, *out)                                                 \
         : launch_k(synth_small_kernel<MV, false>, dim3(B), dim3(kSmallThreads), smem, s, \
                    pdl, D, n, m, *out)
  switch (m) {
    case 1: FAST_SMALL(1); break;
    case 2: FAST_SMALL(2); break;
    case 4: FAST_SMALL(4); break;
    case 8: FAST_SMALL(8); break;
    default: FAST_SMALL(0);
  }
#undef FAST_SMALL
  if (e != cudaSuccess) return FAST_ECUDA;
  return check(cudaGetLastError());
}

bool bad_shape(int B, int n, int m) {
  return B < 0 || n < 2 || n > FAST_MAX_SERVERS || m < 1 ||
         m > FAST_MAX_GPUS_PER_SERVER;
}

}  // namespace

extern "C" {

#ifdef FAST_DEC_PROFILE
int fast_debug_dec_prof(unsigned long long* out8, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out8, g_dec_prof, 8 * sizeof(unsigned long long)) != cudaSuccess)
    return FAST_ECUDA;
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_dec_prof, z, sizeof(z));
  }
  return FAST_OK;
}
#endif

int fast_version(void) { return 200; }

size_t fast_synth_workspace_bytes(int B, int n) {
  if (B <= 0 || n < 1 || n > FAST_MAX_SERVERS) return 0;  // n = 1: decompose only
  return (size_t)B * dec_ws_bytes_per_matrix(n);
}

size_t fast_compact_workspace_bytes(int B) { return (size_t)(B > 0 ? B : 1) * 8 + 256; }

int fast_compact_batch(const fast_sched_bufs* out, int B, int n, int m, int64_t* vals,
                       int64_t* val_base, void* workspace, void* stream) {
  if (bad_shape(B, n, m) || !out || !out->tile_mask || !out->balanced || m > 8 || !val_base ||
      !workspace)
    return FAST_EVALIDATION;
  cudaStream_t s = (cudaStream_t)stream;
  if (B == 0) return check(cudaMemsetAsync(val_base, 0, 8, s));
  int64_t* cnt = (int64_t*)workspace;
  const int T = n * (n - 1);
  compact_count_kernel<<<B, kCompactThreads, 0, s>>>(*out, T, cnt);
  compact_scan_kernel<<<1, kCompactThreads, 0, s>>>(cnt, B, val_base);
  if (vals) compact_pack_kernel<<<B, kCompactThreads, 0, s>>>(*out, n, m, val_base, vals);
  return check(cudaGetLastError());
}

int fast_balance_batch(const int64_t* D, int B, int n, int m,
                       const fast_sched_bufs* out, void* stream) {
  if (bad_shape(B, n, m) || !out) return FAST_EVALIDATION;
  if (B == 0) return FAST_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(out->status, 0, sizeof(int32_t) * B, s) != cudaSuccess)
    return FAST_ECUDA;
  return launch_balance(D, B, n, m, out, s);
}

int fast_decompose_batch(const int64_t* S, int B, int n, int mode,
                         const fast_sched_bufs* out, void* stream) {
  // a 1 x 1 matrix is a valid decompose input (birkhoff.py:140); the
  // synthesis entry points keep the topology's n >= 2 (model.py:55)
  if (B < 0 || n < 1 || n > FAST_MAX_SERVERS || !out) return FAST_EVALIDATION;
  if (mode != FAST_DEC_SERVER && mode != FAST_DEC_DOUBLY_STOCHASTIC)
    return FAST_EVALIDATION;
  if (B == 0) return FAST_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(out->status, 0, sizeof(int32_t) * B, s) != cudaSuccess)
    return FAST_ECUDA;
  return launch_decompose(S, B, n, mode, 0, out, s);
}

int fast_synth_batch_ev(const int64_t* D, int B, int n, int m,
                        const fast_sched_bufs* out, void* stream,
                        void* const* events) {
  if (bad_shape(B, n, m) || !out) return FAST_EVALIDATION;
  if (B == 0) return FAST_OK;
  cudaStream_t s = (cudaStream_t)stream;
  cudaEvent_t const* ev = (cudaEvent_t const*)events;
  if (ev && cudaEventRecord(ev[0], s) != cudaSuccess) return FAST_ECUDA;
  if (!ev) {  // per-kernel events need the separate kernels
    const int rs = launch_synth_small(D, B, n, m, out, s, false);
    if (rs != -1) {
      if (rs != FAST_OK || !out->strip) return rs;
      strip_table_kernel<<<B, kStripThreads, 0, s>>>(n, *out);
      return cudaGetLastError() == cudaSuccess ? FAST_OK : FAST_ECUDA;
    }
  }
  if (cudaMemsetAsync(out->status, 0, sizeof(int32_t) * B, s) != cudaSuccess)
    return FAST_ECUDA;
  int rc = launch_balance(D, B, n, m, out, s);
  if (rc != FAST_OK) return rc;
  if (ev && cudaEventRecord(ev[1], s) != cudaSuccess) return FAST_ECUDA;
  rc = launch_decompose(out->server, B, n, FAST_DEC_SERVER, 1, out, s,
                        ev ? ev[2] : nullptr);
  if (rc != FAST_OK) return rc;
  if (out->strip) {
    strip_table_kernel<<<B, kStripThreads, 0, s>>>(n, *out);
    if (cudaGetLastError() != cudaSuccess) return FAST_ECUDA;
  }
  if (ev && cudaEventRecord(ev[3], s) != cudaSuccess) return FAST_ECUDA;
  return FAST_OK;
}

int fast_synth_batch(const int64_t* D, int B, int n, int m,
                     const fast_sched_bufs* out, void* stream) {
  return fast_synth_batch_ev(D, B, n, m, out, stream, nullptr);
}

}  // extern "C"

int fast_synth_batch_chain(const int64_t* D, int B, int n, int m, const fast_sched_bufs* out,
                           cudaStream_t s, bool pdl) {
  if (bad_shape(B, n, m) || !out) return FAST_EVALIDATION;
  if (B == 0) return FAST_OK;
  const int rs = launch_synth_small(D, B, n, m, out, s, pdl);
  if (rs != -1) return rs;
  int rc = launch_balance(D, B, n, m, out, s, pdl);
  if (rc != FAST_OK) return rc;
  return launch_decompose(out->server, B, n, FAST_DEC_SERVER, 1, out, s, nullptr, pdl);
}

extern "C" {

}  // extern "C"
