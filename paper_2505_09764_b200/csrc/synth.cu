// synth.cu -- batched FAST schedule synthesis on B200 (sm_100a).
//
// Three stream-ordered kernels replace tiersched.synthesize_fast
// (pipeline.py:52-59) for a whole batch of demand matrices:
//
//   balance_kernel   build_balance_plan + reduce_to_server_level
//                    (balance.py:77-174, model.py:169-178).  One CTA per
//                    (server row i, block of J destination servers); the
//                    m rows x J*m columns strip is staged into shared memory
//                    with coalesced loads, one thread balances one m x m
//                    cross tile in place, the strip is written back
//                    coalesced.  HBM-bound: 8*G^2 B read + 8*G^2 B written.
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

namespace {

constexpr int kBalThreads = 256;
constexpr int kDecWarps = 4;  // matrices per CTA in decompose_kernel

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

constexpr int64_t kMaxSafeTotal = int64_t(1) << 62;  // model.py:26

__device__ __forceinline__ int64_t sat_add(int64_t s, int64_t v) {
  // s, v >= 0; saturate at 2^62 so that a later ">= 2^62" test is exact.
  return (v >= kMaxSafeTotal - s) ? kMaxSafeTotal : s + v;
}

__device__ __forceinline__ void raise_status(int32_t* st, int code) {
  atomicMax(st, code);
}

__host__ __device__ __forceinline__ int stage_cap(int n) {
  return n * n - 2 * n + 2;
}

// ---------------------------------------------------------------------------
// balance_senders (balance.py:77-126) on one m x m tile in shared memory.
// Returns the number of moves, or -1 if an invariant breaks.
template <int M>
__device__ int balance_tile(int64_t* __restrict__ t, const int m_rt,
                            fast_move* __restrict__ out, const int slots) {
  constexpr int MM = M ? M : FAST_MAX_GPUS_PER_SERVER;
  const int m = M ? M : m_rt;
  int64_t dev[MM];
  int64_t total = 0;
#pragma unroll
  for (int p = 0; p < MM; ++p) {
    int64_t s = 0;
    if (p < m)
      for (int q = 0; q < m; ++q) s += t[p * m + q];
    dev[p] = s;
    total += s;
  }
  const int64_t base = total / m, extra = total % m;
#pragma unroll
  for (int p = 0; p < MM; ++p)
    if (p < m) dev[p] -= base + (p < extra ? 1 : 0);

  int nmoves = 0;
  for (;;) {
    // over[0]: largest positive deviation, lowest index on ties;
    // under[0]: most negative deviation, lowest index on ties.
    int g = -1, h = -1;
    int64_t dg = 0, dh = 0;
#pragma unroll
    for (int p = 0; p < MM; ++p) {
      if (p < m) {
        const int64_t d = dev[p];
        if (d > dg) { dg = d; g = p; }
        if (d < dh) { dh = d; h = p; }
      }
    }
    if (g < 0) return nmoves;
    if (h < 0 || nmoves >= slots) return -1;
    const int64_t chunk = dg < -dh ? dg : -dh;
    int64_t left = chunk;
    int guard = 0;
    int64_t* rg = t + g * m;
    int64_t* rh = t + h * m;
    while (left > 0) {
      int q = 0;  // np.argmax: first maximum of row g
      int64_t best = rg[0];
      for (int c = 1; c < m; ++c) {
        const int64_t x = rg[c];
        if (x > best) { best = x; q = c; }
      }
      const int64_t take = left < best ? left : best;
      if (take <= 0 || ++guard > m) return -1;
      rg[q] -= take;
      rh[q] += take;
      left -= take;
    }
#pragma unroll
    for (int p = 0; p < MM; ++p) {
      if (p == g) dev[p] -= chunk;
      if (p == h) dev[p] += chunk;
    }
    fast_move mv;
    mv.bytes = chunk;
    mv.from_gpu = g;
    mv.to_gpu = h;
    out[nmoves++] = mv;
  }
}

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
    bool bad = false;
    int64_t s = 0;
    for (int p = 0; p < m; ++p) {
      for (int q = 0; q < m; ++q) {
        const int64_t v = t[p * m + q];
        if (v < 0) { bad = true; continue; }
        if (i == j && p == q && v != 0) bad = true;
        s = sat_add(s, v);
      }
    }
    out.server[(int64_t)b * n * n + i * n + j] = s;
    if (bad) {
      raise_status(st, FAST_EVALIDATION);
    } else if (i != j) {
      const int T = n * (n - 1);
      const int slots = m > 1 ? m - 1 : 1;
      const int tidx = i * (n - 1) + (j < i ? j : j - 1);
      fast_move* mv = out.moves + ((int64_t)b * T + tidx) * slots;
      int nm = balance_tile<M>(t, m, mv, slots);
      if (nm < 0) {
        raise_status(st, FAST_EINVARIANT);
        nm = 0;
      } else {
        // merge_peer row-sum check + per-tile conservation
        // (balance.py:129-136, :157-163)
        int64_t lo = INT64_MAX, hi = INT64_MIN, after = 0;
        for (int p = 0; p < m; ++p) {
          int64_t rs = 0;
          for (int q = 0; q < m; ++q) rs += t[p * m + q];
          lo = rs < lo ? rs : lo;
          hi = rs > hi ? rs : hi;
          after += rs;
        }
        if (hi - lo > 1 || after != s) raise_status(st, FAST_EINVARIANT);
      }
      out.move_count[(int64_t)b * T + tidx] = nm;
    }
  }
  __syncthreads();
  strip_rows<M>(sm, nullptr, Bb, m, G, Jc, false);
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t warp_min_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t x = __shfl_xor_sync(0xffffffffu, v, o);
    v = x < v ? x : v;
  }
  return v;
}
__device__ __forceinline__ int64_t warp_max_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t x = __shfl_xor_sync(0xffffffffu, v, o);
    v = x > v ? x : v;
  }
  return v;
}
__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Per-matrix workspace: work matrix n*n int64, then sort keys (K x u64,
// K x u32) for the kept stages.
__host__ __device__ __forceinline__ size_t dec_ws_bytes_per_matrix(int n) {
  const size_t K = (size_t)stage_cap(n);
  size_t b = (size_t)n * n * 8 + K * 8 + K * 4;
  return (b + 255) & ~(size_t)255;
}

// ---------------------------------------------------------------------------
// Decomposition: one warp per matrix (birkhoff.py:75-252).
//
// State split:
//   shared  sup[u]   support bitset of row u (work[u][v] > 0), NWP words
//           supc[v]  copy of sup[cm[v]]: support of the row matched to v, so
//                    one DFS step is a single 16-B shared load
//           cm[v]    col_match; newcol[u] row's column after re-augmentation
//           pick[k]  DFS stack: column chosen at depth k
//   regs    lane owns rows u = r*32 + lane (r < NW): matched column, work
//           value of its matched cell, and the off-diagonal demand there
//   global  work[u][v] (embedded matrix, written back when a row leaves a
//           non-zero cell) -- only touched when a row's match changes.
// strip_auxiliary (birkhoff.py:225-252) is applied inline with the closed
// form charged = min(w, max(0, work_before - off)): a cell's auxiliary bytes
// are paid first, so aux_left = max(0, aux - peeled) = max(0, work - off).

template <int NW>
struct DecSh {
  static constexpr int NQ = (NW + 1) / 2;   // u64 words per support row
  static constexpr int NWP = 2 * NQ;        // u32 words per support row
  uint32_t* sup;   // [n][NWP]
  uint32_t* supc;  // [n][NWP]
  int64_t* R;      // [n+1]
  int64_t* C;      // [n+1]
  int64_t* auxl;   // [2n+2] aux_left of the NW-corner staircase cells
  int16_t* alo;    // [n] first column of row u's staircase range
  int16_t* ahi;    // [n] last column (alo - 1 when empty)
  int16_t* aoff;   // [n] offset of row u's range in auxl
  int16_t* cm;     // [n]
  int16_t* newcol; // [n]
  int16_t* pick;   // [n]
  int16_t* freed;  // [n]
  uint32_t* chg;   // [NWP] rows whose match changed (bit r%32 of word r/32)
  uint32_t* freeb; // [NWP] free columns (cm < 0), support-bitset layout
};

template <int NW>
__host__ __device__ __forceinline__ size_t dec_smem_bytes_t(int n) {
  constexpr int NWP = 2 * ((NW + 1) / 2);
  size_t b = 2 * (size_t)n * NWP * 4;      // sup, supc
  b += 2 * (size_t)(n + 1) * 8;            // R, C
  b += (size_t)(2 * n + 2) * 8;            // auxl
  b += 3 * (size_t)n * 2 + 16;             // alo ahi aoff
  b += 4 * (size_t)n * 2;                  // cm newcol pick freed
  b += NWP * 4 + 16;                       // chg
  b += NWP * 4 + 16;                       // freeb
  return (b + 15) & ~(size_t)15;
}

template <int NW>
__device__ __forceinline__ DecSh<NW> dec_carve_t(char* p, int n) {
  constexpr int NWP = DecSh<NW>::NWP;
  DecSh<NW> s;
  s.sup = (uint32_t*)p; p += (size_t)n * NWP * 4;
  s.supc = (uint32_t*)p; p += (size_t)n * NWP * 4;
  s.R = (int64_t*)p; p += (size_t)(n + 1) * 8;
  s.C = (int64_t*)p; p += (size_t)(n + 1) * 8;
  s.auxl = (int64_t*)p; p += (size_t)(2 * n + 2) * 8;
  s.chg = (uint32_t*)p; p += NWP * 4 + 16;
  s.freeb = (uint32_t*)p; p += NWP * 4 + 16;
  s.cm = (int16_t*)p; p += n * 2;
  s.newcol = (int16_t*)p; p += n * 2;
  s.pick = (int16_t*)p; p += n * 2;
  s.freed = (int16_t*)p; p += n * 2;
  s.alo = (int16_t*)p; p += n * 2;
  s.ahi = (int16_t*)p; p += n * 2;
  s.aoff = (int16_t*)p;
  return s;
}

// Column layout of the support bitsets: u64 word q holds columns 64q..64q+63
// with column 64q + b at bit 63 - b, so "first column of row & ~seen" is a
// count-leading-zeros per 64-bit half.  In the u32 view that is word
// (v >> 5) ^ 1, bit 31 - (v & 31).
__device__ __forceinline__ int colword(int v) { return (v >> 5) ^ 1; }
__device__ __forceinline__ uint32_t colbit(int v) { return 0x80000000u >> (v & 31); }

template <int NW>
__device__ __forceinline__ void load_row64(const uint32_t* src, uint64_t& r0, uint64_t& r1) {
  if constexpr (DecSh<NW>::NQ == 2) {
    const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(src);
    r0 = x.x;
    r1 = x.y;
  } else {
    r0 = *reinterpret_cast<const uint64_t*>(src);
    r1 = 0ull;
  }
}

// Kuhn augment(root) with a fresh `seen` (birkhoff.py:172-180), one thread.
// When a frame resumes after a failed child every support column left of
// the failed one is already seen, so "first column of support & ~seen" is
// exactly the reference's next v and no resume cursor is needed.  Returns
// the depth of the successful path (pick[k] = column taken at depth k,
// pick[depth] free) or -1.
__device__ __forceinline__ int clz64(uint64_t x) {  // 64 for x == 0
  const uint32_t hi = (uint32_t)(x >> 32), lo = (uint32_t)x;
  return hi ? __clz(hi) : 32 + __clz(lo);
}

template <int NW>
__device__ int dfs_search(const DecSh<NW>& s, const int root, uint64_t free0,
                          uint64_t free1) {
  constexpr int NWP = DecSh<NW>::NWP;
  uint64_t seen0 = 0ull, seen1 = 0ull, r0, r1;
  load_row64<NW>(s.sup + root * NWP, r0, r1);
  int sp = 0;
  for (;;) {
    const int z0 = clz64(r0 & ~seen0), z1 = clz64(r1 & ~seen1);
    const int v = z0 < 64 ? z0 : 64 + z1;  // 128: no unseen support column
    uint64_t n0, n1;
    load_row64<NW>(s.supc + (v & 127) * NWP, n0, n1);  // speculative next row
    if (__builtin_expect(v == 128, 0)) {
      if (sp == 0) return -1;
      --sp;
      load_row64<NW>(sp == 0 ? s.sup + root * NWP : s.supc + s.pick[sp - 1] * NWP, r0, r1);
      continue;
    }
    const uint64_t m = 0x8000000000000000ull >> (v & 63);
    const bool hi = v >= 64;
    const uint64_t fm = (hi ? free1 : free0) & m;
    seen0 |= hi ? 0ull : m;
    seen1 |= hi ? m : 0ull;
    s.pick[sp] = (int16_t)v;
    if (fm) return sp;
    ++sp;
    r0 = n0;
    r1 = n1;
  }
}

// Lane 0 searches, the result is broadcast (the other lanes wait).
template <int NW>
__device__ __forceinline__ int dfs_warp(const DecSh<NW>& s, const int root) {
  int depth = 0;
  if ((threadIdx.x & 31) == 0) {
    const uint64_t* fq = reinterpret_cast<const uint64_t*>(s.freeb);
    depth = dfs_search<NW>(s, root, fq[0], DecSh<NW>::NQ == 2 ? fq[1] : 0ull);
  }
  return __shfl_sync(0xffffffffu, depth, 0);
}

// Apply an augmenting path (warp-wide): cm[pick[k]] = row_k where row_0 =
// root and row_{k+1} = old cm[pick[k]]; record new columns, refresh supc.
template <int NW>
__device__ __forceinline__ void apply_path(const DecSh<NW>& s, const int root,
                                           const int depth, const int lane) {
  constexpr int NWP = DecSh<NW>::NWP;
  __syncwarp();  // lane 0's pick[] writes visible to the warp
  int rows[(FAST_MAX_SERVERS + 31) / 32];
#pragma unroll
  for (int j = 0; j < (FAST_MAX_SERVERS + 31) / 32; ++j) {
    const int k = j * 32 + lane;
    rows[j] = (k <= depth) ? (k == 0 ? root : s.cm[s.pick[k - 1]]) : -1;
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < (FAST_MAX_SERVERS + 31) / 32; ++j) {
    const int k = j * 32 + lane;
    if (k <= depth) {
      const int v = s.pick[k], r = rows[j];
      s.cm[v] = (int16_t)r;
      s.newcol[r] = (int16_t)v;
#pragma unroll
      for (int w = 0; w < NWP; ++w) s.supc[v * NWP + w] = s.sup[r * NWP + w];
      atomicOr(&s.chg[r >> 5], 1u << (r & 31));
      if (k == depth) atomicAnd(&s.freeb[colword(v)], ~colbit(v));  // matched now
    }
  }
  __syncwarp();
}

// aux_left of cell (u, v): a slot of the row's staircase range, or -1.
template <int NW>
__device__ __forceinline__ int aux_slot(const DecSh<NW>& s, int u, int v) {
  return (v >= s.alo[u] && v <= s.ahi[u]) ? s.aoff[u] + v - s.alo[u] : -1;
}

template <int NW>
__global__ void __launch_bounds__(kDecWarps * 32)
    decompose_kernel(const int64_t* __restrict__ S_all, const int B,
                     const int n, const int mode, const int check_total,
                     fast_sched_bufs out) {
  constexpr int NWP = DecSh<NW>::NWP;
  extern __shared__ __align__(16) char dsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * kDecWarps + warp;
  if (b >= B) return;
  const int K = stage_cap(n);
  DecSh<NW> s = dec_carve_t<NW>(dsm + warp * dec_smem_bytes_t<NW>(n), n);
  int64_t* work = (int64_t*)((char*)out.workspace + (size_t)b * dec_ws_bytes_per_matrix(n));
  uint64_t* key_w = (uint64_t*)(work + (size_t)n * n);
  uint32_t* key_t = (uint32_t*)(key_w + K);
  const int64_t* S = S_all + (int64_t)b * n * n;
  int32_t* status = out.status + b;
  int64_t* aux_out = out.aux + (int64_t)b * n * n;

  int st = check_total ? *status : FAST_OK;

  // ---- row/column sums of the off-diagonal demand ------------------------
  int64_t colsum[NW];
  int64_t rowmax = 0, tot = 0, row0 = 0;
  bool neg = false, ds_bad = false;
#pragma unroll
  for (int w = 0; w < NW; ++w) colsum[w] = 0;
  for (int u = 0; u < n; ++u) {
    int64_t rs = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int v = w * 32 + lane;
      if (v < n) {
        int64_t x = S[(int64_t)u * n + v];
        if (x < 0) neg = true;
        tot = sat_add(tot, x < 0 ? 0 : x);
        if (mode == FAST_DEC_SERVER && u == v) x = 0;
        colsum[w] += x;
        rs += x;
      }
    }
    rs = warp_sum_i64(rs);
    if (u == 0) row0 = rs;
    if (mode == FAST_DEC_DOUBLY_STOCHASTIC && rs != row0) ds_bad = true;
    rowmax = rs > rowmax ? rs : rowmax;
    if (lane == 0) s.R[u + 1] = rs;  // row sums; turned into a prefix below
  }
  int64_t colmax = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int v = w * 32 + lane;
    if (v < n) {
      colmax = colsum[w] > colmax ? colsum[w] : colmax;
      if (mode == FAST_DEC_DOUBLY_STOCHASTIC && colsum[w] != row0) ds_bad = true;
    }
  }
  colmax = warp_max_i64(colmax);
  neg = __any_sync(0xffffffffu, neg);
  ds_bad = __any_sync(0xffffffffu, ds_bad);
  int64_t all = 0;
  for (int l = 0; l < 32; ++l) all = sat_add(all, __shfl_sync(0xffffffffu, tot, l));
  if (st == FAST_OK) {
    if (neg || ds_bad) st = FAST_EVALIDATION;
    if (check_total && all >= kMaxSafeTotal) st = FAST_EVALIDATION;
  }
  const int64_t common =
      mode == FAST_DEC_DOUBLY_STOCHASTIC ? row0 : (rowmax > colmax ? rowmax : colmax);
  if (st != FAST_OK) {
    if (lane == 0) {
      *status = st;
      out.common_sum[b] = 0;
      out.n_raw[b] = 0;
      out.n_stages[b] = 0;
    }
    return;
  }

  // ---- embedding: northwest corner == interval overlap of deficit prefixes
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int v = w * 32 + lane;
    if (v < n) s.C[v + 1] = common - colsum[w];
  }
  __syncwarp();
  if (lane == 0) {
    s.R[0] = 0;
    s.C[0] = 0;
    for (int u = 0; u < n; ++u) s.R[u + 1] = s.R[u] + (common - s.R[u + 1]);
    for (int v = 0; v < n; ++v) s.C[v + 1] += s.C[v];
  }
  for (int u = lane; u < n; u += 32) s.cm[u] = -1;
  if (lane < NWP) {
    s.chg[lane] = 0u;
    s.freeb[lane] = 0u;
  }
  __syncwarp();
  for (int v = lane; v < n; v += 32) atomicOr(&s.freeb[colword(v)], colbit(v));
  __syncwarp();
  for (int u = 0; u < n; ++u) {
    const int64_t r0 = s.R[u], r1 = s.R[u + 1];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int v = w * 32 + lane;
      int64_t e = 0;
      if (v < n) {
        int64_t off = S[(int64_t)u * n + v];
        int64_t a = 0;
        if (mode == FAST_DEC_SERVER) {
          if (u == v) off = 0;
          const int64_t lo = r0 > s.C[v] ? r0 : s.C[v];
          const int64_t hi = r1 < s.C[v + 1] ? r1 : s.C[v + 1];
          a = hi > lo ? hi - lo : 0;
        }
        e = off + a;
        aux_out[(int64_t)u * n + v] = a;
        work[(int64_t)u * n + v] = e;
      }
      const uint32_t bits = __brev(__ballot_sync(0xffffffffu, e > 0));
      if (lane == 0) s.sup[u * NWP + (w ^ 1)] = bits;
    }
    if (NWP > NW && lane == 0) s.sup[u * NWP + ((NWP - 1) ^ 1)] = 0u;
  }
  if (lane == 0) {
    out.common_sum[b] = common;
    // NW-corner staircase: row u's aux cells are the contiguous columns whose
    // deficit interval overlaps [R_u, R_u+1); consecutive rows share at most
    // one column, so all of them fit in 2n slots (aux_left lives here).
    int v = 0, at = 0;
    for (int u = 0; u < n; ++u) {
      const int64_t r0 = s.R[u], r1 = s.R[u + 1];
      if (mode != FAST_DEC_SERVER || r1 == r0) {
        s.alo[u] = 0; s.ahi[u] = -1; s.aoff[u] = (int16_t)at;
        continue;
      }
      while (v < n - 1 && s.C[v + 1] <= r0) ++v;
      int e = v;
      while (e < n - 1 && s.C[e + 1] < r1) ++e;
      s.alo[u] = (int16_t)v; s.ahi[u] = (int16_t)e; s.aoff[u] = (int16_t)at;
      for (int c = v; c <= e; ++c) {
        const int64_t lo = r0 > s.C[c] ? r0 : s.C[c];
        const int64_t hi = r1 < s.C[c + 1] ? r1 : s.C[c + 1];
        s.auxl[at++] = hi > lo ? hi - lo : 0;
      }
    }
  }
  __syncwarp();
  if (common == 0) {
    if (lane == 0) {
      out.n_raw[b] = 0;
      out.n_stages[b] = 0;
      *status = FAST_OK;
    }
    return;
  }

  // ---- initial Kuhn matching (birkhoff.py:182-186) -----------------------
  for (int u = 0; u < n; ++u) {
    const int depth = dfs_warp<NW>(s, u);
    if (depth < 0) { st = FAST_EINVARIANT; break; }
    apply_path<NW>(s, u, depth, lane);
  }
  if (st != FAST_OK) {
    if (lane == 0) { *status = st; out.n_raw[b] = 0; out.n_stages[b] = 0; }
    return;
  }
  // lane-owned row state
  int rcol[NW];
  int64_t mv[NW], am[NW];
#pragma unroll
  for (int r = 0; r < NW; ++r) {
    const int u = r * 32 + lane;
    rcol[r] = -1;
    mv[r] = INT64_MAX;
    am[r] = 0;
    if (u < n) {
      const int v = s.newcol[u];
      rcol[r] = v;
      mv[r] = work[(int64_t)u * n + v];
      const int sl = aux_slot<NW>(s, u, v);
      am[r] = sl >= 0 ? s.auxl[sl] : 0;
    }
  }
  if (lane < NWP) s.chg[lane] = 0u;
  __syncwarp();

  // ---- peel loop (birkhoff.py:190-219) fused with strip -----------------
  int64_t remaining = common;
  int k = 0, kept = 0;
  int64_t* wout = out.stage_weight + (int64_t)b * K;
  uint8_t* pout = out.stage_perm + (int64_t)b * K * n;
  int64_t* bout = out.stage_bytes + (int64_t)b * K * n;
  while (remaining > 0) {
    DPROF_T(t0);
    if (k >= K) { st = FAST_EINVARIANT; break; }
    int64_t wl = INT64_MAX;
#pragma unroll
    for (int r = 0; r < NW; ++r) wl = mv[r] < wl ? mv[r] : wl;
    const int64_t weight = warp_min_i64(wl);
    if (weight <= 0) { st = FAST_EINVARIANT; break; }
    remaining -= weight;
    int src0 = -1, nfreed = 0, dst0 = 0;
#pragma unroll
    for (int r = 0; r < NW; ++r) {
      const int u = r * 32 + lane;
      bool real_pos = false, fr = false;
      const int vsave = rcol[r];
      if (u < n) {
        const int v = rcol[r];
        // strip_auxiliary (birkhoff.py:225-252): the cell pays aux first
        const int64_t charged = am[r] < weight ? am[r] : weight;
        const int64_t real = weight - charged;
        am[r] -= charged;
        mv[r] -= weight;
        __stcs(bout + (int64_t)k * n + u, real);
        pout[(int64_t)k * n + u] = (uint8_t)v;
        real_pos = real > 0;
        if (mv[r] == 0) {
          s.sup[u * NWP + colword(v)] &= ~colbit(v);
          fr = remaining > 0;
        }
      }
      const uint32_t rb = __ballot_sync(0xffffffffu, real_pos);
      if (src0 < 0 && rb) {
        src0 = r * 32 + __ffs(rb) - 1;
        dst0 = __shfl_sync(0xffffffffu, vsave, __ffs(rb) - 1);
      }
      const uint32_t fb = __ballot_sync(0xffffffffu, fr);
      if (fr) {
        s.freed[nfreed + __popc(fb & ((1u << lane) - 1u))] = (int16_t)u;
        s.cm[rcol[r]] = -1;  // unmatch (birkhoff.py:210-214)
        atomicOr(&s.freeb[colword(rcol[r])], colbit(rcol[r]));
        rcol[r] = -1;
      }
      nfreed += __popc(fb);
    }
    if (lane == 0) {
      wout[k] = weight;
      if (src0 >= 0) {
        // dst of src0 = the column src0 was matched to in this stage
        key_w[kept] = (uint64_t)weight;
        key_t[kept] = ((uint32_t)src0 << 24) | ((uint32_t)dst0 << 16) | (uint32_t)k;
      }
    }
    if (src0 >= 0) ++kept;
    ++k;
    if (remaining == 0) break;
    __syncwarp();
    DPROF_T(t1);
    DPROF_ADD(0, t1 - t0);
    // re-augment freed rows in index order (birkhoff.py:215-219)
    for (int f = 0; f < nfreed; ++f) {
      const int u = s.freed[f];
      DPROF_T(ta);
      const int depth = dfs_warp<NW>(s, u);
      DPROF_T(tb);
      if (depth < 0) { st = FAST_EINVARIANT; break; }
      apply_path<NW>(s, u, depth, lane);
      DPROF_T(tc);
      DPROF_ADD(1, tb - ta);
      DPROF_ADD(2, tc - tb);
      DPROF_ADD(4, depth + 1);
    }
    if (st != FAST_OK) break;
    DPROF_T(t2);
    // rows whose cell changed: write the old (non-zero) value back, fetch
    // the new cell; all loads are issued before any is consumed.
    uint32_t chg[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) chg[w] = s.chg[w];
    __syncwarp();
    if (lane < NWP) s.chg[lane] = 0u;
    int64_t nv[NW];
    bool moved[NW];
#pragma unroll
    for (int r = 0; r < NW; ++r) {
      const int u = r * 32 + lane;
      const int nc = (u < n && ((chg[r] >> lane) & 1u)) ? s.newcol[u] : rcol[r];
      moved[r] = nc != rcol[r];
      if (moved[r]) {
        if (rcol[r] >= 0) {
          work[(int64_t)u * n + rcol[r]] = mv[r];
          const int so = aux_slot<NW>(s, u, rcol[r]);
          if (so >= 0) s.auxl[so] = am[r];
        }
        rcol[r] = nc;
        nv[r] = work[(int64_t)u * n + nc];
        const int sn = aux_slot<NW>(s, u, nc);
        am[r] = sn >= 0 ? s.auxl[sn] : 0;
      }
    }
#pragma unroll
    for (int r = 0; r < NW; ++r)
      if (moved[r]) mv[r] = nv[r];
    __syncwarp();
    DPROF_T(t3);
    DPROF_ADD(3, t3 - t2);
    DPROF_ADD(5, 1);
  }

  // ---- final invariants (birkhoff.py:216-221, :273-277): every cell peeled
  if (st == FAST_OK) {
    bool left = remaining != 0;
    for (int c = lane; c < n * NWP; c += 32) left |= s.sup[c] != 0u;
    if (__any_sync(0xffffffffu, left)) st = FAST_EINVARIANT;
  }
  // small stage capacity (n <= 6): sort_stages_ascending here with a warp
  // bitonic network on (weight, src0|dst0|raw index) and skip sort_kernel
  if (K <= 32 && st == FAST_OK && kept > 0) {
    __syncwarp();
    uint64_t w = lane < kept ? key_w[lane] : ~0ull;
    uint32_t t = lane < kept ? key_t[lane] : ~0u;
#pragma unroll
    for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
      for (int j = kk >> 1; j > 0; j >>= 1) {
        const uint64_t w2 = __shfl_xor_sync(0xffffffffu, w, j);
        const uint32_t t2 = __shfl_xor_sync(0xffffffffu, t, j);
        const bool asc = (lane & kk) == 0;
        const bool lower = (lane & j) == 0;
        const bool gt = w > w2 || (w == w2 && t > t2);
        if ((lower == asc) ? gt : !gt) { w = w2; t = t2; }
      }
    }
    if (lane < kept) out.stage_order[(int64_t)b * K + lane] = (int32_t)(t & 0xffffu);
  }
  if (lane == 0) {
    *status = st;
    out.n_raw[b] = k;
    out.n_stages[b] = st == FAST_OK ? kept : 0;
  }
}

// ---------------------------------------------------------------------------
// sort_stages_ascending: bitonic sort of (weight, src0<<24|dst0<<16|idx).
__global__ void __launch_bounds__(1024)
    sort_kernel(const int n, fast_sched_bufs out) {
  extern __shared__ __align__(16) char ssm[];
  const int b = blockIdx.x;
  const int K = stage_cap(n);
  int P = 1;
  while (P < K) P <<= 1;
  uint64_t* kw = (uint64_t*)ssm;
  uint32_t* kt = (uint32_t*)(ssm + (size_t)P * 8);
  if (out.status[b] != FAST_OK) return;
  const int kept = out.n_stages[b];
  if (kept <= 0) return;
  int Q = 1;
  while (Q < kept) Q <<= 1;
  const int64_t* work =
      (const int64_t*)((const char*)out.workspace + (size_t)b * dec_ws_bytes_per_matrix(n));
  const uint64_t* key_w = (const uint64_t*)(work + (size_t)n * n);
  const uint32_t* key_t = (const uint32_t*)(key_w + K);
  for (int i = threadIdx.x; i < Q; i += blockDim.x) {
    if (i < kept) {
      kw[i] = key_w[i];
      kt[i] = key_t[i];
    } else {
      kw[i] = ~0ull;
      kt[i] = ~0u;
    }
  }
  __syncthreads();
  for (int kk = 2; kk <= Q; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < Q; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool asc = (i & kk) == 0;
          const uint64_t wa = kw[i], wb = kw[ixj];
          const uint32_t ta = kt[i], tb = kt[ixj];
          const bool gt = wa > wb || (wa == wb && ta > tb);
          if (gt == asc) {
            kw[i] = wb; kw[ixj] = wa;
            kt[i] = tb; kt[ixj] = ta;
          }
        }
      }
      __syncthreads();
    }
  }
  int32_t* ord = out.stage_order + (int64_t)b * K;
  for (int i = threadIdx.x; i < kept; i += blockDim.x) ord[i] = (int32_t)(kt[i] & 0xffffu);
}

size_t sort_smem_bytes(int n) {
  int P = 1;
  while (P < stage_cap(n)) P <<= 1;
  return (size_t)P * 12;
}

int check(cudaError_t e) { return e == cudaSuccess ? FAST_OK : FAST_ECUDA; }

int launch_balance(const int64_t* D, int B, int n, int m,
                   const fast_sched_bufs* out, cudaStream_t s) {
  const size_t tile_bytes = (size_t)(m * m + 1) * 8;
  // ~32 KiB strips: several CTAs per SM overlap the per-tile sequential
  // balancing of one CTA with the HBM traffic of the others.
  int J = (int)((32 * 1024) / tile_bytes);
  if (J > 64) J = 64;
  if (J > n) J = n;
  if (J < 1) J = 1;  // m >= 45: one 16+ KiB tile per CTA
  const size_t smem = (size_t)J * tile_bytes;
  dim3 grid(n, (n + J - 1) / J, B);
  cudaError_t e;
#define FAST_BAL_CASE(MV)                                                    \
  case MV:                                                                   \
    e = cudaFuncSetAttribute(balance_kernel<MV>,                             \
                             cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                             (int)smem);                                     \
    if (e != cudaSuccess) return FAST_ECUDA;                                 \
    balance_kernel<MV><<<grid, kBalThreads, smem, s>>>(D, n, m, J, *out);    \
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
      if (e != cudaSuccess) return FAST_ECUDA;
      balance_kernel<0><<<grid, kBalThreads, smem, s>>>(D, n, m, J, *out);
  }
#undef FAST_BAL_CASE
  return check(cudaGetLastError());
}

template <int NW>
int launch_decompose_t(const int64_t* S, int B, int n, int mode, int check_total,
                       const fast_sched_bufs* out, cudaStream_t s) {
  const size_t smem = dec_smem_bytes_t<NW>(n) * kDecWarps;
  if (cudaFuncSetAttribute(decompose_kernel<NW>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return FAST_ECUDA;
  const int grid = (B + kDecWarps - 1) / kDecWarps;
  decompose_kernel<NW><<<grid, kDecWarps * 32, smem, s>>>(S, B, n, mode,
                                                          check_total, *out);
  return FAST_OK;
}

int launch_decompose(const int64_t* S, int B, int n, int mode, int check_total,
                     const fast_sched_bufs* out, cudaStream_t s,
                     cudaEvent_t after_decompose = nullptr) {
  int rc;
  switch ((n + 31) / 32) {
    case 1: rc = launch_decompose_t<1>(S, B, n, mode, check_total, out, s); break;
    case 2: rc = launch_decompose_t<2>(S, B, n, mode, check_total, out, s); break;
    case 3: rc = launch_decompose_t<3>(S, B, n, mode, check_total, out, s); break;
    default: rc = launch_decompose_t<4>(S, B, n, mode, check_total, out, s); break;
  }
  if (rc != FAST_OK) return rc;
  if (cudaGetLastError() != cudaSuccess) return FAST_ECUDA;
  if (after_decompose && cudaEventRecord(after_decompose, s) != cudaSuccess)
    return FAST_ECUDA;
  if (stage_cap(n) <= 32) return FAST_OK;  // sorted inside decompose_kernel
  const size_t ssmem = sort_smem_bytes(n);
  if (cudaFuncSetAttribute(sort_kernel,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)ssmem) != cudaSuccess)
    return FAST_ECUDA;
  int threads = (int)(ssmem / 12 / 2);
  threads = threads < 32 ? 32 : (threads > 1024 ? 1024 : threads);
  sort_kernel<<<B, threads, ssmem, s>>>(n, *out);
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

int fast_version(void) { return 100; }

size_t fast_synth_workspace_bytes(int B, int n) {
  if (B <= 0 || n < 2 || n > FAST_MAX_SERVERS) return 0;
  return (size_t)B * dec_ws_bytes_per_matrix(n);
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
  if (bad_shape(B, n, 1) || !out) return FAST_EVALIDATION;
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
  if (cudaMemsetAsync(out->status, 0, sizeof(int32_t) * B, s) != cudaSuccess)
    return FAST_ECUDA;
  int rc = launch_balance(D, B, n, m, out, s);
  if (rc != FAST_OK) return rc;
  if (ev && cudaEventRecord(ev[1], s) != cudaSuccess) return FAST_ECUDA;
  rc = launch_decompose(out->server, B, n, FAST_DEC_SERVER, 1, out, s,
                        ev ? ev[2] : nullptr);
  if (rc != FAST_OK) return rc;
  if (ev && cudaEventRecord(ev[3], s) != cudaSuccess) return FAST_ECUDA;
  return FAST_OK;
}

int fast_synth_batch(const int64_t* D, int B, int n, int m,
                     const fast_sched_bufs* out, void* stream) {
  return fast_synth_batch_ev(D, B, n, m, out, stream, nullptr);
}

}  // extern "C"
