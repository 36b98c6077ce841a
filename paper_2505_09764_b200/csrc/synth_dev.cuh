// synth_dev.cuh -- device building blocks of FAST synthesis, shared by the
// batched kernels (synth.cu) and the fused single-matrix executor path
// (exec.cu): balance_senders on one tile, the warp-level Birkhoff
// decomposition with inline strip and (n <= 6) sort.  See synth.cu for the
// design notes; every function cites the reference lines it replaces.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fastb200.h"

#ifndef DPROF_T
#define DPROF_T(var)
#define DPROF_ADD(slot, val)
#endif

namespace {

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
// Returns the number of moves, or -1 if an invariant breaks.  V is the
// arithmetic type of the greedy: int64_t in general, int32_t when the caller
// knows the tile total (hence every cell, row sum, deviation and chunk) is
// below 2^31 -- the same exact integer steps at half the ALU cost.
template <int M, typename V = int64_t>
__device__ __forceinline__ int balance_tile(int64_t* __restrict__ t, const int m_rt,
                            fast_move* __restrict__ out, const int slots,
                            const int64_t* rowsum = nullptr,
                            uint64_t* changed = nullptr) {
  constexpr int MM = M ? M : FAST_MAX_GPUS_PER_SERVER;
  const int m = M ? M : m_rt;
  V dev[MM];
  V total = 0;
#pragma unroll
  for (int p = 0; p < MM; ++p) {
    V s = 0;
    if (p < m) {
      if (rowsum) {
        s = (V)rowsum[p];  // caller already summed the rows
      } else {
        for (int q = 0; q < m; ++q) s += (V)t[p * m + q];
      }
    }
    dev[p] = s;
    total += s;
  }
  const V base = total / m, extra = total % m;
#pragma unroll
  for (int p = 0; p < MM; ++p)
    if (p < m) dev[p] -= base + (p < extra ? 1 : 0);

  int nmoves = 0;
  // cells touched by a transfer (m <= 8): shedding rows only lose and
  // receiving rows only gain bytes, so touched == changed
  uint64_t mk = 0;
  for (;;) {
    // over[0]: largest positive deviation, lowest index on ties;
    // under[0]: most negative deviation, lowest index on ties.
    int g = -1, h = -1;
    V dg = 0, dh = 0;
#pragma unroll
    for (int p = 0; p < MM; ++p) {
      if (p < m) {
        const V d = dev[p];
        if (d > dg) { dg = d; g = p; }
        if (d < dh) { dh = d; h = p; }
      }
    }
    if (g < 0) {
      if (changed) *changed = mk;
      return nmoves;
    }
    if (h < 0 || nmoves >= slots) return -1;
    const V chunk = dg < -dh ? dg : -dh;
    V left = chunk;
    int guard = 0;
    int64_t* rg = t + g * m;
    int64_t* rh = t + h * m;
    while (left > 0) {
      int q = 0;  // np.argmax: first maximum of row g
      V best = (V)rg[0];
      for (int c = 1; c < m; ++c) {
        const V x = (V)rg[c];
        if (x > best) { best = x; q = c; }
      }
      const V take = left < best ? left : best;
      if (take <= 0 || ++guard > m) return -1;
      rg[q] -= take;
      rh[q] += take;
      left -= take;
      if (m <= 8) mk |= (1ull << (g * m + q)) | (1ull << (h * m + q));
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

// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t warp_min_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t x = __shfl_xor_sync(0xffffffffu, v, o);
    v = x < v ? x : v;
  }
  return v;
}
// min of non-negative int64 over the warp with two 32-bit redux.sync ops
// (high words, then the low words of the lanes holding the minimal high word)
__device__ __forceinline__ int64_t warp_min_nonneg_i64(int64_t v) {
  const uint32_t hi = (uint32_t)((uint64_t)v >> 32), lo = (uint32_t)v;
  const uint32_t mh = __reduce_min_sync(0xffffffffu, hi);
  const uint32_t ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xffffffffu);
  return (int64_t)(((uint64_t)mh << 32) | ml);
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
  static constexpr int kRowShift = NWP == 4 ? 4 : 3;  // log2 bytes per row
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
  uint32_t* freeb; // [NWP] free columns (cm < 0), support-bitset layout
  int64_t* nvs;    // [n] value of a rematched row's new cell (cp.async'd in apply_path)
  int64_t* wk;     // [n][n] the work matrix itself when NW == 1 (n <= 32), else unused
};

template <int NW>
__host__ __device__ __forceinline__ size_t dec_smem_bytes_t(int n) {
  constexpr int NWP = 2 * ((NW + 1) / 2);
  size_t b = 2 * (size_t)n * NWP * 4;      // sup, supc
  b += 2 * (size_t)(n + 1) * 8;            // R, C
  b += (size_t)(2 * n + 2) * 8;            // auxl
  b += 3 * (size_t)n * 2 + 16;             // alo ahi aoff
  b += 4 * (size_t)n * 2;                  // cm newcol pick freed
  b += NWP * 4 + 16;                       // freeb
  b += (size_t)n * 8;                      // nvs
  if (NW == 1) b += (size_t)n * n * 8;     // wk: the work matrix (<= 8 KiB)
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
  s.nvs = (int64_t*)p; p += (size_t)n * 8;
  s.wk = (int64_t*)p; p += NW == 1 ? (size_t)n * n * 8 : 0;
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
//
// The search is a dependent chain (next row = supc[first(row & ~seen)]), so
// the loop is written as one PTX block that keeps every step branch-free and
// short: per-word clz -> candidate row addresses -> a two-level selp tree ->
// ld.shared; `seen` is updated from the per-word clz (off the address chain).
// When a frame resumes after a failed child every support column left of the
// failed one is already seen, so "first column of support & ~seen" is exactly
// the reference's next v and no resume cursor is needed.
//
// Free columns are recognised without a per-step test: supc[v] is all-zero
// for a free column v, so stepping onto one ends in the (rare) "no unseen
// column" exit, which tells the two cases apart with the freeb bitmap.
// pick[k] holds the BYTE OFFSET of the k-th column's supc row (column =
// pick >> kRowShift).  Returns the depth of the successful path (pick[depth]
// is the free column) or -1.
#define FAST_DFS_STEP4(R0, R1, R2, R3, N0, N1, N2, N3)                 \
  "and.b32 x0, " R1 ", ns0;\n\t"                                      \
  "and.b32 x1, " R0 ", ns1;\n\t"                                      \
  "and.b32 x2, " R3 ", ns2;\n\t"                                      \
  "and.b32 x3, " R2 ", ns3;\n\t"                                      \
  "bfind.shiftamt.u32 z0, x0;\n\t"                                               \
  "bfind.shiftamt.u32 z1, x1;\n\t"                                               \
  "bfind.shiftamt.u32 z2, x2;\n\t"                                               \
  "bfind.shiftamt.u32 z3, x3;\n\t"                                               \
  "or.b32 t, x0, x1;\n\t"                                             \
  "or.b32 u, x2, x3;\n\t"                                             \
  "or.b32 u, u, t;\n\t"                                               \
  "setp.eq.u32 pn, u, 0;\n\t"                                         \
  "setp.ne.u32 p0, x0, 0;\n\t"                                        \
  "setp.ne.u32 p2, x2, 0;\n\t"                                        \
  "setp.ne.u32 p01, t, 0;\n\t"                                        \
  "mad.lo.u32 a0, z0, 16, bb0;\n\t"                                   \
  "mad.lo.u32 a1, z1, 16, bb1;\n\t"                                   \
  "mad.lo.u32 a2, z2, 16, bb2;\n\t"                                   \
  "mad.lo.u32 a3, z3, 16, bb3;\n\t"                                   \
  "selp.b32 a0, a0, a1, p0;\n\t"                                      \
  "selp.b32 a2, a2, a3, p2;\n\t"                                      \
  "selp.b32 ad, a0, a2, p01;\n\t"                                     \
  "ld.shared.v4.u32 {" N0 ", " N1 ", " N2 ", " N3 "}, [ad];\n\t"     \
  "@pn bra.uni FDFS_BACK;\n\t"                                        \
  "shr.u32 z0, hb, z0;\n\t"                                           \
  "shr.u32 z1, hb, z1;\n\t"                                           \
  "shr.u32 z2, hb, z2;\n\t"                                           \
  "shr.u32 z3, hb, z3;\n\t"                                           \
  "selp.b32 z3, 0, z3, p2;\n\t"                                       \
  "not.b32 z0, z0;\n\t"                                               \
  "not.b32 z1, z1;\n\t"                                               \
  "not.b32 z2, z2;\n\t"                                               \
  "not.b32 z3, z3;\n\t"                                               \
  "and.b32 ns0, ns0, z0;\n\t"                                         \
  "@!p0 and.b32 ns1, ns1, z1;\n\t"                                    \
  "@!p01 and.b32 ns2, ns2, z2;\n\t"                                   \
  "@!p01 and.b32 ns3, ns3, z3;\n\t"                                   \
  "sub.u32 t, ad, bb0;\n\t"                                           \
  "st.shared.u16 [pa], t;\n\t"                                        \
  "add.u32 pa, pa, 2;\n\t"

// Seen update of the selected word.  The visited column's bit z0 is set in
// ns (x = row & ns had it), so clearing it is a subtraction, which ptxas can
// issue on the FMA pipe (IMAD.IADD) instead of the ALU pipe that the
// decomposition saturates at high occupancy (ncu: ALU pipe 70 % of peak with
// 3000 chains resident).  -DFAST_DFS_SEEN_AND: the and-not form.
#ifdef FAST_DFS_SEEN_AND
#define FAST_DFS_SEEN_UPDATE                                            \
  "not.b32 z0, z0;\n\t"                                               \
  "@p0 and.b32 ns0, ns0, z0;\n\t"                                     \
  "@p1 and.b32 ns1, ns1, z0;\n\t"                                     \
  "@p3 and.b32 ns2, ns2, z0;\n\t"                                     \
  "@pz and.b32 ns3, ns3, z0;\n\t"
#else
#define FAST_DFS_SEEN_UPDATE                                            \
  "@p0 sub.u32 ns0, ns0, z0;\n\t"                                     \
  "@p1 sub.u32 ns1, ns1, z0;\n\t"                                     \
  "@p3 sub.u32 ns2, ns2, z0;\n\t"                                     \
  "@pz sub.u32 ns3, ns3, z0;\n\t"
#endif

// v2 step (default): select the first non-empty word (and its row
// base) with predicates first, then ONE bfind on it -- one FLO per step
// instead of four, and the seen update touches only the selected word.
#define FAST_DFS_STEP4_V2(R0, R1, R2, R3, N0, N1, N2, N3)              \
  "and.b32 x0, " R1 ", ns0;\n\t"                                      \
  "and.b32 x1, " R0 ", ns1;\n\t"                                      \
  "and.b32 x2, " R3 ", ns2;\n\t"                                      \
  "and.b32 x3, " R2 ", ns3;\n\t"                                      \
  "setp.ne.u32 p0, x0, 0;\n\t"                                        \
  "setp.ne.u32 p2, x2, 0;\n\t"                                        \
  "or.b32 t, x0, x1;\n\t"                                             \
  "setp.ne.u32 p01, t, 0;\n\t"                                        \
  "selp.b32 a0, x0, x1, p0;\n\t"                                      \
  "selp.b32 a2, x2, x3, p2;\n\t"                                      \
  "selp.b32 a1, bb0, bb1, p0;\n\t"                                    \
  "selp.b32 a3, bb2, bb3, p2;\n\t"                                    \
  "selp.b32 a0, a0, a2, p01;\n\t"                                     \
  "selp.b32 a1, a1, a3, p01;\n\t"                                     \
  "bfind.shiftamt.u32 z0, a0;\n\t"                                    \
  "mad.lo.u32 ad, z0, 16, a1;\n\t"                                    \
  "ld.shared.v4.u32 {" N0 ", " N1 ", " N2 ", " N3 "}, [ad];\n\t"     \
  "setp.eq.u32 pn, a0, 0;\n\t"                                        \
  "@pn bra.uni FDFS_BACK;\n\t"                                        \
  "setp.ne.and.u32 p1, x1, 0, !p0;\n\t"                               \
  "setp.ne.and.u32 p3, x2, 0, !p01;\n\t"                              \
  "or.b32 u, t, x2;\n\t"                                              \
  "setp.eq.u32 pz, u, 0;\n\t"                                         \
  "shr.u32 z0, hb, z0;\n\t"                                           \
  FAST_DFS_SEEN_UPDATE                                                  \
  "sub.u32 t, ad, bb0;\n\t"                                           \
  "st.shared.u16 [pa], t;\n\t"                                        \
  "add.u32 pa, pa, 2;\n\t"

// v3 step (-DFAST_DFS_V3): per-half select, two bfinds in parallel, the
// address selected last (one dependent op less than v2 on the chain).
#define FAST_DFS_STEP4_V3(R0, R1, R2, R3, N0, N1, N2, N3)              \
  "and.b32 x0, " R1 ", ns0;\n\t"                                      \
  "and.b32 x1, " R0 ", ns1;\n\t"                                      \
  "and.b32 x2, " R3 ", ns2;\n\t"                                      \
  "and.b32 x3, " R2 ", ns3;\n\t"                                      \
  "setp.ne.u32 p0, x0, 0;\n\t"                                        \
  "setp.ne.u32 p2, x2, 0;\n\t"                                        \
  "or.b32 t, x0, x1;\n\t"                                             \
  "setp.ne.u32 p01, t, 0;\n\t"                                        \
  "selp.b32 a0, x0, x1, p0;\n\t"                                      \
  "selp.b32 a2, x2, x3, p2;\n\t"                                      \
  "selp.b32 a1, bb0, bb1, p0;\n\t"                                    \
  "selp.b32 a3, bb2, bb3, p2;\n\t"                                    \
  "bfind.shiftamt.u32 z0, a0;\n\t"                                    \
  "bfind.shiftamt.u32 z2, a2;\n\t"                                    \
  "mad.lo.u32 a1, z0, 16, a1;\n\t"                                    \
  "mad.lo.u32 a3, z2, 16, a3;\n\t"                                    \
  "selp.b32 ad, a1, a3, p01;\n\t"                                     \
  "ld.shared.v4.u32 {" N0 ", " N1 ", " N2 ", " N3 "}, [ad];\n\t"     \
  "or.b32 u, t, x2;\n\t"                                              \
  "or.b32 u, u, x3;\n\t"                                              \
  "setp.eq.u32 pn, u, 0;\n\t"                                         \
  "@pn bra.uni FDFS_BACK;\n\t"                                        \
  "setp.ne.and.u32 p1, x1, 0, !p0;\n\t"                               \
  "setp.ne.and.u32 p3, x2, 0, !p01;\n\t"                              \
  "or.b32 u, t, x2;\n\t"                                              \
  "setp.eq.u32 pz, u, 0;\n\t"                                         \
  "selp.b32 z0, z0, z2, p01;\n\t"                                     \
  "shr.u32 z0, hb, z0;\n\t"                                           \
  "not.b32 z0, z0;\n\t"                                               \
  "@p0 and.b32 ns0, ns0, z0;\n\t"                                     \
  "@p1 and.b32 ns1, ns1, z0;\n\t"                                     \
  "@p3 and.b32 ns2, ns2, z0;\n\t"                                     \
  "@pz and.b32 ns3, ns3, z0;\n\t"                                     \
  "sub.u32 t, ad, bb0;\n\t"                                           \
  "st.shared.u16 [pa], t;\n\t"                                        \
  "add.u32 pa, pa, 2;\n\t"

#define FAST_DFS_STEP2(R0, R1, N0, N1)                                 \
  "and.b32 x0, " R1 ", ns0;\n\t"                                      \
  "and.b32 x1, " R0 ", ns1;\n\t"                                      \
  "bfind.shiftamt.u32 z0, x0;\n\t"                                               \
  "bfind.shiftamt.u32 z1, x1;\n\t"                                               \
  "or.b32 t, x0, x1;\n\t"                                             \
  "setp.eq.u32 pn, t, 0;\n\t"                                         \
  "setp.ne.u32 p0, x0, 0;\n\t"                                        \
  "mad.lo.u32 a0, z0, 8, bb0;\n\t"                                    \
  "mad.lo.u32 a1, z1, 8, bb1;\n\t"                                    \
  "selp.b32 ad, a0, a1, p0;\n\t"                                      \
  "ld.shared.v2.u32 {" N0 ", " N1 "}, [ad];\n\t"                     \
  "@pn bra.uni FDFS_BACK;\n\t"                                        \
  "shr.u32 z0, hb, z0;\n\t"                                           \
  "shr.u32 z1, hb, z1;\n\t"                                           \
  "not.b32 z0, z0;\n\t"                                               \
  "not.b32 z1, z1;\n\t"                                               \
  "and.b32 ns0, ns0, z0;\n\t"                                         \
  "@!p0 and.b32 ns1, ns1, z1;\n\t"                                    \
  "sub.u32 t, ad, bb0;\n\t"                                           \
  "st.shared.u16 [pa], t;\n\t"                                        \
  "add.u32 pa, pa, 2;\n\t"

// Shared tail of both widths: the rare exits.  On "no unseen column" the
// last pushed column is either free (success at depth sp-1) or a dead end
// (pop it and resume its parent row); at sp == 0 the root is exhausted.
#define FAST_DFS_BACK(SH, LDROW)                                        \
  "FDFS_BACK:\n\t"                                                      \
  "setp.eq.u32 pz, pa, %2;\n\t"                                         \
  "@pz bra.uni FDFS_FAIL;\n\t"                                          \
  "ld.shared.u16 t, [pa+-2];\n\t"                                       \
  "shr.u32 t, t, " SH ";\n\t"                                           \
  "shr.u32 u, t, 5;\n\t"                                                \
  "xor.b32 u, u, 1;\n\t"                                                \
  "mad.lo.u32 u, u, 4, %3;\n\t"                                         \
  "ld.shared.u32 u, [u];\n\t"                                           \
  "and.b32 t, t, 31;\n\t"                                               \
  "shr.u32 t, hb, t;\n\t"                                               \
  "and.b32 u, u, t;\n\t"                                                \
  "setp.ne.u32 pz, u, 0;\n\t"                                           \
  "@pz bra.uni FDFS_FOUND;\n\t"                                         \
  "sub.u32 pa, pa, 2;\n\t"                                              \
  "setp.eq.u32 pz, pa, %2;\n\t"                                         \
  "mov.b32 ad, %1;\n\t"                                                 \
  "@pz bra.uni FDFS_RELOAD;\n\t"                                        \
  "ld.shared.u16 t, [pa+-2];\n\t"                                       \
  "add.u32 ad, t, bb0;\n\t"                                             \
  "FDFS_RELOAD:\n\t"                                                    \
  LDROW                                                                 \
  "bra.uni FDFS_LOOP;\n\t"                                              \
  "FDFS_FOUND:\n\t"                                                     \
  "sub.u32 t, pa, %2;\n\t"                                              \
  "shr.u32 t, t, 1;\n\t"                                                \
  "sub.u32 %0, t, 1;\n\t"                                               \
  "bra.uni FDFS_END;\n\t"                                               \
  "FDFS_FAIL:\n\t"                                                      \
  "mov.b32 %0, -1;\n\t"                                                 \
  "FDFS_END:\n\t"

// Shared-window addresses are passed by value so that the DecSh of the
// caller never escapes into this (non-inlined) call: otherwise its pointers
// lose their shared address space and every later access becomes generic.
template <int NW>
__device__ __forceinline__ int dfs_search_body(const uint32_t root_a, const uint32_t pick,
                                       const uint32_t freeb, const uint32_t base) {
  constexpr int NWP = DecSh<NW>::NWP;
  int depth;
  if constexpr (NWP == 4) {
    asm volatile(
        "{\n\t"
        ".reg .pred p0, p1, p2, p3, p01, pn, pz;\n\t"
        ".reg .b32 r0, r1, r2, r3, n0, n1, n2, n3, ns0, ns1, ns2, ns3;\n\t"
        ".reg .b32 x0, x1, x2, x3, z0, z1, z2, z3, a0, a1, a2, a3;\n\t"
        ".reg .b32 ad, t, u, pa, hb, bb0, bb1, bb2, bb3;\n\t"
        "mov.b32 ns0, -1;\n\t"
        "mov.b32 ns1, -1;\n\t"
        "mov.b32 ns2, -1;\n\t"
        "mov.b32 ns3, -1;\n\t"
        "mov.b32 hb, 0x80000000;\n\t"
        "mov.b32 pa, %2;\n\t"
        "mov.b32 bb0, %4;\n\t"
        "add.u32 bb1, %4, 512;\n\t"
        "add.u32 bb2, %4, 1024;\n\t"
        "add.u32 bb3, %4, 1536;\n\t"
        "ld.shared.v4.u32 {r0, r1, r2, r3}, [%1];\n\t"
        "FDFS_LOOP:\n\t"
#if defined(FAST_DFS_V1)
        FAST_DFS_STEP4("r0", "r1", "r2", "r3", "n0", "n1", "n2", "n3")
        FAST_DFS_STEP4("n0", "n1", "n2", "n3", "r0", "r1", "r2", "r3")
#elif defined(FAST_DFS_V3)
        FAST_DFS_STEP4_V3("r0", "r1", "r2", "r3", "n0", "n1", "n2", "n3")
        FAST_DFS_STEP4_V3("n0", "n1", "n2", "n3", "r0", "r1", "r2", "r3")
#else  // v2: measured fastest for the batched (contended) case
        FAST_DFS_STEP4_V2("r0", "r1", "r2", "r3", "n0", "n1", "n2", "n3")
        FAST_DFS_STEP4_V2("n0", "n1", "n2", "n3", "r0", "r1", "r2", "r3")
#endif
        "bra.uni FDFS_LOOP;\n\t"
        FAST_DFS_BACK("4", "ld.shared.v4.u32 {r0, r1, r2, r3}, [ad];\n\t")
        "}"
        : "=r"(depth)
        : "r"(root_a), "r"(pick), "r"(freeb), "r"(base)
        : "memory");
  } else {
    asm volatile(
        "{\n\t"
        ".reg .pred p0, pn, pz;\n\t"
        ".reg .b32 r0, r1, n0, n1, ns0, ns1, x0, x1, z0, z1, a0, a1;\n\t"
        ".reg .b32 ad, t, u, pa, hb, bb0, bb1;\n\t"
        "mov.b32 ns0, -1;\n\t"
        "mov.b32 ns1, -1;\n\t"
        "mov.b32 hb, 0x80000000;\n\t"
        "mov.b32 pa, %2;\n\t"
        "mov.b32 bb0, %4;\n\t"
        "add.u32 bb1, %4, 256;\n\t"
        "ld.shared.v2.u32 {r0, r1}, [%1];\n\t"
        "FDFS_LOOP:\n\t"
        FAST_DFS_STEP2("r0", "r1", "n0", "n1")
        FAST_DFS_STEP2("n0", "n1", "r0", "r1")
        "bra.uni FDFS_LOOP;\n\t"
        FAST_DFS_BACK("3", "ld.shared.v2.u32 {r0, r1}, [ad];\n\t")
        "}"
        : "=r"(depth)
        : "r"(root_a), "r"(pick), "r"(freeb), "r"(base)
        : "memory");
  }
  return depth;
}

// Out-of-line copy for the wide rows (n > 64: long paths amortise the call,
// and one copy of the loop keeps the kernel's code compact); n <= 64 inlines
// the body at its call sites (short paths, the call overhead shows).
template <int NW>
__device__ __noinline__ int dfs_search_call(const uint32_t root_a, const uint32_t pick,
                                            const uint32_t freeb, const uint32_t base) {
  return dfs_search_body<NW>(root_a, pick, freeb, base);
}

template <int NW>
__device__ __forceinline__ int dfs_search(const uint32_t root_a, const uint32_t pick,
                                          const uint32_t freeb, const uint32_t base) {
  if constexpr (NW >= 3) return dfs_search_call<NW>(root_a, pick, freeb, base);
  else return dfs_search_body<NW>(root_a, pick, freeb, base);
}

// Lane 0 searches, the result is broadcast (the other lanes wait).
template <int NW>
__device__ __forceinline__ int dfs_warp(const DecSh<NW>& s, const int root) {
  int depth = 0;
  if ((threadIdx.x & 31) == 0)
    depth = dfs_search<NW>((uint32_t)__cvta_generic_to_shared(s.sup + root * DecSh<NW>::NWP),
                           (uint32_t)__cvta_generic_to_shared(s.pick),
                           (uint32_t)__cvta_generic_to_shared(s.freeb),
                           (uint32_t)__cvta_generic_to_shared(s.supc));
  return __shfl_sync(0xffffffffu, depth, 0);
}

// Apply an augmenting path (warp-wide): cm[pick[k]] = row_k where row_0 =
// root and row_{k+1} = old cm[pick[k]]; record new columns, refresh supc.
// JN = number of 32-element rounds of the path (warp-uniform); within the
// rounds everything is branch-free (clamped indices) so the loads of all
// rounds issue back to back.
template <int NW, int JN>
__device__ __forceinline__ void apply_rounds(const DecSh<NW>& s, const int root, const int depth,
                                             const int lane, const int64_t* work, const int n) {
  constexpr int SH = DecSh<NW>::kRowShift;
  int rows[JN], cols[JN];
  bool act[JN];
#pragma unroll
  for (int j = 0; j < JN; ++j) {
    const int k = j * 32 + lane;
    act[j] = k <= depth;
    const int kk = act[j] ? k : depth;
    cols[j] = s.pick[kk] >> SH;
    rows[j] = s.pick[kk > 0 ? kk - 1 : 0] >> SH;  // column of the previous element
  }
#pragma unroll
  for (int j = 0; j < JN; ++j) {
    const int k = j * 32 + lane;
    rows[j] = (k == 0 || !act[j]) ? root : s.cm[rows[j]];
    // the row's new matched cell is read after the re-augmentation (peel
    // loop, "rows whose cell changed"): start copying it into smem now
    if (work && act[j])
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(s.nvs + rows[j])),
                   "l"(work + (int64_t)rows[j] * n + cols[j])
                   : "memory");
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < JN; ++j) {
    const int k = j * 32 + lane;
    const int v = cols[j], r = rows[j];
    if (act[j]) {
      s.cm[v] = (int16_t)r;
      s.newcol[r] = (int16_t)v;
      if constexpr (DecSh<NW>::NWP == 4) {
        *reinterpret_cast<uint4*>(s.supc + v * 4) = *reinterpret_cast<const uint4*>(s.sup + r * 4);
      } else {
        *reinterpret_cast<uint2*>(s.supc + v * 2) = *reinterpret_cast<const uint2*>(s.sup + r * 2);
      }
      if (k == depth) atomicAnd(&s.freeb[colword(v)], ~colbit(v));  // matched now
    }
  }
}

template <int NW>
__device__ __forceinline__ void apply_path(const DecSh<NW>& s, const int root,
                                           const int depth, const int lane,
                                           const int64_t* work = nullptr, const int n = 0) {
  // an earlier path of this peel may still be filling nvs[] (same slots)
  if (work) asm volatile("cp.async.wait_all;" ::: "memory");
  __syncwarp();  // lane 0's pick[] writes visible to the warp
  // path element k = j*32 + lane, k <= depth < n <= 32*NW
  const int jn = depth >> 5;
  if (jn == 0 || NW == 1) apply_rounds<NW, 1>(s, root, depth, lane, work, n);
  else if (jn == 1 || NW == 2) apply_rounds<NW, (NW >= 2 ? 2 : 1)>(s, root, depth, lane, work, n);
  else if (jn == 2 || NW == 3) apply_rounds<NW, (NW >= 3 ? 3 : 1)>(s, root, depth, lane, work, n);
  else apply_rounds<NW, (NW >= 4 ? 4 : 1)>(s, root, depth, lane, work, n);
  __syncwarp();
}

// The whole decomposition of matrix b by one warp; `wsm` is this warp's
// dec_smem_bytes_t<NW>(n) bytes of shared memory.
// WB: write the per-edge stage_bytes (compile-time, so that the compact
// mode's peel loop carries no extra test)
template <int NW, bool WB = true>
__device__ __forceinline__ void decompose_one(char* wsm, const int64_t* __restrict__ S_all, const int b,
                              const int n, const int mode, const int check_total,
                              const fast_sched_bufs& out, const int lane) {
  constexpr int NWP = DecSh<NW>::NWP;
  const int K = stage_cap(n);
  DecSh<NW> s = dec_carve_t<NW>(wsm, n);
  int64_t* const gwork =
      (int64_t*)((char*)out.workspace + (size_t)b * dec_ws_bytes_per_matrix(n));
  // n <= 32: the whole work matrix fits the warp's shared memory, so the
  // rematched-cell reads of the peel loop never leave the SM
  constexpr bool kSmemWork = NW == 1;
  int64_t* const work = kSmemWork ? s.wk : gwork;
  uint64_t* key_w = (uint64_t*)(gwork + (size_t)n * n);
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
  for (int c = lane; c < n * NWP; c += 32) s.supc[c] = 0u;  // free columns: empty row
  if (lane < NWP) s.freeb[lane] = 0u;
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
  // lane-owned row state; the row's staircase range (alo, ahi, aoff) is
  // constant, so aux slots are register arithmetic: slot = v - base if
  // alo <= v <= ahi
  int rcol[NW], alo[NW], ahi[NW], abase[NW];
  int64_t mv[NW], am[NW];
#pragma unroll
  for (int r = 0; r < NW; ++r) {
    const int u = r * 32 + lane;
    rcol[r] = -1;
    mv[r] = INT64_MAX;
    am[r] = 0;
    alo[r] = 0;
    ahi[r] = -1;
    abase[r] = 0;
    if (u < n) {
      const int v = s.newcol[u];
      rcol[r] = v;
      mv[r] = work[(int64_t)u * n + v];
      alo[r] = s.alo[u];
      ahi[r] = s.ahi[u];
      abase[r] = s.aoff[u] - alo[r];
      am[r] = (v >= alo[r] && v <= ahi[r]) ? s.auxl[abase[r] + v] : 0;
    }
  }
  __syncwarp();

  // ---- peel loop (birkhoff.py:190-219) fused with strip -----------------
  int64_t remaining = common;
  int k = 0, kept = 0;
  int64_t* wout = out.stage_weight + (int64_t)b * K;
  uint8_t* pout = out.stage_perm + (int64_t)b * K * n;
  int64_t* bout = WB ? out.stage_bytes + (int64_t)b * K * n : nullptr;
  while (remaining > 0) {
    DPROF_T(t0);
    if (k >= K) { st = FAST_EINVARIANT; break; }
    int64_t wl = INT64_MAX;
#pragma unroll
    for (int r = 0; r < NW; ++r) wl = mv[r] < wl ? mv[r] : wl;
    const int64_t weight = warp_min_nonneg_i64(wl);  // matched cells are > 0
    if (weight <= 0) { st = FAST_EINVARIANT; break; }
    remaining -= weight;
    int src0 = -1, nfreed = 0, dst0 = 0;
#pragma unroll
    for (int r = 0; r < NW; ++r) {
      // rows u >= n carry mv = INT64_MAX - (sum of weights) > 0 and am = 0,
      // so the arithmetic below is harmless for them; only stores are guarded
      const int u = r * 32 + lane;
      const bool valid = u < n;
      const int v = rcol[r];
      // strip_auxiliary (birkhoff.py:225-252): the cell pays aux first
      const int64_t charged = am[r] < weight ? am[r] : weight;
      const int64_t real = weight - charged;
      am[r] -= charged;
      mv[r] -= weight;
      if (valid) {
        if constexpr (WB) __stcs(bout + (int64_t)k * n + u, real);
        pout[(int64_t)k * n + u] = (uint8_t)v;
      }
      const uint32_t rb = __ballot_sync(0xffffffffu, valid && real > 0);
      const uint32_t zb = __ballot_sync(0xffffffffu, valid && mv[r] == 0);
      if (src0 < 0 && rb) {
        src0 = r * 32 + __ffs(rb) - 1;
        dst0 = __shfl_sync(0xffffffffu, v, __ffs(rb) - 1);
      }
      if (zb) {  // warp-uniform: this round holds a peeled-out cell
        if ((zb >> lane) & 1u) {
          s.sup[u * NWP + colword(v)] &= ~colbit(v);
          if (remaining > 0) {  // free the row (birkhoff.py:210-214)
            s.freed[nfreed + __popc(zb & ((1u << lane) - 1u))] = (int16_t)u;
            s.cm[v] = -1;
#pragma unroll
            for (int w = 0; w < NWP; ++w) s.supc[v * NWP + w] = 0u;  // free: empty row
            atomicOr(&s.freeb[colword(v)], colbit(v));
            rcol[r] = -1;
          }
        }
        if (remaining > 0) nfreed += __popc(zb);
      }
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
      apply_path<NW>(s, u, depth, lane, kSmemWork ? nullptr : work, n);
      DPROF_T(tc);
      DPROF_ADD(1, tb - ta);
      DPROF_ADD(2, tc - tb);
      DPROF_ADD(4, depth + 1);
    }
    if (st != FAST_OK) break;
    DPROF_T(t2);
    // rows whose cell changed (newcol != rcol): fetch the new cell's value
    // (nvs, copied by apply_path) and aux_left, then write the old cell's
    // value and aux_left back.  Loads first, stores after: slots of distinct
    // cells never alias.
    int nc[NW], so[NW];
    int64_t na[NW];
#pragma unroll
    for (int r = 0; r < NW; ++r) {
      const int u = r * 32 + lane;
      nc[r] = u < n ? s.newcol[u] : -1;
    }
#pragma unroll
    for (int r = 0; r < NW; ++r) {
      const bool moved = nc[r] != rcol[r];
      const int sn = (moved && nc[r] >= alo[r] && nc[r] <= ahi[r]) ? abase[r] + nc[r] : -1;
      so[r] = (moved && rcol[r] >= alo[r] && rcol[r] <= ahi[r]) ? abase[r] + rcol[r] : -1;
      na[r] = sn >= 0 ? s.auxl[sn] : (moved ? 0 : am[r]);
    }
#pragma unroll
    for (int r = 0; r < NW; ++r) {
      const int u = r * 32 + lane;
      if (nc[r] != rcol[r]) {
        if (rcol[r] >= 0) work[(int64_t)u * n + rcol[r]] = mv[r];
        if (so[r] >= 0) s.auxl[so[r]] = am[r];
      }
    }
    // the new cells' values (nvs, copied by apply_path) are needed last
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
#pragma unroll
    for (int r = 0; r < NW; ++r) {
      const int u = r * 32 + lane;
      if (nc[r] != rcol[r]) {
        rcol[r] = nc[r];
        mv[r] = kSmemWork ? work[(int64_t)u * n + nc[r]] : s.nvs[u];
        am[r] = na[r];
      }
    }
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


}  // namespace
