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

constexpr int kBalThreads = 128;
constexpr int kDecWarps = 4;  // matrices per CTA in decompose_kernel
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
  const int cols = Jc * m;
  const int total = m * cols;
  const int64_t* Db = D + (int64_t)b * G * G + (int64_t)i * m * G + j0 * m;
  int64_t* Bb = out.balanced + (int64_t)b * G * G + (int64_t)i * m * G + j0 * m;

  // Coalesced stage-in of the m x (Jc*m) strip, scattered into tile-major
  // shared memory.
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int r = idx / cols, col = idx - r * cols;
    const int jj = col / m, c = col - jj * m;
    sm[jj * TS + r * m + c] = __ldcs(Db + (int64_t)r * G + col);
  }
  __syncthreads();

  if (threadIdx.x < Jc) {
    const int jj = threadIdx.x, j = j0 + jj;
    int64_t* t = sm + jj * TS;
    int32_t* st = out.status + b;
    bool bad = false;
    int64_t s = 0;
    for (int k = 0; k < m * m; ++k) {
      const int64_t v = t[k];
      if (v < 0) { bad = true; continue; }
      if (i == j && (k / m) == (k % m) && v != 0) bad = true;
      s = sat_add(s, v);
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

  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int r = idx / cols, col = idx - r * cols;
    const int jj = col / m, c = col - jj * m;
    __stcs(Bb + (int64_t)r * G + col, sm[jj * TS + r * m + c]);
  }
}

// ---------------------------------------------------------------------------
// Decomposition: one warp per matrix.

struct DecSmem {
  int64_t* mv;    // [n] work value of each row's matched cell
  int64_t* am;    // [n] aux_left of each row's matched cell
  int64_t* R;     // [n+1] prefix of row deficits (embedding)
  int64_t* C;     // [n+1] prefix of column deficits
  uint32_t* sup;  // [n][W] support bitset: work[u][v] > 0
  uint32_t* seen; // [W]
  int16_t* rm;    // [n] row_match
  int16_t* cm;    // [n] col_match
  int16_t* snap;  // [n] row_match before re-augmentation
  int16_t* su;    // [n] DFS stack: row
  int16_t* sv;    // [n] DFS stack: column taken by that row
  int16_t* freed; // [n]
};

__host__ __device__ __forceinline__ size_t dec_smem_bytes(int n) {
  const int W = (n + 31) / 32;
  size_t b = 0;
  b += 2 * (size_t)n * 8;            // mv, am
  b += 2 * (size_t)(n + 1) * 8;      // R, C
  b += (size_t)n * W * 4 + W * 4;    // sup, seen
  b += 6 * (size_t)n * 2;            // rm cm snap su sv freed
  return (b + 15) & ~(size_t)15;
}

__device__ __forceinline__ DecSmem dec_carve(char* base, int n) {
  const int W = (n + 31) / 32;
  DecSmem s;
  char* p = base;
  s.mv = (int64_t*)p; p += (size_t)n * 8;
  s.am = (int64_t*)p; p += (size_t)n * 8;
  s.R = (int64_t*)p; p += (size_t)(n + 1) * 8;
  s.C = (int64_t*)p; p += (size_t)(n + 1) * 8;
  s.sup = (uint32_t*)p; p += (size_t)n * W * 4;
  s.seen = (uint32_t*)p; p += W * 4;
  s.rm = (int16_t*)p; p += n * 2;
  s.cm = (int16_t*)p; p += n * 2;
  s.snap = (int16_t*)p; p += n * 2;
  s.su = (int16_t*)p; p += n * 2;
  s.sv = (int16_t*)p; p += n * 2;
  s.freed = (int16_t*)p;
  return s;
}

// augment(u, seen) of birkhoff.py:172-180 with a fresh `seen`, as an explicit
// stack.  Columns are scanned in index order via first-set-bit over
// support & ~seen, which visits exactly the v the reference's
// `for v in range(n): if work[u][v] > 0 and not seen[v]` visits.
__device__ bool augment_lane(const DecSmem& s, const int n, const int W,
                             const int root) {
  for (int w = 0; w < W; ++w) s.seen[w] = 0u;
  int sp = 0;
  s.su[0] = (int16_t)root;
  int cur = 0;
  for (;;) {
    const int u = s.su[sp];
    const uint32_t* su = s.sup + u * W;
    int v = -1;
    for (int w = cur >> 5; w < W; ++w) {
      uint32_t bits = su[w] & ~s.seen[w];
      if (w == (cur >> 5)) bits &= 0xffffffffu << (cur & 31);
      if (bits) { v = (w << 5) + __ffs(bits) - 1; break; }
    }
    if (v < 0) {
      if (sp == 0) return false;
      --sp;
      cur = s.sv[sp] + 1;
      continue;
    }
    s.seen[v >> 5] |= 1u << (v & 31);
    s.sv[sp] = (int16_t)v;
    const int c = s.cm[v];
    if (c < 0) {
      for (int k = sp; k >= 0; --k) {
        s.cm[s.sv[k]] = s.su[k];
        s.rm[s.su[k]] = s.sv[k];
      }
      return true;
    }
    ++sp;
    s.su[sp] = (int16_t)c;
    cur = 0;
  }
}

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

struct DecWs {
  int64_t* work;
  int64_t* auxl;
  uint64_t* key_w;
  uint32_t* key_t;
};

__host__ __device__ __forceinline__ size_t dec_ws_bytes_per_matrix(int n) {
  const size_t K = (size_t)stage_cap(n);
  size_t b = 2 * (size_t)n * n * 8 + K * 8 + K * 4;
  return (b + 255) & ~(size_t)255;
}

__device__ __forceinline__ DecWs dec_ws(void* ws, int b, int n) {
  char* p = (char*)ws + (size_t)b * dec_ws_bytes_per_matrix(n);
  const size_t K = (size_t)stage_cap(n);
  DecWs w;
  w.work = (int64_t*)p; p += (size_t)n * n * 8;
  w.auxl = (int64_t*)p; p += (size_t)n * n * 8;
  w.key_w = (uint64_t*)p; p += K * 8;
  w.key_t = (uint32_t*)p;
  return w;
}

// mode FAST_DEC_SERVER: S is a server matrix (diagonal ignored), embed first.
// mode FAST_DEC_DOUBLY_STOCHASTIC: S is decomposed as-is, aux = 0.
// check_total: synthesize path; S holds saturated tile totals and the status
// word already carries the balance kernel's verdict.
__global__ void __launch_bounds__(kDecWarps * 32)
    decompose_kernel(const int64_t* __restrict__ S_all, const int B,
                     const int n, const int mode, const int check_total,
                     fast_sched_bufs out) {
  extern __shared__ __align__(16) char dsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * kDecWarps + warp;
  if (b >= B) return;
  const int W = (n + 31) / 32;
  const int K = stage_cap(n);
  DecSmem s = dec_carve(dsm + warp * dec_smem_bytes(n), n);
  DecWs ws = dec_ws(out.workspace, b, n);
  const int64_t* S = S_all + (int64_t)b * n * n;
  int32_t* status = out.status + b;
  int64_t* aux_out = out.aux + (int64_t)b * n * n;

  int st = check_total ? *status : FAST_OK;

  // ---- row/column sums of the off-diagonal demand --------------------
  int64_t colsum[FAST_MAX_SERVERS / 32];
  int64_t rowmax = 0, tot = 0, row0 = 0;
  bool neg = false, ds_bad = false;
#pragma unroll
  for (int w = 0; w < FAST_MAX_SERVERS / 32; ++w) colsum[w] = 0;
  for (int u = 0; u < n; ++u) {
    int64_t rs = 0;
#pragma unroll
    for (int w = 0; w < FAST_MAX_SERVERS / 32; ++w) {
      const int v = w * 32 + lane;
      if (w < W && v < n) {
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
    if (lane == 0) s.R[u + 1] = rs;  // row sums, turned into a prefix below
  }
  int64_t colmax = 0;
#pragma unroll
  for (int w = 0; w < FAST_MAX_SERVERS / 32; ++w) {
    const int v = w * 32 + lane;
    if (w < W && v < n) {
      colmax = colsum[w] > colmax ? colsum[w] : colmax;
      if (mode == FAST_DEC_DOUBLY_STOCHASTIC && colsum[w] != row0) ds_bad = true;
    }
  }
  colmax = warp_max_i64(colmax);
  neg = __any_sync(0xffffffffu, neg);
  ds_bad = __any_sync(0xffffffffu, ds_bad);
  // matrix total (saturating): lanes hold saturated partial sums
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

  // ---- embedding: northwest corner as interval overlap -----------------
#pragma unroll
  for (int w = 0; w < FAST_MAX_SERVERS / 32; ++w) {
    const int v = w * 32 + lane;
    if (w < W && v < n) s.C[v + 1] = common - colsum[w];
  }
  __syncwarp();
  if (lane == 0) {
    s.R[0] = 0;
    s.C[0] = 0;
    for (int u = 0; u < n; ++u) s.R[u + 1] = s.R[u] + (common - s.R[u + 1]);
    for (int v = 0; v < n; ++v) s.C[v + 1] += s.C[v];
  }
  for (int u = lane; u < n; u += 32) { s.rm[u] = -1; s.cm[u] = -1; }
  __syncwarp();
  for (int u = 0; u < n; ++u) {
    const int64_t r0 = s.R[u], r1 = s.R[u + 1];
    for (int w = 0; w < W; ++w) {
      const int v = w * 32 + lane;
      int64_t e = 0;
      if (v < n) {
        const int64_t x = S[(int64_t)u * n + v];
        int64_t a = 0;
        int64_t off = x;
        if (mode == FAST_DEC_SERVER) {
          if (u == v) off = 0;
          const int64_t lo = r0 > s.C[v] ? r0 : s.C[v];
          const int64_t hi = r1 < s.C[v + 1] ? r1 : s.C[v + 1];
          a = hi > lo ? hi - lo : 0;
        }
        e = off + a;
        aux_out[(int64_t)u * n + v] = a;
        ws.work[(int64_t)u * n + v] = e;
        ws.auxl[(int64_t)u * n + v] = a;
      }
      const uint32_t bits = __ballot_sync(0xffffffffu, e > 0);
      if (lane == 0) s.sup[u * W + w] = bits;
    }
  }
  if (lane == 0) out.common_sum[b] = common;
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
  int ok = 1;
  if (lane == 0) {
    for (int u = 0; u < n && ok; ++u) ok = augment_lane(s, n, W, u);
  }
  ok = __shfl_sync(0xffffffffu, ok, 0);
  __syncwarp();
  if (!ok) {
    if (lane == 0) { *status = FAST_EINVARIANT; out.n_raw[b] = 0; out.n_stages[b] = 0; }
    return;
  }
  for (int u = lane; u < n; u += 32) {
    const int v = s.rm[u];
    s.mv[u] = ws.work[(int64_t)u * n + v];
    s.am[u] = ws.auxl[(int64_t)u * n + v];
  }
  __syncwarp();

  // ---- peel loop (birkhoff.py:190-219) fused with strip (:225-252) -------
  int64_t remaining = common;
  int k = 0, kept = 0;
  int64_t* wout = out.stage_weight + (int64_t)b * K;
  uint8_t* pout = out.stage_perm + (int64_t)b * K * n;
  int64_t* bout = out.stage_bytes + (int64_t)b * K * n;
  while (remaining > 0) {
    if (k >= K) { st = FAST_EINVARIANT; break; }
    int64_t wl = INT64_MAX;
    for (int u = lane; u < n; u += 32) wl = s.mv[u] < wl ? s.mv[u] : wl;
    const int64_t weight = warp_min_i64(wl);
    if (weight <= 0) { st = FAST_EINVARIANT; break; }
    remaining -= weight;
    int src0 = -1;
    int nfreed = 0;
    for (int base = 0; base < n; base += 32) {
      const int u = base + lane;
      bool real_pos = false, fr = false;
      if (u < n) {
        const int v = s.rm[u];
        const int64_t mvu = s.mv[u] - weight;
        const int64_t amu = s.am[u];
        const int64_t charged = amu < weight ? amu : weight;
        const int64_t real = weight - charged;
        s.mv[u] = mvu;
        s.am[u] = amu - charged;
        bout[(int64_t)k * n + u] = real;
        pout[(int64_t)k * n + u] = (uint8_t)v;
        real_pos = real > 0;
        if (mvu == 0) {
          s.sup[u * W + (v >> 5)] &= ~(1u << (v & 31));
          fr = remaining > 0;
        }
      }
      const uint32_t rb = __ballot_sync(0xffffffffu, real_pos);
      if (src0 < 0 && rb) src0 = base + __ffs(rb) - 1;
      const uint32_t fb = __ballot_sync(0xffffffffu, fr);
      if (fr) s.freed[nfreed + __popc(fb & ((1u << lane) - 1u))] = (int16_t)u;
      nfreed += __popc(fb);
    }
    if (lane == 0) {
      wout[k] = weight;
      if (src0 >= 0) {
        ws.key_w[kept] = (uint64_t)weight;
        ws.key_t[kept] = ((uint32_t)src0 << 24) | ((uint32_t)s.rm[src0] << 16) |
                         (uint32_t)k;
      }
    }
    if (src0 >= 0) ++kept;
    ++k;
    if (remaining == 0) break;
    __syncwarp();
    // unmatch freed rows, remember every row's cell
    for (int u = lane; u < n; u += 32) s.snap[u] = s.rm[u];
    __syncwarp();
    for (int f = lane; f < nfreed; f += 32) {
      const int u = s.freed[f];
      const int v = s.rm[u];
      if (s.cm[v] == u) s.cm[v] = -1;
      s.rm[u] = -1;
    }
    __syncwarp();
    if (lane == 0) {
      for (int f = 0; f < nfreed && ok; ++f) {
        const int u = s.freed[f];
        if (s.rm[u] < 0) ok = augment_lane(s, n, W, u);
      }
    }
    ok = __shfl_sync(0xffffffffu, ok, 0);
    __syncwarp();
    if (!ok) { st = FAST_EINVARIANT; break; }
    // rows whose cell changed: write the old cell back, fetch the new one
    for (int u = lane; u < n; u += 32) {
      const int old = s.snap[u], now = s.rm[u];
      if (old != now) {
        ws.work[(int64_t)u * n + old] = s.mv[u];
        ws.auxl[(int64_t)u * n + old] = s.am[u];
        s.mv[u] = ws.work[(int64_t)u * n + now];
        s.am[u] = ws.auxl[(int64_t)u * n + now];
      }
    }
    __syncwarp();
  }

  // ---- final invariants (birkhoff.py:216-221, :250-251, :273-277) --------
  if (st == FAST_OK) {
    for (int u = lane; u < n; u += 32) {
      const int v = s.rm[u];
      ws.work[(int64_t)u * n + v] = s.mv[u];
      ws.auxl[(int64_t)u * n + v] = s.am[u];
    }
    __syncwarp();
    bool left = false;
    for (int c = lane; c < n * n; c += 32)
      left |= (ws.work[c] != 0) | (ws.auxl[c] != 0);
    if (__any_sync(0xffffffffu, left)) st = FAST_EINVARIANT;
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
  DecWs ws = dec_ws(out.workspace, b, n);
  for (int i = threadIdx.x; i < Q; i += blockDim.x) {
    if (i < kept) {
      kw[i] = ws.key_w[i];
      kt[i] = ws.key_t[i];
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
  int J = (int)((96 * 1024) / tile_bytes);
  if (J > kBalThreads) J = kBalThreads;
  if (J > n) J = n;
  if (J < 1) return FAST_EVALIDATION;
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

int launch_decompose(const int64_t* S, int B, int n, int mode, int check_total,
                     const fast_sched_bufs* out, cudaStream_t s,
                     cudaEvent_t after_decompose = nullptr) {
  const size_t smem = dec_smem_bytes(n) * kDecWarps;
  if (cudaFuncSetAttribute(decompose_kernel,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return FAST_ECUDA;
  const int grid = (B + kDecWarps - 1) / kDecWarps;
  decompose_kernel<<<grid, kDecWarps * 32, smem, s>>>(S, B, n, mode,
                                                      check_total, *out);
  if (cudaGetLastError() != cudaSuccess) return FAST_ECUDA;
  if (after_decompose && cudaEventRecord(after_decompose, s) != cudaSuccess)
    return FAST_ECUDA;
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
