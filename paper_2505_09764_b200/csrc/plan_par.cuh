// plan_par.cuh -- CTA-parallel device build of the FAST stage plan.
//
// Produces exactly the op list of the sequential fastplan::plan_compile
// (plan.cuh, which stays the host build and the parity check of this one,
// tests/test_exec_gpu.py::test_parallel_device_plan_equals_host_plan).  The
// sequential walk is one thread doing a long chain of dependent steps per op
// (64-bit divisions, linear take scans); on a GPU one such step costs
// hundreds of cycles, so here the serial depth is kept independent of the
// op count and every op is written straight into its final slot:
//
//   P1  segment offsets             thread per rank (send rows / recv columns)
//   P2  balance replay              thread per tile; per-cell piece lists
//       stage table                 thread per (stage, server): inverse perm
//   P3  balance staging + ops       thread per taker rank (tile j order, take order)
//       intra-server op counts      thread per sender rank
//       window starts               thread per (stage, server): bytes of the
//                                   pair delivered by earlier stages
//   P4  window walk, count          thread per (stage, lane)
//   P5  proxy staging/slot prefix   thread per proxy (j, p), stages in order
//       op positions                block scan over (bucket, stage, pass, lane)
//   P6  window walk, emit           thread per (stage, lane), ops to final slots
//
// Window independence: lane p of pair (i -> j) streams cells (p, 0..m-1),
// each cell = [original part][balanced-in pieces in take order].  Stage s
// moves stream bytes [share(c0), share(c0 + b)) with c0 the pair's bytes in
// earlier stages, so a window locates itself by byte position -- no cursor
// carried between stages -- and visits exactly the pieces (and offsets) the
// sequential cursor walk visits.  Each proxy (j, p) is fed by exactly one
// lane (i, p) per stage (a stage is a permutation), so its sequential
// staging / flag-slot allocation order is the stage order of its feeding
// windows: a per-proxy prefix over per-window needs, without atomics.
#pragma once
#include "plan.cuh"

namespace fastplan {

// Workspace of the parallel build (device global or shared memory).
struct ParWs {
  int64_t* send_off;    // [G][G]
  int64_t* recv_off;    // [G][G]
  Take* takes;          // [T][MT]
  int64_t* orig_len;    // [T][m*m]
  int64_t* tile_sum;    // [T]
  int64_t* stg_top;     // [G]
  int64_t* slot_top;    // [G]
  int64_t* cs0;         // [K][n]   pair bytes delivered before stage s
  int64_t* stg_need;    // [K][G]   staged bytes (16-B aligned) of window -> base
  int64_t* slot_need;   // [K][G]   flag slots of window -> base
  int32_t* ntakes;      // [T]
  int32_t* take_pre;    // [T]      exclusive prefix of ntakes
  int32_t* cell_start;  // [T][m*m+1]
  int32_t* piece_take;  // [T][MT]
  int32_t* direct_pre;  // [G]
  int32_t* inv;         // [K][n]   source server feeding server j at stage s, -1
  int32_t* cnt;         // [3][K][2][G] -> exclusive positions
};

__host__ __device__ inline int64_t par_ws_bytes(int n, int m, int K) {
  const int64_t G = (int64_t)n * m, T = (int64_t)n * (n - 1), MT = max_takes(m);
  int64_t b = 0;
  b += 2 * G * G * 8 + T * MT * (int64_t)sizeof(Take) + T * m * m * 8 + T * 8;
  b += 2 * G * 8 + (int64_t)K * n * 8 + 2 * (int64_t)K * G * 8;
  b += (2 * T + T * (m * m + 1) + T * MT + G + (int64_t)K * n + 6 * (int64_t)K * G) * 4;
  return align16(b + 64);
}

__host__ __device__ inline ParWs par_carve(void* p, int n, int m, int K) {
  const int64_t G = (int64_t)n * m, T = (int64_t)n * (n - 1), MT = max_takes(m);
  char* c = (char*)p;
  ParWs w;
  w.send_off = (int64_t*)c; c += G * G * 8;
  w.recv_off = (int64_t*)c; c += G * G * 8;
  w.takes = (Take*)c; c += T * MT * sizeof(Take);
  w.orig_len = (int64_t*)c; c += T * m * m * 8;
  w.tile_sum = (int64_t*)c; c += T * 8;
  w.stg_top = (int64_t*)c; c += G * 8;
  w.slot_top = (int64_t*)c; c += G * 8;
  w.cs0 = (int64_t*)c; c += (int64_t)K * n * 8;
  w.stg_need = (int64_t*)c; c += (int64_t)K * G * 8;
  w.slot_need = (int64_t*)c; c += (int64_t)K * G * 8;
  w.ntakes = (int32_t*)c; c += T * 4;
  w.take_pre = (int32_t*)c; c += T * 4;
  w.cell_start = (int32_t*)c; c += T * (m * m + 1) * 4;
  w.piece_take = (int32_t*)c; c += T * MT * 4;
  w.direct_pre = (int32_t*)c; c += G * 4;
  w.inv = (int32_t*)c; c += (int64_t)K * n * 4;
  w.cnt = (int32_t*)c;
  return w;
}

#ifdef __CUDACC__

#ifdef FAST_PLAN_PROFILE
__device__ long long g_plan_prof[16];  // clock64 stamps of the last build (thread 0)
#define PLAN_STAMP(k) \
  do { if (threadIdx.x == 0) fastplan::g_plan_prof[k] = clock64(); } while (0)
#else
#define PLAN_STAMP(k) do { } while (0)
#endif

enum : int { kParEarlyVal = 1, kParInvariant = 2, kParLateVal = 4, kParOverflow = 8 };

// Block-wide exclusive scan of a[0, L) in place; returns the total (all threads).
__device__ inline int32_t block_exclusive_scan(int32_t* a, int L) {
  __shared__ int32_t s_part[33];
  const int nt = blockDim.x, t = threadIdx.x;
  const int per = (L + nt - 1) / nt;
  const int lo = min(L, t * per), hi = min(L, lo + per);
  int32_t s = 0;
  for (int i = lo; i < hi; ++i) s += a[i];
  // warp inclusive scan, then across warps
  const int lane = t & 31, wid = t >> 5, nw = (nt + 31) >> 5;
  int32_t x = s;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) s_part[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int32_t v = lane < nw ? s_part[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, v, d);
      if (lane >= d) v += y;
    }
    if (lane < nw) s_part[lane] = v;  // inclusive per warp
    if (lane == 31) s_part[32] = v;
  }
  __syncthreads();
  int32_t run = (wid ? s_part[wid - 1] : 0) + x - s;
  for (int i = lo; i < hi; ++i) {
    const int32_t v = a[i];
    a[i] = run;
    run += v;
  }
  const int32_t total = s_part[32];
  __syncthreads();
  return total;
}

// floor((C + m - 1 - p) / m): lane p's share of the first C bytes (round robin)
__device__ __forceinline__ int64_t lane_share(int64_t C, int m, int p) {
  const int64_t q = C / m;
  return q + ((C - q * m) > p ? 1 : 0);
}

__device__ __forceinline__ int64_t div_chunks(int64_t len, int64_t ch, int ch_shift) {
  return ch_shift >= 0 ? (len + ch - 1) >> ch_shift : (len + ch - 1) / ch;
}

// Window of kept stage s on lane (i, p).  EMIT = false: count its ops per
// (bucket, pass) and its staging / flag-slot needs; EMIT = true: write the
// ops.  Returns false when the window runs past the lane stream.
template <bool EMIT>
__device__ __forceinline__ bool stage_window(const PlanIn& in, const ParWs& w, int s, int i, int p,
                                    fast_op* ops, int32_t op_base, int ch_shift) {
  const int n = in.n, m = in.m, G = n * m, K = in.K, MT = max_takes(m);
  const int k = in.order[s];
  const int64_t b = in.sbytes[(int64_t)k * n + i];
  if (b <= 0) return true;
  const int j = in.perm[(int64_t)k * n + i];
  const int tix = tile_index(n, i, j);
  const int lane = i * m + p, proxy = j * m + p;
  const int64_t c0 = w.cs0[(int64_t)s * n + i];
  const int64_t X0 = lane_share(c0, m, p), X1 = lane_share(c0 + b, m, p);
  const int64_t sp = (int64_t)s * 2;
  const int64_t ix[5] = {(0 * K * 2 + sp + 0) * G + lane, (1 * K * 2 + sp + 0) * G + lane,
                         (0 * K * 2 + sp + 1) * G + lane, (1 * K * 2 + sp + 1) * G + lane,
                         (2 * K * 2 + sp + 0) * G + lane};
  // counters / positions: [pass0 b1, pass0 b2, pass1 b1, pass1 b2, pass0 b3]
  int32_t c[5];
#pragma unroll
  for (int u = 0; u < 5; ++u) c[u] = EMIT ? w.cnt[ix[u]] : 0;
  int64_t stg = EMIT ? w.stg_need[(int64_t)s * G + lane] : 0;
  int64_t slot = EMIT ? w.slot_need[(int64_t)s * G + lane] : 0;
  const Take* tk = w.takes + (int64_t)tix * MT;
  const int32_t* cs = w.cell_start + (int64_t)tix * (m * m + 1);
  const int32_t* pt = w.piece_take + (int64_t)tix * MT;
  const int64_t* ol = w.orig_len + (int64_t)tix * m * m;
  int64_t pos = 0;  // stream offset of the current piece
  for (int q = 0; q < m && pos < X1; ++q) {
    const int cell = p * m + q;
    const int npc = 1 + cs[cell + 1] - cs[cell];
    for (int pc = 0; pc < npc && pos < X1; ++pc) {
      int64_t len, seg_off = 0, loc_off = 0;
      int origin = p, in_stg = 0, wslot = -1;
      if (pc == 0) {
        len = ol[cell];
      } else {
        const Take& t = tk[pt[cs[cell] + pc - 1]];
        len = t.x;
        origin = t.g;
        seg_off = t.seg_off;
        in_stg = 1;
        loc_off = t.stg_off;
        wslot = t.slot;
      }
      const int64_t lo = pos > X0 ? pos : X0, hi = pos + len < X1 ? pos + len : X1;
      pos += len;
      if (hi <= lo) continue;
      const int64_t x = hi - lo, coff = lo - (pos - len);
      const bool staged = q != p;
      const int ci = (staged ? 0 : 2) + in_stg;
      if (EMIT) {
        const int fin = j * m + q, orig = i * m + origin;
        const int64_t src_off =
            in_stg ? loc_off + coff : w.send_off[(int64_t)lane * G + fin] + coff;
        const int64_t fin_off = w.recv_off[(int64_t)orig * G + fin] + seg_off + coff;
        const int ph = in_stg ? FAST_PH_FROM_STAGING : FAST_PH_DIRECT;
        const int sbuf = in_stg ? FAST_BUF_STAGING : FAST_BUF_SEND;
        fast_op o;
        if (!staged) {
          o = make_op(ph, s, lane, sbuf, src_off, proxy, FAST_BUF_RECV, fin_off, x);
        } else {
          o = make_op(ph, s, lane, sbuf, src_off, proxy, FAST_BUF_STAGING, stg, x);
          o.sig_slot = (int32_t)slot;
          fast_op r = make_op(FAST_PH_REDIST, s, proxy, FAST_BUF_STAGING, stg, fin,
                              FAST_BUF_RECV, fin_off, x);
          r.wait_slot = (int32_t)slot;
          ops[op_base + c[4]] = r;
        }
        if (in_stg) {
          o.wait_slot = wslot;
          o.wait_off = coff;
        }
        ops[op_base + c[ci]] = o;
      }
      if (staged) {
        stg += align16(x);
        slot += div_chunks(x, in.chunk, ch_shift);
        c[4] += 1;
      }
      c[ci] += 1;
    }
  }
  if (pos < X1) return false;  // the stream ran out before the window's end
  if (!EMIT) {
#pragma unroll
    for (int u = 0; u < 5; ++u) w.cnt[ix[u]] = c[u];
    w.stg_need[(int64_t)s * G + lane] = stg;
    w.slot_need[(int64_t)s * G + lane] = slot;
  }
  return true;
}

// Whole-CTA plan build.  `ws` holds par_ws_bytes(n, m, in.K); ops are written
// to out.ops directly.  Every thread of the block must call it.
__device__ __forceinline__ void plan_compile_par(const PlanIn& in, const PlanOut& out, void* ws) {
  __shared__ int s_flags;
  __shared__ int32_t s_nbal, s_nint, s_nstage;
  const int n = in.n, m = in.m, G = n * m, T = n * (n - 1), K = in.K, MT = max_takes(m);
  const int S = in.n_stages;
  const int tid = threadIdx.x, nt = blockDim.x;
  const ParWs w = par_carve(ws, n, m, K);
  const int64_t CH = in.chunk > 0 ? in.chunk : ((int64_t)1 << 20);
  const int ch_shift = (CH & (CH - 1)) == 0 ? __ffsll((long long)CH) - 1 : -1;
  PlanIn pin = in;
  pin.chunk = CH;
  if (tid == 0) s_flags = (S > 255 || S > K || m > FAST_MAX_GPUS_PER_SERVER) ? kParEarlyVal : 0;
  __syncthreads();
  if (s_flags) goto done;

  // ---- P1 segment offsets; P2 balance replay per tile; stage table ---------
  PLAN_STAMP(1);
  for (int g = tid; g < G; g += nt) {
    int64_t a = 0;
    for (int h = 0; h < G; ++h) {
      w.send_off[(int64_t)g * G + h] = a;
      a += in.D[(int64_t)g * G + h];
      if (h == g && in.send_self) a += in.send_self[g];
    }
  }
  for (int h = tid; h < G; h += nt) {
    int64_t a = 0;
    for (int g = 0; g < G; ++g) {
      w.recv_off[(int64_t)g * G + h] = a;
      a += in.D[(int64_t)g * G + h];
      if (g == h && in.send_self) a += in.send_self[h];
    }
    if (a > in.recv_cap) atomicOr(&s_flags, kParEarlyVal);
  }
  for (int x = tid; x < K * n; x += nt) w.inv[x] = -1;
  for (int t = tid; t < T; t += nt) {
    const int i = t / (n - 1), jj = t - i * (n - 1), j = jj < i ? jj : jj + 1;
    int64_t* ol = w.orig_len + (int64_t)t * m * m;
    int64_t sum = 0;
    for (int p = 0; p < m; ++p)
      for (int q = 0; q < m; ++q) {
        const int64_t v = in.D[(int64_t)(i * m + p) * G + j * m + q];
        ol[p * m + q] = v;
        sum += v;
      }
    w.tile_sum[t] = sum;
    Take* tk = w.takes + (int64_t)t * MT;
    const int ntk = replay_balance(ol, m, tk, MT);
    if (ntk < 0) {
      atomicOr(&s_flags, kParInvariant);
      w.ntakes[t] = 0;
      continue;
    }
    w.ntakes[t] = ntk;
    // givers and takers are disjoint rows (a giver's excess only shrinks, a
    // taker's deficit only fills), so the replayed tile holds every giver
    // cell's remaining original part; taker rows get their D back
    int32_t* cs = w.cell_start + (int64_t)t * (m * m + 1);
    for (int c = 0; c <= m * m; ++c) cs[c] = 0;
    for (int a = 0; a < ntk; ++a) cs[tk[a].h * m + tk[a].q + 1] += 1;
    for (int a = 0; a < ntk; ++a) {
      const int h = tk[a].h;
      for (int q = 0; q < m; ++q)
        ol[h * m + q] = in.D[(int64_t)(i * m + h) * G + j * m + q];
    }
    for (int c = 0; c < m * m; ++c) cs[c + 1] += cs[c];
    // pieces of cell c in take order: counting sort, cs[c] as fill cursor
    int32_t* pt = w.piece_take + (int64_t)t * MT;
    for (int a = 0; a < ntk; ++a) pt[cs[tk[a].h * m + tk[a].q]++] = a;
    for (int c = m * m; c > 0; --c) cs[c] = cs[c - 1];
    cs[0] = 0;
  }
  __syncthreads();
  if (s_flags) goto done;
  PLAN_STAMP(2);
  for (int t = tid; t < T; t += nt) w.take_pre[t] = w.ntakes[t];
  for (int x = tid; x < S * n; x += nt) {
    const int s = x / n, i = x - s * n, k = in.order[s];
    if (in.sbytes[(int64_t)k * n + i] <= 0) continue;
    const int j = in.perm[(int64_t)k * n + i];
    if (j == i || j >= n) atomicOr(&s_flags, kParInvariant);
    else w.inv[s * n + j] = i;
  }
  __syncthreads();
  {
    const int32_t nbal = block_exclusive_scan(w.take_pre, T);
    if (tid == 0) s_nbal = nbal;
  }
  if (s_flags) goto done;

  // ---- P3 balance staging + ops; intra counts; window starts ---------------
  PLAN_STAMP(3);
  for (int r = tid; r < G; r += nt) {
    const int i = r / m, hl = r - i * m;
    int64_t top = 0, st = 0;
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      const int tix = tile_index(n, i, j);
      Take* tk = w.takes + (int64_t)tix * MT;
      const int ntk = w.ntakes[tix];
      for (int a = 0; a < ntk; ++a) {
        if (tk[a].h != hl) continue;
        const int gi = i * m + tk[a].g, dst = j * m + tk[a].q;
        tk[a].stg_off = top;
        top = align16(top + tk[a].x);
        tk[a].slot = (int32_t)st;
        st += div_chunks(tk[a].x, CH, ch_shift);
        fast_op o = make_op(FAST_PH_BALANCE, 0, gi, FAST_BUF_SEND,
                            w.send_off[(int64_t)gi * G + dst] + tk[a].seg_off, r,
                            FAST_BUF_STAGING, tk[a].stg_off, tk[a].x);
        o.sig_slot = tk[a].slot;
        const int64_t pos = (int64_t)w.take_pre[tix] + a;
        if (pos < in.op_cap) out.ops[pos] = o;
      }
    }
    w.stg_top[r] = top;
    w.slot_top[r] = st;
    int32_t cnt = 0;  // intra-server direct ops of sender r
    for (int q = 0; q < m; ++q) {
      const int h = i * m + q;
      cnt += (h != r && in.D[(int64_t)r * G + h] > 0);
    }
    if (in.copy_self && in.send_self && in.send_self[r] > 0) ++cnt;  // own segment, local
    w.direct_pre[r] = cnt;
  }
  for (int x = tid; x < S * n; x += nt) {  // bytes of (i -> j) in earlier stages
    const int s = x / n, i = x - s * n;
    const int64_t b = in.sbytes[(int64_t)in.order[s] * n + i];
    if (b <= 0) continue;
    const int j = in.perm[(int64_t)in.order[s] * n + i];
    int64_t c0 = 0;
    for (int u = 0; u < s; ++u) {
      const int k = in.order[u];
      if (in.perm[(int64_t)k * n + i] == j) {
        const int64_t bu = in.sbytes[(int64_t)k * n + i];
        c0 += bu > 0 ? bu : 0;
      }
    }
    w.cs0[(int64_t)s * n + i] = c0;
  }
  for (int t = tid; t < T; t += nt) {  // every pair fully delivered (simulate.py:127-142)
    const int i = t / (n - 1), jj = t - i * (n - 1), j = jj < i ? jj : jj + 1;
    int64_t tot = 0;
    for (int s = 0; s < S; ++s) {
      const int k = in.order[s];
      const int64_t b = in.sbytes[(int64_t)k * n + i];
      if (b > 0 && in.perm[(int64_t)k * n + i] == j) tot += b;
    }
    if (tot != w.tile_sum[t]) atomicOr(&s_flags, kParInvariant);
  }
  for (int L = tid; L < 3 * K * 2 * G; L += nt) w.cnt[L] = 0;
  {
    const int32_t nint = block_exclusive_scan(w.direct_pre, G);
    if (tid == 0) s_nint = nint;
  }
  if (s_flags) goto done;

  // ---- P4 window walk (count) -----------------------------------------------
  PLAN_STAMP(4);
  for (int x = tid; x < S * G; x += nt) {
    const int s = x / G, lane = x - s * G;
    if (!stage_window<false>(pin, w, s, lane / m, lane % m, nullptr, 0, ch_shift))
      atomicOr(&s_flags, kParInvariant);
  }
  __syncthreads();
  if (s_flags) goto done;

  // ---- P5 proxy prefixes; op positions -------------------------------------
  PLAN_STAMP(5);
  for (int r = tid; r < G; r += nt) {
    const int j = r / m, p = r - j * m;
    int64_t top = w.stg_top[r], st = w.slot_top[r];
    for (int s = 0; s < S; ++s) {
      const int i = w.inv[s * n + j];
      if (i < 0) continue;
      const int64_t x = (int64_t)s * G + i * m + p;
      const int64_t ns = w.stg_need[x], nsl = w.slot_need[x];
      w.stg_need[x] = top;
      w.slot_need[x] = st;
      top += ns;
      st += nsl;
    }
    out.staging_used[r] = top;
    if (top > in.staging_cap || st > FAST_MAX_SLOTS) atomicOr(&s_flags, kParLateVal);
  }
  {
    const int32_t nstage = block_exclusive_scan(w.cnt, 3 * K * 2 * G);
    if (tid == 0) {
      s_nstage = nstage;
      if ((int64_t)s_nbal + s_nint + nstage > in.op_cap) atomicOr(&s_flags, kParOverflow);
    }
  }
  __syncthreads();
  if (s_flags) goto done;

  // ---- P6 intra-server ops; window walk (emit) ------------------------------
  PLAN_STAMP(6);
  for (int g = tid; g < G; g += nt) {
    const int i = g / m;
    int32_t at = s_nbal + w.direct_pre[g];
    for (int q = 0; q < m; ++q) {
      const int h = i * m + q;
      const int64_t len = h != g ? in.D[(int64_t)g * G + h]
                                 : (in.copy_self && in.send_self ? in.send_self[g] : 0);
      if (len > 0)
        out.ops[at++] = make_op(FAST_PH_DIRECT, FAST_STAGE_INTRA, g, FAST_BUF_SEND, w.send_off[(int64_t)g * G + h],
                                h, FAST_BUF_RECV, w.recv_off[(int64_t)g * G + h], len);
    }
  }
  for (int x = tid; x < S * G; x += nt) {
    const int s = x / G, lane = x - s * G;
    stage_window<true>(pin, w, s, lane / m, lane % m, out.ops, s_nbal + s_nint, ch_shift);
  }

done:
  PLAN_STAMP(7);
  __syncthreads();
  if (tid == 0) {
    const int f = s_flags;
    const int st = (f & kParEarlyVal)   ? FAST_EVALIDATION
                   : (f & kParInvariant) ? FAST_EINVARIANT
                   : (f & kParLateVal)   ? FAST_EVALIDATION
                   : (f & kParOverflow)  ? FAST_EINVARIANT
                                         : FAST_OK;
    *out.n_ops = st == FAST_OK ? s_nbal + s_nint + s_nstage : 0;
    *out.status = st;
  }
  PLAN_STAMP(8);
}

#endif  // __CUDACC__

}  // namespace fastplan
