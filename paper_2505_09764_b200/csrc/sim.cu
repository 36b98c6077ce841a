// sim.cu -- batched analytical cost model.
//
// One CTA per schedule (grid-stride over the batch).  Everything the
// reference computes per schedule in Python (simulate.py:107-242,
// spreadout.py:19-31, bounds.py:27-87) is recomputed here in the same IEEE
// double operation order, so each output is bit-identical:
//
//   t_balance      per (server, gpu) balance send / receive totals, max
//                  (intra_phase_time, simulate.py:69-90)      thread / GPU
//   t_intra        max row / col sum of any non-empty intra tile
//                  (simulate.py:93-104)                       thread / server
//   scale_out[k]   max edge bytes of sorted stage k over m    atomicMax / edge
//   redist[k]      worst row / col sum of the moved part of each pair's
//                  stage-k piece (split_deliveries, balance.py:177-207)
//   spreadout      shifted stages, server-level and demand modes
//   bounds         optimal / worst-case closed forms
//
// split_deliveries is order-free here: a non-final piece is
// floor(cell * r / T) (exact 128-bit product) and the final piece of a pair
// is cell - (sum of the non-final floors), so every non-final edge of every
// stage is handled by its own warp with one atomicAdd per cell, and each
// pair's final piece afterwards; the pair's final stage is the largest
// stage index that carries it (atomicMax).
#include <cuda_runtime.h>
#include <stdint.h>

#include "fastb200.h"

namespace {

constexpr int kSimThreads = 256;
constexpr int kSimWarps = kSimThreads / 32;
constexpr int kSimMaxM = 64;
// CTAs per launch: 4 per SM of the current device (persistent loop over
// schedules); the workspace is sized with the same figure
inline int sim_grid_max() {
  static int g = 0;
  if (!g) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        sms <= 0)
      sms = 148;  // no device (host-side sizing only): B200
    g = 4 * sms;
  }
  return g;
}
constexpr size_t kSimWsBudget = (size_t)2 << 30;

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

__host__ __device__ inline size_t sim_cta_bytes(int n, int m, int K) {
  const size_t P = (size_t)n * n;
  return align256(P * 4) + align256(P * 8) * 2 + align256(P * m * m * 8) +
         2 * align256((size_t)(K > 0 ? K : 1) * 8);
}

inline int sim_grid(int B, int n, int m, int K) {
  const size_t per = sim_cta_bytes(n, m, K);
  const int gmax = sim_grid_max();
  int g = B < gmax ? B : gmax;
  const size_t cap = kSimWsBudget / per;
  if ((size_t)g > cap) g = cap > 0 ? (int)cap : 1;
  return g > 0 ? g : 1;
}

__device__ __forceinline__ double step_cost(double nbytes, double bw, double wake) {
  return nbytes == 0.0 ? 0.0 : wake + nbytes / bw;  // simulate.py:58-66
}

// floor(a * b / d) exactly (a, b >= 0, d > 0, result fits: b <= d)
__device__ __forceinline__ uint64_t muldiv_floor(uint64_t a, uint64_t b, uint64_t d) {
  const uint64_t hi = __umul64hi(a, b), lo = a * b;
  if (hi == 0) return lo / d;
  const unsigned __int128 x = ((unsigned __int128)hi << 64) | lo;
  return (uint64_t)(x / d);
}

// Round-to-nearest-even double of x * 2^-scale given the exact integer
// x (< 2^128) and whether a non-zero remainder lies below it (sticky).
__device__ inline double round_u128(unsigned __int128 x, bool sticky, int scale) {
  const uint64_t hi = (uint64_t)(x >> 64);
  const int L = hi ? 128 - __clzll((long long)hi) : 64 - __clzll((long long)(uint64_t)x);
  if (L <= 53) return ldexp((double)(uint64_t)x, -scale);  // exact (sticky only when
                                                            // scale < 0 is impossible here)
  const int sh = L - 53;
  uint64_t mant = (uint64_t)(x >> sh);
  const unsigned __int128 rem = x & ((((unsigned __int128)1) << sh) - 1);
  const unsigned __int128 half = ((unsigned __int128)1) << (sh - 1);
  if (rem > half || (rem == half && (sticky || (mant & 1)))) mant += 1;
  return ldexp((double)mant, sh - scale);
}

// Python's int / int true division, correctly rounded (a >= 0, d > 0): the
// reference's st.max_edge_bytes() / m (simulate.py:146) and
// max(...) / m (simulate.py:222-224)
__device__ inline double int_div_rn(uint64_t a, uint64_t d) {
  if (a < (1ull << 53)) return (double)a / (double)d;  // both exact: one rounding
  const unsigned __int128 A = (unsigned __int128)a << 64;
  return round_u128(A / d, A % d != 0, 64);
}

// Python's float(int) for a non-negative int < 2^128 (round-half-even)
__device__ inline double u128_to_double(unsigned __int128 x) { return round_u128(x, false, 0); }

// Python 3.12's built-in sum() of floats (start 0): the first item is added
// to int 0 exactly, the rest with Neumaier's compensated summation, and the
// compensation is added at the end when non-zero and finite
// (CPython Python/bltinmodule.c builtin_sum_impl) -- simulate.py:239 sums
// the spreadout stage durations with it.
__device__ inline double py_sum(const double* x, int len) {
  if (len <= 0) return 0.0;
  double f = x[0], c = 0.0;
  for (int k = 1; k < len; ++k) {
    const double v = x[k];
    const double t = __dadd_rn(f, v);
    if (fabs(f) >= fabs(v))
      c = __dadd_rn(c, __dadd_rn(__dsub_rn(f, t), v));
    else
      c = __dadd_rn(c, __dadd_rn(__dsub_rn(v, t), f));
    f = t;
  }
  if (c != 0.0 && isfinite(c)) f = __dadd_rn(f, c);
  return f;
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, v, d);
    v = o > v ? o : v;
  }
  return v;
}

struct SimWs {
  int32_t* last;                 // [n*n] last sorted stage carrying the pair, -1
  unsigned long long* carried;   // [n*n] bytes the stages carry for the pair
  int64_t* tsum;                 // [n*n] table total
  unsigned long long* acc;       // [n*n][m*m] sum over the pair's deliveries of floor(cell*r/T)
  unsigned long long* worst;     // [K] redistribution bottleneck per stage
  unsigned long long* maxedge;   // [K] largest edge per stage
};

__device__ inline SimWs sim_carve(char* p, int n, int m, int K) {
  const size_t P = (size_t)n * n;
  SimWs w;
  w.last = (int32_t*)p; p += align256(P * 4);
  w.carried = (unsigned long long*)p; p += align256(P * 8);
  w.tsum = (int64_t*)p; p += align256(P * 8);
  w.acc = (unsigned long long*)p; p += align256(P * m * m * 8);
  w.worst = (unsigned long long*)p; p += align256((size_t)(K > 0 ? K : 1) * 8);
  w.maxedge = (unsigned long long*)p;
  return w;
}

// Moved-part row / column maxima of one piece of pair (i, j); the warp's
// lanes stride over the m*m cells.  Non-final: piece = floor(cell * r / T),
// accumulated into acc; final: piece = cell - acc (acc then holds every
// earlier delivery's floor -- the final one is never added).
__device__ inline unsigned long long piece_worst(const int64_t* bal, int G, int m, int i, int j,
                                                 uint64_t r, uint64_t T, bool final,
                                                 unsigned long long* acc,
                                                 unsigned long long* rc /*[2][kSimMaxM]*/,
                                                 int lane) {
  for (int c = lane; c < 2 * m; c += 32) rc[c < m ? c : kSimMaxM + c - m] = 0;
  __syncwarp();
  bool any = false;
  for (int c = lane; c < m * m; c += 32) {
    const int p = c / m, q = c - p * m;
    const uint64_t cell = (uint64_t)bal[(int64_t)(i * m + p) * G + j * m + q];
    uint64_t piece;
    if (final) {
      piece = cell - acc[c];
    } else {
      piece = muldiv_floor(cell, r, T);
      atomicAdd(&acc[c], (unsigned long long)piece);
    }
    if (p != q && piece != 0) {
      atomicAdd(&rc[p], (unsigned long long)piece);
      atomicAdd(&rc[kSimMaxM + q], (unsigned long long)piece);
      any = true;
    }
  }
  __syncwarp();
  unsigned long long w = 0;
  if (__any_sync(0xffffffffu, any)) {
    for (int c = lane; c < m; c += 32) {
      const unsigned long long a = rc[c], b = rc[kSimMaxM + c];
      w = a > w ? a : w;
      w = b > w ? b : w;
    }
    w = warp_max_u64(w);
  }
  __syncwarp();
  return w;  // 0 when the moved part is empty (the reference skips it)
}

__global__ void __launch_bounds__(kSimThreads)
    sim_kernel(fast_sim_in in, int B, int n, int m, fast_sim_topo tp, fast_sim_out out,
               char* ws_base, size_t ws_stride) {
  __shared__ unsigned long long s_rc[kSimWarps][2 * kSimMaxM];
  __shared__ int s_flags;
  __shared__ unsigned long long s_wbal, s_wintra, s_rowmax, s_colmax, s_offmax;
  __shared__ int s_ok;
  const int G = n * m, T = n * (n - 1), K = in.stage_stride, MS = in.move_slots;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double b1 = tp.scaleup_bw, b2 = tp.scaleout_bw, wake = tp.wakeup_delay;
  const SimWs w = sim_carve(ws_base + (size_t)blockIdx.x * ws_stride, n, m, K);
  const int P = n * n;
  for (int b = blockIdx.x; b < B; b += gridDim.x) {
    const int st_in = in.status ? in.status[b] : FAST_OK;
    if (st_in != FAST_OK) {
      if (tid == 0) out.status[b] = st_in;
      continue;
    }
    const int S = in.n_stages[b];
    const int64_t* bal = in.balanced + (int64_t)b * G * G;
    const int64_t* srv = in.server + (int64_t)b * P;
    const int32_t* order = in.stage_order + (int64_t)b * K;
    const int64_t* wgt = in.stage_weight + (int64_t)b * K;
    const uint8_t* perm = in.stage_perm + (int64_t)b * K * n;
    const int64_t* sbytes = in.stage_bytes + (int64_t)b * K * n;
    if (tid == 0) {
      s_flags = 0;
      s_wbal = s_wintra = s_rowmax = s_colmax = s_offmax = 0;
      s_ok = 1;
    }
    for (int x = tid; x < P; x += kSimThreads) {
      w.last[x] = -1;
      w.carried[x] = 0;
    }
    for (int x = tid; x < P * m * m; x += kSimThreads) w.acc[x] = 0;
    for (int x = tid; x < S; x += kSimThreads) w.worst[x] = w.maxedge[x] = 0;
    __syncthreads();
    // stages ascending (simulate.py:114-116)
    for (int s = 1 + tid; s < S; s += kSimThreads)
      if (wgt[order[s - 1]] > wgt[order[s]]) atomicOr(&s_flags, 1);
    for (int x = tid; x < P; x += kSimThreads) {  // pair table totals
      const int i = x / n, j = x - i * n;
      int64_t t = 0;
      if (i != j)
        for (int c = 0; c < m * m; ++c) t += bal[(int64_t)(i * m + c / m) * G + j * m + c % m];
      w.tsum[x] = t;
    }
    for (int x = tid; x < S * n; x += kSimThreads) {  // stage edges
      const int s = x / n, i = x - s * n, raw = order[s];
      const int64_t sb = sbytes[(int64_t)raw * n + i];
      if (sb == 0) continue;
      const int j = perm[(int64_t)raw * n + i];
      const unsigned long long r = sb > 0 ? (unsigned long long)sb : 0ull;
      atomicMax(&w.maxedge[s], r);
      if (j == i || j >= n) {
        atomicOr(&s_flags, 2);  // stage edge for an unknown server pair
      } else {
        atomicMax(&w.last[i * n + j], s);
        atomicAdd(&w.carried[i * n + j], r);
      }
    }
    __syncthreads();
    for (int x = tid; x < P; x += kSimThreads) {  // simulate.py:127-142
      const int i = x / n, j = x - i * n;
      if (i == j) continue;
      const bool has = w.last[x] >= 0;
      if (has && (int64_t)w.carried[x] != w.tsum[x]) atomicOr(&s_flags, 2);
      if (!has && w.tsum[x] > 0) atomicOr(&s_flags, 2);
    }
    __syncthreads();
    if (s_flags) {
      if (tid == 0) out.status[b] = (s_flags & 1) ? FAST_EVALIDATION : FAST_EINVARIANT;
      __syncthreads();
      continue;
    }
    // non-final pieces: one warp per stage edge
    for (int x = wid; x < S * n; x += kSimWarps) {
      const int s = x / n, i = x - s * n, raw = order[s];
      const int64_t sb = sbytes[(int64_t)raw * n + i];
      if (sb == 0) continue;
      const int j = perm[(int64_t)raw * n + i];
      const int pr = i * n + j;
      const uint64_t Tt = (uint64_t)w.tsum[pr];
      if (Tt == 0 || w.last[pr] == s) continue;
      const unsigned long long wv =
          piece_worst(bal, G, m, i, j, sb > 0 ? (uint64_t)sb : 0, Tt, false,
                      w.acc + (int64_t)pr * m * m, s_rc[wid], lane);
      if (lane == 0 && wv) atomicMax(&w.worst[s], wv);
    }
    __syncthreads();
    // final pieces: one warp per pair
    for (int pr = wid; pr < P; pr += kSimWarps) {
      const int i = pr / n, j = pr - i * n;
      const int s = w.last[pr];
      if (i == j || s < 0 || w.tsum[pr] == 0) continue;
      const int64_t sb = sbytes[(int64_t)order[s] * n + i];
      const unsigned long long wv =
          piece_worst(bal, G, m, i, j, sb > 0 ? (uint64_t)sb : 0, (uint64_t)w.tsum[pr], true,
                      w.acc + (int64_t)pr * m * m, s_rc[wid], lane);
      if (lane == 0 && wv) atomicMax(&w.worst[s], wv);
    }
    __syncthreads();
    for (int s = tid; s < S; s += kSimThreads) {
      out.scale_out[(int64_t)b * K + s] = step_cost(int_div_rn(w.maxedge[s], m), b2, wake);
      out.redistribution[(int64_t)b * K + s] = step_cost((double)w.worst[s], b1, wake);
    }
    // balance moves: per (server, gpu) send / receive totals
    for (int x = tid; x < G; x += kSimThreads) {
      const int i = x / m, g = x - i * m;
      unsigned long long snd = 0, rcv = 0;
      for (int j = 0; j < n; ++j) {
        if (j == i) continue;
        const int t = i * (n - 1) + (j < i ? j : j - 1);
        const int cnt = in.move_count[(int64_t)b * T + t];
        const fast_move* mv = in.moves + ((int64_t)b * T + t) * MS;
        for (int u = 0; u < cnt; ++u) {
          if (mv[u].from_gpu == g) snd += (unsigned long long)mv[u].bytes;
          if (mv[u].to_gpu == g) rcv += (unsigned long long)mv[u].bytes;
        }
      }
      const unsigned long long v = snd > rcv ? snd : rcv;
      if (v) atomicMax(&s_wbal, v);
    }
    for (int i = tid; i < n; i += kSimThreads) {
      // intra tile (i, i): simulate.py:93-104
      unsigned long long wv = 0;
      bool any = false;
      for (int p = 0; p < m; ++p) {
        unsigned long long rs = 0, cs = 0;
        for (int q = 0; q < m; ++q) {
          const int64_t a = bal[(int64_t)(i * m + p) * G + i * m + q];
          const int64_t c = bal[(int64_t)(i * m + q) * G + i * m + p];
          any |= a != 0;
          rs += (unsigned long long)a;
          cs += (unsigned long long)c;
        }
        wv = rs > wv ? rs : wv;
        wv = cs > wv ? cs : wv;
      }
      if (any) atomicMax(&s_wintra, wv);
      // bounds.py: off-diagonal row / column sums, largest entry, S_i test
      unsigned long long row = 0, col = 0, mx = 0;
      for (int j = 0; j < n; ++j) {
        if (j == i) continue;
        const unsigned long long a = (unsigned long long)srv[i * n + j];
        row += a;
        col += (unsigned long long)srv[j * n + i];
        mx = a > mx ? a : mx;
      }
      atomicMax(&s_rowmax, row);
      atomicMax(&s_colmax, col);
      atomicMax(&s_offmax, mx);
      // numpy int64 product (wraps like the reference's array arithmetic)
      const long long lhs = (long long)((unsigned long long)n * (unsigned long long)srv[i * n + i]);
      if (lhs > (long long)row) atomicAnd(&s_ok, 0);
    }
    // spreadout: shift k moves every server's demand for server (s + k) mod n
    for (int k = 1 + tid; k < n; k += kSimThreads) {
      unsigned long long gov = 0, gd = 0;
      for (int s = 0; s < n; ++s) {
        const int d = (s + k) % n;
        const unsigned long long a = (unsigned long long)srv[s * n + d];
        gov = a > gov ? a : gov;
        if (in.demand) {
          const int64_t* D = in.demand + (int64_t)b * G * G;
          bool any = false;
          unsigned long long wv = 0;
          for (int p = 0; p < m; ++p) {
            unsigned long long rs = 0, cs = 0;
            for (int q = 0; q < m; ++q) {
              const int64_t v = D[(int64_t)(s * m + p) * G + d * m + q];
              any |= v != 0;
              rs += (unsigned long long)v;
              cs += (unsigned long long)D[(int64_t)(s * m + q) * G + d * m + p];
            }
            wv = rs > wv ? rs : wv;
            wv = cs > wv ? cs : wv;
          }
          if (any) gd = wv > gd ? wv : gd;
        }
      }
      const int64_t o = (int64_t)b * (n - 1) + k - 1;
      if (out.so_weight) out.so_weight[o] = (int64_t)gov;
      out.so_server[o] = step_cost(int_div_rn(gov, m), b2, wake);
      if (in.demand && out.so_demand) out.so_demand[o] = step_cost((double)gd, b2, wake);
    }
    __syncthreads();
    if (tid == 0) {
      const double t_bal = step_cost((double)s_wbal, b1, wake);
      const double t_in = step_cost((double)s_wintra, b1, wake);
      out.t_balance[b] = t_bal;
      out.t_intra[b] = t_in;
      int st = FAST_OK;
      double total;
      if (S == 0) {
        total = t_bal + t_in;
      } else {
        const double* so = out.scale_out + (int64_t)b * K;
        const double* rd = out.redistribution + (int64_t)b * K;
        total = t_bal + fmax(so[0], t_in);
        for (int k = 1; k < S; ++k) total += fmax(so[k], rd[k - 1]);
        total += rd[S - 1];
        const double floor_t = (double)in.common_sum[b] / ((double)m * b2);
        if (total < floor_t * (1 - 1e-12)) st = FAST_EINVARIANT;
      }
      out.total[b] = total;
      const unsigned long long mrc = s_rowmax > s_colmax ? s_rowmax : s_colmax;
      out.t_optimal[b] = (double)mrc / ((double)m * b2);
      const double t0 =
          u128_to_double((unsigned __int128)(m - 1) * s_rowmax) / ((double)m * b1);
      const double t1 = (double)s_rowmax / ((double)n * b1);
      const double t2 = (double)mrc / ((double)m * b2);
      const double t3 = (double)s_offmax / ((double)m * b1);
      out.t_worstcase[b] = t0 + t1 + t2 + t3;
      out.assumption_ok[b] = s_ok;
      out.so_total[2 * (int64_t)b] = py_sum(out.so_server + (int64_t)b * (n - 1), n - 1);
      out.so_total[2 * (int64_t)b + 1] =
          in.demand && out.so_demand ? py_sum(out.so_demand + (int64_t)b * (n - 1), n - 1) : 0.0;
      out.status[b] = st;
    }
    __syncthreads();
  }
}

}  // namespace

extern "C" {

size_t fast_sim_workspace_bytes(int B, int n, int m, int stage_stride) {
  if (B <= 0 || n < 1 || m < 1) return 256;
  return (size_t)sim_grid(B, n, m, stage_stride) * sim_cta_bytes(n, m, stage_stride);
}

int fast_simulate_batch(const fast_sim_in* in, int B, int n, int m, const fast_sim_topo* topo,
                        fast_sim_out* out, void* stream) {
  if (!in || !topo || !out || B < 0 || n < 1 || m < 1 || m > kSimMaxM || in->stage_stride < 0 ||
      in->move_slots < 0)
    return FAST_EVALIDATION;
  if (!(topo->scaleup_bw > 0) || !(topo->scaleout_bw > 0) || topo->wakeup_delay < 0)
    return FAST_EVALIDATION;
  if (B == 0) return FAST_OK;
  const int grid = sim_grid(B, n, m, in->stage_stride);
  sim_kernel<<<grid, kSimThreads, 0, (cudaStream_t)stream>>>(
      *in, B, n, m, *topo, *out, (char*)out->workspace, sim_cta_bytes(n, m, in->stage_stride));
  return cudaGetLastError() == cudaSuccess ? FAST_OK : FAST_ECUDA;
}

}  // extern "C"
