// moe.cu -- MoE dispatch front-end on B200 (sm_100a): the traffic-matrix
// builder and token pack/unpack around the FAST alltoallv (BASELINE config
// 3).  None of this exists in the reference ("MoE dispatch
// front-end ... absent"); the paper obtains the matrix from Megatron's
// all-gather of per-expert token counts.
//
//   moe_gate_kernel        deterministic top-k gating: SplitMix64 draws
//                          compared against integer CDF thresholds (exact,
//                          identical to the numpy oracle)
//   moe_route_local_kernel stable counting-sort ranks: __match_any_sync per
//                          warp, per-block expert totals
//   moe_route_scan_kernel  block bases, counts, segment offsets, demand row
//   moe_pack_kernel        one warp per token: the row is read once (16-B
//                          vectors) and written to each of its k destination
//                          rows of the send buffer (grouped by destination,
//                          stable token order)
//   moe_unpack_self_kernel the own segment goes from the send buffer into the
//                          gap the executor leaves at the self slot of the
//                          receive buffer, which then IS the expert input
//                          (source-major, like all_to_all_single)
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fastb200.h"

namespace {

constexpr int kRouteThreads = 1024;
constexpr int kMaxExperts = 64;

__device__ __forceinline__ uint64_t splitmix(uint64_t seed, uint64_t k) {
  uint64_t z = seed + (k + 1) * 0x9E3779B97F4A7C15ull;  // rng.py:20-44
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// searchsorted(thr, r, side="right") == #{i : thr[i] <= r}
__device__ __forceinline__ int count_le(const uint64_t* thr, int E, uint64_t r) {
  int c = 0;
  for (int i = 0; i < E; ++i) c += thr[i] <= r ? 1 : 0;
  return c;
}

__global__ void moe_gate_kernel(int T, uint64_t seed, int E, const uint64_t* __restrict__ thr,
                                const uint64_t* __restrict__ thr2, int32_t* __restrict__ topk) {
  __shared__ uint64_t s_thr[kMaxExperts], s_thr2[kMaxExperts * kMaxExperts];
  for (int i = threadIdx.x; i < E; i += blockDim.x) s_thr[i] = thr[i];
  for (int i = threadIdx.x; i < E * E; i += blockDim.x) s_thr2[i] = thr2[i];
  __syncthreads();
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
    const uint64_t r1 = splitmix(seed, (uint64_t)t) >> 32;
    const uint64_t r2 = splitmix(seed, (uint64_t)T + t) >> 32;
    const int e1 = count_le(s_thr, E, r1);
    const int e2 = count_le(s_thr2 + e1 * E, E, r2);
    topk[2 * t] = e1;
    topk[2 * t + 1] = e2;
  }
}

// entries i = t*k + j in token order; pos[i] <- rank of i among the block's
// entries with the same destination; blk[b][e] <- block totals
// Router-provided top-k ids are validated here: an id outside [0, E) is
// ignored by the histogram and raises `bad` (the scan then poisons the
// demand row, so the alltoallv fails validation instead of dropping tokens).
__global__ void __launch_bounds__(kRouteThreads)
    moe_route_local_kernel(const int32_t* __restrict__ topk, int N, int E,
                           int32_t* __restrict__ pos, int32_t* __restrict__ blk,
                           int32_t* __restrict__ bad) {
  __shared__ int32_t wcnt[kRouteThreads / 32][kMaxExperts];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < (kRouteThreads / 32) * E; i += blockDim.x) (&wcnt[0][0])[(i / E) * kMaxExperts + i % E] = 0;
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + tid;
  int e = i < N ? topk[i] : -1;
  if (i < N && (e < 0 || e >= E)) {
    atomicOr(bad, 1);
    e = -1;
    pos[i] = -1;
  }
  const unsigned peers = __match_any_sync(0xffffffffu, e);
  const int lrank = __popc(peers & ((1u << lane) - 1u));
  if (e >= 0 && lrank == 0) wcnt[warp][e] = __popc(peers);
  __syncthreads();
  // exclusive prefix over warps, per expert; block total
  if (tid < E) {
    int run = 0;
    for (int w = 0; w < kRouteThreads / 32; ++w) {
      const int c = wcnt[w][tid];
      wcnt[w][tid] = run;
      run += c;
    }
    blk[(int64_t)blockIdx.x * E + tid] = run;
  }
  __syncthreads();
  if (e >= 0) pos[i] = wcnt[warp][e] + lrank;
}

// one warp per expert column of blk: 32 block totals per round loaded in
// parallel, warp exclusive scan + carry (no dependent global-load chain)
constexpr int kScanThreads = 1024;
__global__ void __launch_bounds__(kScanThreads)
    moe_route_scan_kernel(int nblocks, int E, int L, int64_t row_bytes, int32_t* __restrict__ blk,
                          const int32_t* __restrict__ bad, int64_t* __restrict__ counts,
                          int64_t* __restrict__ seg_rows, int64_t* __restrict__ demand_row) {
  __shared__ int64_t s_cnt[kMaxExperts];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = warp; e < E; e += kScanThreads / 32) {
    int64_t run = 0;
    for (int b0 = 0; b0 < nblocks; b0 += 32) {
      const int b = b0 + lane;
      const int c = b < nblocks ? blk[(int64_t)b * E + e] : 0;
      int x = c;  // inclusive warp scan
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
      }
      if (b < nblocks) blk[(int64_t)b * E + e] = (int32_t)(run + x - c);  // block base
      run += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) {
      s_cnt[e] = run;
      counts[e] = run;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t a = 0;
    for (int x = 0; x < E; ++x) {
      seg_rows[x] = a;
      a += s_cnt[x];
    }
    // demand row per destination rank: its L consecutive experts
    const bool poisoned = *bad != 0;
    for (int r = 0; r < E / L; ++r) {
      int64_t c = 0;
      for (int x = r * L; x < (r + 1) * L; ++x) c += s_cnt[x];
      demand_row[r] = poisoned ? -1 : c * row_bytes;
    }
  }
}

__device__ __forceinline__ uint4 ldg_nc(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void stg_na(uint4* p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// one warp per token; row_vec = row_bytes / 16 (row_bytes % 16 == 0)
template <int K>
__global__ void __launch_bounds__(256)
    moe_pack_kernel(const uint4* __restrict__ tokens, int T, int64_t row_vec,
                    const int32_t* __restrict__ topk, const int32_t* __restrict__ pos,
                    const int32_t* __restrict__ blkbase, int E,
                    const int64_t* __restrict__ seg_rows, uint4* __restrict__ send) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp; t < T; t += nwarps) {
    uint4* dst[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int i = t * K + j;
      const int e = topk[i];
      // an invalid id (rejected by the route) is not written anywhere
      dst[j] = (e < 0 || e >= E)
                   ? nullptr
                   : send + (seg_rows[e] + blkbase[(int64_t)(i / kRouteThreads) * E + e] + pos[i]) *
                                row_vec;
    }
    const uint4* src = tokens + (int64_t)t * row_vec;
    constexpr int U = 4;
    int64_t v = lane;
    for (; v + (U - 1) * 32 < row_vec; v += U * 32) {
      uint4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) x[u] = ldg_nc(src + v + u * 32);
#pragma unroll
      for (int j = 0; j < K; ++j)
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (dst[j]) stg_na(dst[j] + v + u * 32, x[u]);
    }
    for (; v < row_vec; v += 32) {
      const uint4 x = ldg_nc(src + v);
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (dst[j]) stg_na(dst[j] + v, x);
    }
  }
}

// fused pack -> send: instead of materialising the send buffer, record for
// every send row the token it holds (row_src[row] = t, the pack kernel's
// destination map inverted); the executor then reads token rows through it
template <int K>
__global__ void moe_rowmap_kernel(int T, const int32_t* __restrict__ topk,
                                  const int32_t* __restrict__ pos,
                                  const int32_t* __restrict__ blkbase, int E,
                                  const int64_t* __restrict__ seg_rows,
                                  int32_t* __restrict__ row_src) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < T * K; i += gridDim.x * blockDim.x) {
    const int e = topk[i];
    if (e < 0 || e >= E) continue;  // rejected by the route
    row_src[seg_rows[e] + blkbase[(int64_t)(i / kRouteThreads) * E + e] + pos[i]] = i / K;
  }
}

// own segment of the virtual send buffer (rows row_src[s0 ...]) -> the self
// slot of the receive buffer; one warp per row
__global__ void moe_unpack_self_rows_kernel(const int64_t* __restrict__ D,
                                            const int64_t* __restrict__ self_bytes, int G,
                                            int rank, const uint4* __restrict__ tokens,
                                            const int32_t* __restrict__ row_src, int64_t row_vec,
                                            uint8_t* __restrict__ recv) {
  int64_t soff = 0, roff = 0;
  for (int h = 0; h < rank; ++h) soff += D[(int64_t)rank * G + h];
  for (int g = 0; g < rank; ++g) roff += D[(int64_t)g * G + rank];
  const int64_t RB = row_vec * 16;
  const int64_t s0 = soff / RB, nrows = self_bytes[rank] / RB;
  uint4* d = reinterpret_cast<uint4*>(recv + roff);
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < nrows; r += nwarps) {
    const uint4* src = tokens + (int64_t)row_src[s0 + r] * row_vec;
    for (int64_t v = lane; v < row_vec; v += 32) stg_na(d + r * row_vec + v, ldg_nc(src + v));
  }
}

// own segment: send[sum_{h<rank} D[rank][h] ...] -> recv[sum_{g<rank} D[g][rank] ...]
__global__ void moe_unpack_self_kernel(const int64_t* __restrict__ D,
                                       const int64_t* __restrict__ self_bytes, int G, int rank,
                                       const uint8_t* __restrict__ send, uint8_t* __restrict__ recv) {
  int64_t soff = 0, roff = 0;
  for (int h = 0; h < rank; ++h) soff += D[(int64_t)rank * G + h];
  for (int g = 0; g < rank; ++g) roff += D[(int64_t)g * G + rank];
  const int64_t len = self_bytes[rank];
  const uint8_t* s = send + soff;
  uint8_t* d = recv + roff;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  if ((((uintptr_t)s | (uintptr_t)d) & 15) == 0) {
    const int64_t nv = len >> 4;
    for (int64_t v = tid; v < nv; v += nt)
      stg_na(reinterpret_cast<uint4*>(d) + v, ldg_nc(reinterpret_cast<const uint4*>(s) + v));
    for (int64_t b = (nv << 4) + tid; b < len; b += nt) d[b] = s[b];
  } else {
    for (int64_t b = tid; b < len; b += nt) d[b] = s[b];
  }
}

// Combine (the reverse alltoallv's receive side): token t's output is
// sum_j w[t][j] * row(t, j) over its k experts, in j order with explicit
// round-to-nearest fp32 multiply and add (no FMA contraction, so the numpy
// oracle reproduces it bit for bit), then bf16 round-to-nearest-even.
// row(t, j) of expert e sits at row seg_rows[e] + blkbase + pos of the
// combine receive buffer (segments by expert, forward pack order); the own
// expert's rows were never sent and are read from the expert output buffer.
__device__ __forceinline__ void bf16x8_to_f32(const uint4 v, float (&f)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

template <int K>
__global__ void __launch_bounds__(256)
    moe_combine_kernel(const uint8_t* __restrict__ comb_recv,
                       const uint8_t* __restrict__ expert_out, const int64_t* __restrict__ Dfwd,
                       int G, int me, int T, int64_t row_vec, const int32_t* __restrict__ topk,
                       const int32_t* __restrict__ pos, const int32_t* __restrict__ blkbase,
                       int E, int L, const int64_t* __restrict__ seg_rows,
                       const float* __restrict__ weights, uint4* __restrict__ out) {
  __shared__ int64_t s_self_off;
  if (threadIdx.x == 0) {
    int64_t o = 0;  // self segment of the expert output (forward recv layout)
    for (int g = 0; g < me; ++g) o += Dfwd[(int64_t)g * G + me];
    s_self_off = o;
  }
  const int64_t self_row0 = seg_rows[me * L];  // first send row of my experts
  __syncthreads();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int64_t RB = row_vec * 16;
  for (int t = warp; t < T; t += nwarps) {
    const uint4* src[K];
    float w[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int i = t * K + j;
      const int e = topk[i];
      const int64_t r = blkbase[(int64_t)(i / kRouteThreads) * E + e] + pos[i];
      src[j] = (e / L == me)
                   ? reinterpret_cast<const uint4*>(expert_out + s_self_off +
                                                    (seg_rows[e] - self_row0 + r) * RB)
                   : reinterpret_cast<const uint4*>(comb_recv + (seg_rows[e] + r) * RB);
      w[j] = weights[i];
    }
    for (int64_t v = lane; v < row_vec; v += 32) {
      float acc[8];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        float x[8];
        bf16x8_to_f32(ldg_nc(src[j] + v), x);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float p = __fmul_rn(w[j], x[q]);
          acc[q] = j == 0 ? p : __fadd_rn(acc[q], p);
        }
      }
      uint32_t o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(acc[2 * q], acc[2 * q + 1]);
        o[q] = *reinterpret_cast<const uint32_t*>(&h);
      }
      out[(int64_t)t * row_vec + v] = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

}  // namespace

extern "C" {

size_t fast_moe_route_workspace_bytes(int T, int k, int E) {
  if (T < 0 || k < 1 || E < 1) return 0;
  const int64_t N = (int64_t)T * k;
  const int64_t nb = (N + kRouteThreads - 1) / kRouteThreads;
  return (size_t)((nb > 0 ? nb : 1) * E * 4) + 16;  // + the invalid-id flag
}

static int32_t* route_bad_flag(void* workspace, int T, int k, int E) {
  return (int32_t*)((char*)workspace + fast_moe_route_workspace_bytes(T, k, E) - 16);
}

int fast_moe_gate(int T, uint64_t seed, int E, const uint64_t* thr, const uint64_t* thr2,
                  int32_t* topk, void* stream) {
  if (T < 0 || E < 2 || E > kMaxExperts || !thr || !thr2 || !topk) return FAST_EVALIDATION;
  if (T == 0) return FAST_OK;
  const int blocks = (T + 255) / 256 < 4 * sm_count() ? (T + 255) / 256 : 4 * sm_count();
  moe_gate_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(T, seed, E, thr, thr2, topk);
  return cudaGetLastError() == cudaSuccess ? FAST_OK : FAST_ECUDA;
}

int fast_moe_route_ex(const int32_t* topk, int T, int k, int E, int experts_per_rank,
                      int64_t row_bytes, int32_t* pos, int64_t* counts, int64_t* seg_rows,
                      int64_t* demand_row, void* workspace, void* stream) {
  const int L = experts_per_rank;
  if (T < 0 || k < 1 || E < 1 || E > kMaxExperts || L < 1 || E % L || row_bytes < 0 ||
      !counts || !seg_rows || !demand_row || !workspace)
    return FAST_EVALIDATION;
  cudaStream_t s = (cudaStream_t)stream;
  const int N = T * k;
  const int nb = N > 0 ? (N + kRouteThreads - 1) / kRouteThreads : 0;
  int32_t* bad = route_bad_flag(workspace, T, k, E);
  if (cudaMemsetAsync(bad, 0, 4, s) != cudaSuccess) return FAST_ECUDA;
  if (nb > 0)
    moe_route_local_kernel<<<nb, kRouteThreads, 0, s>>>(topk, N, E, pos, (int32_t*)workspace,
                                                        bad);
  moe_route_scan_kernel<<<1, kScanThreads, 0, s>>>(nb, E, L, row_bytes, (int32_t*)workspace, bad,
                                                   counts, seg_rows, demand_row);
  return cudaGetLastError() == cudaSuccess ? FAST_OK : FAST_ECUDA;
}

int fast_moe_route(const int32_t* topk, int T, int k, int E, int64_t row_bytes, int32_t* pos,
                   int64_t* counts, int64_t* seg_rows, int64_t* demand_row, void* workspace,
                   void* stream) {
  return fast_moe_route_ex(topk, T, k, E, 1, row_bytes, pos, counts, seg_rows, demand_row,
                           workspace, stream);
}

int fast_moe_pack(const void* tokens, int T, int k, int64_t row_bytes, const int32_t* topk,
                  const int32_t* pos, const void* workspace, int E, const int64_t* seg_rows,
                  void* send, void* stream) {
  if (T < 0 || (k != 1 && k != 2 && k != 4 && k != 8) || row_bytes <= 0 || (row_bytes & 15) ||
      ((uintptr_t)tokens & 15) || ((uintptr_t)send & 15))
    return FAST_EVALIDATION;
  if (T == 0) return FAST_OK;
  const int threads = 256;
  int blocks = (int)(((int64_t)T * 32 + threads - 1) / threads);
  if (blocks > 8 * sm_count()) blocks = 8 * sm_count();
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t rv = row_bytes / 16;
  const uint4* tk = (const uint4*)tokens;
  uint4* sd = (uint4*)send;
  const int32_t* bb = (const int32_t*)workspace;
  switch (k) {
    case 1: moe_pack_kernel<1><<<blocks, threads, 0, s>>>(tk, T, rv, topk, pos, bb, E, seg_rows, sd); break;
    case 2: moe_pack_kernel<2><<<blocks, threads, 0, s>>>(tk, T, rv, topk, pos, bb, E, seg_rows, sd); break;
    case 4: moe_pack_kernel<4><<<blocks, threads, 0, s>>>(tk, T, rv, topk, pos, bb, E, seg_rows, sd); break;
    default: moe_pack_kernel<8><<<blocks, threads, 0, s>>>(tk, T, rv, topk, pos, bb, E, seg_rows, sd); break;
  }
  return cudaGetLastError() == cudaSuccess ? FAST_OK : FAST_ECUDA;
}

int fast_moe_unpack_self(const int64_t* D, const int64_t* self_bytes, int G, int rank,
                         const void* send, void* recv, void* stream) {
  if (!D || !self_bytes || G < 1 || rank < 0 || rank >= G || !send || !recv)
    return FAST_EVALIDATION;
  moe_unpack_self_kernel<<<2 * sm_count(), 512, 0, (cudaStream_t)stream>>>(
      D, self_bytes, G, rank, (const uint8_t*)send, (uint8_t*)recv);
  return cudaGetLastError() == cudaSuccess ? FAST_OK : FAST_ECUDA;
}

int fast_moe_rowmap(int T, int k, const int32_t* topk, const int32_t* pos,
                    const void* workspace, int E, const int64_t* seg_rows, int32_t* row_src,
                    void* stream) {
  if (T < 0 || (k != 1 && k != 2 && k != 4 && k != 8) || E < 1 || E > kMaxExperts || !topk ||
      !pos || !workspace || !seg_rows || !row_src)
    return FAST_EVALIDATION;
  if (T == 0) return FAST_OK;
  const int64_t N = (int64_t)T * k;
  int blocks = (int)((N + 255) / 256);
  if (blocks > 4 * sm_count()) blocks = 4 * sm_count();
  cudaStream_t s = (cudaStream_t)stream;
  const int32_t* bb = (const int32_t*)workspace;
  switch (k) {
    case 1: moe_rowmap_kernel<1><<<blocks, 256, 0, s>>>(T, topk, pos, bb, E, seg_rows, row_src); break;
    case 2: moe_rowmap_kernel<2><<<blocks, 256, 0, s>>>(T, topk, pos, bb, E, seg_rows, row_src); break;
    case 4: moe_rowmap_kernel<4><<<blocks, 256, 0, s>>>(T, topk, pos, bb, E, seg_rows, row_src); break;
    default: moe_rowmap_kernel<8><<<blocks, 256, 0, s>>>(T, topk, pos, bb, E, seg_rows, row_src); break;
  }
  return cudaGetLastError() == cudaSuccess ? FAST_OK : FAST_ECUDA;
}

int fast_moe_unpack_self_rows(const int64_t* D, const int64_t* self_bytes, int G, int rank,
                              const void* tokens, const int32_t* row_src, int64_t row_bytes,
                              void* recv, void* stream) {
  if (!D || !self_bytes || G < 1 || rank < 0 || rank >= G || !tokens || !row_src || !recv ||
      row_bytes <= 0 || (row_bytes & 15) || ((uintptr_t)tokens & 15) || ((uintptr_t)recv & 15))
    return FAST_EVALIDATION;
  moe_unpack_self_rows_kernel<<<2 * sm_count(), 512, 0, (cudaStream_t)stream>>>(
      D, self_bytes, G, rank, (const uint4*)tokens, row_src, row_bytes / 16, (uint8_t*)recv);
  return cudaGetLastError() == cudaSuccess ? FAST_OK : FAST_ECUDA;
}

int fast_moe_combine(const void* comb_recv, const void* expert_out, const int64_t* Dfwd, int G,
                     int rank, int T, int k, int64_t row_bytes, const int32_t* topk,
                     const int32_t* pos, const void* workspace, int E, const int64_t* seg_rows,
                     const float* weights, void* out, void* stream) {
  return fast_moe_combine_ex(comb_recv, expert_out, Dfwd, G, rank, T, k, row_bytes, topk, pos,
                             workspace, E, 1, seg_rows, weights, out, stream);
}

int fast_moe_combine_ex(const void* comb_recv, const void* expert_out, const int64_t* Dfwd,
                        int G, int rank, int T, int k, int64_t row_bytes, const int32_t* topk,
                        const int32_t* pos, const void* workspace, int E, int experts_per_rank,
                        const int64_t* seg_rows, const float* weights, void* out, void* stream) {
  const int L = experts_per_rank;
  if (T < 0 || (k != 1 && k != 2 && k != 4 && k != 8) || row_bytes <= 0 || (row_bytes & 15) ||
      !comb_recv || !expert_out || !Dfwd || !topk || !pos || !workspace || !seg_rows ||
      !weights || !out || rank < 0 || rank >= G || ((uintptr_t)out & 15) || L < 1 ||
      E != G * L)
    return FAST_EVALIDATION;
  if (T == 0) return FAST_OK;
  int blocks = (int)(((int64_t)T * 32 + 255) / 256);
  if (blocks > 8 * sm_count()) blocks = 8 * sm_count();
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t rv = row_bytes / 16;
  const uint8_t* cr = (const uint8_t*)comb_recv;
  const uint8_t* eo = (const uint8_t*)expert_out;
  const int32_t* bb = (const int32_t*)workspace;
  uint4* o = (uint4*)out;
  switch (k) {
    case 1: moe_combine_kernel<1><<<blocks, 256, 0, s>>>(cr, eo, Dfwd, G, rank, T, rv, topk, pos, bb, E, L, seg_rows, weights, o); break;
    case 2: moe_combine_kernel<2><<<blocks, 256, 0, s>>>(cr, eo, Dfwd, G, rank, T, rv, topk, pos, bb, E, L, seg_rows, weights, o); break;
    case 4: moe_combine_kernel<4><<<blocks, 256, 0, s>>>(cr, eo, Dfwd, G, rank, T, rv, topk, pos, bb, E, L, seg_rows, weights, o); break;
    default: moe_combine_kernel<8><<<blocks, 256, 0, s>>>(cr, eo, Dfwd, G, rank, T, rv, topk, pos, bb, E, L, seg_rows, weights, o); break;
  }
  return cudaGetLastError() == cudaSuccess ? FAST_OK : FAST_ECUDA;
}

}  // extern "C"
