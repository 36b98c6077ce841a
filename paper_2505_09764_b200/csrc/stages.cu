// stages.cu -- the stage-level building blocks of the reference's Birkhoff
// module as standalone device entry points (the batched synthesis fuses
// them; these serve the drop-in object API):
//
//   fast_match_batch   find_perfect_matching (birkhoff.py:111-137): the
//                      decomposition's warp-level Kuhn DFS (synth_dev.cuh)
//                      on arbitrary boolean supports, one warp per matrix.
//   fast_strip_sort    strip_auxiliary (birkhoff.py:225-252) and / or
//                      sort_stages_ascending (:255-266) on an arbitrary stage
//                      list: one thread per source server walks the stages
//                      in order carrying aux_left per (src, dst) cell (the
//                      reference's own arithmetic), then a block bitonic
//                      sort on (weight, first edge, input position).
#include <cuda_runtime.h>
#include <stdint.h>

#include "fastb200.h"
#include "synth_dev.cuh"

namespace {

constexpr int kMatchWarps = 4;

template <int NW>
__global__ void __launch_bounds__(kMatchWarps * 32)
    match_kernel(const uint8_t* __restrict__ support, int B, int n, int32_t* row_match,
                 int32_t* status) {
  extern __shared__ __align__(16) char msm[];
  constexpr int NWP = DecSh<NW>::NWP;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * kMatchWarps + warp;
  if (b >= B) return;
  DecSh<NW> s = dec_carve_t<NW>(msm + warp * dec_smem_bytes_t<NW>(n), n);
  const uint8_t* sp = support + (int64_t)b * n * n;
  // support bitsets in the DFS layout: u32 word w holds columns 32*(w^1)+t
  // at bit 31 - t (colword / colbit)
  for (int x = lane; x < n * NWP; x += 32) {
    const int u = x / NWP, w = x - u * NWP, cb = (w ^ 1) * 32;
    uint32_t bits = 0;
    for (int t = 0; t < 32; ++t)
      if (cb + t < n && sp[(int64_t)u * n + cb + t]) bits |= 0x80000000u >> t;
    s.sup[x] = bits;
  }
  for (int w = lane; w < NWP; w += 32) {
    const int cb = (w ^ 1) * 32;
    uint32_t bits = 0;
    for (int t = 0; t < 32; ++t)
      if (cb + t < n) bits |= 0x80000000u >> t;
    s.freeb[w] = bits;  // every column starts free
  }
  for (int v = lane; v < n; v += 32) {
    s.cm[v] = -1;
    s.newcol[v] = -1;
  }
  for (int c = lane; c < n * NWP; c += 32) s.supc[c] = 0u;  // free columns: empty row
  __syncwarp();
  int st = FAST_OK;
  for (int u = 0; u < n; ++u) {  // rows in index order, fresh `seen` per root
    const int depth = dfs_warp<NW>(s, u);
    if (depth < 0) {
      st = FAST_EINVARIANT;  // "support matrix has no perfect matching"
      break;
    }
    apply_path<NW>(s, u, depth, lane);
  }
  __syncwarp();
  for (int u = lane; u < n; u += 32)
    row_match[(int64_t)b * n + u] = st == FAST_OK ? s.newcol[u] : -1;
  if (lane == 0) status[b] = st;
}

template <int NW>
int launch_match_t(const uint8_t* support, int B, int n, int32_t* row_match, int32_t* status,
                   cudaStream_t s) {
  const size_t smem = dec_smem_bytes_t<NW>(n) * kMatchWarps;
  static size_t granted = 0;
  if (smem > 48 * 1024 && smem > granted) {
    if (cudaFuncSetAttribute(match_kernel<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return FAST_ECUDA;
    granted = smem;
  }
  match_kernel<NW><<<(B + kMatchWarps - 1) / kMatchWarps, kMatchWarps * 32, smem, s>>>(
      support, B, n, row_match, status);
  return cudaGetLastError() == cudaSuccess ? FAST_OK : FAST_ECUDA;
}

constexpr int kStripThreads = 1024;

__host__ __device__ inline int pow2_at_least(int k) {
  int p = 1;
  while (p < k) p <<= 1;
  return p;
}

__host__ __device__ inline size_t strip_ws_bytes(int K, int n) {
  const size_t P2 = (size_t)pow2_at_least(K > 0 ? K : 1);
  return (size_t)n * n * 8 + 2 * P2 * 8 + (size_t)(K > 0 ? K : 1) * 4 + 256;
}

__global__ void __launch_bounds__(kStripThreads)
    strip_sort_kernel(const int64_t* __restrict__ weight, const int16_t* __restrict__ dst,
                      const int64_t* __restrict__ bytes, const int64_t* __restrict__ aux, int K,
                      int n, int mode, int32_t* order_out, int64_t* real_out, int32_t* n_out,
                      int32_t* status, char* ws) {
  __shared__ int s_bad, s_count;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int P2 = pow2_at_least(K > 0 ? K : 1);
  int64_t* aux_left = (int64_t*)ws;                               // [n][n]
  unsigned long long* khi = (unsigned long long*)(aux_left + (size_t)n * n);  // [P2]
  unsigned long long* klo = khi + P2;                            // [P2]
  int32_t* kept = (int32_t*)(klo + P2);                          // [K]
  if (tid == 0) s_bad = 0, s_count = 0;
  for (int k = tid; k < K; k += nt) kept[k] = (mode & 1) ? 0 : 1;
  if (mode & 1)
    for (int x = tid; x < n * n; x += nt) aux_left[x] = aux[x];
  __syncthreads();
  if (mode & 1) {
    // strip_auxiliary: stages in decomposition order, aux paid first per edge
    for (int u = tid; u < n; u += nt) {
      for (int k = 0; k < K; ++k) {
        const int v = dst[(int64_t)k * n + u];
        if (v < 0) continue;
        const int64_t b = bytes[(int64_t)k * n + u];
        int64_t* al = aux_left + (int64_t)u * n + v;
        const int64_t charged = *al < b ? *al : b;
        *al -= charged;
        const int64_t real = b - charged;
        real_out[(int64_t)k * n + u] = real;
        if (real > 0) kept[k] = 1;
      }
    }
    __syncthreads();
    for (int x = tid; x < n * n; x += nt)
      if (aux_left[x] != 0) atomicOr(&s_bad, 1);  // "auxiliary bytes left unconsumed"
  } else {
    for (int x = tid; x < K * n; x += nt) real_out[x] = dst[x] >= 0 ? bytes[x] : 0;
  }
  __syncthreads();
  if (mode & 2) {
    // key (weight, first edge (src, dst) or (-1, -1), input position)
    for (int k = tid; k < P2; k += nt) {
      unsigned long long hi = ~0ull, lo = ~0ull;
      if (k < K && kept[k]) {
        hi = (unsigned long long)weight[k];
        unsigned long long fe = 0;
        for (int u = 0; u < n; ++u) {
          const int v = dst[(int64_t)k * n + u];
          const bool on = v >= 0 && (!(mode & 1) || real_out[(int64_t)k * n + u] > 0);
          if (on) {
            fe = ((unsigned long long)(u + 1) << 44) | ((unsigned long long)(v + 1) << 24);
            break;
          }
        }
        lo = fe | (unsigned long long)k;
      }
      khi[k] = hi;
      klo[k] = lo;
    }
    __syncthreads();
    for (int size = 2; size <= P2; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = tid; i < P2; i += nt) {
          const int j = i ^ stride;
          if (j > i) {
            const bool up = (i & size) == 0;
            const unsigned long long ah = khi[i], al = klo[i], bh = khi[j], bl = klo[j];
            const bool gt = ah > bh || (ah == bh && al > bl);
            if (gt == up) {
              khi[i] = bh; klo[i] = bl;
              khi[j] = ah; klo[j] = al;
            }
          }
        }
        __syncthreads();
      }
    }
    for (int i = tid; i < K; i += nt)
      if (khi[i] != ~0ull || klo[i] != ~0ull) {
        order_out[i] = (int32_t)(klo[i] & 0xFFFFFF);
        atomicAdd(&s_count, 1);
      }
  } else {
    if (tid == 0) {  // kept stages in decomposition order
      int c = 0;
      for (int k = 0; k < K; ++k)
        if (kept[k]) order_out[c++] = k;
      s_count = c;
    }
  }
  __syncthreads();
  if (tid == 0) {
    *n_out = s_bad ? 0 : s_count;
    *status = s_bad ? FAST_EINVARIANT : FAST_OK;
  }
}

}  // namespace

extern "C" {

int fast_match_batch(const uint8_t* support, int B, int n, int32_t* row_match, int32_t* status,
                     void* stream) {
  if (B < 0 || n < 1 || n > FAST_MAX_SERVERS || !support || !row_match || !status)
    return FAST_EVALIDATION;
  if (B == 0) return FAST_OK;
  cudaStream_t s = (cudaStream_t)stream;
  switch ((n + 31) / 32) {
    case 1: return launch_match_t<1>(support, B, n, row_match, status, s);
    case 2: return launch_match_t<2>(support, B, n, row_match, status, s);
    case 3: return launch_match_t<3>(support, B, n, row_match, status, s);
    default: return launch_match_t<4>(support, B, n, row_match, status, s);
  }
}

size_t fast_strip_sort_workspace_bytes(int K, int n) {
  return K < 0 || n < 1 ? 0 : strip_ws_bytes(K, n);
}

int fast_strip_sort(const int64_t* weight, const int16_t* dst, const int64_t* bytes,
                    const int64_t* aux, int K, int n, int mode, int32_t* order_out,
                    int64_t* real_out, int32_t* n_out, int32_t* status, void* workspace,
                    void* stream) {
  if (K < 0 || K > (1 << 24) || n < 1 || n > (1 << 19) || mode < 1 || mode > 3 || !weight ||
      !dst || !bytes || ((mode & 1) && !aux) || !order_out || !real_out || !n_out || !status ||
      !workspace)
    return FAST_EVALIDATION;
  strip_sort_kernel<<<1, kStripThreads, 0, (cudaStream_t)stream>>>(
      weight, dst, bytes, aux, K, n, mode, order_out, real_out, n_out, status, (char*)workspace);
  return cudaGetLastError() == cudaSuccess ? FAST_OK : FAST_ECUDA;
}

}  // extern "C"
