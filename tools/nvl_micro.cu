// nvl_micro.cu -- NVLink push bandwidth of SM store loops vs TMA bulk stores
// (scratch microbenchmark for the exec kernel's copy primitive).
// One process, G GPUs with peer access; every GPU pushes `bytes` to peer
// (g+1)%G (ring: every GPU sends and receives once, one direction each).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/nvl tools/nvl_micro.cu && /tmp/nvl
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void __launch_bounds__(512) sm_copy(uint4* __restrict__ dst, const uint4* __restrict__ src, int64_t n16) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
  }
  for (; i < n16; i += stride) dst[i] = src[i];
}

// chunked per CTA like the exec kernel: CTA c copies chunks c, c+grid, ...
__global__ void __launch_bounds__(512) sm_copy_chunked(uint8_t* dst, const uint8_t* src, int64_t bytes, int64_t chunk) {
  const int64_t nch = bytes / chunk;
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const uint4* s = reinterpret_cast<const uint4*>(src + c * chunk);
    uint4* d = reinterpret_cast<uint4*>(dst + c * chunk);
    const int64_t n16 = chunk / 16;
    int64_t i = threadIdx.x;
    const int nt = blockDim.x;
    for (; i + 3 * nt < n16; i += 4 * nt) {
      uint4 a = s[i], b = s[i + nt], cc = s[i + 2 * nt], dd = s[i + 3 * nt];
      d[i] = a; d[i + nt] = b; d[i + 2 * nt] = cc; d[i + 3 * nt] = dd;
    }
  }
}

// TMA: one thread per CTA; global -> smem (bulk, mbarrier) -> peer global (bulk store)
template <int TILE, int NBUF>
__global__ void __launch_bounds__(32) tma_copy(uint8_t* dst, const uint8_t* src, int64_t bytes, int64_t chunk) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t mbar[NBUF];
  if (threadIdx.x != 0) return;
  const uint32_t sm0 = (uint32_t)__cvta_generic_to_shared(sm);
  for (int b = 0; b < NBUF; ++b) {
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar[b]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t phase[NBUF];
  for (int b = 0; b < NBUF; ++b) phase[b] = 0;
  const int64_t nch = bytes / chunk;
  int64_t t = 0;  // global tile counter (buffer = t % NBUF)
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    for (int64_t off = 0; off < chunk; off += TILE, ++t) {
      const int b = (int)(t % NBUF);
      const uint32_t sb = sm0 + b * TILE;
      const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar[b]);
      // buffer b free once the store issued NBUF tiles ago has read it
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NBUF - 1) : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(TILE) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sb), "l"(src + c * chunk + off), "r"(TILE), "r"(mb) : "memory");
      // wait for the load, then store
      asm volatile("{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
                   "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                   "@!p bra WAIT_%=;\n\t}" ::"r"(mb), "r"(phase[b]) : "memory");
      phase[b] ^= 1;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   ::"l"(dst + c * chunk + off), "r"(sb), "r"(TILE) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  int G = 0;
  CK(cudaGetDeviceCount(&G));
  if (G < 2) { printf("need 2 GPUs\n"); return 0; }
  const int64_t bytes = 256ll << 20;
  std::vector<uint8_t*> src(G), dst(G);
  std::vector<cudaStream_t> st(G);
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    for (int h = 0; h < G; ++h) if (h != g) cudaDeviceEnablePeerAccess(h, 0);
    CK(cudaMalloc(&src[g], bytes));
    CK(cudaMalloc(&dst[g], bytes));
    CK(cudaMemset(src[g], g + 1, bytes));
    CK(cudaStreamCreate(&st[g]));
  }
  auto run = [&](const char* name, auto launch, int npairs_bidir) {
    // npairs_bidir: 0 = ring (g -> g+1), 1 = 0->1 only, 2 = 0<->1
    for (int rep = 0; rep < 2; ++rep) {
      std::vector<cudaEvent_t> e0(G), e1(G);
      for (int g = 0; g < G; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaDeviceSynchronize());
        cudaEventCreate(&e0[g]); cudaEventCreate(&e1[g]);
      }
      int active = npairs_bidir == 0 ? G : (npairs_bidir == 1 ? 1 : 2);
      for (int g = 0; g < active; ++g) {
        CK(cudaSetDevice(g));
        int peer = npairs_bidir == 0 ? (g + 1) % G : (g == 0 ? 1 : 0);
        cudaEventRecord(e0[g], st[g]);
        for (int it = 0; it < 5; ++it) launch(dst[peer], src[g], st[g]);
        cudaEventRecord(e1[g], st[g]);
      }
      float worst = 0;
      for (int g = 0; g < active; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventSynchronize(e1[g]));
        float ms; cudaEventElapsedTime(&ms, e0[g], e1[g]);
        worst = ms > worst ? ms : worst;
      }
      if (rep == 1) printf("%-44s %s: %.1f GB/s per GPU\n", name,
                           npairs_bidir == 0 ? "ring" : (npairs_bidir == 1 ? "0->1" : "0<->1"),
                           5.0 * bytes / (worst * 1e-3) / 1e9);
    }
  };
  for (int mode = 0; mode < 3; ++mode) {
    run("cudaMemcpyPeerAsync", [&](uint8_t* d, const uint8_t* s, cudaStream_t q) {
      int dd, ss; cudaPointerAttributes a; cudaPointerGetAttributes(&a, d); dd = a.device;
      cudaPointerGetAttributes(&a, s); ss = a.device;
      CK(cudaMemcpyPeerAsync(d, dd, s, ss, bytes, q)); }, mode);
    for (int blocks : {128, 148, 296}) {
      char nm[64]; snprintf(nm, 64, "SM 16B stores, grid-stride, %d x 512", blocks);
      run(nm, [&](uint8_t* d, const uint8_t* s, cudaStream_t q) {
        sm_copy<<<blocks, 512, 0, q>>>((uint4*)d, (const uint4*)s, bytes / 16); }, mode);
    }
    run("SM 16B stores, 1 MiB chunks, 128 x 512", [&](uint8_t* d, const uint8_t* s, cudaStream_t q) {
      sm_copy_chunked<<<128, 512, 0, q>>>(d, s, bytes, 1 << 20); }, mode);
    for (int blocks : {148, 296}) {
      char nm[64]; snprintf(nm, 64, "TMA 16KiB x4 bufs, 1 MiB chunks, %d CTAs", blocks);
      run(nm, [&](uint8_t* d, const uint8_t* s, cudaStream_t q) {
        cudaFuncSetAttribute(tma_copy<16384, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        tma_copy<16384, 4><<<blocks, 32, 65536, q>>>(d, s, bytes, 1 << 20); }, mode);
      snprintf(nm, 64, "TMA 32KiB x6 bufs, 1 MiB chunks, %d CTAs", blocks);
      run(nm, [&](uint8_t* d, const uint8_t* s, cudaStream_t q) {
        cudaFuncSetAttribute(tma_copy<32768, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608);
        tma_copy<32768, 6><<<blocks, 32, 196608, q>>>(d, s, bytes, 1 << 20); }, mode);
    }
  }
  for (int g = 0; g < G; ++g) { cudaSetDevice(g); CK(cudaDeviceSynchronize()); }
  printf("ok\n");
  return 0;
}
