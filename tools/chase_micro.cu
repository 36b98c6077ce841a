// chase_micro.cu -- dependent-chain latency of the DFS step's pieces on
// sm_100a (scratch microbenchmark, see tools/dfs_micro.cu).
#include <cstdio>
#include <cstdint>
#include <vector>
__global__ void k(int variant, const uint32_t* g, int steps, long long* out, int* sink) {
  __shared__ __align__(16) uint32_t sh[128 * 4];
  __shared__ int16_t pick[4096];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) sh[i] = g[i];
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sh);
  uint32_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  uint32_t a = base;
  int acc = 0;
  long long t0 = clock64();
  if (variant == 0) {  // LDS.32 chase
    for (int i = 0; i < steps; ++i) {
      uint32_t x;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(a));
      a = base + (x & 127) * 16;
    }
  } else if (variant == 1) {  // LDS.128 chase + andnot + 4 clz + select, no seen update
    for (int i = 0; i < steps; ++i) {
      uint4 r;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
      const uint32_t x0 = r.y & ~s0, x1 = r.x & ~s1, x2 = r.w & ~s2, x3 = r.z & ~s3;
      const int v = x0 ? __clz(x0) : (x1 ? 32 + __clz(x1) : (x2 ? 64 + __clz(x2) : 96 + (__clz(x3) & 31)));
      a = base + v * 16;
    }
  } else if (variant == 2) {  // + seen update (reset when all seen)
    for (int i = 0; i < steps; ++i) {
      uint4 r;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
      const uint32_t x0 = r.y & ~s0, x1 = r.x & ~s1, x2 = r.w & ~s2, x3 = r.z & ~s3;
      const int v = x0 ? __clz(x0) : (x1 ? 32 + __clz(x1) : (x2 ? 64 + __clz(x2) : 96 + __clz(x3)));
      const uint32_t bit = 0x80000000u >> (v & 31);
      const int w = v >> 5;
      s0 |= w == 0 ? bit : 0u; s1 |= w == 1 ? bit : 0u; s2 |= w == 2 ? bit : 0u; s3 |= w == 3 ? bit : 0u;
      if (v == 128) { s0 = s1 = s2 = s3 = 0; }
      a = base + (v & 127) * 16;
    }
  } else if (variant == 3) {  // + pick store
    for (int i = 0; i < steps; ++i) {
      uint4 r;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
      const uint32_t x0 = r.y & ~s0, x1 = r.x & ~s1, x2 = r.w & ~s2, x3 = r.z & ~s3;
      const int v = x0 ? __clz(x0) : (x1 ? 32 + __clz(x1) : (x2 ? 64 + __clz(x2) : 96 + __clz(x3)));
      const uint32_t bit = 0x80000000u >> (v & 31);
      const int w = v >> 5;
      s0 |= w == 0 ? bit : 0u; s1 |= w == 1 ? bit : 0u; s2 |= w == 2 ? bit : 0u; s3 |= w == 3 ? bit : 0u;
      if (v == 128) { s0 = s1 = s2 = s3 = 0; }
      pick[i & 4095] = (int16_t)v;
      a = base + (v & 127) * 16;
    }
  } else if (variant == 4) {  // 64-bit halves clz (production style)
    uint64_t q0 = 0, q1 = 0;
    for (int i = 0; i < steps; ++i) {
      uint4 r;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
      const uint64_t r0 = ((uint64_t)r.y << 32) | r.x, r1 = ((uint64_t)r.w << 32) | r.z;
      const int z0 = __clzll(r0 & ~q0), z1 = __clzll(r1 & ~q1);
      const int v = z0 < 64 ? z0 : 64 + z1;
      const uint64_t m = 0x8000000000000000ull >> (v & 63);
      q0 |= v < 64 ? m : 0ull; q1 |= (v >= 64 && v < 128) ? m : 0ull;
      if (v == 128) { q0 = q1 = 0; }
      a = base + (v & 127) * 16;
    }
  } else if (variant == 5) {  // clz via float conversion-free: brev-less, branchless min of tagged words
    for (int i = 0; i < steps; ++i) {
      uint4 r;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
      const uint32_t x0 = r.y & ~s0, x1 = r.x & ~s1, x2 = r.w & ~s2, x3 = r.z & ~s3;
      const int z0 = __clz(x0), z1 = __clz(x1), z2 = __clz(x2), z3 = __clz(x3);
      const int c0 = z0 | (x0 ? 0 : 128), c1 = (32 + z1) | (x1 ? 0 : 128), c2 = (64 + z2) | (x2 ? 0 : 128), c3 = 96 + z3;
      const int v = min(min(c0, c1), min(c2, c3));
      const uint32_t bit = 0x80000000u >> (v & 31);
      const int w = v >> 5;
      s0 |= w == 0 ? bit : 0u; s1 |= w == 1 ? bit : 0u; s2 |= w == 2 ? bit : 0u; s3 |= w == 3 ? bit : 0u;
      if (v == 128) { s0 = s1 = s2 = s3 = 0; }
      a = base + (v & 127) * 16;
    }
  }
  long long t1 = clock64();
  out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x] = a + acc + s0 + s1 + s2 + s3;
}
int main() {
  std::vector<uint32_t> g(512);
  srand(3);
  for (auto& x : g) x = (uint32_t)rand() & (uint32_t)rand();
  uint32_t* d; long long* o; int* s;
  cudaMalloc(&d, 2048); cudaMalloc(&o, 8 * 148 * 8); cudaMalloc(&s, 4 * 148 * 8);
  cudaMemcpy(d, g.data(), 2048, cudaMemcpyHostToDevice);
  const int steps = 100000;
  const char* names[] = {"LDS.32 chase", "LDS.128+andnot+4clz+select", "+seen update", "+pick STS", "64-bit halves clzll", "tagged min"};
  for (int v = 0; v < 6; ++v) {
    for (int grid : {148, 148 * 7}) {
      k<<<grid, 32>>>(v, d, steps, o, s);
      k<<<grid, 32>>>(v, d, steps, o, s);
      cudaDeviceSynchronize();
      std::vector<long long> h(grid);
      cudaMemcpy(h.data(), o, 8 * grid, cudaMemcpyDeviceToHost);
      double c = 0; for (auto x : h) c += x;
      printf("%-32s grid %4d: %.1f cycles/step\n", names[v], grid, c / grid / steps);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
