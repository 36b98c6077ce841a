// op_lat.cu -- dependent-chain latency of single SASS ops on sm_100a
// (scratch microbenchmark for the decompose DFS step design).
#include <cstdio>
#include <cstdint>
__global__ void k(int variant, uint32_t seed, int steps, long long* out, uint32_t* sink) {
  uint32_t x = seed | 1u;
  float f = (float)seed;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < steps; ++i) {
    switch (variant) {
      case 0: x = __clz(x) + x; break;                 // FLO + IADD
      case 1: x = __popc(x) + x; break;                // POPC + IADD
      case 2: x = __brev(x) + 1u; break;               // BREV + IADD
      case 3: x = __float_as_uint((float)x) + 1u; break;  // I2F + IADD
      case 4: x = (x ^ 0x1234567u) + 7u; break;        // LOP3 + IADD (2 alu)
      case 5: x = x * 0x9e3779b9u + 7u; break;         // IMAD
      case 6: x = (x & 0xffffu) ? x + 3u : x + 5u; break;  // ISETP + SEL-ish
      case 7: x = __ffs(x) + x; break;                 // BREV+FLO
    }
  }
  long long t1 = clock64();
  out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x] = x;
}
int main() {
  long long* o; uint32_t* s;
  cudaMalloc(&o, 8); cudaMalloc(&s, 4);
  const char* nm[] = {"clz+add", "popc+add", "brev+add", "i2f+add", "xor+add", "imad", "test+sel", "ffs+add"};
  for (int v = 0; v < 8; ++v) {
    k<<<1, 32>>>(v, 12345, 100000, o, s);
    k<<<1, 32>>>(v, 12345, 100000, o, s);
    long long h; cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
    printf("%-10s %.1f cycles/iter\n", nm[v], h / 100000.0);
  }
}
