// chase2_micro.cu -- which part of the DFS step costs the cycles (scratch).
#include <cstdio>
#include <cstdint>
#include <vector>
#define STEP_CORE(R0, R1, R2, R3, N0, N1, N2, N3, LD)               \
  "and.b32 x0, " R1 ", ns0;\n\t"                                      \
  "and.b32 x1, " R0 ", ns1;\n\t"                                      \
  "and.b32 x2, " R3 ", ns2;\n\t"                                      \
  "and.b32 x3, " R2 ", ns3;\n\t"                                      \
  "clz.b32 z0, x0;\n\t"                                               \
  "clz.b32 z1, x1;\n\t"                                               \
  "clz.b32 z2, x2;\n\t"                                               \
  "clz.b32 z3, x3;\n\t"                                               \
  "or.b32 t, x0, x1;\n\t"                                             \
  "setp.ne.u32 p0, x0, 0;\n\t"                                        \
  "setp.ne.u32 p2, x2, 0;\n\t"                                        \
  "setp.ne.u32 p01, t, 0;\n\t"                                        \
  "mad.lo.u32 a0, z0, 16, bb0;\n\t"                                   \
  "mad.lo.u32 a1, z1, 16, bb1;\n\t"                                   \
  "mad.lo.u32 a2, z2, 16, bb2;\n\t"                                   \
  "mad.lo.u32 a3, z3, 16, bb3;\n\t"                                   \
  "selp.b32 s01, a0, a1, p0;\n\t"                                     \
  "selp.b32 s23, a2, a3, p2;\n\t"                                     \
  "selp.b32 ad, s01, s23, p01;\n\t"                                   \
  LD " {" N0 ", " N1 ", " N2 ", " N3 "}, [ad];\n\t"
#define SEEN                                                           \
  "sub.u32 t, ad, bb0;\n\t"                                           \
  "shr.u32 v, t, 4;\n\t"                                              \
  "and.b32 t, v, 31;\n\t"                                             \
  "shr.u32 b, hb, t;\n\t"                                             \
  "shr.u32 w, v, 5;\n\t"                                              \
  "setp.eq.u32 q0, w, 0;\n\t"                                         \
  "setp.eq.u32 q1, w, 1;\n\t"                                         \
  "setp.eq.u32 q2, w, 2;\n\t"                                         \
  "setp.eq.u32 q3, w, 3;\n\t"                                         \
  "not.b32 b, b;\n\t"                                                 \
  "@q0 and.b32 ns0, ns0, b;\n\t"                                      \
  "@q1 and.b32 ns1, ns1, b;\n\t"                                      \
  "@q2 and.b32 ns2, ns2, b;\n\t"                                      \
  "@q3 and.b32 ns3, ns3, b;\n\t"                                      \
  "setp.gt.u32 pn, v, 127;\n\t"                                       \
  "@pn mov.b32 ns0, -1;\n\t"                                          \
  "@pn mov.b32 ns1, -1;\n\t"                                          \
  "@pn mov.b32 ns2, -1;\n\t"                                          \
  "@pn mov.b32 ns3, -1;\n\t"
#define STORE "st.shared.u16 [pa], v;\n\t"
#define BRANCH "setp.eq.u32 ph, v, 1000;\n\t@ph bra.uni L_OUT;\n\t"


#define STEP5(R0, R1, R2, R3, N0, N1, N2, N3)                          \
  "and.b32 x0, " R1 ", ns0;\n\t"                                      \
  "and.b32 x1, " R0 ", ns1;\n\t"                                      \
  "and.b32 x2, " R3 ", ns2;\n\t"                                      \
  "and.b32 x3, " R2 ", ns3;\n\t"                                      \
  "clz.b32 z0, x0;\n\t"                                               \
  "clz.b32 z1, x1;\n\t"                                               \
  "clz.b32 z2, x2;\n\t"                                               \
  "clz.b32 z3, x3;\n\t"                                               \
  "or.b32 t, x0, x1;\n\t"                                             \
  "or.b32 u, x2, x3;\n\t"                                             \
  "or.b32 u, u, t;\n\t"                                               \
  "setp.ne.u32 p0, x0, 0;\n\t"                                        \
  "setp.ne.u32 p2, x2, 0;\n\t"                                        \
  "setp.ne.u32 p01, t, 0;\n\t"                                        \
  "setp.eq.u32 pn, u, 0;\n\t"                                         \
  "mad.lo.u32 a0, z0, 16, bb0;\n\t"                                   \
  "mad.lo.u32 a1, z1, 16, bb1;\n\t"                                   \
  "mad.lo.u32 a2, z2, 16, bb2;\n\t"                                   \
  "mad.lo.u32 a3, z3, 16, bb3;\n\t"                                   \
  "selp.b32 s01, a0, a1, p0;\n\t"                                     \
  "selp.b32 s23, a2, a3, p2;\n\t"                                     \
  "selp.b32 ad, s01, s23, p01;\n\t"                                   \
  "ld.shared.v4.u32 {" N0 ", " N1 ", " N2 ", " N3 "}, [ad];\n\t"     \
  "shr.u32 m0, hb, z0;\n\t"                                           \
  "shr.u32 m1, hb, z1;\n\t"                                           \
  "shr.u32 m2, hb, z2;\n\t"                                           \
  "shr.u32 m3, hb, z3;\n\t"                                           \
  "selp.b32 m1, 0, m1, p0;\n\t"                                       \
  "selp.b32 m2, 0, m2, p01;\n\t"                                      \
  "selp.b32 m3, 0, m3, p01;\n\t"                                      \
  "selp.b32 m3, 0, m3, p2;\n\t"                                       \
  "and.b32 h0, f0, m0;\n\t"                                           \
  "and.b32 h1, f1, m1;\n\t"                                           \
  "and.b32 h2, f2, m2;\n\t"                                           \
  "and.b32 h3, f3, m3;\n\t"                                           \
  "or.b32 h0, h0, h1;\n\t"                                            \
  "or.b32 h2, h2, h3;\n\t"                                            \
  "or.b32 h0, h0, h2;\n\t"                                            \
  "not.b32 m0, m0;\n\t"                                               \
  "not.b32 m1, m1;\n\t"                                               \
  "not.b32 m2, m2;\n\t"                                               \
  "not.b32 m3, m3;\n\t"                                               \
  "and.b32 ns0, ns0, m0;\n\t"                                         \
  "and.b32 ns1, ns1, m1;\n\t"                                         \
  "and.b32 ns2, ns2, m2;\n\t"                                         \
  "and.b32 ns3, ns3, m3;\n\t"                                         \
  "sub.u32 v, ad, bb0;\n\t"                                           \
  "shr.u32 v, v, 4;\n\t"                                              \
  "st.shared.u16 [pa], v;\n\t"                                        \
  "setp.ne.or.u32 ph, h0, 0, pn;\n\t"                                 \
  "@pn mov.b32 ns0, -1;\n\t"                                          \
  "@pn mov.b32 ns1, -1;\n\t"                                          \
  "@pn mov.b32 ns2, -1;\n\t"                                          \
  "@pn mov.b32 ns3, -1;\n\t"                                          \
  "setp.eq.and.u32 ph, v, 1000, ph;\n\t"                              \
  "@ph bra.uni L_OUT;\n\t"

#define KERNEL(NAME, BODY1, BODY2)                                               \
  __global__ void NAME(const uint32_t* g, int steps, long long* out, int* sink) { \
    __shared__ __align__(16) uint32_t sh[128 * 4];                                \
    __shared__ int16_t pk[64];                                                    \
    for (int i = threadIdx.x; i < 512; i += blockDim.x) sh[i] = g[i];            \
    __syncthreads();                                                              \
    if (threadIdx.x != 0) return;                                                 \
    uint32_t base = (uint32_t)__cvta_generic_to_shared(sh);                      \
    uint32_t pka = (uint32_t)__cvta_generic_to_shared(pk);                       \
    uint32_t res = 0;                                                             \
    long long t0 = clock64();                                                     \
    asm volatile("{\n\t"                                                          \
      ".reg .pred p0, p2, p01, q0, q1, q2, q3, pn, ph, pl;\n\t"                   \
      ".reg .b32 r0, r1, r2, r3, n0, n1, n2, n3, ns0, ns1, ns2, ns3, i;\n\t"    \
      ".reg .b32 x0, x1, x2, x3, z0, z1, z2, z3, a0, a1, a2, a3, pa;\n\t"        \
      ".reg .b32 s01, s23, ad, t, v, b, w, hb, bb0, bb1, bb2, bb3, u, m0, m1, m2, m3, h0, h1, h2, h3, f0, f1, f2, f3;\n\t" "mov.b32 f0, 0x10001;\n\tmov.b32 f1, 0x10;\n\tmov.b32 f2, 0x1000;\n\tmov.b32 f3, 0x4;\n\t"          \
      "mov.b32 ns0, -1;\n\tmov.b32 ns1, -1;\n\tmov.b32 ns2, -1;\n\tmov.b32 ns3, -1;\n\t" \
      "mov.b32 hb, 0x80000000;\n\tmov.b32 bb0, %1;\n\tadd.u32 bb1, %1, 512;\n\t" \
      "add.u32 bb2, %1, 1024;\n\tadd.u32 bb3, %1, 1536;\n\tmov.b32 pa, %3;\n\t"  \
      "mov.b32 v, 0;\n\t"                                                         \
      "ld.shared.v4.u32 {r0, r1, r2, r3}, [%1];\n\t"                              \
      "mov.b32 i, %2;\n\t"                                                        \
      "L_LOOP:\n\t"                                                               \
      BODY1 BODY2                                                                 \
      "sub.u32 i, i, 2;\n\t"                                                      \
      "setp.gt.s32 pl, i, 0;\n\t"                                                 \
      "@pl bra.uni L_LOOP;\n\t"                                                   \
      "L_OUT:\n\t"                                                                \
      "add.u32 %0, r0, v;\n\t"                                                    \
      "}" : "=r"(res) : "r"(base), "r"(steps), "r"(pka) : "memory");            \
    long long t1 = clock64();                                                     \
    out[blockIdx.x] = t1 - t0;                                                    \
    sink[blockIdx.x] = res;                                                       \
  }

KERNEL(k_v5, STEP5("r0","r1","r2","r3","n0","n1","n2","n3"), STEP5("n0","n1","n2","n3","r0","r1","r2","r3"))
#define LDN "ld.shared.v4.u32"
#define LDV "ld.volatile.shared.v4.u32"
KERNEL(k_core, STEP_CORE("r0","r1","r2","r3","n0","n1","n2","n3",LDN), STEP_CORE("n0","n1","n2","n3","r0","r1","r2","r3",LDN))
KERNEL(k_seen, STEP_CORE("r0","r1","r2","r3","n0","n1","n2","n3",LDN) SEEN, STEP_CORE("n0","n1","n2","n3","r0","r1","r2","r3",LDN) SEEN)
KERNEL(k_store, STEP_CORE("r0","r1","r2","r3","n0","n1","n2","n3",LDN) SEEN STORE, STEP_CORE("n0","n1","n2","n3","r0","r1","r2","r3",LDN) SEEN STORE)
KERNEL(k_branch, STEP_CORE("r0","r1","r2","r3","n0","n1","n2","n3",LDN) SEEN BRANCH, STEP_CORE("n0","n1","n2","n3","r0","r1","r2","r3",LDN) SEEN BRANCH)
KERNEL(k_all, STEP_CORE("r0","r1","r2","r3","n0","n1","n2","n3",LDN) SEEN STORE BRANCH, STEP_CORE("n0","n1","n2","n3","r0","r1","r2","r3",LDN) SEEN STORE BRANCH)
KERNEL(k_allv, STEP_CORE("r0","r1","r2","r3","n0","n1","n2","n3",LDV) SEEN STORE BRANCH, STEP_CORE("n0","n1","n2","n3","r0","r1","r2","r3",LDV) SEEN STORE BRANCH)

int main() {
  std::vector<uint32_t> g(512);
  srand(3);
  for (auto& x : g) x = (uint32_t)rand() & (uint32_t)rand();
  uint32_t* d; long long* o; int* s;
  cudaMalloc(&d, 2048); cudaMalloc(&o, 8 * 148 * 8); cudaMalloc(&s, 4 * 148 * 8);
  cudaMemcpy(d, g.data(), 2048, cudaMemcpyHostToDevice);
  const int steps = 100000;
  typedef void (*KF)(const uint32_t*, int, long long*, int*);
  KF ks[] = {k_v5, k_core, k_seen, k_store, k_branch, k_all, k_allv};
  const char* names[] = {"v5", "core", "+seen", "+seen+store", "+seen+branch", "+seen+store+branch", "all, volatile ld"};
  for (int v = 0; v < 7; ++v) {
    for (int grid : {148, 148 * 7}) {
      ks[v]<<<grid, 32>>>(d, steps, o, s);
      ks[v]<<<grid, 32>>>(d, steps, o, s);
      cudaDeviceSynchronize();
      std::vector<long long> h(grid);
      cudaMemcpy(h.data(), o, 8 * grid, cudaMemcpyDeviceToHost);
      double c = 0; for (auto x : h) c += x;
      printf("%-22s grid %4d: %.1f cycles/step\n", names[v], grid, c / grid / steps);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
