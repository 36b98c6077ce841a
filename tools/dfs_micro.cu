// dfs_micro.cu -- cycles per Kuhn-DFS step of decompose_kernel's search loop
// (synth_dev.cuh: dfs_search) against candidate rewrites, on random dense
// supports in shared memory.  Each variant must return the same depth and
// pick[] as the production loop.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//     -I include -I paper_2505_09764_b200/csrc -o /tmp/dfs_micro tools/dfs_micro.cu && /tmp/dfs_micro
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "synth_dev.cuh"

namespace {

constexpr int NWv = 4;
using Sh = DecSh<NWv>;
constexpr int NWP = Sh::NWP;

// Variant 1: four 32-bit words, clz per word, predicate select chain; the
// next row address is selected directly.
__device__ int dfs_v1(const Sh& s, const int root, uint32_t f0, uint32_t f1, uint32_t f2,
                      uint32_t f3, long long* iters) {
  // words in column order: c0 = cols 0..31 (u32 word 1), c1 = 32..63 (word 0),
  // c2 = 64..95 (word 3), c3 = 96..127 (word 2); column 32i+b at bit 31-b.
  uint32_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  uint4 r = *reinterpret_cast<const uint4*>(s.sup + root * NWP);
  const char* base = reinterpret_cast<const char*>(s.supc);
  int sp = 0;
  long long it = 0;
  for (;;) {
    ++it;
    const uint32_t x0 = r.y & ~s0, x1 = r.x & ~s1, x2 = r.w & ~s2, x3 = r.z & ~s3;
    const int c0 = __clz(x0), c1 = 32 + __clz(x1), c2 = 64 + __clz(x2), c3 = 96 + __clz(x3);
    const int v = x0 ? c0 : (x1 ? c1 : (x2 ? c2 : c3));  // 128: none
    const uint4 nr = *reinterpret_cast<const uint4*>(base + ((v & 127) << 4) * NWP / 4);
    if (__builtin_expect(v == 128, 0)) {
      if (sp == 0) { *iters += it; return -1; }
      --sp;
      r = *reinterpret_cast<const uint4*>(sp == 0 ? s.sup + root * NWP
                                                  : s.supc + s.pick[sp - 1] * NWP);
      continue;
    }
    const uint32_t bit = 0x80000000u >> (v & 31);
    const int wsel = v >> 5;
    s0 |= wsel == 0 ? bit : 0u;
    s1 |= wsel == 1 ? bit : 0u;
    s2 |= wsel == 2 ? bit : 0u;
    s3 |= wsel == 3 ? bit : 0u;
    const uint32_t fw = wsel == 0 ? f0 : (wsel == 1 ? f1 : (wsel == 2 ? f2 : f3));
    s.pick[sp] = (int16_t)v;
    if (fw & bit) { *iters += it; return sp; }
    ++sp;
    r = nr;
  }
}

// Variant 2: as v1 but the four candidate row addresses are formed from the
// per-word clz in parallel and the address (not the index) is selected.
__device__ int dfs_v2(const Sh& s, const int root, uint32_t f0, uint32_t f1, uint32_t f2,
                      uint32_t f3, long long* iters) {
  uint32_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  uint4 r = *reinterpret_cast<const uint4*>(s.sup + root * NWP);
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(s.supc);
  int sp = 0;
  long long it = 0;
  for (;;) {
    ++it;
    const uint32_t x0 = r.y & ~s0, x1 = r.x & ~s1, x2 = r.w & ~s2, x3 = r.z & ~s3;
    const uint32_t z0 = __clz(x0), z1 = __clz(x1), z2 = __clz(x2), z3 = __clz(x3);
    const uint32_t a0 = base + z0 * 16, a1 = base + 512 + z1 * 16, a2 = base + 1024 + z2 * 16,
                   a3 = base + 1536 + (z3 & 31) * 16;
    const uint32_t a = x0 ? a0 : (x1 ? a1 : (x2 ? a2 : a3));
    uint4 nr;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(nr.x), "=r"(nr.y), "=r"(nr.z), "=r"(nr.w) : "r"(a));
    const int v = x0 ? (int)z0 : (x1 ? 32 + (int)z1 : (x2 ? 64 + (int)z2 : 96 + (int)z3));
    if (__builtin_expect(v == 128, 0)) {
      if (sp == 0) { *iters += it; return -1; }
      --sp;
      r = *reinterpret_cast<const uint4*>(sp == 0 ? s.sup + root * NWP
                                                  : s.supc + s.pick[sp - 1] * NWP);
      continue;
    }
    const uint32_t bit = 0x80000000u >> (v & 31);
    const int wsel = v >> 5;
    s0 |= wsel == 0 ? bit : 0u;
    s1 |= wsel == 1 ? bit : 0u;
    s2 |= wsel == 2 ? bit : 0u;
    s3 |= wsel == 3 ? bit : 0u;
    const uint32_t fw = wsel == 0 ? f0 : (wsel == 1 ? f1 : (wsel == 2 ? f2 : f3));
    s.pick[sp] = (int16_t)v;
    if (fw & bit) { *iters += it; return sp; }
    ++sp;
    r = nr;
  }
}


// Variant 3: the step's select logic as predicated PTX (no branches on the
// address chain): per-word clz -> candidate row addresses -> 2-level selp
// tree -> ld.shared.v4; seen/free bookkeeping hangs off the chain.
__device__ __forceinline__ void dfs_step4(const uint4 r, const uint32_t base, uint32_t& ns0,
                                          uint32_t& ns1, uint32_t& ns2, uint32_t& ns3,
                                          const uint32_t f0, const uint32_t f1,
                                          const uint32_t f2, const uint32_t f3, uint4& nr,
                                          int& v, uint32_t& hit) {
  uint32_t addr, vv, h;
  asm volatile(
      "{\n\t"
      ".reg .pred p0, p2, p01, q0, q1, q2, q3, qlo;\n\t"
      ".reg .b32 x0, x1, x2, x3, z0, z1, z2, z3, a0, a1, a2, a3, s01, s23, t, b, w, fa, fb, fw;\n\t"
      "and.b32 x0, %12, %4;\n\t"
      "and.b32 x1, %11, %5;\n\t"
      "and.b32 x2, %14, %6;\n\t"
      "and.b32 x3, %13, %7;\n\t"
      "clz.b32 z0, x0;\n\t"
      "clz.b32 z1, x1;\n\t"
      "clz.b32 z2, x2;\n\t"
      "clz.b32 z3, x3;\n\t"
      "or.b32 t, x0, x1;\n\t"
      "setp.ne.u32 p0, x0, 0;\n\t"
      "setp.ne.u32 p2, x2, 0;\n\t"
      "setp.ne.u32 p01, t, 0;\n\t"
      "mad.lo.u32 a0, z0, 16, %15;\n\t"
      "add.u32 t, %15, 512;\n\t"
      "mad.lo.u32 a1, z1, 16, t;\n\t"
      "add.u32 t, %15, 1024;\n\t"
      "mad.lo.u32 a2, z2, 16, t;\n\t"
      "add.u32 t, %15, 1536;\n\t"
      "mad.lo.u32 a3, z3, 16, t;\n\t"
      "selp.b32 s01, a0, a1, p0;\n\t"
      "selp.b32 s23, a2, a3, p2;\n\t"
      "selp.b32 %8, s01, s23, p01;\n\t"
      "ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%8];\n\t"
      "sub.u32 t, %8, %15;\n\t"
      "shr.u32 %9, t, 4;\n\t"
      "and.b32 t, %9, 31;\n\t"
      "shr.u32 b, 0x80000000, t;\n\t"
      "shr.u32 w, %9, 5;\n\t"
      "setp.eq.u32 q0, w, 0;\n\t"
      "setp.eq.u32 q1, w, 1;\n\t"
      "setp.eq.u32 q2, w, 2;\n\t"
      "setp.eq.u32 q3, w, 3;\n\t"
      "setp.lt.u32 qlo, w, 2;\n\t"
      "selp.b32 fa, %16, %17, q0;\n\t"
      "selp.b32 fb, %18, %19, q2;\n\t"
      "selp.b32 fw, fa, fb, qlo;\n\t"
      "and.b32 %10, fw, b;\n\t"
      "not.b32 b, b;\n\t"
      "@q0 and.b32 %4, %4, b;\n\t"
      "@q1 and.b32 %5, %5, b;\n\t"
      "@q2 and.b32 %6, %6, b;\n\t"
      "@q3 and.b32 %7, %7, b;\n\t"
      "}"
      : "=r"(nr.x), "=r"(nr.y), "=r"(nr.z), "=r"(nr.w), "+r"(ns0), "+r"(ns1), "+r"(ns2),
        "+r"(ns3), "=r"(addr), "=r"(vv), "=r"(h)
      : "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(base), "r"(f0), "r"(f1), "r"(f2), "r"(f3));
  v = (int)vv;
  hit = h;
}

__device__ int dfs_v3(const Sh& s, const int root, uint32_t f0, uint32_t f1, uint32_t f2,
                      uint32_t f3, long long* iters) {
  uint32_t ns0 = ~0u, ns1 = ~0u, ns2 = ~0u, ns3 = ~0u;
  uint4 r = *reinterpret_cast<const uint4*>(s.sup + root * NWP);
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(s.supc);
  int sp = 0;
  for (;;) {
    uint4 nr;
    int v;
    uint32_t hit;
    dfs_step4(r, base, ns0, ns1, ns2, ns3, f0, f1, f2, f3, nr, v, hit);
    if (__builtin_expect(v >= 128, 0)) {
      if (sp == 0) return -1;
      --sp;
      r = *reinterpret_cast<const uint4*>(sp == 0 ? s.sup + root * NWP
                                                  : s.supc + s.pick[sp - 1] * NWP);
      continue;
    }
    s.pick[sp] = (int16_t)v;
    if (hit) return sp;
    ++sp;
    r = nr;
  }
}


// Variant 4: the whole search loop as one PTX block (2x unrolled, no
// register copies, branch-free step, out-of-line backtrack).
#define DFS_STEP(R0, R1, R2, R3, N0, N1, N2, N3)                      \
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
  "ld.volatile.shared.v4.u32 {" N0 ", " N1 ", " N2 ", " N3 "}, [ad];\n\t"      \
  "sub.u32 t, ad, bb0;\n\t"                                           \
  "shr.u32 v, t, 4;\n\t"                                              \
  "setp.gt.u32 pn, v, 127;\n\t"                                       \
  "@pn bra.uni DFS_BACK;\n\t"                                         \
  "and.b32 t, v, 31;\n\t"                                             \
  "shr.u32 b, hb, t;\n\t"                                             \
  "shr.u32 w, v, 5;\n\t"                                              \
  "setp.eq.u32 q0, w, 0;\n\t"                                         \
  "setp.eq.u32 q1, w, 1;\n\t"                                         \
  "setp.eq.u32 q2, w, 2;\n\t"                                         \
  "setp.eq.u32 q3, w, 3;\n\t"                                         \
  "setp.lt.u32 ql, w, 2;\n\t"                                         \
  "selp.b32 fa, %4, %5, q0;\n\t"                                      \
  "selp.b32 fb, %6, %7, q2;\n\t"                                      \
  "selp.b32 fw, fa, fb, ql;\n\t"                                      \
  "and.b32 fw, fw, b;\n\t"                                            \
  "not.b32 b, b;\n\t"                                                 \
  "@q0 and.b32 ns0, ns0, b;\n\t"                                      \
  "@q1 and.b32 ns1, ns1, b;\n\t"                                      \
  "@q2 and.b32 ns2, ns2, b;\n\t"                                      \
  "@q3 and.b32 ns3, ns3, b;\n\t"                                      \
  "mad.lo.u32 pa, %0, 2, %3;\n\t"                                     \
  "st.shared.u16 [pa], v;\n\t"                                        \
  "setp.ne.u32 ph, fw, 0;\n\t"                                        \
  "@ph bra.uni DFS_DONE;\n\t"                                         \
  "add.u32 %0, %0, 1;\n\t"

__device__ __noinline__ int dfs_v4(uint32_t root_addr, uint32_t base, uint32_t pick_addr,
                                   uint32_t f0, uint32_t f1, uint32_t f2, uint32_t f3) {
  int sp = 0;
  asm volatile(
      "{\n\t"
      ".reg .pred p0, p2, p01, q0, q1, q2, q3, ql, pn, ph, pz;\n\t"
      ".reg .b32 r0, r1, r2, r3, n0, n1, n2, n3, ns0, ns1, ns2, ns3;\n\t"
      ".reg .b32 x0, x1, x2, x3, z0, z1, z2, z3, a0, a1, a2, a3;\n\t"
      ".reg .b32 s01, s23, ad, t, v, b, w, fa, fb, fw, pa, hb, bb0, bb1, bb2, bb3;\n\t"
      "mov.b32 ns0, -1;\n\t"
      "mov.b32 ns1, -1;\n\t"
      "mov.b32 ns2, -1;\n\t"
      "mov.b32 ns3, -1;\n\t"
      "mov.b32 hb, 0x80000000;\n\t"
      "mov.b32 bb0, %2;\n\t"
      "add.u32 bb1, %2, 512;\n\t"
      "add.u32 bb2, %2, 1024;\n\t"
      "add.u32 bb3, %2, 1536;\n\t"
      "ld.shared.v4.u32 {r0, r1, r2, r3}, [%1];\n\t"
      "DFS_LOOP:\n\t"
      DFS_STEP("r0", "r1", "r2", "r3", "n0", "n1", "n2", "n3")
      DFS_STEP("n0", "n1", "n2", "n3", "r0", "r1", "r2", "r3")
      "bra.uni DFS_LOOP;\n\t"
      "DFS_BACK:\n\t"
      "setp.eq.u32 pz, %0, 0;\n\t"
      "@pz bra.uni DFS_FAIL;\n\t"
      "sub.u32 %0, %0, 1;\n\t"
      "setp.eq.u32 pz, %0, 0;\n\t"
      "mov.b32 ad, %1;\n\t"
      "@pz bra.uni DFS_RELOAD;\n\t"
      "mad.lo.u32 pa, %0, 2, %3;\n\t"
      "ld.shared.u16 t, [pa+-2];\n\t"
      "mad.lo.u32 ad, t, 16, bb0;\n\t"
      "DFS_RELOAD:\n\t"
      "ld.shared.v4.u32 {r0, r1, r2, r3}, [ad];\n\t"
      "bra.uni DFS_LOOP;\n\t"
      "DFS_FAIL:\n\t"
      "mov.b32 %0, -1;\n\t"
      "DFS_DONE:\n\t"
      "}"
      : "+r"(sp)
      : "r"(root_addr), "r"(base), "r"(pick_addr), "r"(f0), "r"(f1), "r"(f2), "r"(f3)
      : "memory");
  return sp;
}

__global__ void bench_kernel(int variant, const uint32_t* g_sup, const int16_t* g_cm,
                             const int* roots, int nroots, int n, int reps,
                             long long* cycles, long long* iters, int* depths) {
  extern __shared__ __align__(16) char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Sh s = dec_carve_t<NWv>(sm + warp * dec_smem_bytes_t<NWv>(n), n);
  const int inst = blockIdx.x * (blockDim.x >> 5) + warp;
  const uint32_t* gs = g_sup + (size_t)inst * n * NWP;
  const int16_t* gc = g_cm + (size_t)inst * n;
  for (int i = lane; i < n * NWP; i += 32) s.sup[i] = gs[i];
  for (int v = lane; v < n; v += 32) s.cm[v] = gc[v];
  if (lane < NWP) s.freeb[lane] = 0u;
  __syncwarp();
  for (int v = lane; v < n; v += 32) {
    const int r = s.cm[v];
    for (int w = 0; w < NWP; ++w) s.supc[v * NWP + w] = r >= 0 ? s.sup[r * NWP + w] : 0u;
    if (r < 0) atomicOr(&s.freeb[colword(v)], colbit(v));
  }
  __syncwarp();
  if (lane != 0) return;
  const uint64_t* fq = reinterpret_cast<const uint64_t*>(s.freeb);
  const uint32_t f0 = s.freeb[1], f1 = s.freeb[0], f2 = s.freeb[3], f3 = s.freeb[2];
  long long it = 0;
  int dsum = 0;
  const long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    for (int q = 0; q < nroots; ++q) {
      const int root = roots[(inst * 7 + q) % nroots];
      int d;
      if (variant == 0) {
        d = dfs_search<NWv>(s, root, fq[0], fq[1]);
        it += d + 1;  // path steps only (backtracks not counted here)
      } else if (variant == 1) {
        long long dummy = 0;
        d = dfs_v1(s, root, f0, f1, f2, f3, &dummy);
        it += d + 1;
      } else if (variant == 4) {
        d = dfs_v4((uint32_t)__cvta_generic_to_shared(s.sup + root * NWP),
                   (uint32_t)__cvta_generic_to_shared(s.supc),
                   (uint32_t)__cvta_generic_to_shared(s.pick), f0, f1, f2, f3);
        it += d + 1;
      } else if (variant == 3) {
        long long dummy = 0;
        d = dfs_v3(s, root, f0, f1, f2, f3, &dummy);
        it += d + 1;
      } else {
        long long dummy = 0;
        d = dfs_v2(s, root, f0, f1, f2, f3, &dummy);
        it += d + 1;
      }
      dsum += d * 131 + s.pick[d > 0 ? d : 0];
    }
  }
  const long long t1 = clock64();
  cycles[inst] = t1 - t0;
  iters[inst] = it;
  depths[inst] = dsum;
}

}  // namespace

int main() {
  const int n = 128, ninst = 148 * 7, nroots = 64, reps = 20;
  std::vector<uint32_t> sup((size_t)ninst * n * NWP);
  std::vector<int16_t> cm((size_t)ninst * n);
  std::vector<int> roots(nroots);
  srand(1);
  for (int i = 0; i < ninst; ++i) {
    // random permutation matching with one free column; dense 40% support
    std::vector<int> perm(n);
    for (int v = 0; v < n; ++v) perm[v] = v;
    for (int v = n - 1; v > 0; --v) std::swap(perm[v], perm[rand() % (v + 1)]);
    const int freec = rand() % n;
    for (int v = 0; v < n; ++v) cm[(size_t)i * n + v] = (int16_t)(v == freec ? -1 : perm[v]);
    for (int u = 0; u < n; ++u)
      for (int v = 0; v < n; ++v)
        if ((rand() % 100) < 40) {
          uint32_t* row = &sup[((size_t)i * n + u) * NWP];
          row[(v >> 5) ^ 1] |= 0x80000000u >> (v & 31);
        }
  }
  for (int q = 0; q < nroots; ++q) roots[q] = rand() % n;
  uint32_t* d_sup; int16_t* d_cm; int* d_roots; long long *d_cyc, *d_it; int* d_dep;
  cudaMalloc(&d_sup, sup.size() * 4); cudaMalloc(&d_cm, cm.size() * 2);
  cudaMalloc(&d_roots, nroots * 4);
  cudaMalloc(&d_cyc, ninst * 8); cudaMalloc(&d_it, ninst * 8); cudaMalloc(&d_dep, ninst * 4);
  cudaMemcpy(d_sup, sup.data(), sup.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_cm, cm.data(), cm.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(d_roots, roots.data(), nroots * 4, cudaMemcpyHostToDevice);
  const int wpb = 4;
  const size_t smem = dec_smem_bytes_t<NWv>(n) * wpb;
  std::vector<int> dep0;
  for (int variant = 0; variant < 5; ++variant) {
    for (int pass = 0; pass < 2; ++pass) {
      bench_kernel<<<ninst / wpb, wpb * 32, smem>>>(variant, d_sup, d_cm, d_roots, nroots, n,
                                                     reps, d_cyc, d_it, d_dep);
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<long long> cyc(ninst), it(ninst);
    std::vector<int> dep(ninst);
    cudaMemcpy(cyc.data(), d_cyc, ninst * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(it.data(), d_it, ninst * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(dep.data(), d_dep, ninst * 4, cudaMemcpyDeviceToHost);
    double c = 0, s = 0;
    for (int i = 0; i < ninst; ++i) { c += cyc[i]; s += it[i]; }
    bool same = true;
    if (variant == 0) dep0 = dep;
    else for (int i = 0; i < ninst; ++i) same &= dep[i] == dep0[i];
    printf("variant %d: %.1f cycles/step (%.0f steps/search)%s\n", variant, c / s,
           s / ninst / reps / nroots, same ? "" : "  MISMATCH");
  }
  return 0;
}
