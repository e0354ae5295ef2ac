// fo_tmem.cuh -- tensor-memory (TMEM) load / store helpers for per-thread
// private scratch.  With the 32x32b shape, warp w of a
// warpgroup reads / writes TMEM lanes 32 (w % 4) .. 32 (w % 4) + 31, one lane
// per thread: every thread of the element warpgroup owns one 256-column TMEM
// row (1 KB), measured at 585 B/clk/SM for st + ld against 128 B/clk/SM of
// shared memory (profiles/r02_microbench_tmem.txt).  tcgen05.ld / st are
// warp-collective (.sync.aligned): all 32 lanes execute them convergently.
// Chunk sizes 1..16 doubles (x2..x32 columns); the st/ld variants are written out.
#pragma once
#include <cstdint>

namespace fo {
namespace tmem {

__device__ __forceinline__ uint32_t lo32(double x) { return uint32_t(__double2loint(x)); }
__device__ __forceinline__ uint32_t hi32(double x) { return uint32_t(__double2hiint(x)); }
__device__ __forceinline__ double mk(uint32_t lo, uint32_t hi) { return __hiloint2double(int(hi), int(lo)); }

// store 1 double(s) v[0..1) at TMEM address ta (lane in bits 31:16, column in 15:0)
__device__ __forceinline__ void st1(uint32_t ta, const double* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};"
               :: "r"(ta), "r"(lo32(v[0])), "r"(hi32(v[0])) : "memory");
}
// load 1 double(s) into v[0..1) and wait for them (ld + wait::ld in one statement,
// so no use of the destination registers can be scheduled before the wait)
__device__ __forceinline__ void ld1(uint32_t ta, double* v) {
  uint32_t r[2];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n\t"
               "tcgen05.wait::ld.sync.aligned;"
               : "=r"(r[0]), "=r"(r[1]) : "r"(ta) : "memory");
#pragma unroll
  for (int i = 0; i < 1; ++i) v[i] = mk(r[2 * i], r[2 * i + 1]);
}
// store 2 double(s) v[0..2) at TMEM address ta (lane in bits 31:16, column in 15:0)
__device__ __forceinline__ void st2(uint32_t ta, const double* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};"
               :: "r"(ta), "r"(lo32(v[0])), "r"(hi32(v[0])), "r"(lo32(v[1])), "r"(hi32(v[1])) : "memory");
}
// load 2 double(s) into v[0..2) and wait for them (ld + wait::ld in one statement,
// so no use of the destination registers can be scheduled before the wait)
__device__ __forceinline__ void ld2(uint32_t ta, double* v) {
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n\t"
               "tcgen05.wait::ld.sync.aligned;"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(ta) : "memory");
#pragma unroll
  for (int i = 0; i < 2; ++i) v[i] = mk(r[2 * i], r[2 * i + 1]);
}
// store 4 double(s) v[0..4) at TMEM address ta (lane in bits 31:16, column in 15:0)
__device__ __forceinline__ void st4(uint32_t ta, const double* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "r"(ta), "r"(lo32(v[0])), "r"(hi32(v[0])), "r"(lo32(v[1])), "r"(hi32(v[1])), "r"(lo32(v[2])), "r"(hi32(v[2])), "r"(lo32(v[3])), "r"(hi32(v[3])) : "memory");
}
// load 4 double(s) into v[0..4) and wait for them (ld + wait::ld in one statement,
// so no use of the destination registers can be scheduled before the wait)
__device__ __forceinline__ void ld4(uint32_t ta, double* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t"
               "tcgen05.wait::ld.sync.aligned;"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(ta) : "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = mk(r[2 * i], r[2 * i + 1]);
}
// store 8 double(s) v[0..8) at TMEM address ta (lane in bits 31:16, column in 15:0)
__device__ __forceinline__ void st8(uint32_t ta, const double* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               :: "r"(ta), "r"(lo32(v[0])), "r"(hi32(v[0])), "r"(lo32(v[1])), "r"(hi32(v[1])), "r"(lo32(v[2])), "r"(hi32(v[2])), "r"(lo32(v[3])), "r"(hi32(v[3])), "r"(lo32(v[4])), "r"(hi32(v[4])), "r"(lo32(v[5])), "r"(hi32(v[5])), "r"(lo32(v[6])), "r"(hi32(v[6])), "r"(lo32(v[7])), "r"(hi32(v[7])) : "memory");
}
// load 8 double(s) into v[0..8) and wait for them (ld + wait::ld in one statement,
// so no use of the destination registers can be scheduled before the wait)
__device__ __forceinline__ void ld8(uint32_t ta, double* v) {
  uint32_t r[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
               "tcgen05.wait::ld.sync.aligned;"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) : "r"(ta) : "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = mk(r[2 * i], r[2 * i + 1]);
}
// store 16 double(s) v[0..16) at TMEM address ta (lane in bits 31:16, column in 15:0)
__device__ __forceinline__ void st16(uint32_t ta, const double* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
               :: "r"(ta), "r"(lo32(v[0])), "r"(hi32(v[0])), "r"(lo32(v[1])), "r"(hi32(v[1])), "r"(lo32(v[2])), "r"(hi32(v[2])), "r"(lo32(v[3])), "r"(hi32(v[3])), "r"(lo32(v[4])), "r"(hi32(v[4])), "r"(lo32(v[5])), "r"(hi32(v[5])), "r"(lo32(v[6])), "r"(hi32(v[6])), "r"(lo32(v[7])), "r"(hi32(v[7])), "r"(lo32(v[8])), "r"(hi32(v[8])), "r"(lo32(v[9])), "r"(hi32(v[9])), "r"(lo32(v[10])), "r"(hi32(v[10])), "r"(lo32(v[11])), "r"(hi32(v[11])), "r"(lo32(v[12])), "r"(hi32(v[12])), "r"(lo32(v[13])), "r"(hi32(v[13])), "r"(lo32(v[14])), "r"(hi32(v[14])), "r"(lo32(v[15])), "r"(hi32(v[15])) : "memory");
}
// load 16 double(s) into v[0..16) and wait for them (ld + wait::ld in one statement,
// so no use of the destination registers can be scheduled before the wait)
__device__ __forceinline__ void ld16(uint32_t ta, double* v) {
  uint32_t r[32];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
               "tcgen05.wait::ld.sync.aligned;"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]) : "r"(ta) : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = mk(r[2 * i], r[2 * i + 1]);
}
// N doubles at column offset col (2 columns per double), as power-of-two chunks
template <int N>
__device__ __forceinline__ void st(uint32_t ta, const double* v) {
  if constexpr (N >= 16) { st16(ta, v); st<N - 16>(ta + 32, v + 16); }
  else if constexpr (N >= 8) { st8(ta, v); st<N - 8>(ta + 16, v + 8); }
  else if constexpr (N >= 4) { st4(ta, v); st<N - 4>(ta + 8, v + 4); }
  else if constexpr (N >= 2) { st2(ta, v); st<N - 2>(ta + 4, v + 2); }
  else if constexpr (N == 1) { st1(ta, v); }
}
template <int N>
__device__ __forceinline__ void ld(uint32_t ta, double* v) {
  if constexpr (N >= 16) { ld16(ta, v); ld<N - 16>(ta + 32, v + 16); }
  else if constexpr (N >= 8) { ld8(ta, v); ld<N - 8>(ta + 16, v + 8); }
  else if constexpr (N >= 4) { ld4(ta, v); ld<N - 4>(ta + 8, v + 4); }
  else if constexpr (N >= 2) { ld2(ta, v); ld<N - 2>(ta + 4, v + 2); }
  else if constexpr (N == 1) { ld1(ta, v); }
}
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// allocation (one warp), relinquish, and the fences around the CTA barrier
// that publishes the base address
__device__ __forceinline__ void alloc(uint32_t* smem_dst, uint32_t ncols) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(a), "r"(ncols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

}  // namespace tmem
}  // namespace fo
