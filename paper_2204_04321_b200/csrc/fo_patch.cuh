// fo_patch.cuh -- pieces shared by the owner-computes patch kernels of the
// wedge path (fo_owner.cu) and of the hexahedral path (fo_hex.cu): the view of
// the patch plan, the one-shot bulk copy of a patch's plan into shared memory,
// and the emission of one (column, slot) pair's sums into the CSR values
// ("KA-patch").
#pragma once
#include <cuda_runtime.h>

#include "fo_internal.h"

namespace fo {

struct PlanView {
  const int32_t* __restrict__ t_begin;
  const int32_t* __restrict__ col_ptr;
  const int32_t* __restrict__ pair_ptr;
  const int32_t* __restrict__ nedge;
  const uint8_t* __restrict__ blob;      // per-patch plan blobs (fo_plan.cpp)
  const int64_t* __restrict__ blob_off;
  double* partials;   // multi columns' partial blocks (fo_plan.cpp)
  int p_off;          // patch of block 0 (a launch covers patches p_off .. p_off + gridDim.x - 1)
  // KA-ws in-kernel zero fill (inkz != 0, single launch over all patches):
  // patches are taken in ticket order (flags[n_patches]), each zero-fills the
  // boundary columns it leads (zl), raises flags[p], and waits for the flags
  // of the leads of its other boundary columns (wl)
  const int32_t* __restrict__ zl;
  const int32_t* __restrict__ zl_ptr;
  const int32_t* __restrict__ wl;
  const int32_t* __restrict__ wl_ptr;
  int32_t* flags;     // [n_patches + 3]: per-patch zero-fill flags | ticket | boundary-done count | ready
  int inkz;
  int n_patches;
  // fused halo (trig != 0, fo_assemble_jacobian_halo): the last of the n_bnd
  // boundary patches (tickets 0 .. n_bnd-1) runs the fix-up of the multi
  // records 0 .. n_multi_bnd-1 and raises flags[n_patches + 2], which the
  // halo's side stream waits on before sending the ghost rows
  const MultiRec* __restrict__ multi;
  int trig, n_bnd, n_multi_bnd;
};

// one-shot bulk copy global -> shared with an mbarrier (TMA, non-tensor):
// bulk_init by one thread, a CTA barrier, then bulk_load by that thread
__device__ __forceinline__ void bulk_init(uint64_t* bar) {
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(d), "l"(src), "r"(bytes), "r"(b) : "memory");
}
__device__ __forceinline__ void bulk_wait(uint64_t* bar) {
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(b) : "memory");
}

// L2 eviction-priority hints (FO_L2HINT bits, default 1 | 8): 1 = the
// interior stores stream (evict_first: never re-read by the kernel; C3 DRAM
// 3.07 -> 2.77 GB per launch, 1.301 -> 1.294 ms), 8 = the wedge kernel's
// in-kernel zero fill stays (evict_last: a later patch's RED reads the line;
// 2.76 -> 2.62 GB, 1.276 -> 1.273 ms; not for the hexahedral kernel, 5.32 ->
// 5.37 ms), 2 = the zero fill and the REDs evict_last (2.65 GB but 1.308 ms,
// not kept); profiles/r02ah_variants_l2hint.txt, r02aj_variants_zl.txt
#ifndef FO_L2HINT
#define FO_L2HINT 9
#endif
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void red_add(double* p, double v) {
  if (FO_L2HINT & 2)
    asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v),
                 "l"(l2_policy_last()) : "memory");
  else
    asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
// the in-kernel zero fill's stores
__device__ __forceinline__ void zero2(double2* p) {
  if (FO_L2HINT & (2 | 8))   // 8: the zero fill alone (experiment)
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %1}, %2;" ::"l"(p), "d"(0.0), "l"(l2_policy_last())
                 : "memory");
  else
    *p = make_double2(0.0, 0.0);
}

// The patch's plan in shared memory.
struct SmemPlan {
  const PlanCol* cols;
  const PlanPair* pairs;
  const uint32_t* contrib;
  int ncols, npairs;
  int nedge;   // pairs [0, nedge): edge slots, exactly two entries each
};

__device__ __forceinline__ void put2(double* dst, double x, double y, bool interior) {
  if (interior) {
    if (FO_L2HINT & 1)
      asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(dst), "d"(x), "d"(y),
                   "l"(l2_policy_first()) : "memory");
    else
      *reinterpret_cast<double2*>(dst) = make_double2(x, y);
  } else {
    red_add(dst, x);
    red_add(dst + 1, y);
  }
}

// The 12 sums of one (column, slot) pair: level-kk rows x column level kk
// (dg, from D), level-kk rows x level kk+1 (up, from O), level-kk+1 rows x
// level kk (nx, from O transposed); [row comp a][column comp b].
struct PairSums {
  double dg[4], up[4], nx[4];
};

// write one pair's sums: plain stores (interior column) or RED (boundary),
// or the patch's partial block (self slot of a multi column)
template <bool UP>
__device__ __forceinline__ void emit(const PlanPair& pp, const PlanCol& pc, const PairSums& s, int kk, int L,
                                     double* __restrict__ vals, double* __restrict__ partials) {
  const int m0 = (kk == 0 || kk == L) ? 2 : 3;           // column groups of level-kk rows
  const int m1 = (kk + 1 == L) ? 2 : 3;                   // column groups of level-kk+1 rows
  const int P0 = kk == 0 ? 0 : 3 * kk - 1, P1 = 3 * kk + 2;
  const int g0 = kk == 0 ? 0 : 2;                          // offset of group kk in a kk-row slot
  const int nc = pc.info & 255;
  const bool interior = (pc.info >> 8) & 1;
  if (((pc.info >> 30) & 1) && pp.slot == ((pc.info >> 9) & 255)) {
    double2* q = reinterpret_cast<double2*>(partials + (int64_t(pc.pad) * (L + 1) + kk) * kPartialStride);
    q[0] = make_double2(s.dg[0], s.dg[1]);
    q[1] = make_double2(s.dg[2], s.dg[3]);
    if (UP) {
      q[2] = make_double2(s.up[0], s.up[1]);
      q[3] = make_double2(s.up[2], s.up[3]);
      q[4] = make_double2(s.nx[0], s.nx[1]);
      q[5] = make_double2(s.nx[2], s.nx[3]);
    }
    return;
  }
  double* d0 = vals + pc.colstart + int64_t(4 * nc) * P0 + int64_t(pp.slot) * (2 * m0) + g0;
  double* d1 = d0 + 2 * nc * m0;
  put2(d0, s.dg[0], s.dg[1], interior);
  put2(d1, s.dg[2], s.dg[3], interior);
  if (UP) {
    put2(d0 + 2, s.up[0], s.up[1], interior);
    put2(d1 + 2, s.up[2], s.up[3], interior);
    double* e0 = vals + pc.colstart + int64_t(4 * nc) * P1 + int64_t(pp.slot) * (2 * m1);
    put2(e0, s.nx[0], s.nx[1], interior);
    put2(e0 + 2 * nc * m1, s.nx[2], s.nx[3], interior);
  }
}


}  // namespace fo
