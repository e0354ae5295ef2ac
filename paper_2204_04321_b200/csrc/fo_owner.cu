// fo_owner.cu -- KA-patch: owner-computes residual (+ Jacobian) assembly
// (DESIGN.md "KA-patch").  PAPER.md P:177-183 (gather, interpolate,
// evaluate, scatter) fused into one kernel; the scatter writes every CSR value
// of an interior column exactly once with coalesced plain stores (the
// overwrite semantics of fo_assemble_jacobian), boundary columns with RED.
//
// One CTA = one patch of <= kPatchTris consecutive triangles, one thread per
// triangle column, layers k = 0..L-1 in order.  Per layer:
//   phase A  each thread evaluates wedge (t,k) in registers (fo_element.cuh)
//            and publishes to shared memory (SoA, [entry][triangle]):
//              D  += bottom-bottom block + bottom residual  (D already holds
//                    the top-top block + top residual of wedge k-1: the
//                    vertical merge of the shared level k)
//              O[k&1] = bottom-top block (rows level k, columns level k+1)
//   phase B  every warp takes whole columns of the patch; lanes walk the
//            contiguous level-k segment of the column's two rows (u, v) and
//            gather each double2 (b = 0,1) from D / O[k&1] / O[(k-1)&1]^T
//            through the plan's per-slot contribution lists.
//   then the thread stores its held top-top block into D for layer k+1.
// A final phase B writes the surface level L.
#include <cuda_runtime.h>

#include "fo_element.cuh"
#include "fo_element_v4.cuh"
#include "fo_element_tet.cuh"
#include "fo_element_ws.cuh"

#include <functional>
#include <type_traits>
#include "fo_internal.h"
#include "fo_kernels.cuh"
#include "fo_patch.cuh"

namespace fo {




constexpr int TP = kPatchStride;   // SoA row stride (threads per CTA: kPatchTris)
constexpr int kD = 27;   // level-k diagonal block (21, 2x2-block layout) + 6 residual
constexpr int kO = 36;   // 6x6 bottom-top block of wedge k
constexpr int kC = 36;   // compact per-point scratch (6 x 6 quadrature points)
constexpr int kSlotsPerTri = kD + kO + kC;
// byte offset of the plan in dynamic shared memory (16-byte aligned for the bulk copy)
constexpr int kPlanOffset = (kSlotsPerTri * TP * 8 + 15) / 16 * 16;
// residual only (KR): the residual slots of D (6) and the compact scratch, so
// three CTAs fit an SM (shared memory and <= 168 registers)
constexpr int kDR = 6;
constexpr int kPlanOffsetR = ((kDR + kC) * TP * 8 + 15) / 16 * 16;
constexpr int kPatchCtasPerSmR = 3;





// Phase B for wedge layer k (kk = k < L) or the surface (kk = L, D only).
// One thread per (column, slot) pair walks the slot's contributions once and
// gathers: level-kk rows, column level kk (from D) and kk+1 (from O); level
// kk+1 rows, column level kk (from O transposed).  The level-kk rows' column
// level kk-1 part was written by the previous call (partial rows, completed
// in L2).  Edge pairs (1-2 contributions) come first in the plan, self pairs
// (one contribution per fan triangle) last, so loop lengths in a warp are
// nearly uniform; consecutive slots of a column sit on consecutive lanes.

// one gather step over the two contributions c2: FIRST sets s = a + b (the
// same double as (0 + a) + b, one add fewer), later steps add a, then b
template <bool UP, bool FIRST>
__device__ __forceinline__ void gather2(uint2 c2, const double* D, const double* O, PairSums& s) {
  const int tla = int(c2.x & 255), tlb = int(c2.y & 255);
  const int pata = int((c2.x >> 13) & 3), patb = int((c2.y >> 13) & 3);
  const int saa = pata == 1 ? 2 * TP : TP, sba = pata == 2 ? 2 * TP : TP;
  const int sab = patb == 1 ? 2 * TP : TP, sbb = patb == 2 ? 2 * TP : TP;
  const double* Da = D + int((c2.x >> 8) & 31) * TP + tla;
  const double* Db = D + int((c2.y >> 8) & 31) * TP + tlb;
  if (FIRST) {
    s.dg[0] = Da[0] + Db[0];
    s.dg[1] = Da[sba] + Db[sbb];
    s.dg[2] = Da[saa] + Db[sab];
    s.dg[3] = Da[saa + sba] + Db[sab + sbb];
  } else {
    s.dg[0] = (s.dg[0] + Da[0]) + Db[0];
    s.dg[1] = (s.dg[1] + Da[sba]) + Db[sbb];
    s.dg[2] = (s.dg[2] + Da[saa]) + Db[sab];
    s.dg[3] = (s.dg[3] + Da[saa + sba]) + Db[sab + sbb];
  }
  if (UP) {
    const double* Oua = O + int((c2.x >> 15) & 31) * TP + tla;
    const double* Ona = O + int((c2.x >> 20) & 31) * TP + tla;
    const double* Oub = O + int((c2.y >> 15) & 31) * TP + tlb;
    const double* Onb = O + int((c2.y >> 20) & 31) * TP + tlb;
    constexpr int ou[4] = {0, TP, 6 * TP, 7 * TP}, on[4] = {0, 6 * TP, TP, 7 * TP};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (FIRST) {
        s.up[i] = Oua[ou[i]] + Oub[ou[i]];
        s.nx[i] = Ona[on[i]] + Onb[on[i]];
      } else {
        s.up[i] = (s.up[i] + Oua[ou[i]]) + Oub[ou[i]];
        s.nx[i] = (s.nx[i] + Ona[on[i]]) + Onb[on[i]];
      }
    }
  }
}

template <bool UP>
__device__ __forceinline__ void phase_b_j(const SmemPlan& sp, int kk, int L, const double* D,
                                          const double* O, double* __restrict__ vals,
                                          double* __restrict__ partials, int tid, int nthr) {
  // edge pairs (exactly two entries) first, then self pairs (one entry per
  // fan triangle, padded to even); a variant gathering two edge pairs per
  // thread at a time measured slower (1.98 vs 1.91 ms)
  for (int pi = tid; pi < sp.npairs; pi += nthr) {
    const PlanPair pp = sp.pairs[pi];
    PairSums s;
    const uint32_t* cp = sp.contrib + pp.off - 2;   // even count >= 2, 8-byte aligned
    gather2<UP, true>(make_uint2(pp.c0, pp.c1), D, O, s);
    for (int e = 2; e < pp.cnt; e += 2) gather2<UP, false>(*reinterpret_cast<const uint2*>(cp + e), D, O, s);
    emit<UP>(pp, sp.cols[pp.col], s, kk, L, vals, partials);
  }
}

// Dr: the residual slots (D + 21 TP in the R + J layout, the whole D of KR)
__device__ __forceinline__ void phase_b_r(const SmemPlan& sp, int kk, int L, const double* Dr,
                                          double* __restrict__ R, double* __restrict__ partials, int tid,
                                          int nthr) {
  for (int ci = tid; ci < sp.ncols; ci += nthr) {
    const PlanCol& pc = sp.cols[ci];
    double r0, r1;
    {   // self lists hold >= 2 entries (padded to even): first step r = a + b
      const uint2 c2 = *reinterpret_cast<const uint2*>(sp.contrib + pc.self_off);
      const double* Da = Dr + 2 * int((c2.x >> 25) & 3) * TP + int(c2.x & 255);
      const double* Db = Dr + 2 * int((c2.y >> 25) & 3) * TP + int(c2.y & 255);
      r0 = Da[0] + Db[0];
      r1 = Da[TP] + Db[TP];
    }
    for (int e = pc.self_off + 2; e < pc.self_off + pc.self_cnt; e += 2) {
      const uint2 c2 = *reinterpret_cast<const uint2*>(sp.contrib + e);
      const double* Da = Dr + 2 * int((c2.x >> 25) & 3) * TP + int(c2.x & 255);
      const double* Db = Dr + 2 * int((c2.y >> 25) & 3) * TP + int(c2.y & 255);
      r0 += Da[0];
      r1 += Da[TP];
      r0 += Db[0];
      r1 += Db[TP];
    }
    if ((pc.info >> 30) & 1)
      *reinterpret_cast<double2*>(partials + (int64_t(pc.pad) * (L + 1) + kk) * kPartialStride + 12) =
          make_double2(r0, r1);
    else
      put2(R + 2 * (int64_t(pc.c) * (L + 1) + kk), r0, r1, (pc.info >> 8) & 1);
  }
}

template <bool NEED_J>
__device__ __forceinline__ void phase_b(const SmemPlan& sp, int kk, int L, const double* D,
                                        const double* O, double* __restrict__ R,
                                        double* __restrict__ vals, double* __restrict__ partials,
                                        int tid, int nthr) {
  if (NEED_J) {
    if (kk < L) phase_b_j<true>(sp, kk, L, D, O, vals, partials, tid, nthr);
    else phase_b_j<false>(sp, kk, L, D, O, vals, partials, tid, nthr);
  }
  phase_b_r(sp, kk, L, NEED_J ? D + 21 * TP : D, R, partials, tid, nthr);
}

// Sink of wedge_element_v4: bottom parts added to D and O in shared memory,
// the top (level k+1) block and residual held in registers.
struct PatchSink {
  double* D;
  double* O;
  int tl;
  double held[27];   // dmap layout
  __device__ __forceinline__ void r_bot_add(int p, double v) { D[(21 + p) * TP + tl] += v; }
  __device__ __forceinline__ void bot_add(int p, int p2, double v) { D[dmap(p, p2) * TP + tl] += v; }
  __device__ __forceinline__ void off(int p, int p2, double v) { O[(6 * p + p2) * TP + tl] = v; }
  __device__ __forceinline__ void off_add(int p, int p2, double v) { O[(6 * p + p2) * TP + tl] += v; }
  __device__ __forceinline__ double off_get(int p, int p2) const { return O[(6 * p + p2) * TP + tl]; }
  __device__ __forceinline__ double bot_get(int p, int p2) const { return D[dmap(p, p2) * TP + tl]; }
  __device__ __forceinline__ void bot_set(int p, int p2, double v) { D[dmap(p, p2) * TP + tl] = v; }
  __device__ __forceinline__ double top_get(int i) const {
    double v = 0.0;
#pragma unroll
    for (int p = 0; p < 6; ++p)
#pragma unroll
      for (int p2 = p; p2 < 6; ++p2)
        if (pk6(p, p2) == i) v = held[dmap(p, p2)];
    return v;
  }
  __device__ __forceinline__ void top(int i, double v) {
    // i is the packed upper-triangle index pk6(p, p2)
#pragma unroll
    for (int p = 0; p < 6; ++p)
#pragma unroll
      for (int p2 = p; p2 < 6; ++p2)
        if (pk6(p, p2) == i) held[dmap(p, p2)] = v;
  }
  __device__ __forceinline__ void top_add(int i, double v) {
#pragma unroll
    for (int p = 0; p < 6; ++p)
#pragma unroll
      for (int p2 = p; p2 < 6; ++p2)
        if (pk6(p, p2) == i) held[dmap(p, p2)] += v;
  }
  __device__ __forceinline__ void r_top(int p, double v) { held[21 + p] = v; }
  __device__ __forceinline__ void r_top_add(int p, double v) { held[21 + p] += v; }
};

// residual-only sink: the Jacobian parts of the element are dead code; D is
// the compact KR layout (the 6 residual slots only)
struct PatchSinkR {
  double* D;
  int tl;
  double held[27];
  __device__ __forceinline__ void r_bot_add(int p, double v) { D[p * TP + tl] += v; }
  __device__ __forceinline__ void bot_add(int, int, double) {}
  __device__ __forceinline__ void off(int, int, double) {}
  __device__ __forceinline__ void off_add(int, int, double) {}
  __device__ __forceinline__ double off_get(int, int) const { return 0.0; }
  __device__ __forceinline__ double bot_get(int, int) const { return 0.0; }
  __device__ __forceinline__ void bot_set(int, int, double) {}
  __device__ __forceinline__ double top_get(int) const { return 0.0; }
  __device__ __forceinline__ void top(int, double) {}
  __device__ __forceinline__ void top_add(int, double) {}
  __device__ __forceinline__ void r_top(int p, double v) { held[21 + p] = v; }
  __device__ __forceinline__ void r_top_add(int p, double v) { held[21 + p] += v; }
};

// the thread's compact per-point scratch: 42 doubles at base[i * TP + tl]
struct SmemCmp {
  double* base;
  int tl;
  __device__ __forceinline__ double& operator()(int i) { return base[i * TP + tl]; }
};

template <bool NEED_J, bool N3, bool TET>
__global__ void __launch_bounds__(kPatchTris, NEED_J ? kPatchCtasPerSm : kPatchCtasPerSmR)
ka_patch_kernel(const ColRec* __restrict__ col, const TriRec* __restrict__ tris,
                const double* __restrict__ sigma, const double* __restrict__ Aw, KParams kp,
                PlanView pv, const double* __restrict__ U, double* __restrict__ R,
                double* __restrict__ vals) {
  extern __shared__ __align__(16) double smem[];
  double* const D = smem;                                       // [kD][TP] (KR: [kDR][TP])
  double* const O = smem + kD * TP;                             // [kO][TP] (KR: unused)
  double* const C = smem + (NEED_J ? kD + kO : kDR) * TP;       // [kC][TP]
  const int p = pv.p_off + int(blockIdx.x);
  const int t0 = __ldg(pv.t_begin + p), nt = __ldg(pv.t_begin + p + 1) - t0;
  // the patch's plan -> shared memory (after the value buffers): one bulk
  // copy, issued now and waited for before the first gather phase
  __shared__ uint64_t plan_bar;
  SmemPlan sp;
  {
    const int c0 = __ldg(pv.col_ptr + p), c1 = __ldg(pv.col_ptr + p + 1);
    const int q0 = __ldg(pv.pair_ptr + p), q1 = __ldg(pv.pair_ptr + p + 1);
    const int64_t b0 = __ldg(pv.blob_off + p), b1 = __ldg(pv.blob_off + p + 1);
    char* base = reinterpret_cast<char*>(smem) + (NEED_J ? kPlanOffset : kPlanOffsetR);
    sp.pairs = reinterpret_cast<const PlanPair*>(base);
    sp.cols = reinterpret_cast<const PlanCol*>(base + (q1 - q0) * sizeof(PlanPair));
    sp.contrib = reinterpret_cast<const uint32_t*>(base + (c1 - c0) * sizeof(PlanCol) + (q1 - q0) * sizeof(PlanPair));
    sp.ncols = c1 - c0; sp.npairs = q1 - q0;
    sp.nedge = __ldg(pv.nedge + p);
    if (threadIdx.x == 0) bulk_init(&plan_bar);
    // the mbarrier is initialised before any warp can wait on it (warps without
    // triangles reach the first bulk_wait at once) and before the copy arrives on it
    __syncthreads();
    if (threadIdx.x == 0) bulk_load(base, pv.blob + b0, unsigned(b1 - b0), &plan_bar);
  }
  const int L = kp.L;
  const int tl = threadIdx.x;
  const bool active = tl < nt;
  TriRec tr;
  tr.v[0] = tr.v[1] = tr.v[2] = 0;
  if (active) {
    const int* tp = reinterpret_cast<const int*>(tris + (t0 + tl));
    const int2 v01 = __ldg(reinterpret_cast<const int2*>(tp));
    tr.v[0] = v01.x; tr.v[1] = v01.y; tr.v[2] = __ldg(tp + 2);
#pragma unroll
    for (int i = 0; i < (NEED_J ? kD : kDR); ++i) D[i * TP + tl] = 0.0;
  }
  // triangle slot kPatchTris: the zero column the plan's pad entries read
  if (threadIdx.x < (NEED_J ? kD : kDR)) D[threadIdx.x * TP + kPatchTris] = 0.0;
  if (NEED_J && threadIdx.x < kO) O[threadIdx.x * TP + kPatchTris] = 0.0;
  for (int k = 0; k < L; ++k) {
    typename std::conditional<NEED_J, PatchSink, PatchSinkR>::type sk;
    sk.D = D;
    sk.tl = tl;
    if constexpr (NEED_J) sk.O = O;
    if (active) {
      // re-gather the (L1-resident) column records every layer instead of
      // keeping ~60 registers of triangle geometry live across the layer loop
      const ColRec* colk = col;
      asm volatile("" : "+l"(colk));
      TriGeo geo;
      load_tri_geo(colk, tr, geo);
      const double Afac = wedge_afac(kp, Aw, t0 + tl, k);
      WedgeIn w;
      wedge_input(geo, tr, sigma, Afac, U, L, k, w, kp.go != 0);
      SmemCmp cmp{C, tl};
      if constexpr (TET) tet3_element<N3, true>(w, 0, kp.rg, kp.eps, kp.glen_n, sk);
      else wedge_element_v4<N3>(w, kp.rg, kp.eps, kp.glen_n, sk, cmp);
    }
    if (k == 0) bulk_wait(&plan_bar);
    __syncthreads();
    phase_b<NEED_J>(sp, k, L, D, O, R, vals, pv.partials, threadIdx.x, blockDim.x);
    __syncthreads();
    if (active) {   // the held top block becomes level k+1's diagonal block
      if (NEED_J) {
#pragma unroll
        for (int i = 0; i < kD; ++i) D[i * TP + tl] = sk.held[i];
      } else {
#pragma unroll
        for (int i = 21; i < kD; ++i) D[(i - 21) * TP + tl] = sk.held[i];
      }
    }
  }
  if (L == 0) bulk_wait(&plan_bar);
  __syncthreads();
  phase_b<NEED_J>(sp, L, L, D, O, R, vals, pv.partials, threadIdx.x, blockDim.x);
}

// multi columns: add the patches' partial blocks in patch order and store the
// self-slot entries and the residual; item i = (record i / (L+1), row level)
__device__ __forceinline__ void multi_fixup_one(const MultiRec* __restrict__ mr, int i, int L,
                                                const double* __restrict__ partials, double* __restrict__ R,
                                                double* __restrict__ vals) {
  const int mc = i / (L + 1), kk = i - mc * (L + 1);
  const MultiRec r = mr[mc];
  const bool up = vals && kk < L;
  double s[14];
#pragma unroll
  for (int e = 0; e < 14; ++e) s[e] = 0.0;
  for (int b = 0; b < r.cnt; ++b) {
    const double* q = partials + (int64_t(r.base + b) * (L + 1) + kk) * kPartialStride;
    s[12] += q[12];
    s[13] += q[13];
    if (vals) {
#pragma unroll
      for (int e = 0; e < 4; ++e) s[e] += q[e];
    }
    if (up) {
#pragma unroll
      for (int e = 4; e < 12; ++e) s[e] += q[e];
    }
  }
  *reinterpret_cast<double2*>(R + 2 * (int64_t(r.c) * (L + 1) + kk)) = make_double2(s[12], s[13]);
  if (!vals) return;
  const int nc = r.nc_self & 255, slot = r.nc_self >> 8;
  const int m0 = (kk == 0 || kk == L) ? 2 : 3, m1 = (kk + 1 == L) ? 2 : 3;
  const int P0 = kk == 0 ? 0 : 3 * kk - 1, P1 = 3 * kk + 2;
  const int g0 = kk == 0 ? 0 : 2;
  double* d0 = vals + r.colstart + int64_t(4 * nc) * P0 + int64_t(slot) * (2 * m0) + g0;
  double* d1 = d0 + 2 * nc * m0;
  *reinterpret_cast<double2*>(d0) = make_double2(s[0], s[1]);
  *reinterpret_cast<double2*>(d1) = make_double2(s[2], s[3]);
  if (up) {
    *reinterpret_cast<double2*>(d0 + 2) = make_double2(s[4], s[5]);
    *reinterpret_cast<double2*>(d1 + 2) = make_double2(s[6], s[7]);
    double* e0 = vals + r.colstart + int64_t(4 * nc) * P1 + int64_t(slot) * (2 * m1);
    *reinterpret_cast<double2*>(e0) = make_double2(s[8], s[9]);
    *reinterpret_cast<double2*>(e0 + 2 * nc * m1) = make_double2(s[10], s[11]);
  }
}

// ---------------------------------------------------------------------------
// KA-ws: the warp-specialised patch kernel ("KA-ws").
// Same patch plan, shared layout and scatter (phase B) as ka_patch_kernel, but
// the element and scatter phases run in two warpgroups that overlap:
//   WG0 (threads 0..127, one per triangle, up to kWsRegsE registers): wedge
//        element k+1 (fo_element_ws.cuh) with all its intermediate blocks in
//        the thread's private TMEM row, while
//   WG1 (threads 128..255, kWsRegsB registers): phase B of level k from the
//        shared D / O arrays.
// Handshake per level with two named barriers of 256 threads: EMPTY (WG1
// arrives after its phase B; WG0 waits before overwriting D / O) and FULL (WG0
// arrives after publishing D(k) / O(k); WG1 waits before its phase B).
// element threads per CTA (one per triangle of a patch, rounded up to
// warpgroups) and as many scatter threads; 128-triangle patches: 2 CTAs per
// SM; 255-triangle patches (FO_EXPERIMENT_PATCH255): one 512-thread CTA
constexpr int kWsHalf = kPatchTris <= 128 ? 128 : 256;
constexpr int kWsThreads = 2 * kWsHalf;
constexpr int kWsCtas = kWsHalf == 128 ? 2 : 1;
constexpr uint32_t kWsAlloc = kTmCols * (kWsHalf / 128);   // TMEM columns per CTA
#ifndef FO_WS_REGS_E
#define FO_WS_REGS_E 192
#endif
// setmaxnreg split: E + B = 2 x 128.  192 / 64 (session 3 of round 2): no
// spills in either warpgroup of either instance -- wedges 1.293 -> 1.280 ms
// against 200 / 56 (which left the tetrahedral instance's scatter spilling:
// C3-tet 1.418 -> 1.244 ms), profiles/r02ai_ab_regs.txt, r02ai_ab_tet.txt.
// Earlier kernels: 200 / 56 vs 208 / 48 1.403 vs 1.471 ms (scatter spills),
// 192 / 64 then 1.496 ms (element spills)
constexpr int kWsRegsE = FO_WS_REGS_E, kWsRegsB = 256 - FO_WS_REGS_E;
constexpr int kPlanOffsetWS = ((kD + kO) * TP * 8 + 15) / 16 * 16;
constexpr int kUbufOffsetWS = (kPlanOffsetWS + kPlanBytes + 15) / 16 * 16;   // [3 levels x 3 nodes][TP] double2
constexpr int kWsSmem = kUbufOffsetWS + 9 * TP * 16;
constexpr int kBarEmpty = 1, kBarFull = 2, kBarElem = 3, kBarScat = 4;

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <bool N3, bool TET>
__global__ void __launch_bounds__(kWsThreads, kWsCtas)
ka_ws_kernel(const ColRec* __restrict__ col, const TriRec* __restrict__ tris,
             const double* __restrict__ sigma, const double* __restrict__ Aw, KParams kp, PlanView pv,
             const double* __restrict__ U, double* __restrict__ R, double* __restrict__ vals) {
  extern __shared__ __align__(16) double smem[];
  double* const D = smem;              // [kD][TP]
  double* const O = smem + kD * TP;    // [kO][TP]
  __shared__ uint64_t plan_bar;
  __shared__ uint32_t tmem_base;
  __shared__ int ticket;
  __shared__ int last_bnd;
  if (pv.inkz && threadIdx.x == 0) ticket = atomicAdd(pv.flags + pv.n_patches, 1);
  __syncthreads();
  // with the in-kernel zero fill a CTA's patch is its ticket: a lead patch
  // (lower ticket) belongs to a CTA that is already running, so waiting for it
  // cannot deadlock
  const int p = pv.inkz ? ticket : pv.p_off + int(blockIdx.x);
  const int t0 = __ldg(pv.t_begin + p), nt = __ldg(pv.t_begin + p + 1) - t0;
  SmemPlan sp;
  char* const base = reinterpret_cast<char*>(smem) + kPlanOffsetWS;
  const int64_t b0 = __ldg(pv.blob_off + p), b1 = __ldg(pv.blob_off + p + 1);
  {
    const int c0 = __ldg(pv.col_ptr + p), c1 = __ldg(pv.col_ptr + p + 1);
    const int q0 = __ldg(pv.pair_ptr + p), q1 = __ldg(pv.pair_ptr + p + 1);
    sp.pairs = reinterpret_cast<const PlanPair*>(base);
    sp.cols = reinterpret_cast<const PlanCol*>(base + (q1 - q0) * sizeof(PlanPair));
    sp.contrib = reinterpret_cast<const uint32_t*>(base + (c1 - c0) * sizeof(PlanCol) + (q1 - q0) * sizeof(PlanPair));
    sp.ncols = c1 - c0; sp.npairs = q1 - q0;
    sp.nedge = __ldg(pv.nedge + p);
  }
  if (threadIdx.x == 0) bulk_init(&plan_bar);
  if (threadIdx.x < 32) tmem::alloc(&tmem_base, kWsAlloc);   // warp 0 owns the TMEM allocation
  {   // triangle slot kPatchTris: the zero column the plan's pad entries read
    const int i = int(threadIdx.x) - kWsHalf;
    if (i >= 0 && i < kD) D[i * TP + kPatchTris] = 0.0;
    if (i >= 0 && i < kO) O[i * TP + kPatchTris] = 0.0;
  }
  tmem::fence_before();
  __syncthreads();
  tmem::fence_after();
  if (threadIdx.x == 0) bulk_load(base, pv.blob + b0, unsigned(b1 - b0), &plan_bar);
  const int L = kp.L;
  if (threadIdx.x < kWsHalf) {
    // ---------------- WG0: elements ----------------
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kWsRegsE));
    const int tl = threadIdx.x;
    const bool active = tl < nt;
    // tcgen05.ld / st are warp-collective: lanes without a triangle evaluate a
    // copy of the patch's last one and publish nothing
    const int te = active ? tl : nt - 1;
    // this warp's TMEM lane quarter (and, for a second element warpgroup, its column half)
    const uint32_t tm = tmem_base + (uint32_t(tl & 127 & ~31) << 16) + uint32_t(tl >> 7) * kTmCols;
    TriRec tr;
    {
      const int* tp = reinterpret_cast<const int*>(tris + (t0 + te));
      const int2 v01 = __ldg(reinterpret_cast<const int2*>(tp));
      tr.v[0] = v01.x; tr.v[1] = v01.y; tr.v[2] = __ldg(tp + 2);
    }
    {
      double z[27];
#pragma unroll
      for (int i = 0; i < 27; ++i) z[i] = 0.0;
      tmem::st<27>(tm + kTmHeld, z);   // no wedge below the bed
    }
    // the velocities one layer ahead: level k + 2 is copied global -> shared
    // with cp.async (no registers held) while wedge k is computed, into a
    // three-level ring per thread (the gather otherwise waits on L2 every layer)
    double2* const ub2 = reinterpret_cast<double2*>(smem + kUbufOffsetWS / 8);
    auto u_copy = [&](int lev) {
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(ub2 + ((lev % 3) * 3 + j) * TP + tl));
        const double2* src = reinterpret_cast<const double2*>(U) + int64_t(tr.v[j]) * (L + 1) + lev;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
      }
    };
    u_copy(0);
    u_copy(1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    for (int k = 0; k < L; ++k) {
      double acc[36];
      {
        if (k + 2 <= L) u_copy(k + 2);
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");   // levels k, k + 1 are in
        const ColRec* colk = col;
        asm volatile("" : "+l"(colk));
        TriGeo geo;
        load_tri_geo(colk, tr, geo);
        const double Afac = wedge_afac(kp, Aw, t0 + te, k);
        WedgeIn w;
        {
          double2 ucur[3], utop[3];
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            ucur[j] = ub2[((k % 3) * 3 + j) * TP + tl];
            utop[j] = ub2[(((k + 1) % 3) * 3 + j) * TP + tl];
          }
          wedge_input_u(geo, sigma, Afac, ucur, utop, k, w, kp.go != 0);
        }
        if constexpr (TET) tet3_element_ws<N3>(w, kp.rg, kp.eps, kp.glen_n, tm, acc);
        else wedge_element_ws<N3>(w, kp.rg, kp.eps, kp.glen_n, tm, acc);
      }
      double dk[27];
      tmem::wait_st();
      tmem::ld<27>(tm + kTmBB, dk);
      named_sync(kBarEmpty, kWsThreads);   // phase B of level k-1 has released D / O
      if (active) {
#pragma unroll
        for (int q = 0; q < 6; ++q)
#pragma unroll
          for (int q2 = 0; q2 < 6; ++q2) O[(6 * q + q2) * TP + tl] = acc[oidx(q, q2)];
#pragma unroll
        for (int i = 0; i < kD; ++i) D[i * TP + tl] = dk[i];
      }
      named_arrive(kBarFull, kWsThreads);   // level k published
    }
    {   // the surface level L: D(L) = the top block of wedge L-1
      double hd[27];
      tmem::wait_st();
      tmem::ld<27>(tm + kTmHeld, hd);
      named_sync(kBarEmpty, kWsThreads);
      if (active) {
#pragma unroll
        for (int i = 0; i < kD; ++i) D[i * TP + tl] = hd[i];
      }
      named_arrive(kBarFull, kWsThreads);
    }
    tmem::fence_before();
    named_sync(kBarElem, kWsHalf);   // every element warp is done with TMEM
    tmem::fence_after();
    if (tl < 32) tmem::dealloc(tmem_base, kWsAlloc);
  } else {
    // ---------------- WG1: scatter (phase B) ----------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kWsRegsB));
    const int tb = int(threadIdx.x) - kWsHalf;
    if (pv.inkz) {
      // while the element warps compute layer 0: zero-fill the boundary
      // columns this patch leads (a warp per column), publish, then wait for
      // the leads of the other boundary columns before the first RED
      const int z0 = __ldg(pv.zl_ptr + p), z1 = __ldg(pv.zl_ptr + p + 1);
      const int lane = tb & 31;
      for (int i = z0 + (tb >> 5); i < z1; i += kWsHalf / 32) {
        const int c = __ldg(pv.zl + i);
        for (int j = lane; j < L + 1; j += 32) zero2(reinterpret_cast<double2*>(R + 2 * (int64_t(c) * (L + 1) + j)));
        const long long csn = __double_as_longlong(__ldg(reinterpret_cast<const double*>(col + c) + 5));
        double2* v = reinterpret_cast<double2*>(vals + (csn >> 8));
        const int64_t len2 = int64_t(2 * (csn & 255)) * (3 * L + 1);
        for (int64_t j = lane; j < len2; j += 32) zero2(v + j);
      }
      named_sync(kBarScat, kWsHalf);
      if (tb == 0) {
        __threadfence();   // the scatter warps' zero stores (ordered by the barrier) before the flag
        asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(pv.flags + p), "r"(1) : "memory");
      }
      const int w0 = __ldg(pv.wl_ptr + p), w1 = __ldg(pv.wl_ptr + p + 1);
      for (int i = w0 + tb; i < w1; i += kWsHalf) {
        const int32_t* f = pv.flags + __ldg(pv.wl + i);
        int v = 0;
        for (;;) {
          asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
          if (v) break;
          __nanosleep(64);
        }
      }
      named_sync(kBarScat, kWsHalf);
    }
    bulk_wait(&plan_bar);
    named_arrive(kBarEmpty, kWsThreads);   // D / O start free
    for (int kk = 0; kk <= L; ++kk) {
      named_sync(kBarFull, kWsThreads);
      phase_b<true>(sp, kk, L, D, O, R, vals, pv.partials, tb, kWsHalf);
      if (kk < L) named_arrive(kBarEmpty, kWsThreads);
    }
    if (pv.trig && p < pv.n_bnd) {
      // fused halo: count the finished boundary patches; the last one runs the
      // fix-up of the multi columns only they touch and raises the ready flag
      named_sync(kBarScat, kWsHalf);
      if (tb == 0) {
        __threadfence();   // this patch's stores (ordered by the barrier) before the count
        last_bnd = atomicAdd(pv.flags + pv.n_patches + 1, 1) == pv.n_bnd - 1;
        __threadfence();   // and every other boundary patch's before the fix-up reads
      }
      named_sync(kBarScat, kWsHalf);
      if (last_bnd) {
        for (int i = tb; i < pv.n_multi_bnd * (L + 1); i += kWsHalf)
          multi_fixup_one(pv.multi, i, L, pv.partials, R, vals);
        named_sync(kBarScat, kWsHalf);
        if (tb == 0) {
          // system scope: the flag releases the ghost rows to the side stream's
          // copy engine / NCCL kernels, not only to this GPU's SMs
          __threadfence_system();
          asm volatile("st.relaxed.sys.global.b32 [%0], %1;" ::"l"(pv.flags + pv.n_patches + 2), "r"(1) : "memory");
        }
      }
    }
  }
}


// zero the rows (CSR values and residual) of boundary columns
__global__ void zero_boundary_kernel(const ColRec* __restrict__ col, const int32_t* __restrict__ zc,
                                     int n, int L, double* __restrict__ R, double* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n; w += (gridDim.x * blockDim.x) >> 5) {
    const int c = zc[w];
    if (R)
      for (int i = lane; i < 2 * (L + 1); i += 32) R[2 * int64_t(c) * (L + 1) + i] = 0.0;
    if (vals) {
      const long long csn = __double_as_longlong(__ldg(reinterpret_cast<const double*>(col + c) + 5));
      const int64_t b = csn >> 8;
      const int64_t len = int64_t(4 * (csn & 255)) * (3 * L + 1);
      for (int64_t i = lane; i < len / 2; i += 32)
        reinterpret_cast<double2*>(vals + b)[i] = make_double2(0.0, 0.0);
    }
  }
}

// multi columns: add the patches' partial blocks in patch order and store the
// self-slot entries and the residual (one thread per column and row level)
// (the fix-up kernel: eight threads per (record, row level), thread `part` < 7
// sums the double2 `part` of the 14 sums -- dg 0-1, up 2-3, nx 4-5, residual 6
// -- over the partial blocks in patch order, bitwise the same as
// multi_fixup_one, with one serial load chain of cnt double2 per thread:
// C3 R + J 1.279 -> 1.274 ms, profiles/r02ai_ab_fixup.txt; FO_FIXUP_ONE: one
// thread per item)
__device__ __forceinline__ void multi_fixup_part(const MultiRec* __restrict__ mr, int i, int part, int L,
                                                 const double* __restrict__ partials, double* __restrict__ R,
                                                 double* __restrict__ vals) {
  const int mc = i / (L + 1), kk = i - mc * (L + 1);
  const MultiRec r = mr[mc];
  if (part != 6 && (!vals || (part >= 2 && kk == L))) return;
  double2 a = make_double2(0.0, 0.0);
  for (int b = 0; b < r.cnt; ++b) {
    const double2 q = __ldg(reinterpret_cast<const double2*>(partials + (int64_t(r.base + b) * (L + 1) + kk) *
                                                                            kPartialStride) + part);
    a.x += q.x;
    a.y += q.y;
  }
  if (part == 6) {
    *reinterpret_cast<double2*>(R + 2 * (int64_t(r.c) * (L + 1) + kk)) = a;
    return;
  }
  const int nc = r.nc_self & 255, slot = r.nc_self >> 8;
  double* dst;
  if (part < 4) {
    const int m0 = (kk == 0 || kk == L) ? 2 : 3, P0 = kk == 0 ? 0 : 3 * kk - 1, g0 = kk == 0 ? 0 : 2;
    dst = vals + r.colstart + int64_t(4 * nc) * P0 + int64_t(slot) * (2 * m0) + g0 + (part & 1) * (2 * nc * m0) +
          (part >> 1) * 2;
  } else {
    const int m1 = (kk + 1 == L) ? 2 : 3, P1 = 3 * kk + 2;
    dst = vals + r.colstart + int64_t(4 * nc) * P1 + int64_t(slot) * (2 * m1) + (part & 1) * (2 * nc * m1);
  }
  *reinterpret_cast<double2*>(dst) = a;
}

__global__ void multi_fixup_kernel(const MultiRec* __restrict__ mr, int n, int L,
                                   const double* __restrict__ partials, double* __restrict__ R,
                                   double* __restrict__ vals) {
#ifdef FO_FIXUP_ONE
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n * (L + 1)) multi_fixup_one(mr, i, L, partials, R, vals);
#else
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = t >> 3, part = t & 7;
  if (i < n * (L + 1) && part < 7) multi_fixup_part(mr, i, part, L, partials, R, vals);
#endif
}

static size_t smem_bytes(bool need_j) { return size_t(need_j ? kPlanOffset : kPlanOffsetR) + kPlanBytes; }

template <bool N3, bool TET>
static fo_status launch_ws(fo_mesh m, const double* U, double* R, double* vals, cudaStream_t s, int p0, int np,
                           bool inkz, bool trig = false) {
  const size_t sm = size_t(kWsSmem);
  fo_status st = cuda_status(cudaFuncSetAttribute(ka_ws_kernel<N3, TET>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  int(sm)), "cudaFuncSetAttribute");
  if (st) return st;
  PlanView pv{m->d_plan.t_begin, m->d_plan.col_ptr, m->d_plan.pair_ptr, m->d_plan.nedge, m->d_plan.blob,
              m->d_plan.blob_off, m->d_plan.partials, p0, m->d_plan.zl, m->d_plan.zl_ptr, m->d_plan.wl,
              m->d_plan.wl_ptr, m->d_plan.flags, inkz ? 1 : 0, m->plan.n_patches,
              m->d_plan.multi, trig ? 1 : 0, m->plan.n_bnd_patches, m->plan.n_multi_bnd};
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (m->timing) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
  }
  ka_ws_kernel<N3, TET><<<np, kWsThreads, sm, s>>>(m->d_col, m->d_tri, m->d_sigma, m->d_A, make_kparams(m), pv, U, R,
                                              vals);
  if (m->timing) {
    cudaEventRecord(e1, s);
    m->timed.push_back({e0, e1});
  }
  return cuda_status(cudaGetLastError(), "ka_ws_kernel launch");
}

template <bool NEED_J, bool N3, bool TET>
static fo_status launch_patch(fo_mesh m, const double* U, double* R, double* vals, cudaStream_t s, int p0,
                              int np) {
  // the shared-memory opt-in is per device: set it on every call (cheap), so
  // meshes on different devices of one process, and concurrent callers, are safe
  const size_t sm = smem_bytes(NEED_J);
  {
    fo_status st = cuda_status(cudaFuncSetAttribute(ka_patch_kernel<NEED_J, N3, TET>,
                                                    cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)),
                               "cudaFuncSetAttribute");
    if (st) return st;
  }
  PlanView pv{m->d_plan.t_begin, m->d_plan.col_ptr, m->d_plan.pair_ptr, m->d_plan.nedge, m->d_plan.blob,
              m->d_plan.blob_off, m->d_plan.partials, p0, m->d_plan.zl, m->d_plan.zl_ptr, m->d_plan.wl,
              m->d_plan.wl_ptr, m->d_plan.flags, 0, m->plan.n_patches, m->d_plan.multi, 0, 0, 0};
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (m->timing) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
  }
  ka_patch_kernel<NEED_J, N3, TET><<<np, kPatchTris, sm, s>>>(m->d_col, m->d_tri, m->d_sigma, m->d_A,
                                                              make_kparams(m), pv, U, R, vals);
  if (m->timing) {
    cudaEventRecord(e1, s);
    m->timed.push_back({e0, e1});
  }
  return cuda_status(cudaGetLastError(), "ka_patch_kernel launch");
}

namespace {
// The pieces of one owner-computes assembly: the
// prologue (class-C residual zero, boundary-column zero fill), the patch
// kernel over a range of patches, the multi-column fix-up over a range of
// its records.
struct OwnerCall {
  fo_mesh m;
  const double* U;
  double* R;
  double* vals;   // nullptr: residual only
  int launches = 0;
};

fo_status owner_begin(OwnerCall& c, fo_mesh m, const double* d_U, double* d_R, double* d_vals) {
  c.m = m;
  c.U = d_U;
  c.vals = d_vals;
  // R is always produced by the kernel; use a scratch vector when the caller passes none
  c.R = d_R;
  if (!c.R) {
    if (!m->d_scratch_R) {
      fo_status st = cuda_status(cudaMalloc(&m->d_scratch_R, sizeof(double) * m->n_dof), "cudaMalloc");
      if (st) return st;
    }
    c.R = m->d_scratch_R;
  }
  return FO_OK;
}

// the wedge R + J path runs the warp-specialised kernel unless the round-1 kernel is asked for
bool uses_ws(const OwnerCall& c) {
  return c.vals != nullptr && (c.m->scatter == FO_SCATTER_OWNER || c.m->scatter == FO_SCATTER_OWNER_WS);
}

// inkz: the warp-specialised kernel zero-fills the boundary columns itself
// (single launch over all patches): reset its flags and ticket instead of
// launching zero_boundary_kernel
fo_status owner_prologue(OwnerCall& c, cudaStream_t s, bool inkz = false) {
  fo_mesh m = c.m;
  if (inkz) {
    fo_status st = cuda_status(cudaMemsetAsync(m->d_plan.flags, 0, sizeof(int32_t) * (m->plan.n_patches + 3), s),
                               "cudaMemsetAsync");
    if (st) return st;
  }
  const int64_t nk_dof = 2 * (m->nA + m->nB) * (m->L + 1);
  if (nk_dof < m->n_dof) {   // column-only (class C) DOFs: residual 0
    fo_status st = cuda_status(cudaMemsetAsync(c.R + nk_dof, 0, sizeof(double) * (m->n_dof - nk_dof), s),
                               "cudaMemsetAsync");
    if (st) return st;
  }
  const int nz = int(m->plan.zero_cols.size());
  if (nz > 0 && !inkz) {
    const int blocks = int(std::min<int64_t>((int64_t(nz) * 32 + 255) / 256, 148 * 16));
    zero_boundary_kernel<<<blocks, 256, 0, s>>>(m->d_col, m->d_plan.zero_cols, nz, m->L, c.R, c.vals);
    fo_status st = cuda_status(cudaGetLastError(), "zero_boundary_kernel launch");
    if (st) return st;
    ++c.launches;
  }
  return FO_OK;
}

fo_status owner_patches(OwnerCall& c, cudaStream_t s, int p0, int p1, bool inkz = false, bool trig = false) {
  if (p1 <= p0) return FO_OK;
  fo_mesh m = c.m;
  const bool need_j = c.vals != nullptr, n3 = m->p.glen_n == 3.0, tet = m->elem_type == FO_ELEM_TET3;
  const int np = p1 - p0;
  fo_status st;
  if (uses_ws(c))
    st = tet ? (n3 ? launch_ws<true, true>(m, c.U, c.R, c.vals, s, p0, np, inkz, trig)
                   : launch_ws<false, true>(m, c.U, c.R, c.vals, s, p0, np, inkz, trig))
             : (n3 ? launch_ws<true, false>(m, c.U, c.R, c.vals, s, p0, np, inkz, trig)
                   : launch_ws<false, false>(m, c.U, c.R, c.vals, s, p0, np, inkz, trig));
  else if (need_j)
    st = tet ? (n3 ? launch_patch<true, true, true>(m, c.U, c.R, c.vals, s, p0, np)
                   : launch_patch<true, false, true>(m, c.U, c.R, c.vals, s, p0, np))
             : (n3 ? launch_patch<true, true, false>(m, c.U, c.R, c.vals, s, p0, np)
                   : launch_patch<true, false, false>(m, c.U, c.R, c.vals, s, p0, np));
  else
    st = tet ? (n3 ? launch_patch<false, true, true>(m, c.U, c.R, nullptr, s, p0, np)
                   : launch_patch<false, false, true>(m, c.U, c.R, nullptr, s, p0, np))
             : (n3 ? launch_patch<false, true, false>(m, c.U, c.R, nullptr, s, p0, np)
                   : launch_patch<false, false, false>(m, c.U, c.R, nullptr, s, p0, np));
  if (st) return st;
  ++c.launches;
  return FO_OK;
}

fo_status owner_multi(OwnerCall& c, cudaStream_t s, int r0, int r1) {
  if (r1 <= r0) return FO_OK;
  fo_mesh m = c.m;
  const int n = (r1 - r0) * (m->L + 1);
#ifdef FO_FIXUP_ONE
  const int nthreads = n;
#else
  const int nthreads = 8 * n;
#endif
  multi_fixup_kernel<<<(nthreads + 127) / 128, 128, 0, s>>>(m->d_plan.multi + r0, r1 - r0, m->L, m->d_plan.partials,
                                                     c.R, c.vals);
  fo_status st = cuda_status(cudaGetLastError(), "multi_fixup_kernel launch");
  if (st) return st;
  ++c.launches;
  return FO_OK;
}
}  // namespace

// the owner-computes prologue / epilogue for the hexahedral patch kernel
// (fo_hex.cu): class-C residual zero + boundary-column zero fill (inkz: the
// kernel's flags and ticket reset instead), and the multi-column fix-up;
// `launches` counts the kernels enqueued
fo_status launch_owner_prologue(fo_mesh m, double* R, double* vals, cudaStream_t s, int* launches, bool inkz) {
  OwnerCall c;
  c.m = m;
  c.R = R;
  c.vals = vals;
  fo_status st = owner_prologue(c, s, inkz);
  *launches += c.launches;
  return st;
}
fo_status launch_owner_fixup(fo_mesh m, double* R, double* vals, cudaStream_t s, int* launches) {
  OwnerCall c;
  c.m = m;
  c.R = R;
  c.vals = vals;
  fo_status st = owner_multi(c, s, 0, int(m->plan.multi.size()));
  *launches += c.launches;
  return st;
}

fo_status launch_owner(fo_mesh m, const double* d_U, double* d_R, double* d_vals, cudaStream_t s) {
  OwnerCall c;
  fo_status st = owner_begin(c, m, d_U, d_R, d_vals);
  // one launch over all patches: the warp-specialised kernel zero-fills in-kernel
  const bool inkz = !st && uses_ws(c);
  if (!st) st = owner_prologue(c, s, inkz);
  if (!st) st = owner_patches(c, s, 0, m->plan.n_patches, inkz);
  if (!st) st = owner_multi(c, s, 0, int(m->plan.multi.size()));
  if (st) return st;
  m->last_launches = c.launches;
  return FO_OK;
}

// Boundary-first assembly of a part mesh with the ghost-row sum overlapped
// (fo_assemble_jacobian_halo): ONE warp-specialised launch over all patches
// with the in-kernel zero fill; a part mesh orders its ghost-touching
// triangles first, so the boundary patches draw tickets 0 .. K-1, and the
// last of them to finish runs the fix-up of the multi columns only they touch
// and raises the ready flag.  The halo's side stream waits for that flag
// (stream memory operation `wait_value`) and sends the final ghost rows while
// the interior patches are still running; the remaining fix-up follows the
// kernel on `s`.  Returns FO_ESTATE when this path does not apply (not the
// warp-specialised kernel, or no boundary patches): the caller then runs the
// sequential order.
fo_status launch_owner_overlap(fo_mesh m, const double* d_U, double* d_R, double* d_vals, cudaStream_t s,
                               cudaStream_t side, cudaEvent_t ev0, const std::function<fo_status(
                                   cudaStream_t, const int32_t*)>& wait_ready) {
  OwnerCall c;
  fo_status st = owner_begin(c, m, d_U, d_R, d_vals);
  if (st) return st;
  const int K = m->plan.n_bnd_patches, nmb = m->plan.n_multi_bnd;
  if (!uses_ws(c) || K == 0) return FO_ESTATE;
  st = owner_prologue(c, s, true);
  if (!st) st = cuda_status(cudaEventRecord(ev0, s), "cudaEventRecord");
  if (!st) st = cuda_status(cudaStreamWaitEvent(side, ev0, 0), "cudaStreamWaitEvent");
  if (!st) st = wait_ready(side, m->d_plan.flags + m->plan.n_patches + 2);
  if (!st) st = owner_patches(c, s, 0, m->plan.n_patches, true, true);
  if (!st) st = owner_multi(c, s, nmb, int(m->plan.multi.size()));
  if (st) return st;
  m->last_launches = c.launches;
  return FO_OK;
}

}  // namespace fo
