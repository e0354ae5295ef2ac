// fo_kernels.cu -- sm_100a kernels of libfo: residual (KR) and residual +
// Jacobian (KA) assembly of the FO-Stokes equations.
//
// Two scatter strategies for KA:
//   KA-atomic: one thread per wedge, fp64 RED into zero-filled outputs;
//   KA-owner : column-patch owner-computes (fo_owner.cu), every CSR value
//              written exactly once with coalesced plain stores.
// CSR positions are computed from the column structure (TriRec slots and the
// ColRec value offsets); col_idx is never read.
#include <cuda_runtime.h>

#include <cmath>

#include "fo_element.cuh"
#include "fo_internal.h"
#include "fo_kernels.cuh"

namespace fo {

// ---------------------------------------------------------------- KR / KA-atomic
template <bool NEED_J, bool N3>
__global__ void __launch_bounds__(128)
assemble_atomic_kernel(const ColRec* __restrict__ col, const TriRec* __restrict__ tris,
                       const double* __restrict__ sigma, const double* __restrict__ Aw,
                       KParams kp, const double* __restrict__ U, double* __restrict__ R,
                       double* __restrict__ vals) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= kp.n_elem) return;
  const int L = kp.L;
  const int64_t t = e / L;
  const int k = int(e - t * L);
  WedgeIn w;
  TriRec tr;
  ColRec cr[3];
  load_wedge(col, tris, sigma, Aw, kp, U, t, k, w, tr, cr);
  double r[12];
  double J[NEED_J ? 78 : 1];
  wedge_element<NEED_J, N3>(w, kp.rg, kp.eps, kp.glen_n, r, J);
  // scatter
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const int j = i % 3, l = i / 3;
    const int64_t node = int64_t(tr.v[j]) * (L + 1) + k + l;
    if (R) {
      atomicAdd(R + 2 * node, r[2 * i]);
      atomicAdd(R + 2 * node + 1, r[2 * i + 1]);
    }
  }
  if (NEED_J) {
#pragma unroll
    for (int p = 0; p < 12; ++p) {
      const int i = p >> 1, ca = p & 1, j = i % 3, l = i / 3;
      const int kk = k + l;
      const int64_t cs = cr[j].cs_n >> 8;
      const int nc = int(cr[j].cs_n & 255);
      const int m = (kk == 0 || kk == L) ? 2 : 3;
      const int64_t row = cs + int64_t(4 * nc) * (kk == 0 ? 0 : 3 * kk - 1) + ca * (2 * nc * m);
#pragma unroll
      for (int q = 0; q < 12; ++q) {
        const int i2 = q >> 1, cb = q & 1, j2 = i2 % 3, l2 = i2 / 3;
        const int off = (kk == 0) ? l2 : (l2 - l + 1);
        const int64_t pos = row + tr.slot[3 * j + j2] * (2 * m) + 2 * off + cb;
        const double v = p <= q ? J[jidx(p, q)] : J[jidx(q, p)];
        atomicAdd(vals + pos, v);
      }
    }
  }
}

template <bool NEED_J>
static fo_status launch_atomic(fo_mesh m, const double* d_U, double* d_R, double* d_vals,
                               cudaStream_t s) {
  const KParams kp = make_kparams(m);
  const int bs = 128;
  const int64_t nb = (m->n_elem + bs - 1) / bs;
  const bool n3 = m->p.glen_n == 3.0;
  if (n3)
    assemble_atomic_kernel<NEED_J, true><<<unsigned(nb), bs, 0, s>>>(m->d_col, m->d_tri, m->d_sigma, m->d_A, kp, d_U, d_R, d_vals);
  else
    assemble_atomic_kernel<NEED_J, false><<<unsigned(nb), bs, 0, s>>>(m->d_col, m->d_tri, m->d_sigma, m->d_A, kp, d_U, d_R, d_vals);
  return cuda_status(cudaGetLastError(), "assemble_atomic_kernel launch");
}

fo_status launch_residual(fo_mesh m, const double* d_U, double* d_R, void* stream) {
  fo_status st = cuda_status(cudaSetDevice(m->device), "cudaSetDevice");
  if (st) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  m->last_launches = 0;
  if (m->n_dof == 0) return FO_OK;
  if (m->quad) return launch_hex(m, d_U, d_R, nullptr, s);
  if (m->scatter != FO_SCATTER_ATOMIC && m->plan.n_patches > 0) {
    st = launch_owner(m, d_U, d_R, nullptr, s);
  } else {
    st = cuda_status(cudaMemsetAsync(d_R, 0, sizeof(double) * m->n_dof, s), "cudaMemsetAsync");
    if (st || m->n_elem == 0) return st;
    st = launch_atomic<false>(m, d_U, d_R, nullptr, s);
    m->last_launches = 1;
  }
  if (!st) st = launch_lateral(m, d_R, s);
  return st;
}

fo_status launch_jacobian(fo_mesh m, const double* d_U, double* d_R, double* d_vals,
                          void* stream) {
  fo_status st = cuda_status(cudaSetDevice(m->device), "cudaSetDevice");
  if (st) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  m->last_launches = 0;
  if (m->n_dof == 0) return FO_OK;
  if (m->quad) return launch_hex(m, d_U, d_R, d_vals, s);
  if (m->scatter != FO_SCATTER_ATOMIC && m->plan.n_patches > 0) {
    st = launch_owner(m, d_U, d_R, d_vals, s);
  } else {
    if (d_R) st = cuda_status(cudaMemsetAsync(d_R, 0, sizeof(double) * m->n_dof, s), "cudaMemsetAsync");
    if (!st && m->nnz > 0)
      st = cuda_status(cudaMemsetAsync(d_vals, 0, sizeof(double) * m->nnz, s), "cudaMemsetAsync");
    if (st || m->n_elem == 0) return st;
    st = launch_atomic<true>(m, d_U, d_R, d_vals, s);
    m->last_launches = 1;
  }
  if (!st) st = launch_lateral(m, d_R, s);
  return st;
}

}  // namespace fo
