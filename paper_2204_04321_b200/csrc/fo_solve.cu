// fo_solve.cu -- NEXT-f2: the Newton consumer of the assembled Jacobian
// (PAPER.md eq:linearsystem P:160-165: J(U) dU = -F(U), solved by
// preconditioned GMRES).  Kernels:
//   * fo_spmv           y = J x on the library's CSR values; every position comes
//                       from the column structure (row (c,k,a): slot s of c's
//                       coupling list, level k' in [k-1, k+1], comp b), so
//                       col_idx is never read (4 B/nnz less than plain CSR);
//   * fo_line_factor /  the vertical-line preconditioner: for every column the
//     fo_line_solve     2x2-block tridiagonal block of J coupling its own 2(L+1)
//                       DOFs (the self slot), factored by block Thomas; applying
//                       all columns' exact solves is block Jacobi over vertical
//                       lines, the B200 analogue of the semicoarsening /
//                       line smoothers of the paper's multigrid;
//   * fo_krylov_dots /  deterministic V^T w and w -= V h for the GMRES basis
//     fo_krylov_update  (fixed-order reductions: bitwise reproducible).
// The damped Newton / GMRES(m) driver is paper_2204_04321_b200/newton.py.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "fo_internal.h"

namespace fo {

namespace {

constexpr int kDotBlocks = 296;   // 2 x 148 SMs
constexpr int kDotThreads = 256;

// one thread per row of a column with rows
__global__ void spmv_kernel(const ColRec* __restrict__ col, const int64_t* __restrict__ nptr,
                            const int32_t* __restrict__ nbr, int64_t n_rows, int L,
                            const double* __restrict__ vals, const double* __restrict__ x,
                            double* __restrict__ y) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  const int64_t node = r >> 1;
  const int a = int(r & 1);
  const int64_t c = node / (L + 1);
  const int k = int(node - c * (L + 1));
  const long long csn = __double_as_longlong(__ldg(reinterpret_cast<const double*>(col + c) + 5));
  const int64_t cs = csn >> 8;
  const int nc = int(csn & 255);
  const int m = (k == 0 || k == L) ? 2 : 3;
  const int P = k == 0 ? 0 : 3 * k - 1;
  const int kmin = k == 0 ? 0 : k - 1;
  const double2* seg = reinterpret_cast<const double2*>(vals + cs + int64_t(4 * nc) * P + int64_t(a) * 2 * nc * m);
  const double2* x2 = reinterpret_cast<const double2*>(x);
  const int64_t nb = __ldg(nptr + c);
  double acc = 0.0;
  for (int s = 0; s < nc; ++s) {
    const int64_t cn = __ldg(nbr + nb + s);
    const double2* xs = x2 + cn * (L + 1) + kmin;
    for (int g = 0; g < m; ++g) {
      const double2 v = __ldg(seg + s * m + g);
      const double2 xv = __ldg(xs + g);
      acc = fma(v.x, xv.x, acc);
      acc = fma(v.y, xv.y, acc);
    }
  }
  y[r] = acc;
}

// per column: block Thomas factorisation of the 2x2-block tridiagonal
// A_k = J[(c,k),(c,k)], B_k = J[(c,k),(c,k+1)], C_k = J[(c,k+1),(c,k)]:
//   S_0 = A_0, S_k = A_k - C_{k-1} S_{k-1}^-1 B_{k-1};
// stored per (column, level): inv(S_k) (4) and G_k = S_k^-1 B_k (4)
__device__ __forceinline__ void inv2(const double* a, double* o) {
  const double d = a[0] * a[3] - a[1] * a[2];
  const double id = 1.0 / d;
  o[0] = a[3] * id; o[1] = -a[1] * id; o[2] = -a[2] * id; o[3] = a[0] * id;
}
__device__ __forceinline__ void mul2(const double* a, const double* b, double* o) {
  o[0] = a[0] * b[0] + a[1] * b[2]; o[1] = a[0] * b[1] + a[1] * b[3];
  o[2] = a[2] * b[0] + a[3] * b[2]; o[3] = a[2] * b[1] + a[3] * b[3];
}

// J entry block (rows (c,k,a=0,1), columns (c,k2,b=0,1)) with |k2 - k| <= 1
__device__ __forceinline__ void self_block(const double* __restrict__ vals, int64_t cs, int nc, int self,
                                           int L, int k, int k2, double* o) {
  const int m = (k == 0 || k == L) ? 2 : 3;
  const int P = k == 0 ? 0 : 3 * k - 1;
  const int kmin = k == 0 ? 0 : k - 1;
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const double* row = vals + cs + int64_t(4 * nc) * P + int64_t(a) * 2 * nc * m;
    const double2 v = *reinterpret_cast<const double2*>(row + self * 2 * m + 2 * (k2 - kmin));
    o[2 * a] = v.x;
    o[2 * a + 1] = v.y;
  }
}

__global__ void line_factor_kernel(const ColRec* __restrict__ col, const int32_t* __restrict__ self_slot,
                                   int64_t n_cols, int L, const double* __restrict__ vals,
                                   double* __restrict__ fac) {
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= n_cols) return;
  const long long csn = __double_as_longlong(__ldg(reinterpret_cast<const double*>(col + c) + 5));
  const int64_t cs = csn >> 8;
  const int nc = int(csn & 255);
  const int self = __ldg(self_slot + c);
  double* f = fac + c * (L + 1) * 8;
  double S[4], Si[4], B[4], Cm[4], T[4], G[4] = {0, 0, 0, 0};
  for (int k = 0; k <= L; ++k) {
    self_block(vals, cs, nc, self, L, k, k, S);
    if (k > 0) {   // S_k = A_k - C_{k-1} G_{k-1}
      self_block(vals, cs, nc, self, L, k, k - 1, Cm);
      mul2(Cm, G, T);
#pragma unroll
      for (int i = 0; i < 4; ++i) S[i] -= T[i];
    }
    inv2(S, Si);
    if (k < L) {
      self_block(vals, cs, nc, self, L, k, k + 1, B);
      mul2(Si, B, G);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[8 * k + i] = Si[i];
      f[8 * k + 4 + i] = k < L ? G[i] : 0.0;
    }
  }
}

// z = M^-1 r, M = block diagonal of the columns' tridiagonal blocks
__global__ void line_solve_kernel(const ColRec* __restrict__ col, const int32_t* __restrict__ self_slot,
                                  int64_t n_cols, int L, const double* __restrict__ vals,
                                  const double* __restrict__ fac, const double* __restrict__ r,
                                  double* __restrict__ z) {
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= n_cols) return;
  const long long csn = __double_as_longlong(__ldg(reinterpret_cast<const double*>(col + c) + 5));
  const int64_t cs = csn >> 8;
  const int nc = int(csn & 255);
  const int self = __ldg(self_slot + c);
  const double* f = fac + c * (L + 1) * 8;
  const double2* r2 = reinterpret_cast<const double2*>(r) + c * (L + 1);
  double2* z2 = reinterpret_cast<double2*>(z) + c * (L + 1);
  // forward: y_k = S_k^-1 (r_k - C_{k-1} y_{k-1})
  double yp0 = 0.0, yp1 = 0.0;
  for (int k = 0; k <= L; ++k) {
    double2 rk = r2[k];
    if (k > 0) {
      double Cm[4];
      self_block(vals, cs, nc, self, L, k, k - 1, Cm);
      rk.x -= Cm[0] * yp0 + Cm[1] * yp1;
      rk.y -= Cm[2] * yp0 + Cm[3] * yp1;
    }
    const double* Si = f + 8 * k;
    yp0 = Si[0] * rk.x + Si[1] * rk.y;
    yp1 = Si[2] * rk.x + Si[3] * rk.y;
    z2[k] = make_double2(yp0, yp1);
  }
  // backward: z_k = y_k - G_k z_{k+1}
  double zn0 = 0.0, zn1 = 0.0;
  for (int k = L; k >= 0; --k) {
    double2 zk = z2[k];
    if (k < L) {
      const double* G = f + 8 * k + 4;
      zk.x -= G[0] * zn0 + G[1] * zn1;
      zk.y -= G[2] * zn0 + G[3] * zn1;
    }
    z2[k] = zk;
    zn0 = zk.x;
    zn1 = zk.y;
  }
}

// partial dot products: part[j * kDotBlocks + block] = sum over the block's
// grid-stride range of V_j . w   (fixed order: thread-strided, then a tree)
__global__ void dots_partial_kernel(int64_t n, int kv, const double* __restrict__ V, int64_t ldv,
                                    const double* __restrict__ w, double* __restrict__ part) {
  __shared__ double red[kDotThreads];
  for (int j = 0; j < kv; ++j) {
    const double* v = V + int64_t(j) * ldv;
    double s = 0.0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
      s = fma(v[i], w[i], s);
    red[threadIdx.x] = s;
    __syncthreads();
    for (int h = blockDim.x / 2; h > 0; h >>= 1) {
      if (int(threadIdx.x) < h) red[threadIdx.x] += red[threadIdx.x + h];
      __syncthreads();
    }
    if (threadIdx.x == 0) part[j * gridDim.x + blockIdx.x] = red[0];
    __syncthreads();
  }
}

__global__ void dots_final_kernel(int kv, int nb, const double* __restrict__ part, double* __restrict__ out) {
  const int j = threadIdx.x;
  if (j >= kv) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += part[j * nb + b];
  out[j] = s;
}

// w -= sum_j h_j V_j (h on the device)
__global__ void update_kernel(int64_t n, int kv, const double* __restrict__ V, int64_t ldv,
                              const double* __restrict__ h, double* __restrict__ w) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double s = w[i];
    for (int j = 0; j < kv; ++j) s = fma(-__ldg(h + j), V[int64_t(j) * ldv + i], s);
    w[i] = s;
  }
}

fo_status ensure_solver_data(fo_mesh m) {
  // keyed on the LAST allocation: a call that failed half way is redone
  if (m->d_kry_work) return FO_OK;
  cudaFree(m->d_nbr_ptr); cudaFree(m->d_self_slot); cudaFree(m->d_nbr); cudaFree(m->d_line_fac);
  m->d_nbr_ptr = nullptr; m->d_self_slot = nullptr; m->d_nbr = nullptr; m->d_line_fac = nullptr;
  const int64_t nk = m->nA + m->nB;
  std::vector<int32_t> self(static_cast<size_t>(nk));
  for (int64_t c = 0; c < nk; ++c) {
    const int32_t* b = m->nbr.data() + m->nbr_ptr[size_t(c)];
    const int32_t* e = m->nbr.data() + m->nbr_ptr[size_t(c) + 1];
    self[size_t(c)] = int32_t(std::lower_bound(b, e, int32_t(c)) - b);
  }
  auto up = [](void** dst, const void* src, size_t bytes) {
    fo_status st = cuda_status(cudaMalloc(dst, bytes), "cudaMalloc");
    if (!st) st = cuda_status(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
    return st;
  };
  fo_status st = up(reinterpret_cast<void**>(&m->d_nbr_ptr), m->nbr_ptr.data(), m->nbr_ptr.size() * sizeof(int64_t));
  if (!st) st = up(reinterpret_cast<void**>(&m->d_self_slot), self.data(), self.size() * sizeof(int32_t));
  if (!st) st = up(reinterpret_cast<void**>(&m->d_nbr), m->nbr.data(), m->nbr.size() * sizeof(int32_t));
  if (!st)
    st = cuda_status(cudaMalloc(reinterpret_cast<void**>(&m->d_line_fac), sizeof(double) * 8 * size_t(nk) * (m->L + 1)),
                     "cudaMalloc");
  if (!st) st = cuda_status(cudaMalloc(reinterpret_cast<void**>(&m->d_kry_work), sizeof(double) * kDotBlocks * 64), "cudaMalloc");
  return st;
}

fo_status fail(fo_status st, const char* msg) {
  set_error(msg);
  return st;
}

fo_status single_domain(fo_mesh m) {
  if (m->n_parts != 1) return fail(FO_ESTATE, "the Newton consumer (NEXT-f2) runs on single-domain meshes");
  return FO_OK;
}

}  // namespace
}  // namespace fo

using namespace fo;

extern "C" {

fo_status fo_spmv(fo_mesh m, fo_graph g, const double* d_vals, const double* d_x, double* d_y, void* stream) {
  if (!m || !g) return fail(FO_EINVAL, "mesh or graph is NULL");
  if (g->mesh != m) return fail(FO_ESTATE, "graph was built for another mesh");
  fo_status st = single_domain(m);
  if (st) return st;
  if (m->n_dof == 0) return FO_OK;
  if (!d_vals || !d_x || !d_y) return fail(FO_EINVAL, "NULL device buffer");
  st = cuda_status(cudaSetDevice(m->device), "cudaSetDevice");
  if (!st) st = ensure_solver_data(m);
  if (st) return st;
  const int64_t n_rows = 2 * (m->nA + m->nB) * (m->L + 1);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  spmv_kernel<<<unsigned((n_rows + 255) / 256), 256, 0, s>>>(m->d_col, m->d_nbr_ptr, m->d_nbr, n_rows, m->L,
                                                             d_vals, d_x, d_y);
  return cuda_status(cudaGetLastError(), "spmv_kernel launch");
}

fo_status fo_line_factor(fo_mesh m, fo_graph g, const double* d_vals, void* stream) {
  if (!m || !g) return fail(FO_EINVAL, "mesh or graph is NULL");
  if (g->mesh != m) return fail(FO_ESTATE, "graph was built for another mesh");
  fo_status st = single_domain(m);
  if (st) return st;
  if (m->n_dof == 0) return FO_OK;
  if (!d_vals) return fail(FO_EINVAL, "NULL device buffer");
  st = cuda_status(cudaSetDevice(m->device), "cudaSetDevice");
  if (!st) st = ensure_solver_data(m);
  if (st) return st;
  const int64_t nk = m->nA + m->nB;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  line_factor_kernel<<<unsigned((nk + 127) / 128), 128, 0, s>>>(m->d_col, m->d_self_slot, nk, m->L, d_vals,
                                                                m->d_line_fac);
  m->line_vals = d_vals;
  return cuda_status(cudaGetLastError(), "line_factor_kernel launch");
}

fo_status fo_line_solve(fo_mesh m, const double* d_r, double* d_z, void* stream) {
  if (!m) return fail(FO_EINVAL, "mesh is NULL");
  if (m->n_dof == 0) return FO_OK;
  if (!m->line_vals) return fail(FO_ESTATE, "fo_line_factor has not been called");
  if (!d_r || !d_z) return fail(FO_EINVAL, "NULL device buffer");
  fo_status st = cuda_status(cudaSetDevice(m->device), "cudaSetDevice");
  if (st) return st;
  const int64_t nk = m->nA + m->nB;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  line_solve_kernel<<<unsigned((nk + 127) / 128), 128, 0, s>>>(m->d_col, m->d_self_slot, nk, m->L, m->line_vals,
                                                               m->d_line_fac, d_r, d_z);
  return cuda_status(cudaGetLastError(), "line_solve_kernel launch");
}

fo_status fo_krylov_dots(fo_mesh m, int64_t n, int32_t k, const double* d_V, int64_t ldv, const double* d_w,
                         double* d_out, void* stream) {
  if (!m) return fail(FO_EINVAL, "mesh is NULL");
  if (k < 1 || k > 64 || n < 0 || ldv < n) return fail(FO_EINVAL, "need 1 <= k <= 64 and ldv >= n");
  if (!d_V || !d_w || !d_out) return fail(FO_EINVAL, "NULL device buffer");
  fo_status st = cuda_status(cudaSetDevice(m->device), "cudaSetDevice");
  if (!st) st = ensure_solver_data(m);
  if (st) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  dots_partial_kernel<<<kDotBlocks, kDotThreads, 0, s>>>(n, k, d_V, ldv, d_w, m->d_kry_work);
  dots_final_kernel<<<1, 64, 0, s>>>(k, kDotBlocks, m->d_kry_work, d_out);
  return cuda_status(cudaGetLastError(), "krylov dots launch");
}

fo_status fo_krylov_update(fo_mesh m, int64_t n, int32_t k, const double* d_V, int64_t ldv, const double* d_h,
                           double* d_w, void* stream) {
  if (!m) return fail(FO_EINVAL, "mesh is NULL");
  if (k < 1 || n < 0 || ldv < n) return fail(FO_EINVAL, "need k >= 1 and ldv >= n");
  if (!d_V || !d_h || !d_w) return fail(FO_EINVAL, "NULL device buffer");
  fo_status st = cuda_status(cudaSetDevice(m->device), "cudaSetDevice");
  if (st) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  update_kernel<<<kDotBlocks * 4, 256, 0, s>>>(n, k, d_V, ldv, d_h, d_w);
  return cuda_status(cudaGetLastError(), "krylov update launch");
}

}  // extern "C"
