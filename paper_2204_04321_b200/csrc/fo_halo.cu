// fo_halo.cu -- footprint-partitioned assembly across GPUs: the paper's
// Tpetra Import (U owned -> overlapped) and Export (R, J overlapped ->
// owned with summation), rebuilt on NCCL over NVLink.
//
// Plan: every rank derives every part's local
// numbering from the global footprint and the triangle partition, so no
// metadata is exchanged.  The ghost (class B) columns of a part are numbered
// last and grouped by owner, so the rows a part sends to owner q are ONE
// contiguous slice of its R and CSR values (zero-copy sends).  The owner adds
// the received slices into its owned rows with a precomputed position map,
// one sender at a time in ascending rank order (deterministic).
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "fo_internal.h"

namespace fo {
namespace {

inline int64_t m_of(int64_t k, int64_t L) { return (k == 0 || k == L) ? 2 : 3; }
inline int64_t P_of(int64_t k) { return k == 0 ? 0 : 3 * k - 1; }

fo_status fail(fo_status st, const std::string& msg) {
  set_error(msg);
  return st;
}

fo_status nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return FO_OK;
  return fail(FO_ENCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

std::vector<int32_t> owners(int64_t n_vert, int64_t n_tri, const int32_t* tri, const int32_t* part) {
  std::vector<int32_t> own(size_t(n_vert), INT32_MAX);
  for (int64_t t = 0; t < n_tri; ++t)
    for (int i = 0; i < 3; ++i) own[tri[3 * t + i]] = std::min(own[tri[3 * t + i]], part[t]);
  return own;
}

// What part p sends to owner q (contiguous slices of p's arrays) and where
// each value lands in q's local arrays.
struct SendSlice {
  int32_t q = -1;
  int64_t col0 = 0, col1 = 0;        // p-local B column range owned by q
  int64_t row0 = 0, nrows = 0;       // R slice (DOF offsets in p)
  int64_t val0 = 0, nvals = 0;       // CSR value slice in p
  std::vector<int64_t> dest_rows;    // [nrows] DOF offsets in q
  std::vector<int64_t> dest_vals;    // [nvals] CSR positions in q
  std::vector<int64_t> import_src;   // [nrows] DOF offsets in q's U feeding p's ghosts
};

std::vector<int64_t> local_index(const Topo& T, int64_t n_vert) {
  std::vector<int64_t> loc(size_t(n_vert), -1);
  for (size_t i = 0; i < T.glob.size(); ++i) loc[size_t(T.glob[i])] = int64_t(i);
  return loc;
}

// sends of part p (topology Tp) to part q (topology Tq)
SendSlice plan_sends(const Topo& Tp, const Topo& Tq, const std::vector<int64_t>& locq,
                     const std::vector<int32_t>& own, int32_t q, int32_t L) {
  SendSlice S;
  S.q = q;
  int64_t c0 = -1, c1 = -1;
  for (int64_t c = Tp.nA; c < Tp.nA + Tp.nB; ++c)
    if (own[size_t(Tp.glob[size_t(c)])] == q) {
      if (c0 < 0) c0 = c;
      c1 = c + 1;
    }
  if (c0 < 0) return S;
  S.col0 = c0; S.col1 = c1;
  S.row0 = 2 * c0 * (L + 1);
  S.nrows = 2 * (c1 - c0) * (L + 1);
  S.val0 = Tp.colstart[size_t(c0)];
  S.nvals = Tp.colstart[size_t(c1)] - S.val0;
  S.dest_rows.reserve(size_t(S.nrows));
  S.dest_vals.reserve(size_t(S.nvals));
  for (int64_t c = c0; c < c1; ++c) {
    const int64_t cq = locq[size_t(Tp.glob[size_t(c)])];
    const int64_t np = Tp.nbr_ptr[size_t(c) + 1] - Tp.nbr_ptr[size_t(c)];
    const int64_t nq = Tq.nbr_ptr[size_t(cq) + 1] - Tq.nbr_ptr[size_t(cq)];
    const int32_t* lq = Tq.nbr.data() + Tq.nbr_ptr[size_t(cq)];
    std::vector<int64_t> slot_q(static_cast<size_t>(np));
    for (int64_t s = 0; s < np; ++s) {
      const int64_t cpp = Tp.nbr[size_t(Tp.nbr_ptr[size_t(c)] + s)];
      const int32_t cqq = int32_t(locq[size_t(Tp.glob[size_t(cpp)])]);
      slot_q[size_t(s)] = std::lower_bound(lq, lq + nq, cqq) - lq;
    }
    for (int64_t k = 0; k <= L; ++k) {
      const int64_t m = m_of(k, L);
      for (int a = 0; a < 2; ++a) {
        S.dest_rows.push_back(2 * (cq * (L + 1) + k) + a);
        S.import_src.push_back(2 * (cq * (L + 1) + k) + a);
        const int64_t rq = Tq.colstart[size_t(cq)] + 4 * nq * P_of(k) + a * 2 * nq * m;
        for (int64_t s = 0; s < np; ++s)
          for (int64_t g = 0; g < m; ++g)
            for (int b = 0; b < 2; ++b) S.dest_vals.push_back(rq + slot_q[size_t(s)] * 2 * m + 2 * g + b);
      }
    }
  }
  return S;
}

__global__ void gather_kernel(const double* __restrict__ src, const int64_t* __restrict__ idx,
                              double* __restrict__ out, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = src[idx[i]];
}

__global__ void scatter_add_kernel(const double* __restrict__ buf, const int64_t* __restrict__ idx,
                                   double* __restrict__ dst, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[idx[i]] += buf[i];
}

unsigned grid_for(int64_t n) { return unsigned(std::min<int64_t>((n + 255) / 256, 148 * 8)); }

template <class T>
fo_status dev_copy(T** dst, const std::vector<T>& v) {
  *dst = nullptr;
  if (v.empty()) return FO_OK;
  fo_status st = cuda_status(cudaMalloc(reinterpret_cast<void**>(dst), v.size() * sizeof(T)), "cudaMalloc");
  if (st) return st;
  return cuda_status(cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "cudaMemcpy");
}

}  // namespace
}  // namespace fo

namespace fo {
// Loopback transport: the P parts of a partitioned mesh held by ONE process
// (one device), for running the halo code path without a second GPU.  It
// stands in for NCCL's point-to-point calls only -- the plans, staging
// buffers, gather / unpack-add kernels and the sender order of fo_halo_import
// and fo_halo_sum are the same code.  A send is eager (copied into a
// stream-ordered scratch buffer on the sender's stream, an event recorded); a
// recv is completed, on the receiver's stream after that event, as soon as
// the matching send exists (the k-th send p -> q matches the k-th recv of q
// from p, NCCL's ordering).  Work that depends on a recv (the unpack-add) is
// enqueued when the last recv of its group completes, which may happen inside
// a later part's call: every part must enter a phase (import, sum) before
// work that depends on it is enqueued on any part.
struct LoopOp {                 // one group of a halo call
  int pending = 0;
  bool ended = false;
  std::function<fo_status()> cont;   // enqueued when all recvs completed
};
struct LoopSend { double* buf; int64_t n; cudaEvent_t ev; };
struct LoopRecv { double* dst; int64_t n; cudaStream_t s; std::shared_ptr<LoopOp> op; };
struct LoopGroup {
  std::mutex mu;
  int device = 0;
  std::map<std::pair<int32_t, int32_t>, std::deque<LoopSend>> sends;   // (from, to)
  std::map<std::pair<int32_t, int32_t>, std::deque<LoopRecv>> recvs;
  fo_status error = FO_OK;
};
}  // namespace fo

struct fo_halo_s {
  int device = 0;
  int32_t rank = 0, n_ranks = 1, L = 0;
  ncclComm_t comm = nullptr;
  std::shared_ptr<fo::LoopGroup> loop;    // loopback transport, else NCCL
  std::shared_ptr<fo::LoopOp> op;         // the loopback group being posted
  // owners q of my ghost columns: sum sends my slices to q, import receives
  // q's U into my ghost slice [row0, row0 + nrows)
  struct Owner { int32_t q; int64_t row0, nrows, val0, nvals; };
  // parts p holding ghosts of columns I own: sum receives + adds p's slices,
  // import gathers my U for p's ghosts (p's order) and sends it
  struct Holder {
    int32_t p; int64_t nrows, nvals;
    int64_t* d_rows; int64_t* d_vals;      // destination maps into my R / vals
    double* d_buf_r; double* d_buf_v;      // receive staging
    int64_t* d_imp_idx; double* d_imp_buf; // import gather map + buffer
  };
  std::vector<Owner> owners;
  std::vector<Holder> holders;
  // fo_assemble_jacobian_halo: the boundary patches and the transfers run on
  // `side` (higher priority than the caller's stream), joined back by events
  cudaStream_t side = nullptr;
  cudaEvent_t ev0 = nullptr, ev_b = nullptr, ev_sum = nullptr;
};

namespace fo {
namespace {

// ---- point-to-point transport: NCCL, or the loopback group ----
fo_status loop_match(LoopGroup& G, std::pair<int32_t, int32_t> ch) {
  auto& S = G.sends[ch];
  auto& Rq = G.recvs[ch];
  while (!S.empty() && !Rq.empty()) {
    LoopSend sd = S.front();
    LoopRecv rv = Rq.front();
    S.pop_front();
    Rq.pop_front();
    if (sd.n != rv.n) return fail(FO_ESTATE, "loopback: send / recv sizes differ");
    fo_status st = cuda_status(cudaStreamWaitEvent(rv.s, sd.ev, 0), "cudaStreamWaitEvent");
    if (!st) st = cuda_status(cudaMemcpyAsync(rv.dst, sd.buf, sizeof(double) * size_t(sd.n),
                                              cudaMemcpyDeviceToDevice, rv.s), "cudaMemcpyAsync");
    if (!st) st = cuda_status(cudaFreeAsync(sd.buf, rv.s), "cudaFreeAsync");
    cudaEventDestroy(sd.ev);
    if (st) return st;
    if (--rv.op->pending == 0 && rv.op->ended && rv.op->cont) {
      st = rv.op->cont();
      rv.op->cont = nullptr;
      if (st) return st;
    }
  }
  return FO_OK;
}

fo_status xp_group_start(fo_halo h) {
  if (h->loop) {
    h->op = std::make_shared<LoopOp>();
    return FO_OK;
  }
  return nccl_status(ncclGroupStart(), "ncclGroupStart");
}

fo_status xp_send(fo_halo h, const double* buf, int64_t n, int32_t peer, cudaStream_t s) {
  if (!h->loop) return nccl_status(ncclSend(buf, size_t(n), ncclDouble, peer, h->comm, s), "ncclSend");
  LoopGroup& G = *h->loop;
  std::lock_guard<std::mutex> lk(G.mu);
  LoopSend sd{nullptr, n, nullptr};
  fo_status st = cuda_status(cudaMallocAsync(reinterpret_cast<void**>(&sd.buf),
                                             sizeof(double) * size_t(std::max<int64_t>(n, 1)), s),
                             "cudaMallocAsync");
  if (!st && n > 0)
    st = cuda_status(cudaMemcpyAsync(sd.buf, buf, sizeof(double) * size_t(n), cudaMemcpyDeviceToDevice, s),
                     "cudaMemcpyAsync");
  if (!st) st = cuda_status(cudaEventCreateWithFlags(&sd.ev, cudaEventDisableTiming), "cudaEventCreate");
  if (!st) st = cuda_status(cudaEventRecord(sd.ev, s), "cudaEventRecord");
  if (st) return st;
  const auto ch = std::make_pair(h->rank, peer);
  G.sends[ch].push_back(sd);
  return loop_match(G, ch);
}

fo_status xp_recv(fo_halo h, double* buf, int64_t n, int32_t peer, cudaStream_t s) {
  if (!h->loop) return nccl_status(ncclRecv(buf, size_t(n), ncclDouble, peer, h->comm, s), "ncclRecv");
  LoopGroup& G = *h->loop;
  std::lock_guard<std::mutex> lk(G.mu);
  ++h->op->pending;
  const auto ch = std::make_pair(peer, h->rank);
  G.recvs[ch].push_back({buf, n, s, h->op});
  return loop_match(G, ch);
}

// ends the group; `cont` (the work that consumes the received data) is
// enqueued now (NCCL: stream order covers the recvs) or, on the loopback,
// when the group's last recv completes
fo_status xp_group_end(fo_halo h, std::function<fo_status()> cont) {
  if (!h->loop) {
    fo_status st = nccl_status(ncclGroupEnd(), "ncclGroupEnd");
    if (st) return st;
    return cont ? cont() : FO_OK;
  }
  LoopGroup& G = *h->loop;
  std::lock_guard<std::mutex> lk(G.mu);
  auto op = h->op;
  h->op.reset();
  op->ended = true;
  if (op->pending == 0) return cont ? cont() : FO_OK;
  op->cont = std::move(cont);
  return FO_OK;
}

}  // namespace
}  // namespace fo

using namespace fo;

extern "C" {

fo_status fo_part_graph_host(int64_t n_vert, int64_t n_tri, const int32_t* tri, int32_t n_layers,
                             const int32_t* part_of_tri, int32_t n_parts, int32_t my_part,
                             int64_t* n_cols, int64_t* n_owned, int64_t* n_ghost, int64_t* nnz,
                             int64_t* glob, int64_t* row_ptr, int32_t* col_idx) {
  if (n_layers < 1 || !part_of_tri || n_parts < 1 || my_part < 0 || my_part >= n_parts || !tri)
    return fail(FO_EINVAL, "bad arguments");
  for (int64_t t = 0; t < n_tri; ++t)
    if (part_of_tri[t] < 0 || part_of_tri[t] >= n_parts) return fail(FO_EINVAL, "part out of range");
  for (int64_t t = 0; t < 3 * n_tri; ++t)
    if (tri[t] < 0 || tri[t] >= n_vert) return fail(FO_EMESH, "vertex index out of range");
  Topo T;
  fo_status st = build_topology(n_vert, n_tri, tri, n_layers, part_of_tri, my_part, T);
  if (st) return st;
  if (n_cols) *n_cols = int64_t(T.glob.size());
  if (n_owned) *n_owned = T.nA;
  if (n_ghost) *n_ghost = T.nB;
  if (nnz) *nnz = T.colstart.back();
  if (glob) std::copy(T.glob.begin(), T.glob.end(), glob);
  if (row_ptr || col_idx) {
    std::vector<int64_t> rp;
    std::vector<int32_t> ci;
    build_csr(T, n_layers, row_ptr ? &rp : nullptr, col_idx ? &ci : nullptr, nullptr);
    if (row_ptr) std::copy(rp.begin(), rp.end(), row_ptr);
    if (col_idx) std::copy(ci.begin(), ci.end(), col_idx);
  }
  return FO_OK;
}

fo_status fo_halo_plan_host(int64_t n_vert, int64_t n_tri, const int32_t* tri, int32_t n_layers,
                            const int32_t* part_of_tri, int32_t n_parts, int32_t my_part,
                            int64_t* counts, int64_t* vcounts, int64_t* send_rows,
                            int64_t* dest_rows, int64_t* send_vals, int64_t* dest_vals) {
  if (n_layers < 1 || !part_of_tri || !tri || n_parts < 1 || my_part < 0 || my_part >= n_parts)
    return fail(FO_EINVAL, "bad arguments");
  for (int64_t t = 0; t < n_tri; ++t)
    if (part_of_tri[t] < 0 || part_of_tri[t] >= n_parts) return fail(FO_EINVAL, "part out of range");
  for (int64_t t = 0; t < 3 * n_tri; ++t)
    if (tri[t] < 0 || tri[t] >= n_vert) return fail(FO_EMESH, "vertex index out of range");
  const auto own = owners(n_vert, n_tri, tri, part_of_tri);
  Topo Tp;
  fo_status st = build_topology(n_vert, n_tri, tri, n_layers, part_of_tri, my_part, Tp);
  if (st) return st;
  int64_t ro = 0, vo = 0;
  for (int32_t q = 0; q < n_parts; ++q) {
    if (counts) counts[q] = 0;
    if (vcounts) vcounts[q] = 0;
    if (q == my_part) continue;
    bool any = false;
    for (int64_t c = Tp.nA; c < Tp.nA + Tp.nB && !any; ++c) any = own[size_t(Tp.glob[size_t(c)])] == q;
    if (!any) continue;
    Topo Tq;
    st = build_topology(n_vert, n_tri, tri, n_layers, part_of_tri, q, Tq);
    if (st) return st;
    const auto locq = local_index(Tq, n_vert);
    SendSlice S = plan_sends(Tp, Tq, locq, own, q, n_layers);
    if (counts) counts[q] = S.nrows;
    if (vcounts) vcounts[q] = S.nvals;
    for (int64_t i = 0; i < S.nrows; ++i) {
      if (send_rows) send_rows[ro + i] = S.row0 + i;
      if (dest_rows) dest_rows[ro + i] = S.dest_rows[size_t(i)];
    }
    for (int64_t i = 0; i < S.nvals; ++i) {
      if (send_vals) send_vals[vo + i] = S.val0 + i;
      if (dest_vals) dest_vals[vo + i] = S.dest_vals[size_t(i)];
    }
    ro += S.nrows;
    vo += S.nvals;
  }
  return FO_OK;
}

fo_status fo_nccl_unique_id(void* id128) {
  if (!id128) return fail(FO_EINVAL, "NULL id buffer");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  fo_status st = nccl_status(ncclGetUniqueId(&id), "ncclGetUniqueId");
  if (!st) std::memcpy(id128, &id, sizeof(id));
  return st;
}

}  // extern "C"

namespace fo {
namespace {
// the plan of one rank (owners / holders, device maps and staging), shared by
// the NCCL and the loopback transports
fo_status halo_plan(fo_halo h, fo_mesh local) {
  const int64_t nv = local->global_n_vert, nt = int64_t(local->global_tri.size() / 3);
  const int32_t* gtri = local->global_tri.data();
  const int32_t* part = local->global_part.data();
  const int32_t n_ranks = h->n_ranks, rank = h->rank;
  const auto own = owners(nv, nt, gtri, part);
  std::vector<Topo> T(static_cast<size_t>(n_ranks));
  fo_status st = FO_OK;
  for (int32_t p = 0; p < n_ranks && !st; ++p) st = build_topology(nv, nt, gtri, h->L, part, p, T[size_t(p)]);
  if (st) return st;
  std::vector<std::vector<int64_t>> loc(static_cast<size_t>(n_ranks));
  for (int32_t p = 0; p < n_ranks; ++p) loc[size_t(p)] = local_index(T[size_t(p)], nv);
  for (int32_t q = 0; q < n_ranks; ++q) {
    if (q == rank) continue;
    SendSlice S = plan_sends(T[size_t(rank)], T[size_t(q)], loc[size_t(q)], own, q, h->L);
    if (S.nrows > 0) h->owners.push_back({q, S.row0, S.nrows, S.val0, S.nvals});
  }
  for (int32_t p = 0; p < n_ranks && !st; ++p) {
    if (p == rank) continue;
    SendSlice S = plan_sends(T[size_t(p)], T[size_t(rank)], loc[size_t(rank)], own, rank, h->L);
    if (S.nrows == 0) continue;
    fo_halo_s::Holder hd{p, S.nrows, S.nvals, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    st = dev_copy(&hd.d_rows, S.dest_rows);
    if (!st) st = dev_copy(&hd.d_vals, S.dest_vals);
    if (!st) st = dev_copy(&hd.d_imp_idx, S.import_src);
    if (!st) st = cuda_status(cudaMalloc(&hd.d_buf_r, sizeof(double) * S.nrows), "cudaMalloc");
    if (!st) st = cuda_status(cudaMalloc(&hd.d_imp_buf, sizeof(double) * S.nrows), "cudaMalloc");
    if (!st) st = cuda_status(cudaMalloc(&hd.d_buf_v, sizeof(double) * std::max<int64_t>(1, S.nvals)), "cudaMalloc");
    h->holders.push_back(hd);
  }
  return st;
}
// cuStreamWaitValue32 from the driver (no libcuda link): the side stream
// waits on the kernel's ready flag
typedef CUresult (*WaitValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitValueFn wait_value_fn() {
  static WaitValueFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<WaitValueFn>(p);
    else
      cudaGetLastError();
  });
  return fn;
}

fo_status halo_streams(fo_halo h) {
  int lo = 0, hi = 0;
  fo_status st = cuda_status(cudaDeviceGetStreamPriorityRange(&lo, &hi), "cudaDeviceGetStreamPriorityRange");
  if (!st) st = cuda_status(cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, hi), "cudaStreamCreate");
  for (cudaEvent_t* e : {&h->ev0, &h->ev_b, &h->ev_sum})
    if (!st) st = cuda_status(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "cudaEventCreate");
  return st;
}

// Export: send my ghost slices of R / CSR values to their owners and
// add the slices I receive into my owned rows, senders in ascending rank
// order.  Transfers go on `sx`; the unpack-add on `su` once they are in
// (joined by an event when the streams differ).
fo_status halo_sum_impl(fo_halo h, double* d_R, double* d_vals, cudaStream_t sx, cudaStream_t su) {
  fo_status st = xp_group_start(h);
  for (auto& o : h->owners) {
    if (st) break;
    if (d_R) st = xp_send(h, d_R + o.row0, o.nrows, o.q, sx);
    if (!st && d_vals && o.nvals > 0) st = xp_send(h, d_vals + o.val0, o.nvals, o.q, sx);
  }
  for (auto& hd : h->holders) {
    if (st) break;
    if (d_R) st = xp_recv(h, hd.d_buf_r, hd.nrows, hd.p, sx);
    if (!st && d_vals && hd.nvals > 0) st = xp_recv(h, hd.d_buf_v, hd.nvals, hd.p, sx);
  }
  // deterministic unpack once every slice is in: senders in ascending rank order
  fo_status st2 = xp_group_end(h, [h, d_R, d_vals, sx, su]() -> fo_status {
    if (su != sx) {
      fo_status e = cuda_status(cudaEventRecord(h->ev_sum, sx), "cudaEventRecord");
      if (!e) e = cuda_status(cudaStreamWaitEvent(su, h->ev_sum, 0), "cudaStreamWaitEvent");
      if (e) return e;
    }
    for (auto& hd : h->holders) {
      if (d_R) scatter_add_kernel<<<grid_for(hd.nrows), 256, 0, su>>>(hd.d_buf_r, hd.d_rows, d_R, hd.nrows);
      if (d_vals && hd.nvals > 0)
        scatter_add_kernel<<<grid_for(hd.nvals), 256, 0, su>>>(hd.d_buf_v, hd.d_vals, d_vals, hd.nvals);
    }
    return cuda_status(cudaGetLastError(), "scatter_add_kernel");
  });
  return st ? st : st2;
}
}  // namespace
}  // namespace fo

extern "C" {

fo_status fo_halo_create(fo_mesh local, fo_graph local_g, const void* nccl_unique_id, int32_t rank,
                         int32_t n_ranks, fo_halo* out) {
  if (!local || !local_g || !nccl_unique_id || !out) return fail(FO_EINVAL, "NULL argument");
  *out = nullptr;
  if (local_g->mesh != local) return fail(FO_ESTATE, "graph was built for another mesh");
  if (n_ranks != local->n_parts || rank != local->part)
    return fail(FO_ESTATE, "rank / n_ranks do not match the local mesh's part / n_parts");
  if (!local->global_tri.size() && n_ranks > 1)
    return fail(FO_ESTATE, "mesh has no global footprint (create it with fo_mesh_create_part)");
  fo_status st = cuda_status(cudaSetDevice(local->device), "cudaSetDevice");
  if (st) return st;
  fo_halo h = new fo_halo_s();
  h->device = local->device;
  h->rank = rank;
  h->n_ranks = n_ranks;
  h->L = local->L;
  if (n_ranks > 1) {
    st = halo_plan(h, local);
    if (!st) {
      ncclUniqueId id;
      std::memcpy(&id, nccl_unique_id, sizeof(id));
      st = nccl_status(ncclCommInitRank(&h->comm, n_ranks, id, rank), "ncclCommInitRank");
    }
    if (!st) st = halo_streams(h);
    if (st) { fo_halo_destroy(h); return st; }
  }
  *out = h;
  return FO_OK;
}

fo_status fo_halo_create_loopback(const fo_mesh* parts, const fo_graph* graphs, int32_t n_parts,
                                  fo_halo* out) {
  if (!parts || !graphs || !out || n_parts < 1) return fail(FO_EINVAL, "NULL argument or n_parts < 1");
  for (int32_t p = 0; p < n_parts; ++p) out[p] = nullptr;
  for (int32_t p = 0; p < n_parts; ++p) {
    if (!parts[p] || !graphs[p]) return fail(FO_EINVAL, "NULL mesh or graph");
    if (graphs[p]->mesh != parts[p]) return fail(FO_ESTATE, "graph was built for another mesh");
    if (parts[p]->n_parts != n_parts || parts[p]->part != p)
      return fail(FO_ESTATE, "parts[p] must be the local mesh of part p of an n_parts partition");
    if (parts[p]->device != parts[0]->device) return fail(FO_EINVAL, "loopback parts must share one device");
    if (n_parts > 1 && (parts[p]->global_tri != parts[0]->global_tri ||
                        parts[p]->global_part != parts[0]->global_part))
      return fail(FO_ESTATE, "parts come from different footprints or partitions");
  }
  fo_status st = cuda_status(cudaSetDevice(parts[0]->device), "cudaSetDevice");
  if (st) return st;
  auto G = std::make_shared<LoopGroup>();
  G->device = parts[0]->device;
  for (int32_t p = 0; p < n_parts && !st; ++p) {
    fo_halo h = new fo_halo_s();
    h->device = parts[p]->device;
    h->rank = p;
    h->n_ranks = n_parts;
    h->L = parts[p]->L;
    h->loop = G;
    out[p] = h;
    if (n_parts > 1) st = halo_plan(h, parts[p]);
    if (!st && n_parts > 1) st = halo_streams(h);
  }
  if (st)
    for (int32_t p = 0; p < n_parts; ++p) { fo_halo_destroy(out[p]); out[p] = nullptr; }
  return st;
}

fo_status fo_halo_import(fo_halo h, double* d_U, void* stream) {
  NvtxRange nvtx("fo_halo_import");
  if (!h) return fail(FO_EINVAL, "halo is NULL");
  if (h->n_ranks == 1) return FO_OK;
  if (!d_U) return fail(FO_EINVAL, "d_U is NULL");
  fo_status st = cuda_status(cudaSetDevice(h->device), "cudaSetDevice");
  if (st) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (auto& hd : h->holders)
    gather_kernel<<<grid_for(hd.nrows), 256, 0, s>>>(d_U, hd.d_imp_idx, hd.d_imp_buf, hd.nrows);
  st = cuda_status(cudaGetLastError(), "gather_kernel");
  if (st) return st;
  st = xp_group_start(h);
  for (auto& hd : h->holders)
    if (!st) st = xp_send(h, hd.d_imp_buf, hd.nrows, hd.p, s);
  for (auto& o : h->owners)
    if (!st) st = xp_recv(h, d_U + o.row0, o.nrows, o.q, s);
  fo_status st2 = xp_group_end(h, nullptr);
  return st ? st : st2;
}

fo_status fo_halo_sum(fo_halo h, double* d_R, double* d_vals, void* stream) {
  NvtxRange nvtx("fo_halo_sum");
  if (!h) return fail(FO_EINVAL, "halo is NULL");
  if (h->n_ranks == 1) return FO_OK;
  fo_status st = cuda_status(cudaSetDevice(h->device), "cudaSetDevice");
  if (st) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return halo_sum_impl(h, d_R, d_vals, s, s);
}

fo_status fo_assemble_jacobian_halo(fo_mesh m, fo_graph g, fo_halo h, const double* d_U, double* d_R,
                                    double* d_vals, void* stream) {
  NvtxRange nvtx("fo_assemble_jacobian_halo");
  if (!m || !h) return fail(FO_EINVAL, "mesh or halo is NULL");
  if (!d_U || !d_R) return fail(FO_EINVAL, "d_U or d_R is NULL");
  if (d_vals && (!g || g->mesh != m)) return fail(FO_ESTATE, "graph is NULL or was built for another mesh");
  if (h->rank != m->part || h->n_ranks != m->n_parts) return fail(FO_ESTATE, "halo was built for another mesh");
  if (m->quad) return fail(FO_EINVAL, "fo_assemble_jacobian_halo: wedge / tetrahedral meshes only");
  fo_status st = cuda_status(cudaSetDevice(m->device), "cudaSetDevice");
  if (st) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // sequential fallbacks: one part; the atomic ablation; the lateral term (it
  // adds into ghost rows after every patch, so nothing can be sent earlier)
  if (h->n_ranks == 1 || m->scatter == FO_SCATTER_ATOMIC || m->lateral || m->plan.n_patches == 0) {
    st = d_vals ? launch_jacobian(m, d_U, d_R, d_vals, s) : launch_residual(m, d_U, d_R, s);
    if (!st && h->n_ranks > 1) st = halo_sum_impl(h, d_R, d_vals, s, s);
    return st;
  }
  WaitValueFn wv = wait_value_fn();
  if (wv) {
    st = launch_owner_overlap(m, d_U, d_R, d_vals, s, h->side, h->ev0,
                              [wv](cudaStream_t side, const int32_t* flag) -> fo_status {
                                const CUresult r = wv(reinterpret_cast<CUstream>(side),
                                                      reinterpret_cast<CUdeviceptr>(flag), 1,
                                                      CU_STREAM_WAIT_VALUE_GEQ);
                                return r == CUDA_SUCCESS ? FO_OK : fail(FO_ECUDA, "cuStreamWaitValue32 failed");
                              });
    // the side stream sends the ghost rows once the boundary patches raised
    // the ready flag, while the interior patches run on s; the unpack-add
    // joins s after both
    if (st == FO_OK) return halo_sum_impl(h, d_R, d_vals, h->side, s);
    if (st != FO_ESTATE) return st;
  }
  // no overlap available: the sequential order
  st = d_vals ? launch_jacobian(m, d_U, d_R, d_vals, s) : launch_residual(m, d_U, d_R, s);
  return st ? st : halo_sum_impl(h, d_R, d_vals, s, s);
}

fo_status fo_halo_info(fo_halo h, int32_t* n_neighbors, int64_t* recv_rows, int64_t* recv_vals) {
  if (!h) return fail(FO_EINVAL, "halo is NULL");
  int64_t rr = 0, rv = 0;
  for (auto& hd : h->holders) { rr += hd.nrows; rv += hd.nvals; }
  int32_t nn = 0;
  std::vector<int32_t> peers;
  for (auto& o : h->owners) peers.push_back(o.q);
  for (auto& hd : h->holders) peers.push_back(hd.p);
  std::sort(peers.begin(), peers.end());
  nn = int32_t(std::unique(peers.begin(), peers.end()) - peers.begin());
  if (n_neighbors) *n_neighbors = nn;
  if (recv_rows) *recv_rows = rr;
  if (recv_vals) *recv_vals = rv;
  return FO_OK;
}

void fo_halo_destroy(fo_halo h) {
  if (!h) return;
  cudaSetDevice(h->device);
  for (auto& hd : h->holders) {
    cudaFree(hd.d_rows); cudaFree(hd.d_vals); cudaFree(hd.d_buf_r); cudaFree(hd.d_buf_v);
    cudaFree(hd.d_imp_idx); cudaFree(hd.d_imp_buf);
  }
  if (h->comm) ncclCommDestroy(h->comm);
  if (h->side) cudaStreamDestroy(h->side);
  for (cudaEvent_t e : {h->ev0, h->ev_b, h->ev_sum})
    if (e) cudaEventDestroy(e);
  delete h;
}

}  // extern "C"
