"""Thin ctypes binding of libfo.so (include/fo.h).

Argument marshalling only: every step of the assembly runs in libfo's CUDA
kernels.  PyTorch provides device memory and streams.  There is no CPU
fallback: if libfo.so is missing or no CUDA device is present, the calls
raise.

    mesh = Mesh.from_footprint(fp)            # fo_mesh_create
    graph = mesh.graph()                        # fo_graph_build
    R = mesh.residual(U)                        # fo_assemble_residual
    R, vals = mesh.jacobian(U, graph)           # fo_assemble_jacobian
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libfo.so")
ROOT = os.path.dirname(_PKG)
HEADER = os.path.join(ROOT, "include", "fo.h")

FO_OK, FO_EINVAL, FO_EMESH, FO_ECUDA, FO_ENCCL, FO_ENOMEM, FO_ESTATE = 0, -1, -2, -3, -4, -5, -6
SCATTER_OWNER, SCATTER_ATOMIC, SCATTER_OWNER_WS, SCATTER_OWNER_1WG = 0, 1, 2, 3
_NAMES = {0: "FO_OK", -1: "FO_EINVAL", -2: "FO_EMESH", -3: "FO_ECUDA", -4: "FO_ENCCL",
          -5: "FO_ENOMEM", -6: "FO_ESTATE"}


class FoError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: {_NAMES.get(status, status)}: {msg}")
        self.status = status


class Params(C.Structure):
    _fields_ = [("rho", C.c_double), ("g", C.c_double), ("rho_w", C.c_double),
                ("glen_n", C.c_double), ("eps_reg", C.c_double), ("A", C.c_double),
                ("H_min", C.c_double)]


_lib = None
P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double

_SIGS = {
    "fo_params_default": [P],
    "fo_mesh_create": [P, I64, P, I64, P, I32, P, P, P, P, P, P, C.c_int, P],
    "fo_mesh_create_part": [P, I64, P, I64, P, I32, P, P, P, P, P, P, P, I32, I32, C.c_int, P],
    "fo_mesh_create_quad": [P, I64, P, I64, P, I32, P, P, P, P, P, P, C.c_int, P],
    "fo_partition": [I64, I32, P],
    "fo_mesh_info": [P, P, P, P, P],
    "fo_mesh_columns": [P, P, P, P, P, P],
    "fo_graph_build": [P, P],
    "fo_graph_info": [P, P, P],
    "fo_graph_arrays": [P, P, P],
    "fo_graph_to_host": [P, P, P],
    "fo_graph_host": [I64, I64, P, I32, P, P, P],
    "fo_assemble_residual": [P, P, P, P],
    "fo_assemble_jacobian": [P, P, P, P, P, P],
    "fo_assemble_jacobian_host": [P, P, P, P, P, P],
    "fo_set_scatter": [P, C.c_int],
    "fo_mesh_set_temperature": [P, P, C.c_double, C.c_double],
    "fo_set_lateral": [P, C.c_int],
    "fo_set_element": [P, C.c_int],
    "fo_spmv": [P, P, P, P, P, P],
    "fo_line_factor": [P, P, P, P],
    "fo_line_solve": [P, P, P, P],
    "fo_krylov_dots": [P, I64, I32, P, I64, P, P, P],
    "fo_krylov_update": [P, I64, I32, P, I64, P, P, P],
    "fo_last_launch_count": [P, P],
    "fo_kernel_timing": [P, I32],
    "fo_kernel_time_ms": [P, P, P],
    "fo_nccl_unique_id": [P],
    "fo_halo_create": [P, P, P, I32, I32, P],
    "fo_halo_create_loopback": [P, P, I32, P],
    "fo_halo_import": [P, P, P],
    "fo_halo_sum": [P, P, P, P],
    "fo_assemble_jacobian_halo": [P, P, P, P, P, P, P],
    "fo_halo_info": [P, P, P, P],
    "fo_halo_plan_host": [I64, I64, P, I32, P, I32, I32, P, P, P, P, P, P],
    "fo_part_graph_host": [I64, I64, P, I32, P, I32, I32, P, P, P, P, P, P, P],
    "fo_plan_check_host": [I64, P, I64, P, I32, P, I32, I32, P],
    "fo_plan_check_quad_host": [I64, P, I64, P, I32, P],
}
_VOID = ["fo_mesh_destroy", "fo_graph_destroy", "fo_halo_destroy"]


def declared_symbols() -> list[str]:
    """every function declared in include/fo.h (parsed from the header)."""
    import re
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"FO_API\s+[\w\s\*]*?\b(fo_\w+)\s*\(", txt)))


def lib():
    """load libfo.so; raises if it is missing (no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FoError(FO_ESTATE, "load", f"{LIB_PATH} missing: run paper_2204_04321_b200._build")
        L = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        for name in _VOID:
            getattr(L, name).argtypes = [P]
            getattr(L, name).restype = None
        L.fo_last_error.argtypes = []
        L.fo_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def check(status: int, where: str):
    if status != FO_OK:
        raise FoError(status, where, lib().fo_last_error().decode())


def default_params(**over) -> Params:
    p = Params()
    check(lib().fo_params_default(C.byref(p)), "fo_params_default")
    for k, v in over.items():
        setattr(p, k, float(v))
    return p


def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return C.c_void_p(a.ctypes.data)


def _stream_ptr(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def partition(n_tri: int, n_parts: int) -> np.ndarray:
    part = np.zeros(n_tri, dtype=np.int32)
    check(lib().fo_partition(n_tri, n_parts, _ptr(part)), "fo_partition")
    return part


def graph_host(n_vert, tri, n_layers):
    """library's CSR pattern built on the host (no device needed)."""
    tri = np.ascontiguousarray(tri, dtype=np.int32)
    n_tri = tri.shape[0]
    n_dof = 2 * n_vert * (n_layers + 1)
    row_ptr = np.zeros(n_dof + 1, dtype=np.int64)
    nnz = C.c_int64(0)
    check(lib().fo_graph_host(n_vert, n_tri, _ptr(tri), n_layers, None, None, C.byref(nnz)), "fo_graph_host")
    col = np.zeros(nnz.value, dtype=np.int32)
    check(lib().fo_graph_host(n_vert, n_tri, _ptr(tri), n_layers, _ptr(row_ptr), _ptr(col), C.byref(nnz)),
          "fo_graph_host")
    return row_ptr, col


def plan_check_host(xy, tri, n_layers, part=None, n_parts=1, my_part=0):
    """host-only coverage check of the owner-computes plan (no device): dict of
    patches, pairs, contributions, zero_cols, multi, bad_slots, bad_entries, plan_bytes."""
    xy = np.ascontiguousarray(xy, dtype=np.float64)
    tri = np.ascontiguousarray(tri, dtype=np.int32)
    st = np.zeros(8, dtype=np.int64)
    pt = None if part is None else np.ascontiguousarray(part, dtype=np.int32)
    check(lib().fo_plan_check_host(xy.shape[0], _ptr(xy), tri.shape[0], _ptr(tri), n_layers, _ptr(pt),
                                   my_part, n_parts, _ptr(st)), "fo_plan_check_host")
    keys = ["patches", "pairs", "contributions", "zero_cols", "multi", "bad_slots", "bad_entries", "plan_bytes"]
    return dict(zip(keys, st.tolist()))


def plan_check_quad_host(xy, quad, n_layers):
    """host-only coverage check of the hexahedral (quad-patch) plan: dict as
    plan_check_host."""
    xy = np.ascontiguousarray(xy, dtype=np.float64)
    quad = np.ascontiguousarray(quad, dtype=np.int32)
    st = np.zeros(8, dtype=np.int64)
    check(lib().fo_plan_check_quad_host(xy.shape[0], _ptr(xy), quad.shape[0], _ptr(quad), n_layers, _ptr(st)),
          "fo_plan_check_quad_host")
    keys = ["patches", "pairs", "contributions", "zero_cols", "multi", "bad_slots", "bad_entries", "plan_bytes"]
    return dict(zip(keys, st.tolist()))


def part_graph_host(n_vert, tri, n_layers, part, n_parts, my_part):
    """local numbering and CSR pattern of one part (no device): returns
    (glob, n_owned, n_ghost, row_ptr, col_idx)."""
    tri = np.ascontiguousarray(tri, dtype=np.int32)
    part = np.ascontiguousarray(part, dtype=np.int32)
    nc, na, nb, nnz = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    args = (n_vert, tri.shape[0], _ptr(tri), n_layers, _ptr(part), n_parts, my_part)
    check(lib().fo_part_graph_host(*args, C.byref(nc), C.byref(na), C.byref(nb), C.byref(nnz),
                                   None, None, None), "fo_part_graph_host")
    glob = np.zeros(nc.value, dtype=np.int64)
    row_ptr = np.zeros(2 * nc.value * (n_layers + 1) + 1, dtype=np.int64)
    col = np.zeros(nnz.value, dtype=np.int32)
    check(lib().fo_part_graph_host(*args, None, None, None, None, _ptr(glob), _ptr(row_ptr), _ptr(col)),
          "fo_part_graph_host")
    return glob, na.value, nb.value, row_ptr, col


def halo_plan_host(n_vert, tri, n_layers, part, n_parts, my_part):
    """what part my_part sends to every other part: dict q -> (send_rows,
    dest_rows, send_vals, dest_vals) (offsets in the sender's / owner's arrays)."""
    tri = np.ascontiguousarray(tri, dtype=np.int32)
    part = np.ascontiguousarray(part, dtype=np.int32)
    counts = np.zeros(n_parts, dtype=np.int64)
    vcounts = np.zeros(n_parts, dtype=np.int64)
    args = (n_vert, tri.shape[0], _ptr(tri), n_layers, _ptr(part), n_parts, my_part)
    check(lib().fo_halo_plan_host(*args, _ptr(counts), _ptr(vcounts), None, None, None, None),
          "fo_halo_plan_host")
    sr = np.zeros(counts.sum(), dtype=np.int64); dr = np.zeros_like(sr)
    sv = np.zeros(vcounts.sum(), dtype=np.int64); dv = np.zeros_like(sv)
    check(lib().fo_halo_plan_host(*args, _ptr(counts), _ptr(vcounts), _ptr(sr), _ptr(dr), _ptr(sv), _ptr(dv)),
          "fo_halo_plan_host")
    out, ro, vo = {}, 0, 0
    for q in range(n_parts):
        if counts[q] == 0:
            continue
        out[q] = (sr[ro:ro + counts[q]], dr[ro:ro + counts[q]], sv[vo:vo + vcounts[q]], dv[vo:vo + vcounts[q]])
        ro += counts[q]
        vo += vcounts[q]
    return out


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    check(lib().fo_nccl_unique_id(buf), "fo_nccl_unique_id")
    return bytes(buf)


class Halo:
    """Ghost import / ghost-row sum of a partitioned mesh: NCCL (collective,
    one rank per GPU) or, with Halo.loopback, all parts in one process."""

    def __init__(self, mesh: "Mesh", uid: bytes | None, rank: int, n_ranks: int, _handle=None):
        self.mesh = mesh
        if _handle is not None:
            self.handle = _handle
            return
        buf = (C.c_char * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        check(lib().fo_halo_create(mesh.handle, mesh.graph().handle, buf, rank, n_ranks, C.byref(h)),
              "fo_halo_create")
        self.handle = h

    @classmethod
    def loopback(cls, meshes) -> list["Halo"]:
        """fo_halo_create_loopback: the halos of all parts (meshes[p] = part p)
        of one partition on one device."""
        n = len(meshes)
        parts = (C.c_void_p * n)(*[m.handle.value for m in meshes])
        graphs = (C.c_void_p * n)(*[m.graph().handle.value for m in meshes])
        out = (C.c_void_p * n)()
        check(lib().fo_halo_create_loopback(parts, graphs, n, out), "fo_halo_create_loopback")
        return [cls(m, None, p, n, _handle=C.c_void_p(out[p])) for p, m in enumerate(meshes)]

    def info(self):
        nn, rr, rv = C.c_int32(), C.c_int64(), C.c_int64()
        check(lib().fo_halo_info(self.handle, C.byref(nn), C.byref(rr), C.byref(rv)), "fo_halo_info")
        return nn.value, rr.value, rv.value

    def import_(self, U, stream=None):
        check(lib().fo_halo_import(self.handle, _ptr(U), _stream_ptr(stream)), "fo_halo_import")

    def sum(self, R=None, vals=None, stream=None):
        check(lib().fo_halo_sum(self.handle, _ptr(R), _ptr(vals), _stream_ptr(stream)), "fo_halo_sum")

    def assemble(self, U, R, vals=None, stream=None):
        """fo_assemble_jacobian_halo: assembly of the local mesh (R, and the
        CSR values if vals is given) with the ghost-row sum overlapped; the
        ghost U must be imported first.  R / vals are overwritten."""
        g = self.mesh.graph() if vals is not None else None
        check(lib().fo_assemble_jacobian_halo(self.mesh.handle, g.handle if g is not None else None, self.handle,
                                              _ptr(U), _ptr(R), _ptr(vals), _stream_ptr(stream)),
              "fo_assemble_jacobian_halo")

    def close(self):
        if self.handle:
            lib().fo_halo_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Graph:
    def __init__(self, mesh: "Mesh"):
        self.mesh = mesh
        h = C.c_void_p()
        check(lib().fo_graph_build(mesh.handle, C.byref(h)), "fo_graph_build")
        self.handle = h
        n_rows, nnz = C.c_int64(), C.c_int64()
        check(lib().fo_graph_info(h, C.byref(n_rows), C.byref(nnz)), "fo_graph_info")
        self.n_rows, self.nnz = n_rows.value, nnz.value

    def row_ptr_host(self):
        row_ptr = np.zeros(self.n_rows + 1, dtype=np.int64)
        check(lib().fo_graph_to_host(self.handle, _ptr(row_ptr), None), "fo_graph_to_host")
        return row_ptr

    def to_host(self):
        row_ptr = np.zeros(self.n_rows + 1, dtype=np.int64)
        col = np.zeros(self.nnz, dtype=np.int32)
        check(lib().fo_graph_to_host(self.handle, _ptr(row_ptr), _ptr(col)), "fo_graph_to_host")
        return row_ptr, col

    def close(self):
        if self.handle:
            lib().fo_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Mesh:
    """fo_mesh handle + sizes.  Construct with from_footprint / from_arrays."""

    def __init__(self, handle, device: int):
        self.handle = handle
        self.device = device
        n_nodes, n_dofs, n_elems, n_owned = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().fo_mesh_info(handle, C.byref(n_nodes), C.byref(n_dofs), C.byref(n_elems),
                                 C.byref(n_owned)), "fo_mesh_info")
        self.n_nodes, self.n_dofs, self.n_elems, self.n_owned_dofs = (
            n_nodes.value, n_dofs.value, n_elems.value, n_owned.value)
        self._graph = None

    @staticmethod
    def _arrays(fp):
        arr = dict(
            xy=np.ascontiguousarray(fp.xy, dtype=np.float64),
            tri=np.ascontiguousarray(fp.tri, dtype=np.int32),
            sigma=np.ascontiguousarray(fp.sigma, dtype=np.float64),
            H=np.ascontiguousarray(fp.thickness, dtype=np.float64),
            s=np.ascontiguousarray(fp.surface, dtype=np.float64),
            b=None if fp.bed is None else np.ascontiguousarray(fp.bed, dtype=np.float64),
            beta=np.ascontiguousarray(fp.beta, dtype=np.float64),
            A=None if getattr(fp, "A_elem", None) is None else np.ascontiguousarray(fp.A_elem, dtype=np.float64),
        )
        return arr

    @classmethod
    def from_footprint(cls, fp, device: int = 0, params: dict | None = None, part=None,
                       my_part: int = 0, n_parts: int = 1) -> "Mesh":
        prm = dict(fp.params)
        if params:
            prm.update(params)
        p = default_params(**prm)
        a = cls._arrays(fp)
        h = C.c_void_p()
        n_vert, n_tri, L = a["xy"].shape[0], a["tri"].shape[0], a["sigma"].size - 1
        if getattr(fp, "elem_type", 0) == 2:   # NEXT-f4: quadrilateral footprint, hexahedra
            if part is not None:
                raise FoError(FO_EINVAL, "fo_mesh_create_quad", "hexahedral meshes are single-domain")
            st = lib().fo_mesh_create_quad(C.byref(p), n_vert, _ptr(a["xy"]), n_tri, _ptr(a["tri"]), L,
                                           _ptr(a["sigma"]), _ptr(a["H"]), _ptr(a["s"]), _ptr(a["b"]),
                                           _ptr(a["beta"]), _ptr(a["A"]), device, C.byref(h))
            check(st, "fo_mesh_create_quad")
        elif part is None:
            st = lib().fo_mesh_create(C.byref(p), n_vert, _ptr(a["xy"]), n_tri, _ptr(a["tri"]), L,
                                      _ptr(a["sigma"]), _ptr(a["H"]), _ptr(a["s"]), _ptr(a["b"]),
                                      _ptr(a["beta"]), _ptr(a["A"]), device, C.byref(h))
            check(st, "fo_mesh_create")
        else:
            part = np.ascontiguousarray(part, dtype=np.int32)
            st = lib().fo_mesh_create_part(C.byref(p), n_vert, _ptr(a["xy"]), n_tri, _ptr(a["tri"]), L,
                                           _ptr(a["sigma"]), _ptr(a["H"]), _ptr(a["s"]), _ptr(a["b"]),
                                           _ptr(a["beta"]), _ptr(a["A"]), _ptr(part), my_part, n_parts,
                                           device, C.byref(h))
            check(st, "fo_mesh_create_part")
        return cls(h, device)

    def columns(self):
        n, a, b, c = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().fo_mesh_columns(self.handle, C.byref(n), C.byref(a), C.byref(b), C.byref(c), None),
              "fo_mesh_columns")
        glob = np.zeros(n.value, dtype=np.int64)
        check(lib().fo_mesh_columns(self.handle, None, None, None, None, _ptr(glob)), "fo_mesh_columns")
        return glob, a.value, b.value, c.value

    def graph(self) -> Graph:
        if self._graph is None:
            self._graph = Graph(self)
        return self._graph

    def set_temperature(self, T_star, A0: float = 0.0, Q: float = 0.0):
        """NEXT-f3: A = A0 exp(-Q / (R T*)) per wedge; T_star is a
        host array [n_tri*L] of the (global) footprint, None reverts."""
        if T_star is None:
            check(lib().fo_mesh_set_temperature(self.handle, None, 0.0, 0.0), "fo_mesh_set_temperature")
            return
        T = np.ascontiguousarray(T_star, dtype=np.float64)
        check(lib().fo_mesh_set_temperature(self.handle, T.ctypes.data, float(A0), float(Q)),
              "fo_mesh_set_temperature")

    def set_element(self, elem_type: int):
        """NEXT-f4: 0 = wedge (default), 1 = three P1 tetrahedra per prism."""
        check(lib().fo_set_element(self.handle, int(elem_type)), "fo_set_element")

    def set_lateral(self, on: bool = True):
        """NEXT-f1: include the lateral margin term in R."""
        check(lib().fo_set_lateral(self.handle, 1 if on else 0), "fo_set_lateral")

    def set_scatter(self, mode: int):
        check(lib().fo_set_scatter(self.handle, int(mode)), "fo_set_scatter")

    def kernel_timing(self, on: bool):
        check(lib().fo_kernel_timing(self.handle, 1 if on else 0), "fo_kernel_timing")

    def kernel_time_ms(self):
        """(summed ms, launches) of the main kernel since the last call."""
        ms, n = C.c_double(), C.c_int32()
        check(lib().fo_kernel_time_ms(self.handle, C.byref(ms), C.byref(n)), "fo_kernel_time_ms")
        return ms.value, n.value

    def last_launch_count(self) -> int:
        n = C.c_int32()
        check(lib().fo_last_launch_count(self.handle, C.byref(n)), "fo_last_launch_count")
        return n.value

    def _alloc(self, n):
        import torch
        return torch.empty(n, dtype=torch.float64, device=f"cuda:{self.device}")

    def residual(self, U, R=None, stream=None):
        """R = F(U) on the device (U: float64 CUDA tensor [n_dofs])."""
        if R is None:
            R = self._alloc(self.n_dofs)
        self._check_vec(U, self.n_dofs)
        self._check_vec(R, self.n_dofs)
        check(lib().fo_assemble_residual(self.handle, _ptr(U), _ptr(R), _stream_ptr(stream)),
              "fo_assemble_residual")
        return R

    def jacobian(self, U, graph: Graph | None = None, R=None, vals=None, stream=None, want_R=True):
        graph = graph or self.graph()
        if vals is None:
            vals = self._alloc(graph.nnz)
        if R is None and want_R:
            R = self._alloc(self.n_dofs)
        self._check_vec(U, self.n_dofs)
        self._check_vec(vals, graph.nnz)
        if R is not None:
            self._check_vec(R, self.n_dofs)
        check(lib().fo_assemble_jacobian(self.handle, graph.handle, _ptr(U), _ptr(R), _ptr(vals),
                                         _stream_ptr(stream)), "fo_assemble_jacobian")
        return R, vals

    def jacobian_host(self, U_host, R_host, vals_host, graph: Graph | None = None, stream=None):
        """host-buffer entry point (copies in and out inside the call)."""
        graph = graph or self.graph()
        check(lib().fo_assemble_jacobian_host(self.handle, graph.handle, _ptr(U_host), _ptr(R_host),
                                              _ptr(vals_host), _stream_ptr(stream)),
              "fo_assemble_jacobian_host")

    def _check_vec(self, t, n):
        import torch
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64
                and t.is_contiguous() and t.numel() == n and t.device.index == self.device):
            raise FoError(FO_EINVAL, "argument", f"need a contiguous float64 CUDA tensor of {n} "
                                                 f"elements on cuda:{self.device}")

    def close(self):
        if self._graph is not None:
            self._graph.close()
            self._graph = None
        if self.handle:
            lib().fo_mesh_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
