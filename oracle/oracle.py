"""ctypes wrapper of the serial CPU oracle (liboracle.so, fo_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package never
imports this module.  It imports nothing from the product package: a workload
is passed duck-typed (attributes xy, tri, sigma, thickness, surface, bed, beta,
A_elem, params -- e.g. a meshgen.Footprint).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

VISC, BODY, BASAL, ALL, LATERAL = 1, 2, 4, 7, 8


def build(force: bool = False) -> str:
    """compile liboracle.so with g++ -O2 (no fast-math, no threads)."""
    src = os.path.join(_HERE, "fo_oracle.cpp")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "fo_oracle.h"))):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-Wall", "-fPIC", "-shared",
                               "-o", _LIB_PATH, src])
    return _LIB_PATH


class _Params(C.Structure):
    _fields_ = [("rho", C.c_double), ("g", C.c_double), ("rho_w", C.c_double),
                ("glen_n", C.c_double), ("eps_reg", C.c_double), ("A", C.c_double),
                ("H_min", C.c_double)]


class _Mesh(C.Structure):
    _fields_ = [("n_vert", C.c_int64), ("xy", C.c_void_p), ("n_tri", C.c_int64),
                ("tri", C.c_void_p), ("n_layers", C.c_int32), ("sigma", C.c_void_p),
                ("thickness", C.c_void_p), ("surface", C.c_void_p), ("bed", C.c_void_p),
                ("beta", C.c_void_p), ("A_elem", C.c_void_p), ("p", _Params),
                ("T_star", C.c_void_p), ("A0", C.c_double), ("Q_act", C.c_double),
                ("elem_type", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        P = C.c_void_p
        L.ora_validate.argtypes = [P]
        L.ora_graph.argtypes = [P, P, P, P]
        L.ora_residual.argtypes = [P, C.c_int, P, P, P, P]
        L.ora_jacobian.argtypes = [P, C.c_int, P, P, P, P, P]
        L.ora_energy.argtypes = [P, C.c_int, P, C.c_int64, P]
        L.ora_element.argtypes = [P, C.c_int, P, C.c_int64, C.c_int32, P, P, P]
        for f in (L.ora_validate, L.ora_graph, L.ora_residual, L.ora_jacobian,
                  L.ora_energy, L.ora_element):
            f.restype = C.c_int
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


class OracleError(RuntimeError):
    pass


class Oracle:
    """Holds contiguous copies of one workload's arrays and calls the oracle."""

    def __init__(self, fp, params: dict | None = None):
        prm = dict(fp.params)
        if params:
            prm.update(params)
        self.xy = np.ascontiguousarray(fp.xy, dtype=np.float64)
        self.tri = np.ascontiguousarray(fp.tri, dtype=np.int32)
        self.sigma = np.ascontiguousarray(fp.sigma, dtype=np.float64)
        self.H = np.ascontiguousarray(fp.thickness, dtype=np.float64)
        self.s = np.ascontiguousarray(fp.surface, dtype=np.float64)
        self.b = None if fp.bed is None else np.ascontiguousarray(fp.bed, dtype=np.float64)
        self.beta = np.ascontiguousarray(fp.beta, dtype=np.float64)
        self.A_elem = None if getattr(fp, "A_elem", None) is None else \
            np.ascontiguousarray(fp.A_elem, dtype=np.float64)
        # NEXT-f3: per-wedge temperature T* with the Arrhenius constants
        self.T_star = None if getattr(fp, "T_star", None) is None else \
            np.ascontiguousarray(fp.T_star, dtype=np.float64)
        arr = getattr(fp, "arrhenius", None) or {}
        self.params = prm
        self.L = int(self.sigma.size - 1)
        self.n_vert = int(self.xy.shape[0])
        self.n_tri = int(self.tri.shape[0])
        self.n_dof = 2 * self.n_vert * (self.L + 1)
        self._m = _Mesh(self.n_vert, _ptr(self.xy), self.n_tri, _ptr(self.tri), self.L,
                        _ptr(self.sigma), _ptr(self.H), _ptr(self.s), _ptr(self.b),
                        _ptr(self.beta), _ptr(self.A_elem),
                        _Params(prm["rho"], prm["g"], prm["rho_w"], prm["glen_n"],
                                prm["eps_reg"], prm["A"], prm["H_min"]),
                        _ptr(self.T_star), float(arr.get("A0", 0.0)), float(arr.get("Q", 0.0)),
                        int(getattr(fp, "elem_type", 0) or 0))
        self._graph = None

    @property
    def mp(self):
        return C.byref(self._m)

    def _check(self, st, what):
        if st != 0:
            raise OracleError(f"{what} failed with status {st}")

    def validate(self) -> int:
        return lib().ora_validate(self.mp)

    def graph(self):
        if self._graph is None:
            row_ptr = np.zeros(self.n_dof + 1, dtype=np.int64)
            nnz = C.c_int64(0)
            self._check(lib().ora_graph(self.mp, _ptr(row_ptr), None, C.byref(nnz)), "graph")
            col = np.zeros(int(nnz.value), dtype=np.int32)
            self._check(lib().ora_graph(self.mp, _ptr(row_ptr), _ptr(col), C.byref(nnz)), "graph")
            self._graph = (row_ptr, col)
        return self._graph

    def residual(self, U, terms=ALL):
        U = np.ascontiguousarray(U, dtype=np.float64)
        R = np.zeros(self.n_dof)
        M = np.zeros(self.n_dof)
        pi = C.c_double(0.0)
        self._check(lib().ora_residual(self.mp, terms, _ptr(U), _ptr(R), _ptr(M), C.byref(pi)),
                    "residual")
        return R, M, pi.value

    def jacobian(self, U, terms=ALL):
        """returns (R, vals) with vals in the CSR order of graph()."""
        row_ptr, col = self.graph()
        U = np.ascontiguousarray(U, dtype=np.float64)
        R = np.zeros(self.n_dof)
        vals = np.zeros(col.size)
        self._check(lib().ora_jacobian(self.mp, terms, _ptr(U), _ptr(row_ptr), _ptr(col),
                                       _ptr(R), _ptr(vals)), "jacobian")
        return R, vals

    def energy(self, U, dof=-1, terms=ALL):
        U = np.ascontiguousarray(U, dtype=np.float64)
        pi = C.c_double(0.0)
        self._check(lib().ora_energy(self.mp, terms, _ptr(U), dof, C.byref(pi)), "energy")
        return pi.value

    def element(self, U, t, k, terms=ALL):
        U = np.ascontiguousarray(U, dtype=np.float64)
        r = np.zeros(12)
        Je = np.zeros(144)
        g = np.zeros(12, dtype=np.int64)
        self._check(lib().ora_element(self.mp, terms, _ptr(U), t, k, _ptr(r), _ptr(Je), _ptr(g)),
                    "element")
        return r, Je.reshape(12, 12), g

    def dense_jacobian(self, U, terms=ALL):
        row_ptr, col = self.graph()
        _, vals = self.jacobian(U, terms)
        J = np.zeros((self.n_dof, self.n_dof))
        rows = np.repeat(np.arange(self.n_dof), np.diff(row_ptr))
        J[rows, col] = vals
        return J
