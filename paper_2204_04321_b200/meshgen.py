"""Seeded synthetic inputs: footprints, fields and velocities.

This module is the ONE piece of code shared by the oracle side (tests, bench's
cpu_baseline) and the CUDA side.  It holds none of the method's arithmetic: it
never extrudes, never evaluates a basis function, strain rate, viscosity or any
residual/Jacobian term.  It only produces arrays:

    xy[n_vert, 2] (m), tri[n_tri, 3] (int32, CCW), sigma[L+1],
    thickness H, surface s, bed b, beta (per vertex), A (scalar),
    U[2 * n_vert * (L+1)] with DOF = 2*(c*(L+1)+k) + a  (a = 0: u, 1: v).

The velocity U is an analytic shallow-ice-like guess evaluated in sigma
coordinates (u(sigma) = u_b + u_d (1 - (1-sigma)^(n+1))), so it needs no node
heights.  Workload recipes (configs of BASELINE.json):

    C1  ismip_hom_a()        ISMIP-HOM A slab, 80 km, 20x20 quads -> 800 tri, L=5
    C2  greenland_like(16)   450x1200 km star-shaped ellipse, uniform 16 km, L=10
    C3  greenland_like_1_10  graded 1-10 km, N_t tuned to 479,930 +- 2%
    C4  greenland_like_1_10(scale=n)  N_t ~ n * 479,930 (weak scaling)
    C5  antarctica_like()    2100 km disc, 4-20 km, two floating embayments

Random numbers: splitmix64 -> 53-bit uniform -> Box-Muller (the SPEC.md S:429,
S:442 pipeline), so every array is bit-reproducible from its seed.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

DEFAULT_PARAMS = dict(rho=910.0, g=9.81, rho_w=1028.0, glen_n=3.0, eps_reg=1e-10,
                      A=1e-16, H_min=1.0)

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


class SplitMix64:
    """splitmix64 stream (Steele et al.); uniform() uses the top 53 bits."""

    def __init__(self, seed: int):
        self.state = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)

    def next_u64(self, n: int) -> np.ndarray:
        with np.errstate(over="ignore"):
            inc = np.uint64(0x9E3779B97F4A7C15)
            steps = (np.arange(1, n + 1, dtype=np.uint64) * inc) + self.state
            self.state = steps[-1] if n > 0 else self.state
            z = steps.copy()
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
        return z

    def uniform(self, n: int) -> np.ndarray:
        """n uniforms in (0, 1): (top 53 bits + 0.5) * 2^-53."""
        z = self.next_u64(n) >> np.uint64(11)
        return (z.astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)

    def normal(self, n: int) -> np.ndarray:
        """n standard normals, Box-Muller on consecutive uniform pairs."""
        m = (n + 1) // 2
        u = self.uniform(2 * m)
        u1, u2 = u[0::2], u[1::2]
        r = np.sqrt(-2.0 * np.log(u1))
        z = np.empty(2 * m)
        z[0::2] = r * np.cos(2.0 * math.pi * u2)
        z[1::2] = r * np.sin(2.0 * math.pi * u2)
        return z[:n]


@dataclasses.dataclass
class Footprint:
    """One extruded-mesh workload: footprint + fields + a velocity state."""
    name: str
    xy: np.ndarray          # float64 [n_vert, 2]
    tri: np.ndarray         # int32 [n_tri, 3], CCW
    sigma: np.ndarray       # float64 [L+1]
    thickness: np.ndarray   # float64 [n_vert]
    surface: np.ndarray
    bed: np.ndarray | None
    beta: np.ndarray
    U: np.ndarray           # float64 [2*n_vert*(L+1)]
    params: dict
    A_elem: np.ndarray | None = None
    T_star: np.ndarray | None = None    # NEXT-f3: per-wedge temperature (K)
    arrhenius: dict | None = None       # {"A0": Pa^-n a^-1, "Q": J/mol}
    elem_type: int = 0                  # NEXT-f4: 0 wedge, 1 three P1 tetrahedra per prism,
                                        # 2 quadrilateral footprint (tri = [n, 4]) and hexahedra

    @property
    def n_vert(self) -> int:
        return int(self.xy.shape[0])

    @property
    def n_tri(self) -> int:
        return int(self.tri.shape[0])

    @property
    def n_layers(self) -> int:
        return int(self.sigma.shape[0] - 1)

    @property
    def n_elem(self) -> int:
        return self.n_tri * self.n_layers

    @property
    def n_dof(self) -> int:
        return 2 * self.n_vert * (self.n_layers + 1)


# --------------------------------------------------------------------------
# velocity guess (analytic, sigma coordinates)
# --------------------------------------------------------------------------

def _sia_velocity(H, grad_s, beta, sigma, params, rng, rel_noise, abs_noise,
                  slide_cap=5000.0):
    """u(sigma) = u_b + u_d (1 - (1-sigma)^(n+1)) at every (column, level).

    u_d = -(2 A (rho g)^n / (n+1)) |grad s|^(n-1) grad s H^(n+1)  (SIA),
    u_b = -rho g H grad s / beta (beta = 0 -> cap); |u_d| and |u_b| are each
    capped at slide_cap m/a.
    """
    n = params["glen_n"]
    rg = params["rho"] * params["g"]
    gs = np.hypot(grad_s[:, 0], grad_s[:, 1])
    coef = -(2.0 * params["A"] * rg ** n / (n + 1.0)) * gs ** (n - 1.0) * H ** (n + 1.0)
    ud = coef[:, None] * grad_s
    mag_d = np.hypot(ud[:, 0], ud[:, 1])
    ud = ud * np.where(mag_d > slide_cap, slide_cap / np.maximum(mag_d, 1e-300), 1.0)[:, None]
    with np.errstate(divide="ignore", invalid="ignore"):
        ub = -(rg * H / np.where(beta > 0, beta, np.inf))[:, None] * grad_s
    ub = np.where((beta > 0)[:, None], ub, -np.sign(grad_s) * slide_cap)
    mag = np.hypot(ub[:, 0], ub[:, 1])
    scale = np.where(mag > slide_cap, slide_cap / np.maximum(mag, 1e-300), 1.0)
    ub = ub * scale[:, None]
    L = sigma.shape[0] - 1
    prof = 1.0 - (1.0 - sigma) ** (n + 1.0)                  # [L+1]
    U = ub[:, None, :] + ud[:, None, :] * prof[None, :, None]  # [nv, L+1, 2]
    noise = rng.normal(U.size).reshape(U.shape)
    U = U + noise * (rel_noise * np.abs(U) + abs_noise)
    return np.ascontiguousarray(U.reshape(-1))


def _fd_grad(fun, xy, h=1.0):
    """central-difference gradient of an analytic scalar field fun(x, y)."""
    x, y = xy[:, 0], xy[:, 1]
    gx = (fun(x + h, y) - fun(x - h, y)) / (2 * h)
    gy = (fun(x, y + h) - fun(x, y - h)) / (2 * h)
    return np.stack([gx, gy], axis=1)


# --------------------------------------------------------------------------
# C1: ISMIP-HOM experiment A geometry
# --------------------------------------------------------------------------

def ismip_hom_a(nx: int = 20, n_layers: int = 5, length: float = 80e3, seed: int = 42,
                params: dict | None = None) -> Footprint:
    """[0, length]^2, nx x nx quads split along (i,j)->(i+1,j+1), vertex id
    i*(nx+1)+j at (x, y) = (i, j) * length/nx.  s = -x tan(0.5 deg),
    b = s - 1000 + 500 sin(wx) sin(wy), w = 2 pi / length; beta = 1000 + 1000
    sin(wx) sin(wy) (ISMIP-HOM C's field); uniform sigma."""
    params = dict(DEFAULT_PARAMS, **(params or {}))
    rng = SplitMix64(seed)
    h = length / nx
    ii, jj = np.meshgrid(np.arange(nx + 1), np.arange(nx + 1), indexing="ij")
    xy = np.stack([ii.reshape(-1) * h, jj.reshape(-1) * h], axis=1).astype(np.float64)
    tris = []
    for i in range(nx):
        for j in range(nx):
            v00, v10 = i * (nx + 1) + j, (i + 1) * (nx + 1) + j
            v11, v01 = (i + 1) * (nx + 1) + j + 1, i * (nx + 1) + j + 1
            tris.append((v00, v10, v11))
            tris.append((v00, v11, v01))
    tri = np.array(tris, dtype=np.int32)
    w = 2.0 * math.pi / length
    alpha = math.radians(0.5)
    s_fun = lambda x, y: -x * math.tan(alpha)
    b_fun = lambda x, y: s_fun(x, y) - 1000.0 + 500.0 * np.sin(w * x) * np.sin(w * y)
    x, y = xy[:, 0], xy[:, 1]
    s = s_fun(x, y)
    b = b_fun(x, y)
    H = s - b
    beta = 1000.0 + 1000.0 * np.sin(w * x) * np.sin(w * y)
    sigma = np.linspace(0.0, 1.0, n_layers + 1)
    sigma[-1] = 1.0
    grad_s = _fd_grad(lambda X, Y: s_fun(X, Y) + 0.0 * Y, xy)
    U = _sia_velocity(H, grad_s, beta, sigma, params, rng, rel_noise=0.0, abs_noise=1.0)
    return Footprint("C1-ismip-hom-a", xy, tri, sigma, H, s, None, beta, U, params)


def slab(nx: int = 20, n_layers: int = 5, length: float = 80e3, H0: float = 1000.0,
         seed: int = 42, distort: float = 0.0, params: dict | None = None,
         velocity: str = "random") -> Footprint:
    """Flat slab (s = 0, H = H0) on the C1 footprint (C1' variants for the pins).
    distort > 0 moves interior vertices by up to distort*h (seeded) and makes
    the thickness vary, so columns are not right prisms."""
    params = dict(DEFAULT_PARAMS, **(params or {}))
    fp = ismip_hom_a(nx, n_layers, length, seed, params)
    rng = SplitMix64(seed + 1000)
    xy = fp.xy.copy()
    h = length / nx
    if distort > 0:
        interior = (xy[:, 0] > 0) & (xy[:, 0] < length) & (xy[:, 1] > 0) & (xy[:, 1] < length)
        d = (rng.uniform(2 * xy.shape[0]).reshape(-1, 2) - 0.5) * 2.0 * distort * h
        xy[interior] += d[interior]
    nv = xy.shape[0]
    H = np.full(nv, H0)
    if distort > 0:
        H = H0 * (1.0 + 0.3 * (rng.uniform(nv) - 0.5))
    s = np.zeros(nv)
    beta = 500.0 + 1000.0 * rng.uniform(nv)
    sigma = fp.sigma
    if distort > 0:
        sigma = np.linspace(0.0, 1.0, n_layers + 1) ** 1.5
    if velocity == "random":
        U = 10.0 * rng.normal(2 * nv * (n_layers + 1)) + 50.0
    else:
        U = np.zeros(2 * nv * (n_layers + 1))
    return Footprint("slab", xy, fp.tri.copy(), sigma, H, s, None, beta, U, params)


def to_quads(fp: Footprint, nx: int) -> Footprint:
    """NEXT-f4 hexahedral workload: the (nx+1)^2 grid of an ismip_hom_a / slab
    footprint as nx^2 CCW quadrilaterals (v(i,j), v(i+1,j), v(i+1,j+1), v(i,j+1)),
    vertex id i*(nx+1)+j; fields and U unchanged."""
    q = []
    for i in range(nx):
        for j in range(nx):
            q.append((i * (nx + 1) + j, (i + 1) * (nx + 1) + j, (i + 1) * (nx + 1) + j + 1, i * (nx + 1) + j + 1))
    out = Footprint(fp.name + "-quads", fp.xy.copy(), np.array(q, dtype=np.int32), fp.sigma.copy(),
                    fp.thickness.copy(), fp.surface.copy(), None if fp.bed is None else fp.bed.copy(),
                    fp.beta.copy(), fp.U.copy(), dict(fp.params))
    out.elem_type = 2
    return out


# --------------------------------------------------------------------------
# ring / zipper footprints for star-shaped domains
# --------------------------------------------------------------------------

class _Domain:
    """Star-shaped domain x = rho*Rx*m(th) cos th, y = rho*Ry*m(th) sin th,
    m(th) = 1 + 0.05 * sum_{m=2..6} c_m cos(m th + phi_m), c_m in [-1, 1]."""

    def __init__(self, Rx, Ry, rng: SplitMix64):
        u = rng.uniform(10)
        self.Rx, self.Ry = Rx, Ry
        self.c = 2.0 * u[:5] - 1.0
        self.phi = 2.0 * math.pi * u[5:]
        # arc-length table of the boundary curve
        th = np.linspace(0.0, 2.0 * math.pi, 20001)
        p = self.boundary(th)
        seg = np.hypot(np.diff(p[:, 0]), np.diff(p[:, 1]))
        self._th = th
        self._arc = np.concatenate([[0.0], np.cumsum(seg)])
        self.perimeter = float(self._arc[-1])
        self.R_eff = math.sqrt(Rx * Ry)

    def m(self, th):
        th = np.asarray(th, dtype=np.float64)
        out = np.ones_like(th)
        for k in range(5):
            out = out + 0.05 * self.c[k] * np.cos((k + 2) * th + self.phi[k])
        return out

    def boundary(self, th):
        mm = self.m(th)
        return np.stack([self.Rx * mm * np.cos(th), self.Ry * mm * np.sin(th)], axis=1)

    def theta_of_arc(self, t):
        """boundary parameter th for normalised arc length t in [0, 1)."""
        return np.interp(t * self.perimeter, self._arc, self._th)

    def map(self, rho, t):
        th = self.theta_of_arc(t)
        mm = self.m(th)
        return np.stack([rho * self.Rx * mm * np.cos(th), rho * self.Ry * mm * np.sin(th)], axis=1)

    def rho_theta(self, x, y):
        th = np.arctan2(y / self.Ry, x / self.Rx)
        r = np.hypot(x / self.Rx, y / self.Ry) / self.m(th)
        return r, th


def _spacing(d, h_min, h_max, D):
    return h_min + (h_max - h_min) * np.minimum(1.0, d / D)


def _ring_radii(dom: _Domain, h_min, h_max, D):
    """normalised ring radii from the margin (rho = 1) inwards, and the
    physical spacing on each ring."""
    rhos, hs = [1.0], [_spacing(0.0, h_min, h_max, D)]
    while True:
        d = (1.0 - rhos[-1]) * dom.R_eff
        h = float(_spacing(d, h_min, h_max, D))
        nxt = rhos[-1] - h / dom.R_eff
        if nxt * dom.perimeter / h < 6.0 or nxt <= 0.0:
            break
        d2 = (1.0 - nxt) * dom.R_eff
        rhos.append(nxt)
        hs.append(float(_spacing(d2, h_min, h_max, D)))
    return np.array(rhos), np.array(hs)


def _ring_counts(dom, h_min, h_max, D):
    rhos, hs = _ring_radii(dom, h_min, h_max, D)
    n = np.maximum(6, np.round(rhos * dom.perimeter / hs)).astype(np.int64)
    return rhos, n


def _predicted_ntri(dom, h_min, h_max, D):
    _, n = _ring_counts(dom, h_min, h_max, D)
    return int(np.sum(n[:-1] + n[1:]) + n[-1])


def _zipper(inner_ids, t_in, outer_ids, t_out):
    """triangulate the annulus between two rings (params t in [0,1), ascending).
    Emits (inner_p, outer_q, inner_p+1) or (inner_p, outer_q, outer_q+1), CCW."""
    ni, no = len(t_in), len(t_out)
    # outer start: last outer point with t <= t_in[0] (cyclically)
    q0 = int(np.searchsorted(t_out, t_in[0], side="right")) - 1
    A_in = lambda p: t_in[p % ni] + (p // ni)
    A_out = lambda q: t_out[q % no] + (q // no) if q >= 0 else t_out[q % no] - 1.0
    tris = np.empty((ni + no, 3), dtype=np.int64)
    p, q, e = 0, q0, 0
    while p < ni or q < q0 + no:
        adv_inner = (q >= q0 + no) or (p < ni and A_in(p + 1) <= A_out(q + 1))
        if adv_inner:
            tris[e] = (inner_ids[p % ni], outer_ids[q % no], inner_ids[(p + 1) % ni])
            p += 1
        else:
            tris[e] = (inner_ids[p % ni], outer_ids[q % no], outer_ids[(q + 1) % no])
            q += 1
        e += 1
    return tris[:e]


def _ring_mesh(dom: _Domain, h_min, h_max, D, rng: SplitMix64):
    rhos, n = _ring_counts(dom, h_min, h_max, D)
    pts, params_t, ids = [], [], []
    base = 0
    for j, (rho, nj) in enumerate(zip(rhos, n)):
        off = rng.uniform(1)[0] / nj              # seeded per-ring phase
        t = (np.arange(nj) / nj + off) % 1.0
        t.sort()
        pts.append(dom.map(rho, t))
        params_t.append(t)
        ids.append(np.arange(base, base + nj))
        base += nj
    centre = base
    xy = np.concatenate(pts + [np.zeros((1, 2))], axis=0)
    tris = []
    for j in range(len(rhos) - 1):     # ring j is outer, ring j+1 is inner
        tris.append(_zipper(ids[j + 1], params_t[j + 1], ids[j], params_t[j]))
    last = ids[-1]
    fan = np.stack([np.full(len(last), centre), last, np.roll(last, -1)], axis=1)
    tris.append(fan)
    tri = np.concatenate(tris, axis=0)
    return xy, tri


# --------------------------------------------------------------------------
# canonicalisation: Hilbert order of vertices and triangles
# --------------------------------------------------------------------------

def _hilbert_key(xy, order=20):
    lo = xy.min(axis=0)
    span = max(float((xy.max(axis=0) - lo).max()), 1e-300)
    n = 1 << order
    X = np.minimum(((xy[:, 0] - lo[0]) / span * (n - 1)).astype(np.int64), n - 1)
    Y = np.minimum(((xy[:, 1] - lo[1]) / span * (n - 1)).astype(np.int64), n - 1)
    d = np.zeros(xy.shape[0], dtype=np.int64)
    s = n >> 1
    while s > 0:
        rx = ((X & s) > 0).astype(np.int64)
        ry = ((Y & s) > 0).astype(np.int64)
        d += s * s * ((3 * rx) ^ ry)
        # rotate
        flip = ry == 0
        swap_and_flip = flip & (rx == 1)
        X = np.where(swap_and_flip, s - 1 - X, X)
        Y = np.where(swap_and_flip, s - 1 - Y, Y)
        Xn = np.where(flip, Y, X)
        Yn = np.where(flip, X, Y)
        X, Y = Xn, Yn
        s >>= 1
    return d


def canonicalise(xy, tri):
    """Hilbert-sort vertices (ties: old id) and triangles (ties: sorted ids),
    rotate each triangle so its smallest vertex id comes first (keeps CCW)."""
    tri = np.asarray(tri, dtype=np.int64)
    # orient CCW
    p0, p1, p2 = xy[tri[:, 0]], xy[tri[:, 1]], xy[tri[:, 2]]
    cross = (p1[:, 0] - p0[:, 0]) * (p2[:, 1] - p0[:, 1]) - (p2[:, 0] - p0[:, 0]) * (p1[:, 1] - p0[:, 1])
    cw = cross < 0
    tri[cw] = tri[cw][:, [0, 2, 1]]
    kv = _hilbert_key(xy)
    vperm = np.lexsort((np.arange(xy.shape[0]), kv))
    inv = np.empty_like(vperm)
    inv[vperm] = np.arange(vperm.size)
    xy2 = xy[vperm]
    t2 = inv[tri]
    # rotate so the smallest id is first
    r = np.argmin(t2, axis=1)
    idx = (np.arange(3)[None, :] + r[:, None]) % 3
    t2 = np.take_along_axis(t2, idx, axis=1)
    cen = xy2[t2].mean(axis=1)
    kt = _hilbert_key(cen)
    st = np.sort(t2, axis=1)
    tperm = np.lexsort((st[:, 2], st[:, 1], st[:, 0], kt))
    return xy2, t2[tperm].astype(np.int32), vperm


def _smooth_field(rng: SplitMix64, xy, n_modes=32, lam_min=50e3, lam_max=500e3):
    """zero-mean, unit-variance sum of n_modes random plane waves."""
    u = rng.uniform(3 * n_modes).reshape(n_modes, 3)
    lam = lam_min * (lam_max / lam_min) ** u[:, 0]
    ang = 2.0 * math.pi * u[:, 1]
    ph = 2.0 * math.pi * u[:, 2]
    k = (2.0 * math.pi / lam)[:, None] * np.stack([np.cos(ang), np.sin(ang)], axis=1)

    def f(x, y):
        arg = np.outer(x, k[:, 0]) + np.outer(y, k[:, 1]) + ph[None, :]
        return math.sqrt(2.0 / n_modes) * np.cos(arg).sum(axis=1)
    return f


def _ice_sheet(name, dom, h_min, h_max, D, n_layers, seed, H0, b0, b1, params,
               embayments=0):
    params = dict(DEFAULT_PARAMS, **(params or {}))
    rng = SplitMix64(seed * 7919 + 17)
    xy, tri = _ring_mesh(dom, h_min, h_max, D, rng)
    xy, tri, _ = canonicalise(xy, tri)
    xi_b = _smooth_field(rng, xy)
    xi_beta = _smooth_field(rng, xy)
    emb = rng.uniform(2) * 2.0 * math.pi
    rho, rho_w = params["rho"], params["rho_w"]

    def emb_weight(th):
        w = np.zeros_like(th)
        for c in emb[:embayments]:
            dth = np.angle(np.exp(1j * (th - c)))
            w = np.maximum(w, np.clip(1.0 - np.abs(dth) / math.radians(15.0), 0.0, 1.0))
        return w

    def fields(x, y):
        r, th = dom.rho_theta(x, y)
        r = np.clip(r, 0.0, 1.0)
        H = H0 * np.clip(1.0 - r ** (4.0 / 3.0), 0.0, 1.0) ** (3.0 / 8.0)
        b = b0 - b1 * r ** 2 + 150.0 * xi_b(x, y)
        if embayments:
            w = emb_weight(th) * np.clip((r - 0.6) / 0.4, 0.0, 1.0)
            H_shelf = 300.0 + (H0 * 0.3 - 300.0) * np.clip((1.0 - r) / 0.4, 0.0, 1.0)
            H = (1.0 - w) * H + w * H_shelf
            b = (1.0 - w) * b + w * (-800.0)
        H = np.maximum(H, 10.0)
        grounded = rho * H >= -rho_w * b
        s = np.where(grounded, b + H, H * (1.0 - rho / rho_w))
        beta = 10.0 ** (1.0 + 3.0 * (1.0 - r) + 0.5 * xi_beta(x, y))
        return H, s, b, beta

    H, s, b, beta = fields(xy[:, 0], xy[:, 1])
    sigma = np.linspace(0.0, 1.0, n_layers + 1) ** 1.5
    sigma[0], sigma[-1] = 0.0, 1.0
    grad_s = _fd_grad(lambda X, Y: fields(X, Y)[1], xy, h=1.0)
    beta_eff = np.where(rho * H < -rho_w * b, 0.0, beta)
    U = _sia_velocity(H, grad_s, beta_eff, sigma, params, rng, rel_noise=0.01, abs_noise=0.1)
    return Footprint(name, xy, tri, sigma, H, s, b, beta, U, params)


def greenland_like(h_km: float = 16.0, n_layers: int = 10, seed: int = 1,
                   params: dict | None = None) -> Footprint:
    """C2: 450 x 1200 km star-shaped ellipse, uniform spacing h_km."""
    dom = _Domain(450e3, 1200e3, SplitMix64(seed))
    return _ice_sheet(f"C2-greenland-like-{h_km:g}km", dom, h_km * 1e3, h_km * 1e3, 1.0,
                      n_layers, seed, 3000.0, 300.0, 600.0, params)


C3_TARGET_NTRI = 479_930          # P:596 (Greenland 1-7 km mesh triangle count)


def tune_grading(dom, h_min, h_max, target, tol=0.02):
    """bisection on D so that the predicted triangle count hits target."""
    lo, hi = 1e3, 5e6
    for _ in range(80):
        mid = math.sqrt(lo * hi)
        nt = _predicted_ntri(dom, h_min, h_max, mid)
        if abs(nt - target) <= tol * 0.25 * target:
            return mid
        if nt > target:      # larger D -> finer mesh -> more triangles
            hi = mid
        else:
            lo = mid
    return math.sqrt(lo * hi)


def greenland_like_1_10(scale: float = 1.0, n_layers: int = 10, seed: int = 1,
                        params: dict | None = None, target: int | None = None) -> Footprint:
    """C3 (scale=1) / C4 (scale=n): graded 1-10 km ring mesh, spacing scaled by
    1/sqrt(scale), D tuned so N_t = scale * 479,930 +- 2%."""
    dom = _Domain(450e3, 1200e3, SplitMix64(seed))
    f = 1.0 / math.sqrt(scale)
    h_min, h_max = 1e3 * f, 10e3 * f
    tgt = target if target is not None else int(round(scale * C3_TARGET_NTRI))
    D = tune_grading(dom, h_min, h_max, tgt)
    return _ice_sheet(f"C3-greenland-like-1-10km-x{scale:g}", dom, h_min, h_max, D,
                      n_layers, seed, 3000.0, 300.0, 600.0, params)


def antarctica_like(n_layers: int = 10, seed: int = 2, D_km: float = 600.0,
                    params: dict | None = None) -> Footprint:
    """C5: 2100 km disc with margin modes, 4-20 km, two floating embayments."""
    dom = _Domain(2100e3, 2100e3, SplitMix64(seed))
    return _ice_sheet("C5-antarctica-like-4-20km", dom, 4e3, 20e3, D_km * 1e3, n_layers,
                      seed, 4000.0, 200.0, 700.0, params, embayments=2)


def sub_footprint(fp: Footprint, t0: int, t1: int) -> Footprint:
    """Triangles [t0, t1) with their vertices (ascending old id) and the
    matching slices of every field and of U.  Pure data slicing."""
    tri = fp.tri[t0:t1]
    verts = np.unique(tri.reshape(-1))
    remap = -np.ones(fp.n_vert, dtype=np.int64)
    remap[verts] = np.arange(verts.size)
    L1 = fp.n_layers + 1
    Uv = fp.U.reshape(fp.n_vert, L1, 2)[verts].reshape(-1).copy()
    return Footprint(fp.name + f"[{t0}:{t1}]", fp.xy[verts].copy(),
                     remap[tri].astype(np.int32), fp.sigma.copy(), fp.thickness[verts].copy(),
                     fp.surface[verts].copy(), None if fp.bed is None else fp.bed[verts].copy(),
                     fp.beta[verts].copy(), Uv, dict(fp.params),
                     None if fp.A_elem is None else fp.A_elem.reshape(fp.n_tri, -1)[t0:t1].reshape(-1).copy(),
                     None if fp.T_star is None else fp.T_star.reshape(fp.n_tri, -1)[t0:t1].reshape(-1).copy(),
                     None if fp.arrhenius is None else dict(fp.arrhenius), fp.elem_type)


def sub_footprint_tris(fp: Footprint, tri_ids) -> Footprint:
    """The triangles tri_ids (kept in ascending order) with their vertices
    (ascending old id, so sorted neighbour lists keep their order).  Pure slicing."""
    tri_ids = np.unique(np.asarray(tri_ids, dtype=np.int64))
    tri = fp.tri[tri_ids]
    verts = np.unique(tri.reshape(-1))
    remap = -np.ones(fp.n_vert, dtype=np.int64)
    remap[verts] = np.arange(verts.size)
    L1 = fp.n_layers + 1
    Uv = fp.U.reshape(fp.n_vert, L1, 2)[verts].reshape(-1).copy()
    A = None if fp.A_elem is None else fp.A_elem.reshape(fp.n_tri, -1)[tri_ids].reshape(-1).copy()
    sub = Footprint(fp.name + "[subset]", fp.xy[verts].copy(), remap[tri].astype(np.int32),
                    fp.sigma.copy(), fp.thickness[verts].copy(), fp.surface[verts].copy(),
                    None if fp.bed is None else fp.bed[verts].copy(), fp.beta[verts].copy(), Uv,
                    dict(fp.params), A,
                    None if fp.T_star is None else fp.T_star.reshape(fp.n_tri, -1)[tri_ids].reshape(-1).copy(),
                    None if fp.arrhenius is None else dict(fp.arrhenius), fp.elem_type)
    sub.vertex_ids = verts
    return sub


# Arrhenius constants of the synthetic temperature recipe (cold-ice branch of
# the Paterson-Budd fit, converted to years): A0 = 3.61e-13 Pa^-3 s^-1, Q = 60 kJ/mol
ARRHENIUS_COLD = dict(A0=3.61e-13 * 31556926.0, Q=6.0e4)


def with_temperature(fp: Footprint, seed: int = 7, T_surf: float = 243.0,
                     T_bed: float = 268.0, noise: float = 2.0) -> Footprint:
    """NEXT-f3 input recipe: per-wedge T* linear in the mid-layer sigma,
    T_surf at the surface to T_bed at the bed, plus seeded noise (+-noise K);
    sets fp.T_star and fp.arrhenius in place and returns fp."""
    rng = SplitMix64(seed)
    sm = 0.5 * (fp.sigma[:-1] + fp.sigma[1:])
    T = (T_bed + (T_surf - T_bed) * sm)[None, :] + noise * (2.0 * rng.uniform(fp.n_elem).reshape(fp.n_tri, -1) - 1.0)
    fp.T_star = T.reshape(-1)
    fp.arrhenius = dict(ARRHENIUS_COLD)
    return fp


def by_name(name: str) -> Footprint:
    """workload by config id: C1, C2, C3, C4x<n>, C5."""
    if name == "C1":
        return ismip_hom_a()
    if name == "C2":
        return greenland_like(16.0)
    if name == "C3":
        return greenland_like_1_10(1.0)
    if name.startswith("C4x"):
        return greenland_like_1_10(float(name[3:]))
    if name == "C5":
        return antarctica_like()
    raise ValueError(name)
