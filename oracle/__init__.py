"""FP64 CPU oracle for the compressed view-factor hot path (PAPER.md = P:<line>).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_2209_07632_b200`` (the product):
neither imports the other; both take their inputs from ``scenegen``.

Contents
  * vf_oracle.c (ctypes): facet data, visibility V_ij,
    F_ij (P:134-136 eq. FF-def), insolation, dense/CSR apply.
  * this module: the Jacobi radiosity solve (P:40-43 eq. radiosity-system,
    P:143), the thermal equilibrium chain (P:62-74, P:110-115,
    P:282-290), a dense LU reference solve, the analytic cap-crater
    equilibrium.
  * ``oracle.hmatrix``: the paper's Alg. 2-5 written out step by
    step with numpy's SVD as the truncated-SVD primitive; it writes its
    compressed matrix in the HVFM container (include/vf.h) so the GPU path
    can apply exactly the same blocks.

Every function is pinned in tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "vf_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

SIGMA_SB = 5.670374419e-8  # Stefan-Boltzmann, W m^-2 K^-4 (CODATA 2018)


def build(force: bool = False) -> str:
    """Compile vf_oracle.c -> liboracle.so (gcc, -O2, OpenMP, no FP contraction)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
                               "-std=c11", "-D_GNU_SOURCE", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        i = ctypes.c_int
        d = ctypes.c_double
        L.or_facet_data.argtypes = [I, P, P, i, P, P, P]
        L.or_facet_data.restype = i
        L.or_visibility_rows.argtypes = [I, P, P, I, P, I, P, P, i, i, I, P, P]
        L.or_viewfactor_dense.argtypes = [I, P, P, P, I, P, I, P, P, i, i, P]
        L.or_viewfactor_csr_rows.argtypes = [I, P, P, P, I, P, I, P, P, i, i, I, P]
        L.or_viewfactor_csr_rows.restype = P
        L.or_csr_nnz.argtypes = [P]
        L.or_csr_nnz.restype = I
        L.or_csr_fetch.argtypes = [P, P, P, P]
        L.or_csr_free.argtypes = [P]
        L.or_insolation.argtypes = [I, P, P, I, P, I, P, P, i, I, P, d, P]
        L.or_apply_dense.argtypes = [I, P, I, P, P]
        L.or_apply_csr.argtypes = [I, P, P, P, I, I, P, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ------------------------------------------------------------------ geometry

def facet_data(V, F, orient_up: bool = True):
    """centroid x_i, unit normal n_i (n_z > 0 if orient_up), area A_i."""
    V = _f64(V)
    F = np.ascontiguousarray(F, dtype=np.int32)
    nf = F.shape[0]
    x = np.empty((nf, 3)); n = np.empty((nf, 3)); A = np.empty(nf)
    bad = lib().or_facet_data(nf, _p(V), _p(F), int(orient_up), _p(x), _p(n), _p(A))
    if bad:
        raise ValueError(f"{bad} degenerate (zero-area) faces")
    return x, n, A


def default_grid(nt: int) -> int:
    """Grid resolution for the xy accelerator (0 = brute force)."""
    return 0 if nt <= 800 else max(1, int(math.sqrt(nt / 2.0)))


class Scene:
    """A triangle mesh with its oracle facet data.  Occluders are the mesh
    triangles themselves (facet f <-> triangle f)."""

    def __init__(self, V, F, orient_up: bool = True, grid: int | None = None):
        self.V = _f64(V)
        self.T = np.ascontiguousarray(F, dtype=np.int32)
        self.x, self.n, self.A = facet_data(self.V, self.T, orient_up)
        self.N = self.T.shape[0]
        self.grid = default_grid(self.N) if grid is None else grid
        self.tri_of = np.arange(self.N, dtype=np.int64)

    def _occ(self):
        return (self.V.shape[0], _p(self.V), self.T.shape[0], _p(self.T), _p(self.tri_of))

    def visibility_rows(self, rows, cull_only=False, grid=None):
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        out = np.zeros((rows.size, self.N), dtype=np.uint8)
        nv, pV, nt, pT, pto = self._occ()
        lib().or_visibility_rows(self.N, _p(self.x), _p(self.n), nv, pV, nt, pT, pto, int(cull_only),
                                 self.grid if grid is None else grid, rows.size, _p(rows), _p(out))
        return out

    def F_dense(self, cull_only=False, grid=None):
        """Dense F (eq. FF-def), row-major N x N."""
        out = np.empty((self.N, self.N))
        nv, pV, nt, pT, pto = self._occ()
        lib().or_viewfactor_dense(self.N, _p(self.x), _p(self.n), _p(self.A), nv, pV, nt, pT, pto,
                                  int(cull_only), self.grid if grid is None else grid, _p(out))
        return out

    def F_csr_rows(self, rows=None, cull_only=False, grid=None):
        """Exact CSR rows of F (Alg. 1): (rowptr, cols, vals)."""
        rows = np.arange(self.N, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
        nv, pV, nt, pT, pto = self._occ()
        L = lib()
        h = L.or_viewfactor_csr_rows(self.N, _p(self.x), _p(self.n), _p(self.A), nv, pV, nt, pT, pto,
                                     int(cull_only), self.grid if grid is None else grid, rows.size, _p(rows))
        nnz = L.or_csr_nnz(h)
        rowptr = np.empty(rows.size + 1, dtype=np.int64)
        cols = np.empty(max(nnz, 1), dtype=np.int64)
        vals = np.empty(max(nnz, 1))
        L.or_csr_fetch(h, _p(rowptr), _p(cols), _p(vals))
        L.or_csr_free(h)
        return rowptr, cols[:nnz], vals[:nnz]

    def insolation(self, suns, S: float = 1365.0, grid=None):
        """Q_dir column-major N x k for unit sun dirs (k, 3)."""
        suns = _f64(np.atleast_2d(suns))
        k = suns.shape[0]
        Q = np.empty((self.N, k), order="F")
        nv, pV, nt, pT, pto = self._occ()
        lib().or_insolation(self.N, _p(self.x), _p(self.n), nv, pV, nt, pT, pto,
                            self.grid if grid is None else grid, k, _p(suns), float(S), _p(Q))
        return Q


def insolation_disk(scene, dirs, w, S: float = 1365.0):
    """Finite solar disk as a sum over point sources: each source
    contributes eq. insolation-for-point-sun with weight w_p;
    Q[:, c] = sum_p w_p Q_point(dirs[c P + p]) summed in p order."""
    w = np.asarray(w, dtype=np.float64).reshape(-1)
    P = w.size
    Qp = scene.insolation(dirs, S)                 # N x (k P)
    k = Qp.shape[1] // P
    Q = np.zeros((scene.N, k), order="F")
    for c in range(k):
        for p in range(P):
            Q[:, c] += w[p] * Qp[:, c * P + p]
    return Q


def F_dense_facets(x, n, A, cull_only=True):
    """Dense F from facet data alone (no occluding mesh): used with
    sphere-exact facet data (pin P1/P4) where V_ij is the culling test."""
    x = _f64(x); n = _f64(n); A = _f64(A)
    N = x.shape[0]
    out = np.empty((N, N))
    lib().or_viewfactor_dense(N, _p(x), _p(n), _p(A), 0, None, 0, None, None, int(cull_only), 0, _p(out))
    return out


# ------------------------------------------------------------------ applies

def apply_dense(F, X):
    """Y = F X (row by row, P:134 operator).  X column-major N x k."""
    F = _f64(F)
    X = np.asfortranarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X[:, None]
    N, k = X.shape
    Y = np.empty((F.shape[0], k), order="F")
    lib().or_apply_dense(N, _p(F), k, _p(X), _p(Y))
    return Y


def apply_csr(csr, X):
    rowptr, cols, vals = csr
    X = np.asfortranarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X[:, None]
    N, k = X.shape
    nr = rowptr.size - 1
    Y = np.empty((nr, k), order="F")
    lib().or_apply_csr(nr, _p(np.ascontiguousarray(rowptr)), _p(np.ascontiguousarray(cols)),
                       _p(np.ascontiguousarray(vals)), N, k, _p(X), _p(Y))
    return Y


# ------------------------------------------------------------------- solves

def jacobi(apply, E, rho, tol: float, iters: int, clamp: bool = True):
    """Jacobi / Neumann iteration for B = E + diag(rho) F B.

    Readings (DESIGN.md R-JAC, R-CLAMP): B_0 = E; each iteration is one
    F-apply: Q_k = F B_k, Q_k <- max(Q_k, 0) if clamp,
    B_{k+1} = E + rho * Q_k; r_k = ||B_{k+1} - B_k||_2 / ||E||_2 per column
    (||E|| = 0 -> r = 0); stop when every column has r_k <= tol or after
    ``iters`` iterations.  Returns (B_{k+1}, Q_k, iterations, r_k)."""
    E = np.asfortranarray(E, dtype=np.float64)
    if E.ndim == 1:
        E = E[:, None]
    rho = np.asarray(rho, dtype=np.float64).reshape(-1)
    nE = np.sqrt(np.sum(E * E, axis=0))
    B = E.copy(order="F")
    Q = np.zeros_like(B)
    r = np.zeros(E.shape[1])
    it = 0
    for it in range(1, iters + 1):
        Q = apply(B)
        if clamp:
            Q = np.maximum(Q, 0.0)
        Bn = E + rho[:, None] * Q
        dB = np.sqrt(np.sum((Bn - B) ** 2, axis=0))
        r = np.where(nE > 0, dB / np.where(nE > 0, nE, 1.0), 0.0)
        B = np.asfortranarray(Bn)
        if np.all(r <= tol):
            break
    return B, np.asfortranarray(Q), it, r


def thermal(apply, Qdir, albedo, emiss, tol: float, iters: int, clamp: bool = True):
    """Equilibrium temperature (eq. 3d-equilbr).

    Stage 1 (eq. time-indep-system-1 as eq. (1) with rho = alpha, reading
    R-A14): B = alpha Q_dir + alpha F B; Q_refl = F B_k (the last apply);
    Q_vis = Q_dir + Q_refl.
    Stage 2 (eq. time-indep-system-2 / eq. QIR with H = 0): W = (1-alpha)
    Q_vis + F W; Q_IR = F W_k (the last apply).
    T = (((1-alpha) Q_vis + eps Q_IR) / (eps sigma))^(1/4).
    Returns dict(T, Qvis, Qir, Qrefl, it1, it2, r1, r2)."""
    Qdir = np.asfortranarray(Qdir, dtype=np.float64)
    if Qdir.ndim == 1:
        Qdir = Qdir[:, None]
    a = np.asarray(albedo, dtype=np.float64).reshape(-1)[:, None]
    e = np.asarray(emiss, dtype=np.float64).reshape(-1)[:, None]
    B, Qrefl, it1, r1 = jacobi(apply, a * Qdir, a[:, 0], tol, iters, clamp)
    Qvis = Qdir + Qrefl
    W, Qir, it2, r2 = jacobi(apply, (1.0 - a) * Qvis, np.ones(a.shape[0]), tol, iters, clamp)
    Qabs = (1.0 - a) * Qvis + e * Qir
    T = (Qabs / (e * SIGMA_SB)) ** 0.25
    return dict(T=T, Qvis=Qvis, Qir=Qir, Qrefl=Qrefl, B=B, W=W, it1=it1, it2=it2, r1=r1, r2=r2)


def lu_radiosity(F, E, rho):
    """Direct solve of (I - diag(rho) F) B = E by LU (numpy.linalg.solve)."""
    F = _f64(F)
    rho = np.asarray(rho, dtype=np.float64).reshape(-1)
    M = np.eye(F.shape[0]) - rho[:, None] * F
    return np.linalg.solve(M, np.asarray(E, dtype=np.float64))


# --------------------------------------------------- analytic cap crater (§7)

def cap_f(D_over_d: float) -> float:
    """1/f = 1 + (D/d)^2 / 4."""
    return 1.0 / (1.0 + 0.25 * D_over_d * D_over_d)


def cap_b(f: float, albedo: float, emiss: float) -> float:
    """b = f (eps + alpha (1 - f)) / (1 - alpha f)."""
    return f * (emiss + albedo * (1.0 - f)) / (1.0 - albedo * f)


def cap_shadow_T_p361(S: float, e_sun_deg: float, f: float, albedo: float, emiss: float) -> float:
    """sigma T^4 = S sin(e) f (1-alpha)/(1-alpha f) [1 + alpha (1-f)/eps]."""
    s = S * math.sin(math.radians(e_sun_deg)) * f * (1 - albedo) / (1 - albedo * f) * (1 + albedo * (1 - f) / emiss)
    return (s / SIGMA_SB) ** 0.25


def cap_T_global(S: float, e_sun_deg: float, f: float, albedo: float, emiss: float,
                 region: str, sin_e_local: float = 0.0) -> float:
    """P:370-377 eq. globalsolution: eps sigma T^4 = (1 - alpha) S x
    {sin e_sun (sunlit, outside) | sin e + b sin e_sun (sunlit, in crater) |
     b sin e_sun (shadowed, in crater)}."""
    b = cap_b(f, albedo, emiss)
    se = math.sin(math.radians(e_sun_deg))
    fac = {"outside": se, "lit": sin_e_local + b * se, "shadow": b * se}[region]
    return ((1 - albedo) * S * fac / (emiss * SIGMA_SB)) ** 0.25
