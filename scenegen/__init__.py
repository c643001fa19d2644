"""Seeded synthetic inputs shared by ``oracle/`` and the product path.

This module is INPUT GENERATION ONLY.  It holds none of the method's
arithmetic: no facet centroids/normals/areas, no view factors, no
visibility, no insolation, no solves.  It produces vertex/face arrays,
sun directions and random right-hand sides with the shapes and value
distributions of the paper's workloads (§7 spherical-cap crater,
P:331-456; §8 rough DEM terrain), using the recipes fixed in
DESIGN.md §"Input recipe" (BASELINE.json configs[0..4]).

Vertex arrays are float64 (nv, 3) in metres (or sphere-radius units);
face arrays are int32 (nf, 3), 0-based.  Height-field meshes are emitted
counter-clockwise in the xy projection; closed bodies are emitted
counter-clockwise seen from outside (outward right-hand-rule normals),
or clockwise when ``inward=True``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "CapGeometry", "cap_geometry", "cfg1_mesh", "cfg2_mesh", "cfg3_mesh",
    "fbm_heightfield", "grid_mesh", "sun_dirs", "random_rhs",
    "flat_plane_mesh", "closed_sphere_mesh", "sphere_exact_facets",
    "facing_plates_mesh", "rough_small_mesh", "blocked_plates_mesh",
    "cap_mesh", "sun_disk_points", "SUN_ANGULAR_RADIUS", "bilobed_body_mesh",
]

SEED_MESH = 1   # mesh jitter seed
SEED_FBM = 2    # fBm phases
SEED_X = 3      # matvec right-hand sides


@dataclass(frozen=True)
class CapGeometry:
    """Spherical-cap crater geometry (Fig. 1 caption).

    R: sphere radius; beta: rim-to-axis angle; rc = R sin(beta): rim radius;
    Hc = R cos(beta): sphere-centre height above the ground plane;
    depth = R - Hc; D = 2 rc: crater diameter.
    """
    R: float
    beta: float
    rc: float
    Hc: float
    depth: float
    D: float


def cap_geometry(R: float = 1.0, d_over_D: float = 0.2) -> CapGeometry:
    # depth/diameter = (1 - cos b) / (2 sin b) = tan(b/2) / 2
    beta = 2.0 * math.atan(2.0 * d_over_D)
    rc = R * math.sin(beta)
    Hc = R * math.cos(beta)
    return CapGeometry(R=R, beta=beta, rc=rc, Hc=Hc, depth=R - Hc, D=2.0 * rc)


def _cap_z(geo: CapGeometry, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Surface height of the cap crater inset in the z=0 plane."""
    r2 = x * x + y * y
    z = np.zeros_like(x)
    inside = r2 < geo.rc * geo.rc
    z[inside] = geo.Hc - np.sqrt(geo.R * geo.R - r2[inside])
    return np.minimum(z, 0.0)


def _delaunay_ccw(xy: np.ndarray) -> np.ndarray:
    from scipy.spatial import Delaunay
    tri = Delaunay(xy).simplices.astype(np.int64)
    a, b, c = xy[tri[:, 0]], xy[tri[:, 1]], xy[tri[:, 2]]
    cross = (b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (b[:, 1] - a[:, 1]) * (c[:, 0] - a[:, 0])
    flip = cross < 0
    tri[flip] = tri[flip][:, [0, 2, 1]]
    cross = np.abs(cross)
    keep = cross > 1e-12 * cross.max()
    return np.ascontiguousarray(tri[keep].astype(np.int32))


def cap_mesh(n_fib: int = 706, n_rim: int = 90, jitter: float = 0.3,
             seed: int = SEED_MESH, R: float = 1.0, d_over_D: float = 0.2):
    """Spherical-cap crater alone (BASELINE configs[0]).

    Jittered Fibonacci points on the cap (cos t_k = 1 - (1 - cos b)(k+1/2)/n,
    phi_k = k pi (3 - sqrt 5)), Gaussian xy jitter of ``jitter`` x spacing,
    plus ``n_rim`` points on the rim circle; Delaunay in xy; z on the sphere.
    """
    geo = cap_geometry(R, d_over_D)
    rng = np.random.default_rng(seed)
    k = np.arange(n_fib, dtype=np.float64)
    cos_t = 1.0 - (1.0 - math.cos(geo.beta)) * (k + 0.5) / n_fib
    sin_t = np.sqrt(np.maximum(0.0, 1.0 - cos_t * cos_t))
    phi = k * math.pi * (3.0 - math.sqrt(5.0))
    x = R * sin_t * np.cos(phi)
    y = R * sin_t * np.sin(phi)
    h = math.sqrt(math.pi * geo.rc ** 2 / n_fib)
    x = x + jitter * h * rng.standard_normal(n_fib)
    y = y + jitter * h * rng.standard_normal(n_fib)
    keep = np.hypot(x, y) < geo.rc - 0.5 * h
    x, y = x[keep], y[keep]
    th = 2.0 * math.pi * np.arange(n_rim) / n_rim
    xr, yr = geo.rc * np.cos(th), geo.rc * np.sin(th)
    xy = np.concatenate([np.stack([x, y], 1), np.stack([xr, yr], 1)])
    tri = _delaunay_ccw(xy)
    z = _cap_z(geo, xy[:, 0], xy[:, 1])
    z[len(x):] = 0.0
    V = np.ascontiguousarray(np.column_stack([xy, z]))
    return V, tri


def cfg1_mesh(seed: int = SEED_MESH):
    """BASELINE configs[0]: cap crater alone, R = 1, d/D = 0.2, ~1,500 facets."""
    return cap_mesh(770, 90, 0.3, seed)


def cfg2_mesh(seed: int = SEED_MESH, n_side: int = 98, jitter: float = 0.3,
              R: float = 1.0, d_over_D: float = 0.2):
    """BASELINE configs[1]: the cap crater inset in a square plain of side 4D.

    Uniform jittered grid of n_side^2 points (minus a 0.5h band around the
    rim and the square boundary), rim points and square-boundary points at
    spacing ~h; Delaunay in xy.  ~20,000 facets, ~1,000 of them in the crater.
    """
    geo = cap_geometry(R, d_over_D)
    L = 4.0 * geo.D
    h = L / n_side
    rng = np.random.default_rng(seed)
    g = (np.arange(n_side) + 0.5) * h - 0.5 * L
    X, Y = np.meshgrid(g, g, indexing="ij")
    x = X.ravel() + jitter * h * rng.standard_normal(X.size)
    y = Y.ravel() + jitter * h * rng.standard_normal(Y.size)
    r = np.hypot(x, y)
    keep = (np.abs(r - geo.rc) > 0.5 * h) & (np.abs(x) < 0.5 * L - 0.5 * h) & (np.abs(y) < 0.5 * L - 0.5 * h)
    x, y = x[keep], y[keep]
    n_rim = int(round(2 * math.pi * geo.rc / h))
    th = 2.0 * math.pi * np.arange(n_rim) / n_rim
    rim = np.stack([geo.rc * np.cos(th), geo.rc * np.sin(th)], 1)
    nb = n_side
    s = np.linspace(-0.5 * L, 0.5 * L, nb + 1)[:-1]
    bnd = np.concatenate([
        np.stack([s, np.full(nb, -0.5 * L)], 1),
        np.stack([np.full(nb, 0.5 * L), s], 1),
        np.stack([-s, np.full(nb, 0.5 * L)], 1),
        np.stack([np.full(nb, -0.5 * L), -s], 1),
    ])
    xy = np.concatenate([np.stack([x, y], 1), rim, bnd])
    tri = _delaunay_ccw(xy)
    z = _cap_z(geo, xy[:, 0], xy[:, 1])
    z[len(x):] = 0.0
    V = np.ascontiguousarray(np.column_stack([xy, z]))
    return V, tri


def fbm_heightfield(n: int, spacing: float, hurst: float = 0.8,
                    rms_slope_deg: float = 15.0, seed: int = SEED_FBM) -> np.ndarray:
    """(n+1) x (n+1) vertex heights: FFT spectral synthesis, amplitude
    |k|^-(H+1), random phases, scaled so sqrt(mean |grad z|^2) (central
    differences over vertices) = tan(rms_slope)."""
    m = n + 1
    rng = np.random.default_rng(seed)
    kx = np.fft.fftfreq(m)[:, None]
    ky = np.fft.rfftfreq(m)[None, :]
    kk = np.sqrt(kx * kx + ky * ky)
    kk[0, 0] = 1.0
    amp = kk ** (-(hurst + 1.0))
    amp[0, 0] = 0.0
    phase = rng.uniform(0.0, 2.0 * math.pi, amp.shape)
    spec = amp * np.exp(1j * phase)
    z = np.fft.irfft2(spec, s=(m, m))
    gx = (z[2:, 1:-1] - z[:-2, 1:-1]) / (2 * spacing)
    gy = (z[1:-1, 2:] - z[1:-1, :-2]) / (2 * spacing)
    rms = math.sqrt(float(np.mean(gx * gx + gy * gy)))
    return z * (math.tan(math.radians(rms_slope_deg)) / rms)


def grid_mesh(z: np.ndarray, spacing: float):
    """Regular grid of (n+1)^2 vertices, two triangles per cell, diagonal
    (i, j) -> (i+1, j+1); centred on the origin."""
    m = z.shape[0]
    n = m - 1
    c = (np.arange(m) - 0.5 * n) * spacing
    X, Y = np.meshgrid(c, c, indexing="ij")
    V = np.ascontiguousarray(np.column_stack([X.ravel(), Y.ravel(), z.ravel()]))
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    v00 = (i * m + j).ravel()
    v10 = ((i + 1) * m + j).ravel()
    v01 = (i * m + j + 1).ravel()
    v11 = ((i + 1) * m + j + 1).ravel()
    t1 = np.stack([v00, v10, v11], 1)
    t2 = np.stack([v00, v11, v01], 1)
    F = np.empty((2 * n * n, 3), dtype=np.int32)
    F[0::2] = t1
    F[1::2] = t2
    return V, F


def cfg3_mesh(n: int = 256, spacing: float = 10.0, crater_D: float = 1000.0,
              d_over_D: float = 0.2, seed: int = SEED_FBM):
    """BASELINE configs[2] (n=256) / configs[3] (n=1024, crater_D=5000):
    fBm (H = 0.8, RMS slope 15 deg) + a spherical-cap crater at the centre."""
    z = fbm_heightfield(n, spacing, 0.8, 15.0, seed)
    V, F = grid_mesh(z, spacing)
    geo = cap_geometry(R=1.0, d_over_D=d_over_D)
    scale = 0.5 * crater_D / geo.rc
    geo = cap_geometry(R=scale, d_over_D=d_over_D)
    V[:, 2] += _cap_z(geo, V[:, 0], V[:, 1])
    return V, F


def sun_dirs(elev_deg: float, n: int, phase0: float = 0.0) -> np.ndarray:
    """n unit sun directions s_j = (cos e cos phi_j, cos e sin phi_j, sin e),
    phi_j = phase0 + 2 pi j / n.  Returns (n, 3) float64."""
    e = math.radians(elev_deg)
    phi = phase0 + 2.0 * math.pi * np.arange(n) / n
    return np.ascontiguousarray(np.stack([math.cos(e) * np.cos(phi),
                                          math.cos(e) * np.sin(phi),
                                          np.full(n, math.sin(e))], 1))


SUN_ANGULAR_RADIUS = math.radians(0.2666)   # solar disk seen from 1 AU (~16 arcmin)


def sun_disk_points(suns, radius: float = SUN_ANGULAR_RADIUS, P: int = 16):
    """Point sources sampling the solar disk around each sun direction
    ("a disk of finite extent ... a sum over point sources"):
    a sunflower pattern in the disk's tangent plane, offset angle
    r_p = radius sqrt((p + 1/2)/P), position angle p * golden angle, equal
    weights 1/P (uniform disk).  Input shaping only: returns (k*P, 3) unit
    directions (sun c's points at rows c*P .. c*P+P-1) and the (P,) weights."""
    suns = np.atleast_2d(np.asarray(suns, dtype=np.float64))
    ga = math.pi * (3.0 - math.sqrt(5.0))
    p = np.arange(P, dtype=np.float64)
    rp = radius * np.sqrt((p + 0.5) / P)
    th = p * ga
    out = np.empty((suns.shape[0] * P, 3))
    for c, s in enumerate(suns):
        s = s / np.linalg.norm(s)
        a = np.array([0.0, 0.0, 1.0]) if abs(s[2]) < 0.9 else np.array([1.0, 0.0, 0.0])
        u = np.cross(s, a); u /= np.linalg.norm(u)
        v = np.cross(s, u)
        d = (np.cos(rp)[:, None] * s[None, :] + np.sin(rp)[:, None] *
             (np.cos(th)[:, None] * u[None, :] + np.sin(th)[:, None] * v[None, :]))
        out[c * P:(c + 1) * P] = d / np.linalg.norm(d, axis=1)[:, None]
    return np.ascontiguousarray(out), np.full(P, 1.0 / P)


def random_rhs(N: int, k: int, seed: int = SEED_X) -> np.ndarray:
    """U[0,1) right-hand sides, column-major N x k (Fortran order)."""
    rng = np.random.default_rng(seed)
    return np.asfortranarray(rng.random((N, k)))


# ---------------------------------------------------------------- test scenes

def bilobed_body_mesh(n_pts: int = 800, neck: float = 0.45, elong: float = 1.6, seed: int = SEED_MESH):
    """Closed bilobed body, a synthetic stand-in for the 67P shape model
    (the Rosetta model is not in the container): Fibonacci
    points on the unit sphere (seeded tangential jitter), convex hull
    triangulation (outward, counter-clockwise seen from outside), then the
    radial map p = r(u) (u_x, u_y, elong u_z) with r = 1 - neck exp(-(u_z/0.35)^2):
    a concave neck between two lobes, so facets see each other across it and
    shadow each other (a closed body needs the octree)."""
    from scipy.spatial import ConvexHull
    rng = np.random.default_rng(seed)
    k = np.arange(n_pts) + 0.5
    z = 1.0 - 2.0 * k / n_pts
    phi = k * math.pi * (3.0 - math.sqrt(5.0)) + 0.2 * rng.standard_normal(n_pts) / math.sqrt(n_pts)
    r = np.sqrt(1.0 - z * z)
    U = np.stack([r * np.cos(phi), r * np.sin(phi), z], 1)
    U /= np.linalg.norm(U, axis=1)[:, None]
    hull = ConvexHull(U)
    F = hull.simplices.astype(np.int32).copy()
    a, b, c = U[F[:, 0]], U[F[:, 1]], U[F[:, 2]]
    flip = np.einsum("ij,ij->i", np.cross(b - a, c - a), a + b + c) < 0
    F[flip] = F[flip][:, [0, 2, 1]]
    rad = 1.0 - neck * np.exp(-(U[:, 2] / 0.35) ** 2)
    V = np.stack([rad * U[:, 0], rad * U[:, 1], rad * elong * U[:, 2]], 1)
    return np.ascontiguousarray(V), np.ascontiguousarray(F)


def flat_plane_mesh(n: int = 8, size: float = 1.0):
    return grid_mesh(np.zeros((n + 1, n + 1)), size / n)


def closed_sphere_mesh(n_pts: int = 200, R: float = 1.0, inward: bool = False):
    """Convex hull of Fibonacci sphere points; faces CCW from outside
    (outward normals) or CW (inward normals) when ``inward``."""
    from scipy.spatial import ConvexHull
    k = np.arange(n_pts) + 0.5
    z = 1.0 - 2.0 * k / n_pts
    r = np.sqrt(1.0 - z * z)
    phi = k * math.pi * (3.0 - math.sqrt(5.0))
    P = R * np.stack([r * np.cos(phi), r * np.sin(phi), z], 1)
    hull = ConvexHull(P)
    F = hull.simplices.astype(np.int64)
    a, b, c = P[F[:, 0]], P[F[:, 1]], P[F[:, 2]]
    out = np.einsum("ij,ij->i", np.cross(b - a, c - a), a + b + c) > 0
    F[~out] = F[~out][:, [0, 2, 1]]
    if inward:
        F = F[:, [0, 2, 1]]
    return np.ascontiguousarray(P), np.ascontiguousarray(F.astype(np.int32))


def sphere_exact_facets(n: int = 400, R: float = 1.0, cap_cos: float = -1.0,
                        seed: int = SEED_MESH):
    """Facet data placed exactly on a sphere: centroids x_i (Fibonacci points
    with z/R >= cap_cos), radial INWARD unit normals, positive random areas.
    Returns (x, nrm, A).  These are inputs for the facet-level entry points
    (pins P1/P4), not a triangle mesh."""
    rng = np.random.default_rng(seed)
    k = np.arange(n) + 0.5
    z = 1.0 - (1.0 - cap_cos) * k / n
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    phi = k * math.pi * (3.0 - math.sqrt(5.0))
    u = np.stack([r * np.cos(phi), r * np.sin(phi), z], 1)
    u /= np.linalg.norm(u, axis=1)[:, None]
    x = R * u
    nrm = -u
    A = (4.0 * math.pi * R * R / n) * (0.5 + rng.random(n))
    return np.ascontiguousarray(x), np.ascontiguousarray(nrm), np.ascontiguousarray(A)


def facing_plates_mesh(d: float = 1.0, s: float = 0.01):
    """Two small triangles with centroids on the z axis at z=0 and z=d,
    facing each other (normals +z and -z as wound)."""
    h = s * math.sqrt(3.0) / 2.0
    tri = np.array([[-s / 2, -h / 3, 0.0], [s / 2, -h / 3, 0.0], [0.0, 2 * h / 3, 0.0]])
    top = tri.copy()
    top[:, 2] = d
    V = np.concatenate([tri, top])
    F = np.array([[0, 1, 2], [3, 5, 4]], dtype=np.int32)
    return V, F


def blocked_plates_mesh(d: float = 1.0, s: float = 0.01, blocker: float = 0.2):
    """facing_plates_mesh plus a large horizontal triangle at z = d/2 that
    crosses the segment between the two centroids."""
    V, F = facing_plates_mesh(d, s)
    b = blocker
    wall = np.array([[-b, -b, d / 2], [b, -b, d / 2], [0.0, b, d / 2]])
    V = np.concatenate([V, wall])
    F = np.concatenate([F, np.array([[6, 7, 8]], dtype=np.int32)])
    return V, F


def rough_small_mesh(n: int = 10, seed: int = SEED_MESH, amp: float = 0.35):
    """Small rough height field (2 n^2 facets, 200 at n=10) with occlusion."""
    rng = np.random.default_rng(seed)
    z = amp * rng.standard_normal((n + 1, n + 1))
    return grid_mesh(z, 1.0 / n)
