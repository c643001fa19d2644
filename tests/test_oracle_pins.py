"""Pins of the FP64 oracle against things other than itself (closed forms,
invariants, printed worked values, independent brute force).  CPU only.

PAPER.md = P:<line>; pin ids P1..P10 follow SURVEY.md §8(c) / DESIGN.md §Pins.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import oracle.hmatrix as hm
import scenegen as sg

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------- facet data

def test_facet_data_unit_triangles():
    # unit right triangle -> area 1/2, normal +z, centroid (1/3,1/3,0);
    # equilateral of side 2 -> area sqrt(3).
    V = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [2, 0, 1], [1, math.sqrt(3), 1]], float)
    F = np.array([[0, 1, 2], [3, 5, 4]], np.int32)   # second one wound clockwise in xy
    x, n, A = oracle.facet_data(V, F, orient_up=True)
    assert np.allclose(A, [0.5, math.sqrt(3)], rtol=1e-15)
    assert np.allclose(n, [[0, 0, 1], [0, 0, 1]])
    assert np.allclose(x[0], [1 / 3, 1 / 3, 0])
    x2, n2, _ = oracle.facet_data(V, F, orient_up=False)   # right-hand rule kept
    assert np.allclose(n2[1], [0, 0, -1])
    with pytest.raises(ValueError):
        oracle.facet_data(V, np.array([[0, 0, 1]], np.int32))


# ------------------------------------------------------------ P1 sphere-exact

@pytest.mark.parametrize("n", [150, 600])
def test_P1_sphere_exact_F_is_Aj_over_4piR2(n):
    # Two points on a sphere with inward normals: cos(th_i) = cos(th_j) = r/(2R),
    # so F(x,y) = 1/(4 pi R^2) and F_ij = A_j / (4 pi R^2).
    R = 2.5
    x, nrm, A = sg.sphere_exact_facets(n, R)
    F = oracle.F_dense_facets(x, nrm, A, cull_only=True)
    c = 1.0 / (4 * math.pi * R * R)
    expect = c * np.tile(A, (n, 1))
    np.fill_diagonal(expect, 0.0)
    assert np.max(np.abs(F - expect) / expect.max()) < 1e-13
    rs = F.sum(1)
    assert np.allclose(rs, c * (A.sum() - A), rtol=1e-13, atol=0)


def test_P2_closed_planar_sphere_rowsums_tend_to_one():
    # Enclosure: a closed surface sees itself entirely, row sums -> 1 under
    # refinement (midpoint rule, A20).  Convex body: every culled-in pair visible.
    errs = []
    for npts in (200, 800):
        S = oracle.Scene(*sg.closed_sphere_mesh(npts, 1.0, inward=True), orient_up=False, grid=0)
        F = S.F_dense()
        off = ~np.eye(S.N, dtype=bool)
        assert np.all(F[off] > 0)
        errs.append(np.max(np.abs(F.sum(1) - 1)))
    assert errs[0] < 0.03 and errs[1] < 0.008 and errs[1] < errs[0] / 2


def test_P9_outward_sphere_and_flat_plane_are_zero():
    S = oracle.Scene(*sg.closed_sphere_mesh(200, 1.0, inward=False), orient_up=False, grid=0)
    assert np.count_nonzero(S.F_dense()) == 0
    P = oracle.Scene(*sg.flat_plane_mesh(6), grid=0)
    assert np.count_nonzero(P.F_dense()) == 0          # coplanar -> n.d = 0


def test_facing_plates_closed_form_and_blocker():
    d, s = 1.7, 1e-3
    S = oracle.Scene(*sg.facing_plates_mesh(d, s), orient_up=False, grid=0)
    F = S.F_dense()
    # both cosines are 1: F_01 = A_1 / (pi d^2)
    assert F[0, 1] == pytest.approx(S.A[1] / (math.pi * d * d), rel=1e-14)
    assert F[1, 0] == pytest.approx(S.A[0] / (math.pi * d * d), rel=1e-14)
    B = oracle.Scene(*sg.blocked_plates_mesh(d, s), orient_up=False, grid=0)
    vis = B.visibility_rows(np.arange(B.N))
    assert vis[0, 1] == 0 and vis[1, 0] == 0
    assert B.F_dense()[0, 1] == 0.0


def test_P3_reciprocity():
    for V, Fc in (sg.cfg1_mesh(), sg.rough_small_mesh(10)):
        S = oracle.Scene(V, Fc)
        F = S.F_dense()
        AF = S.A[:, None] * F
        assert np.max(np.abs(AF - AF.T)) <= 1e-14 * np.max(AF)


# ---------------------------------------------------- P7 brute force / grid

def _seg_tri_numpy(P0, D, a, b, c):
    """Independent predicate: solve P0 + t D = a + u (b-a) + v (c-a) with a
    3x3 linear solve (not Moller-Trumbore); open segment t in (1e-9, 1-1e-9),
    inclusive barycentrics."""
    M = np.column_stack([D, -(b - a), -(c - a)])
    if abs(np.linalg.det(M)) < 1e-300:
        return False
    t, u, v = np.linalg.solve(M, a - P0)
    return (1e-9 < t < 1 - 1e-9) and u >= 0 and v >= 0 and u + v <= 1


def test_P7_visibility_matches_independent_bruteforce():
    S = oracle.Scene(*sg.rough_small_mesh(7), grid=0)   # 98 facets
    vis = S.visibility_rows(np.arange(S.N))
    tri = S.V[S.T]
    ref = np.zeros_like(vis)
    for i in range(S.N):
        for j in range(S.N):
            if i == j:
                continue
            d = S.x[j] - S.x[i]
            if not (S.n[i] @ d > 0 and -(S.n[j] @ d) > 0):
                continue
            hit = any(_seg_tri_numpy(S.x[i], d, *tri[k]) for k in range(S.N) if k != i and k != j)
            ref[i, j] = 0 if hit else 1
    assert np.array_equal(vis, ref)
    assert np.array_equal(vis, vis.T)                  # S:156 symmetry
    assert 0 < vis.sum() < S.N * (S.N - 1)             # some occlusion, some visibility


@pytest.mark.parametrize("mesh", ["rough20", "cfg1"])
def test_P7_grid_equals_bruteforce(mesh):
    V, F = sg.rough_small_mesh(20) if mesh == "rough20" else sg.cfg1_mesh()
    S = oracle.Scene(V, F)
    rows = np.random.default_rng(0).choice(S.N, size=min(S.N, 120), replace=False)
    g = S.visibility_rows(rows, grid=max(4, S.grid))
    b = S.visibility_rows(rows, grid=0)
    assert np.array_equal(g, b)
    suns = sg.sun_dirs(10.0, 6)
    assert np.array_equal(S.insolation(suns, grid=max(4, S.grid)), S.insolation(suns, grid=0))


def test_P7_cos_form_equals_dot_form():
    S = oracle.Scene(*sg.rough_small_mesh(10))
    F = S.F_dense()
    vis = S.visibility_rows(np.arange(S.N))
    d = S.x[None, :, :] - S.x[:, None, :]
    r = np.linalg.norm(d, axis=2)
    np.fill_diagonal(r, 1.0)
    cos_i = np.einsum("ik,ijk->ij", S.n, d) / r          # theta(x_i, x_j)
    cos_j = -np.einsum("jk,ijk->ij", S.n, d) / r
    Fc = cos_i * cos_j / (math.pi * r * r) * vis * S.A[None, :]
    assert np.max(np.abs(Fc - F)) <= 1e-14 * F.max()


# ---------------------------------------------------------------- insolation

def test_insolation_flat_plane_and_horizon():
    S = oracle.Scene(*sg.flat_plane_mesh(5), grid=0)
    Q = S.insolation(np.array([[0, 0, 1.0], [1.0, 0, 0], [0.6, 0, -0.8]]), S=1361.0)
    assert np.allclose(Q[:, 0], 1361.0) and np.all(Q[:, 1] == 0) and np.all(Q[:, 2] == 0)


def test_insolation_cap_shadow_matches_geometric_silhouette():
    # A point p inside the sphere is lit iff the ray p + t s leaves the sphere
    # above the rim plane z = 0 (P:388-396 silhouette geometry).
    geo = sg.cap_geometry()
    S = oracle.Scene(*sg.cfg1_mesh())
    s = sg.sun_dirs(10.0, 1)[0]
    Q = S.insolation(s[None, :])[:, 0]
    c = np.array([0, 0, geo.Hc])
    p = S.x - c
    b = p @ s
    t = -b + np.sqrt(b * b - (np.sum(p * p, 1) - geo.R ** 2))
    z_exit = S.x[:, 2] + t * s[2]
    lit_geo = (z_exit > 0) & (S.n @ s > 0)
    lit = Q > 0
    band = np.abs(z_exit) < 0.01                            # facets straddling the shadow line
    assert np.array_equal(lit[~band], lit_geo[~band])
    assert band.mean() < 0.05


def test_insolation_cap_mean_flux_identity():
    # All flux through the opening lands on the cap: sum A_i Q_i -> S sin(e) pi rc^2
    geo = sg.cap_geometry()
    errs = []
    for nfib in (300, 1200):
        S = oracle.Scene(*sg.cap_mesh(nfib, int(round(90 * math.sqrt(nfib / 770)))))
        Q = S.insolation(sg.sun_dirs(10.0, 1))[:, 0]
        errs.append(abs(S.A @ Q / (1365 * math.sin(math.radians(10)) * math.pi * geo.rc ** 2) - 1))
    assert errs[1] < 0.03 and errs[1] < errs[0]


# ---------------------------------------------------------------- solvers

def test_jacobi_fixed_point_examples():
    # K = 0 -> x = rhs after one iteration; scalar K = 0.5, rhs = 1 -> 2.
    E = np.array([[1.0], [2.0]])
    B, Q, it, r = oracle.jacobi(lambda X: np.zeros_like(X), E, [0.3, 0.3], 1e-14, 50)
    assert it == 1 and np.array_equal(B, E) and np.all(r == 0)
    B, Q, it, r = oracle.jacobi(lambda X: 0.5 * X, np.array([[1.0]]), [1.0], 1e-15, 200)
    assert B[0, 0] == pytest.approx(2.0, rel=1e-14)
    # rho = 0 -> B = E (P9)
    B, *_ = oracle.jacobi(lambda X: X, E, [0.0, 0.0], 1e-14, 10)
    assert np.array_equal(B, E)


def _sherman_morrison(A, rho, E, c):
    # F = c (1 A^T - diag A): (I - diag(rho) F) = D - c rho A^T, D = diag(1 + c rho_i A_i)
    Dg = 1.0 + c * rho * A
    y = E / Dg[:, None]
    u = rho / Dg
    return y + u[:, None] * (c * (A @ y)) / (1.0 - c * (A @ u))


def test_P4_sherman_morrison_jacobi_and_lu():
    R = 1.0
    x, nrm, A = sg.sphere_exact_facets(300, R, cap_cos=0.2)
    F = oracle.F_dense_facets(x, nrm, A)
    c = 1 / (4 * math.pi * R * R)
    rng = np.random.default_rng(5)
    rho = 0.05 + 0.9 * rng.random(300)
    E = np.asfortranarray(rng.random((300, 3)))
    exact = _sherman_morrison(A, rho, E, c)
    B_lu = oracle.lu_radiosity(F, E, rho)
    assert np.max(np.abs(B_lu - exact)) / np.max(np.abs(exact)) < 1e-13
    B, Q, it, r = oracle.jacobi(lambda X: oracle.apply_dense(F, X), E, rho, 1e-14, 200)
    assert np.max(np.abs(B - exact)) / np.max(np.abs(exact)) < 1e-13
    assert it < 60 and np.all(r <= 1e-14)


def test_thermal_special_cases():
    N = 5
    Qdir = np.linspace(0, 1000, N)[:, None]
    alb, em = np.full(N, 0.2), np.full(N, 0.9)
    out = oracle.thermal(lambda X: np.zeros_like(X), Qdir, alb, em, 1e-12, 20)
    assert np.allclose(out["T"][:, 0], ((1 - alb) * Qdir[:, 0] / (em * oracle.SIGMA_SB)) ** 0.25, rtol=1e-15)
    out = oracle.thermal(lambda X: 0.1 * X, np.zeros((N, 1)), alb, em, 1e-12, 20)
    assert np.all(out["T"] == 0)


def test_thermal_W_form_equals_T_form_iteration():
    # c1 item 6: T_k -> eps sigma T_k^4 = (1-a)Qvis + eps Q_IR,k ->
    # Q_IR,k+1 = F[eps sigma T_k^4 + (1-eps) Q_IR,k] (eq. QIR-integral-equation,
    # P:93) is iterate-for-iterate the W iteration of eq. QIR.
    S = oracle.Scene(*sg.cap_mesh(200, 40))
    F = S.F_dense()
    a, e = 0.12, 0.95
    Qvis = S.insolation(sg.sun_dirs(10, 1))
    E2 = (1 - a) * Qvis
    W = E2.copy()
    Qir_T = np.zeros_like(Qvis)
    for _ in range(6):
        Qir_W = F @ W
        W = E2 + Qir_W
        T4 = ((1 - a) * Qvis + e * Qir_T) / (e * oracle.SIGMA_SB)
        Qir_T = F @ (e * oracle.SIGMA_SB * T4 + (1 - e) * Qir_T)
        assert np.allclose(Qir_T, Qir_W, rtol=1e-12, atol=1e-12 * Qvis.max())


# ---------------------------------------------------- P6 analytic cap crater

def test_P6_analytic_formulas_spec_worked_values():
    g = json.load(open(os.path.join(GOLD, "cap_analytic_spec.json")))
    beta = math.radians(g["beta_deg"])
    D_over_d = 2 * math.sin(beta) / (1 - math.cos(beta))
    f = oracle.cap_f(D_over_d)
    b = oracle.cap_b(f, g["albedo"], g["emiss"])
    assert abs(f - g["f"]) < g["f_abs_tol"] and abs(b - g["b"]) < g["b_abs_tol"]
    T361 = oracle.cap_shadow_T_p361(g["S"], g["e_sun_deg"], f, g["albedo"], g["emiss"])
    Tglob = oracle.cap_T_global(g["S"], g["e_sun_deg"], f, g["albedo"], g["emiss"], "shadow")
    assert abs(T361 - g["T_shadow_K"]) < g["T_abs_tol"]
    assert T361 == pytest.approx(Tglob, rel=1e-14)        # P:361 and P:370-380 agree


def test_P6_cfg1_values():
    g = json.load(open(os.path.join(GOLD, "cap_cfg1_survey.json")))
    f = oracle.cap_f(g["D_over_d"])
    assert f == pytest.approx(g["f"], rel=1e-15)
    b = oracle.cap_b(f, g["albedo"], g["emiss"])
    assert abs(b - g["b"]) < g["b_abs_tol"]
    T = oracle.cap_T_global(g["S"], g["e_sun_deg"], f, g["albedo"], g["emiss"], "shadow")
    assert abs(T - g["T_shadow_K"]) < g["T_abs_tol"]


@pytest.mark.slow
def test_P6_shadow_temperature_approached_under_refinement():
    g = json.load(open(os.path.join(GOLD, "cap_cfg1_survey.json")))
    Tex = oracle.cap_T_global(g["S"], g["e_sun_deg"], oracle.cap_f(5.0), g["albedo"], g["emiss"], "shadow")
    errs, errs_lit = [], []
    for nfib in (180, 770, 3000):
        S = oracle.Scene(*sg.cap_mesh(nfib, int(round(90 * math.sqrt(nfib / 770)))))
        F = S.F_dense()
        Q = S.insolation(sg.sun_dirs(g["e_sun_deg"], 1), S=g["S"])
        out = oracle.thermal(lambda X: oracle.apply_dense(F, X), Q, np.full(S.N, g["albedo"]),
                             np.full(S.N, g["emiss"]), 1e-10, 100)
        sh = Q[:, 0] == 0
        T = out["T"][sh, 0]
        errs.append(np.linalg.norm(T - Tex) / (math.sqrt(T.size) * Tex))
        # sunlit crater facets: P:370-377 'lit' branch, sin e_local = n_i.s = Q_i / S
        lit = ~sh
        Tl = np.array([oracle.cap_T_global(g["S"], g["e_sun_deg"], oracle.cap_f(5.0), g["albedo"], g["emiss"],
                                           "lit", q / g["S"]) for q in Q[lit, 0]])
        errs_lit.append(np.linalg.norm(out["T"][lit, 0] - Tl) / np.linalg.norm(Tl))
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] < 0.02
    assert errs_lit[0] > errs_lit[1] > errs_lit[2] and errs_lit[2] < 5e-4


# --------------------------------------------------------- hierarchical (Alg. 2-5)

def test_quadtree_partition():
    xy = np.array([[0.25, 0.25], [0.25, 0.75], [0.75, 0.25], [0.75, 0.75]])
    root, perm = hm.quadtree(xy, 8, 1)
    assert len(root.children) == 4 and all(c.size == 1 for c in root.children)
    rng = np.random.default_rng(1)
    xy = rng.random((500, 2))
    root, perm = hm.quadtree(xy, 6, 8)
    assert np.array_equal(np.sort(perm), np.arange(500))

    def check(nd):
        if nd.children:
            assert nd.children[0].start == nd.start and nd.children[-1].stop == nd.stop
            for a, b in zip(nd.children[:-1], nd.children[1:]):
                assert a.stop == b.start
            for c in nd.children:
                pts = xy[perm[c.start:c.stop]]
                par = xy[perm[nd.start:nd.stop]]
                assert np.all(pts.min(0) >= par.min(0)) and np.all(pts.max(0) <= par.max(0))
                check(c)
    check(root)


def test_nbytes_examples_and_rank():
    assert hm.nbytes_dense(100, 100, 4) == 40000
    assert hm.nbytes_csr(10, 0, 4) == 88
    rng = np.random.default_rng(2)
    a, b = rng.random(300), rng.random(200)
    q, *_ = hm.estimate_rank(np.outer(a, b), 1e-2, 8)       # rank-1 -> q = 1
    assert q == 1
    assert hm.estimate_rank(np.eye(64), 1e-2, 8) is None    # flat spectrum fails


@pytest.mark.parametrize("eps", [1e-2, 1e-5])
def test_P8_svd_block_bound_and_10tol(eps):
    S = oracle.Scene(*sg.cfg1_mesh())
    F = S.F_dense()
    H = hm.compress(S.x, F, eps, min_size=4096)
    Fp = F[np.ix_(H.perm, H.perm)]
    nsvd = 0
    for b in H.leaves():
        if b.kind == hm.SVD:
            nsvd += 1
            blk = Fp[b.row0:b.row0 + b.m, b.col0:b.col0 + b.n]
            q, ur, vr, U, Sg, V = b.data
            approx = np.zeros_like(blk)
            approx[np.ix_(ur, vr)] = (U * Sg) @ V.T
            s = np.linalg.svd(blk, compute_uv=False)
            err = np.linalg.norm(blk - approx, 2)
            sq1 = s[q] if q < s.size else 0.0
            assert err <= sq1 * (1 + 1e-8) + 1e-15 * s[0]
            assert err < eps * s[0]
    assert nsvd > 0
    D = hm.densify(H)
    assert np.linalg.norm(D - F) / np.linalg.norm(F) <= 10 * eps
    X = sg.random_rhs(S.N, 20)
    Y = hm.hmatvec(H, X)
    Y0 = oracle.apply_dense(F, X)
    assert np.linalg.norm(Y - Y0) / np.linalg.norm(Y0) <= 10 * eps
    # DP dominance: never more than the full CSR + node overheads
    nnz = np.count_nonzero(F)
    assert H.nbytes <= hm.nbytes_csr(S.N, nnz, 8) * 1.05


def test_sphere_exact_blocks_are_rank_one():
    x, nrm, A = sg.sphere_exact_facets(800, 1.0, cap_cos=0.3)
    F = oracle.F_dense_facets(x, nrm, A)
    H = hm.compress(x, F, 1e-10, min_size=2048)
    ks = [b.data[0] for b in H.leaves() if b.kind == hm.SVD]
    assert ks and all(k == 1 for k in ks)                   # P4: off-diagonal blocks c 1 A^T
    assert np.allclose(hm.hmatvec(H, np.ones((800, 1)))[:, 0], F.sum(1), rtol=1e-12)


def test_hmatvec_zero_cases():
    S = oracle.Scene(*sg.flat_plane_mesh(12))
    F = S.F_dense()
    H = hm.compress(S.x, F, 1e-5, min_size=256)
    assert H.leaves() == [] and H.nbytes == 0
    assert np.all(hm.hmatvec(H, np.ones((S.N, 2))) == 0)


# ------------------------------------------------------------ round-2 pins

def test_alg3_accepts_rank_above_half_min():
    """Alg. 3 ("Increase k ... jump back") has no k >= min(m,n)/2
    stop: a 100 x 100 block whose 50 x 50 nonzero core has exactly 33 unit
    singular values (rank 33 > 50/2) is accepted at q = 33, because its SVD
    (w q (m'+n') + w q + 4 (m'+n') = 26400 + 264 + 400 = 27,064 B, reading A7/A8)
    is smaller than its CSR (8 (100+1) + 12 x 2500 = 30,808 B)."""
    rng = np.random.default_rng(11)
    Qa, _ = np.linalg.qr(rng.standard_normal((50, 50)))
    Qb, _ = np.linalg.qr(rng.standard_normal((50, 50)))
    core = Qa[:, :33] @ Qb[:, :33].T                       # singular values: 33 x 1.0, 17 x 0
    B = np.zeros((100, 100))
    rows, cols = rng.choice(100, 50, replace=False), rng.choice(100, 50, replace=False)
    B[np.ix_(np.sort(rows), np.sort(cols))] = core
    assert np.count_nonzero(B) == 2500
    assert hm.nbytes_csr(100, 2500, 8) == 30808
    assert hm.nbytes_svd(33, 50, 50, 8) == 27064
    out = hm.estimate_rank(B, 1e-5, 8)
    assert out is not None
    q, ur, vr, U, S, V = out
    assert q == 33
    assert np.array_equal(ur, np.sort(rows)) and np.array_equal(vr, np.sort(cols))
    R = np.zeros_like(B)
    R[np.ix_(ur, vr)] = (U * S) @ V.T
    assert np.abs(R - B).max() < 1e-12


def test_alg3_rejects_when_factor_bytes_reach_csr_bytes():
    """The one stop rule left (A5): w k (m'+n') >= nbytes(F_IJ) -> no q > k can
    pass eq. nbytes-comparison.  A full-rank 40 x 40 random block never passes."""
    rng = np.random.default_rng(12)
    assert hm.estimate_rank(rng.random((40, 40)), 1e-5, 8) is None


def test_F_csr_rows_and_apply_csr_match_dense():
    """or_viewfactor_csr_rows / or_apply_csr (the exact-F reference of the
    full-size GPU parity and of bench.py's parity) on a rows subset that is
    neither 0..n nor sorted: every stored row equals the dense row (pinned by
    P1/P3/P7) and holds every nonzero of it; the apply equals numpy's product."""
    S = oracle.Scene(*sg.rough_small_mesh(14, amp=0.3))        # 392 facets, occluded
    Fd = S.F_dense()
    rng = np.random.default_rng(5)
    rows = rng.choice(S.N, 97, replace=False)                  # unsorted, gaps
    rows[3] = rows[0]                                          # a repeated row
    rowptr, cols, vals = S.F_csr_rows(rows)
    assert rowptr[0] == 0 and rowptr.size == rows.size + 1
    for i, r in enumerate(rows):
        c, v = cols[rowptr[i]:rowptr[i + 1]], vals[rowptr[i]:rowptr[i + 1]]
        dense_row = np.zeros(S.N)
        dense_row[c] = v
        assert np.array_equal(dense_row, Fd[r]), r             # bitwise, incl. the zero pattern
        assert np.all(v != 0) and np.all(np.diff(c) > 0)
    assert rowptr[-1] == np.count_nonzero(Fd[rows])
    # the grid accelerator and brute force give the same rows
    rp2, c2, v2 = S.F_csr_rows(rows, grid=0)
    assert np.array_equal(rp2, rowptr) and np.array_equal(c2, cols) and np.array_equal(v2, vals)
    X = sg.random_rhs(S.N, 3)
    Y = oracle.apply_csr((rowptr, cols, vals), X)
    Yn = Fd[rows] @ X
    assert np.abs(Y - Yn).max() <= 1e-14 * np.abs(Yn).max()
    assert np.array_equal(Y, oracle.apply_dense(Fd, X)[rows])  # same per-row order -> bitwise


def test_quadtree_splits_at_midpoint_not_median():
    """Reading A1: split at x_mid = (x_min + x_max)/2,
    y_mid likewise, a coordinate equal to mid goes to the upper half.  On this
    asymmetric set the median split would put 2 points on each side of x."""
    xy = np.array([[0.0, 0.0], [0.1, 0.3], [0.2, 0.1], [0.3, 0.2], [10.0, 10.0]])
    root, perm = hm.quadtree(xy, 8, 1)
    # x_mid = y_mid = 5: four points lower-left (I1), one upper-right (I4)
    assert [c.size for c in root.children] == [4, 1]
    assert sorted(perm[root.children[0].start:root.children[0].stop].tolist()) == [0, 1, 2, 3]
    assert perm[root.children[1].start] == 4
    # ties: x = x_mid and y = y_mid go to the upper halves
    xy = np.array([[0.0, 0.0], [4.0, 4.0], [8.0, 8.0], [4.0, 0.0], [0.0, 4.0]])
    root, perm = hm.quadtree(xy, 8, 1)
    sets = [sorted(perm[c.start:c.stop].tolist()) for c in root.children]
    # I1 = {x<4,y<4}: 0; I2 = {x<4,y>=4}: 4; I3 = {x>=4,y<4}: 3; I4 = {x>=4,y>=4}: 1, 2
    assert sets == [[0], [4], [3], [1, 2]]


def test_cap_T_global_outside_is_flat_plane_equilibrium():
    """P:370-377 'outside' branch: eps sigma T^4 = (1 - alpha) S sin e for a
    facet that sees no other facet -- the oracle's thermal chain on a flat
    plane (F = 0, P9) must give exactly this temperature."""
    S = oracle.Scene(*sg.flat_plane_mesh(6))
    F = S.F_dense()
    e = 23.0
    Q = S.insolation(sg.sun_dirs(e, 1), S=1365.0)
    out = oracle.thermal(lambda X: oracle.apply_dense(F, X), Q, np.full(S.N, 0.12), np.full(S.N, 0.95), 1e-12, 20)
    Tout = oracle.cap_T_global(1365.0, e, 0.1, 0.12, 0.95, "outside")
    assert np.allclose(out["T"][:, 0], Tout, rtol=1e-13)


def test_insolation_disk_point_limit_and_flat_plane():
    """Finite solar disk: P = 1 at radius 0 is the point sun; on an
    unoccluded flat plane the sum over the sunflower sources equals
    S sum_p w_p sin(e_p) with sin(e_p) = d_p.z, whose mean over a disk uniform
    in the tangent plane (r^2 uniform) is sin(e) 2 (cos rho + rho sin rho - 1)/rho^2
    to the quadrature error; the azimuthal terms cancel."""
    S = oracle.Scene(*sg.flat_plane_mesh(5))
    suns = sg.sun_dirs(30.0, 3)
    d1, w1 = sg.sun_disk_points(suns, radius=0.0, P=1)
    np.testing.assert_array_equal(oracle.insolation_disk(S, d1, w1, 1000.0), S.insolation(suns, 1000.0))
    rho = math.radians(5.0)
    mean_cos = 2.0 * (math.cos(rho) + rho * math.sin(rho) - 1.0) / rho ** 2
    exact = 1000.0 * math.sin(math.radians(30.0)) * mean_cos
    errs = []
    for P in (100, 400, 1600):                       # quadrature error ~ 1/P
        d, w = sg.sun_disk_points(suns, radius=rho, P=P)
        errs.append(np.abs(oracle.insolation_disk(S, d, w, 1000.0) / exact - 1.0).max())
    assert errs[0] > errs[1] > errs[2] and errs[2] < 1e-4
    assert abs(mean_cos - 1.0) > 1e-3                # the disk effect is resolved, not rounding


def test_insolation_disk_penumbra_between_zero_and_point_flux():
    """Facets near the cap's shadow edge see part of the disk: 0 <= Q_disk <= S n.s_max,
    and far from the edge the disk and point fluxes agree closely."""
    S = oracle.Scene(*sg.cfg1_mesh())
    suns = sg.sun_dirs(10.0, 1)
    d, w = sg.sun_disk_points(suns, radius=0.03, P=24)
    Qd = oracle.insolation_disk(S, d, w)[:, 0]
    Qp = S.insolation(suns)[:, 0]
    mu_max = np.max(S.n @ d.T, axis=1).clip(0) * 1365.0
    assert np.all(Qd >= 0) and np.all(Qd <= mu_max + 1e-9)
    part = (Qd > 0) & (Qd < 0.9 * (S.n @ suns[0]).clip(0) * 1365.0)
    assert part.sum() > 0
    # facets that see every source: Qd = S sum_p w_p n.d_p, within S rho of the point flux
    unocc = np.abs(Qd - 1365.0 * (np.clip(S.n @ d.T, 0, None) @ w)) < 1e-9
    full = unocc & (Qp > 0) & (Qd > 0)
    assert full.sum() > 0.15 * S.N
    assert np.all(np.abs(Qd[full] - Qp[full]) <= 1365.0 * 0.03)


def test_octree_partition_and_midpoint_rule():
    """Octree: <= 8 children split at the x/y/z midpoints (reading
    A1 in 3D, ties to the upper half), children in (x, y, z) order, x slowest;
    nested, contiguous tree-order ranges."""
    pts = np.array([[0, 0, 0], [0, 0, 4.0], [0, 4.0, 0], [0, 4, 4], [4, 0, 0], [4, 0, 4], [4, 4, 0], [8, 8, 8.0],
                    [0.1, 0.2, 0.3]])
    root, perm = hm.octree(pts, 8, 1)
    sets = [sorted(perm[c.start:c.stop].tolist()) for c in root.children]
    # mid = 4 on every axis: the 4's go up; (0.1,0.2,0.3) joins the origin's octant
    assert sets == [[0, 8], [1], [2], [3], [4], [5], [6], [7]]
    rng = np.random.default_rng(3)
    xyz = rng.random((700, 3)) ** 2                          # skewed: midpoint != median
    root, perm = hm.octree(xyz, 6, 8)
    assert np.array_equal(np.sort(perm), np.arange(700))
    assert len(root.children) == 8

    def check(nd):
        if nd.children:
            assert len(nd.children) <= 8
            assert nd.children[0].start == nd.start and nd.children[-1].stop == nd.stop
            par = xyz[perm[nd.start:nd.stop]]
            mid = 0.5 * (par.min(0) + par.max(0))
            for c in nd.children:
                pts_c = xyz[perm[c.start:c.stop]]
                hi = pts_c >= mid
                assert np.all(hi == hi[0])                     # one octant per child
                check(c)
    check(root)


def test_octree_closed_body_reciprocity_and_compression():
    """Closed bilobed body (67P stand-in): the exact F satisfies reciprocity
    (P3), is nonzero only across the concave neck region, and the octree
    compression reproduces it within 10 eps."""
    V, F = sg.bilobed_body_mesh(800)
    S = oracle.Scene(V, F, orient_up=False)
    Fd = S.F_dense()
    AF = S.A[:, None] * Fd
    assert np.abs(AF - AF.T).max() <= 1e-14 * AF.max()
    assert 0 < np.count_nonzero(Fd) < 0.1 * Fd.size
    H = hm.compress(S.x, Fd, 1e-5, min_size=2048, tree="oct")
    assert len(H.tops) <= 64
    assert np.linalg.norm(hm.densify(H) - Fd) / np.linalg.norm(Fd) <= 1e-4
