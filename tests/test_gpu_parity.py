"""GPU parity: the CUDA path through the C ABI vs the FP64 oracle.

  * same blocks:  GPU apply/solves of an oracle-built F-hat (written by
    oracle/hmatrix.py as HVFM, loaded with vf_load) vs the oracle's Alg. 5
    apply and Jacobi/thermal solves of the same blocks:  rel. L2 <= 1e-12
    (f64), <= 1e-5 (f32), identical iteration counts (BASELINE north_star
    tolerances);
  * whole pipeline: the product's own vf_build F-hat on the GPU vs the
    oracle's exact F:  <= 10 tol, Sherman-Morrison closed form;
  * full size (BASELINE configs[1], the bench workload): sampled rows of the
    exact F and the thermal solve of the bench's launch configuration.
"""
import math

import numpy as np
import pytest

import oracle
import oracle.hmatrix as hm
import paper_2209_07632_b200 as vf
import scenegen as sg

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def dev(a, dtype=np.float64):
    a = np.asarray(a, dtype=dtype)
    if a.ndim == 1:
        return torch.from_numpy(a.copy()).cuda()
    return torch.from_numpy(np.ascontiguousarray(a.T)).cuda().T        # (N, k), strides (1, N)


def empty(N, k, dtype=torch.float64):
    return torch.empty((k, N), dtype=dtype, device="cuda").T


def host(t):
    return t.cpu().numpy().astype(np.float64)


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


# ----------------------------------------------------------------- fixtures

@pytest.fixture(scope="module")
def cap():
    V, F = sg.cfg1_mesh()
    S = oracle.Scene(V, F)
    return V, F, S, S.F_dense()


@pytest.fixture(scope="module")
def rough():
    V, F = sg.rough_small_mesh(24, amp=0.05)   # 1152 facets, occluded: CSR leaves
    S = oracle.Scene(V, F)
    return V, F, S, S.F_dense()


def oracle_handle(S, Fd, tmp_path_factory, eps, dtype="f64", min_size=16384, tag=""):
    H = hm.compress(S.x, Fd, eps, dtype=dtype, min_size=min_size)
    p = str(tmp_path_factory.mktemp("hv") / f"o{tag}{dtype}.hvfm")
    hm.write_hvfm(H, p)
    return H, vf.ViewFactorMatrix.load(p, device=0)


CASES = [("cap", 1e-5, 16384), ("cap", 1e-7, 2048), ("rough", 1e-5, 2048), ("rough", 1e-14, 16384)]


@pytest.mark.parametrize("which,eps,min_size", CASES)
@pytest.mark.parametrize("k", [1, 2, 3, 8, 17, 64, 130, 300])
def test_matvec_same_blocks_f64(cap, rough, tmp_path_factory, which, eps, min_size, k):
    V, F, S, Fd = cap if which == "cap" else rough
    H, M = oracle_handle(S, Fd, tmp_path_factory, eps, "f64", min_size, f"{which}{eps}{min_size}")
    kinds = {b.kind for b in H.leaves()}
    assert kinds
    X = sg.random_rhs(S.N, k, seed=3 + k)
    Y = empty(S.N, k)
    M.matvec(dev(X), Y)
    assert rel(host(Y), hm.hmatvec(H, X)) <= 1e-12


def test_block_kinds_covered(cap, rough, tmp_path_factory):
    seen = set()
    for which, eps, ms in CASES:
        V, F, S, Fd = cap if which == "cap" else rough
        H = hm.compress(S.x, Fd, eps, min_size=ms)
        seen |= {b.kind for b in H.leaves()}
    assert seen == {hm.DENSE, hm.CSR, hm.SVD}


@pytest.mark.parametrize("k", [1, 4, 64])
def test_matvec_same_blocks_f32(cap, rough, tmp_path_factory, k):
    for which in ("cap", "rough"):
        V, F, S, Fd = cap if which == "cap" else rough
        H, M = oracle_handle(S, Fd, tmp_path_factory, 1e-5, "f32", 2048, which)
        X = sg.random_rhs(S.N, k).astype(np.float32).astype(np.float64)
        Y = empty(S.N, k, torch.float32)
        M.matvec(dev(X, np.float32), Y)
        assert rel(host(Y), hm.hmatvec(H, X)) <= 1e-5


def test_host_pointers_equal_device_and_deterministic(cap, tmp_path_factory):
    V, F, S, Fd = cap
    H, M = oracle_handle(S, Fd, tmp_path_factory, 1e-5, "f64", 4096, "hp")
    X = sg.random_rhs(S.N, 5)
    Yh = np.empty((S.N, 5), order="F")
    M.matvec(np.asfortranarray(X), Yh)
    Yd = empty(S.N, 5)
    M.matvec(dev(X), Yd)
    Yd2 = empty(S.N, 5)
    M.matvec(dev(X), Yd2)
    assert np.array_equal(Yh, host(Yd)) and torch.equal(Yd, Yd2)


@pytest.mark.parametrize("k", [1, 3, 64])
def test_radiosity_same_blocks(cap, rough, tmp_path_factory, k):
    for which in ("cap", "rough"):
        V, F, S, Fd = cap if which == "cap" else rough
        H, M = oracle_handle(S, Fd, tmp_path_factory, 1e-6, "f64", 2048, "rad" + which)
        rng = np.random.default_rng(11)
        E = np.asfortranarray(1000 * rng.random((S.N, k)))
        # keep the spectral radius of diag(rho) F below 0.9 (rough midpoint-rule
        # meshes have row sums > 1)
        rho = (0.05 + 0.9 * rng.random(S.N)) / max(1.0, np.abs(Fd).sum(1).max())
        B0, Q0, it0, r0 = oracle.jacobi(lambda X: hm.hmatvec(H, X), E, rho, 1e-13, 200)
        B = empty(S.N, k)
        M.solve_radiosity(dev(E), dev(rho), B, iters=200, tol=1e-13)
        st = M.stats()
        assert st["iters1"] == it0
        assert rel(host(B), B0) <= 1e-12


@pytest.mark.parametrize("k", [1, 64])
def test_thermal_same_blocks(cap, tmp_path_factory, k):
    V, F, S, Fd = cap
    H, M = oracle_handle(S, Fd, tmp_path_factory, 1e-5, "f64", 16384, "th")
    Q = S.insolation(sg.sun_dirs(10.0, k, 0.1))
    alb, emi = np.full(S.N, 0.12), np.full(S.N, 0.95)
    ref = oracle.thermal(lambda X: hm.hmatvec(H, X), Q, alb, emi, 1e-12, 100)
    T, Qv, Qi = empty(S.N, k), empty(S.N, k), empty(S.N, k)
    M.solve_thermal(dev(Q), dev(alb), dev(emi), T, Qv, Qi, iters=100, tol=1e-12)
    st = M.stats()
    assert (st["iters1"], st["iters2"]) == (ref["it1"], ref["it2"])
    assert rel(host(Qv), ref["Qvis"]) <= 1e-12
    assert rel(host(Qi), ref["Qir"]) <= 1e-12
    assert rel(host(T), ref["T"]) <= 1e-12


def test_noconv_keeps_last_iterate(cap, tmp_path_factory):
    V, F, S, Fd = cap
    H, M = oracle_handle(S, Fd, tmp_path_factory, 1e-5, "f64", 16384, "nc")
    E = np.asfortranarray(np.random.default_rng(1).random((S.N, 2)))
    rho = np.full(S.N, 0.9)
    B0, *_ = oracle.jacobi(lambda X: hm.hmatvec(H, X), E, rho, 1e-300, 2)
    B = empty(S.N, 2)
    with pytest.raises(vf.VFError) as e:
        M.solve_radiosity(dev(E), dev(rho), B, iters=2, tol=1e-300)
    assert e.value.code == vf.VF_ENOCONV
    assert rel(host(B), B0) <= 1e-12


# ----------------------------------------------------------- whole pipeline

@pytest.mark.parametrize("tol", [1e-3, 1e-5])
def test_product_build_matvec_vs_exact_F(cap, tol):
    V, F, S, Fd = cap
    M = vf.ViewFactorMatrix.build(V, F, tol)
    X = sg.random_rhs(S.N, 20)
    Y = empty(S.N, 20)
    M.matvec(dev(X), Y)
    assert rel(host(Y), oracle.apply_dense(Fd, X)) <= 10 * tol


def test_product_build_f32(cap):
    V, F, S, Fd = cap
    M = vf.ViewFactorMatrix.build(V, F, 1e-5, dtype=vf.VF_F32)
    X = sg.random_rhs(S.N, 8)
    Y = empty(S.N, 8, torch.float32)
    M.matvec(dev(X, np.float32), Y)
    assert rel(host(Y), oracle.apply_dense(Fd, X)) <= 1e-4


def test_sherman_morrison_pipeline():
    R = 1.0
    x, n, A = sg.sphere_exact_facets(1200, R, cap_cos=0.2)
    M = vf.ViewFactorMatrix.build_facets(x, n, A, 1e-10, min_block=4096)
    c = 1 / (4 * math.pi * R * R)
    rng = np.random.default_rng(5)
    rho = 0.05 + 0.9 * rng.random(1200)
    E = np.asfortranarray(rng.random((1200, 4)))
    Dg = 1.0 + c * rho * A
    y = E / Dg[:, None]
    u = rho / Dg
    exact = y + u[:, None] * (c * (A @ y)) / (1.0 - c * (A @ u))
    B = empty(1200, 4)
    M.solve_radiosity(dev(E), dev(rho), B, iters=100, tol=1e-15, clamp=True)
    assert rel(host(B), exact) <= 1e-12


def test_product_thermal_vs_exact_F_cfg1(cap):
    V, F, S, Fd = cap
    M = vf.ViewFactorMatrix.build(V, F, 1e-5)
    Q = S.insolation(sg.sun_dirs(10.0, 1))
    alb, emi = np.full(S.N, 0.12), np.full(S.N, 0.95)
    ref = oracle.thermal(lambda X: oracle.apply_dense(Fd, X), Q, alb, emi, 1e-10, 100)
    T = empty(S.N, 1)
    M.solve_thermal(dev(Q), dev(alb), dev(emi), T, iters=100, tol=1e-10)
    assert rel(host(T), ref["T"]) <= 10 * 1e-5


# ------------------------------------------------------------- edge cases

def test_empty_operator_flat_plane():
    V, F = sg.flat_plane_mesh(16)
    M = vf.ViewFactorMatrix.build(V, F, 1e-5)
    N = F.shape[0]
    X = sg.random_rhs(N, 3)
    Y = empty(N, 3)
    M.matvec(dev(X), Y)
    assert torch.count_nonzero(Y) == 0
    B = empty(N, 3)
    M.solve_radiosity(dev(X), dev(np.full(N, 0.3)), B, iters=10, tol=1e-12)
    assert np.array_equal(host(B), X) and M.stats()["iters1"] == 1


def test_zero_inputs_and_rho_zero(cap, tmp_path_factory):
    V, F, S, Fd = cap
    H, M = oracle_handle(S, Fd, tmp_path_factory, 1e-5, "f64", 16384, "z")
    Y = empty(S.N, 2)
    M.matvec(dev(np.zeros((S.N, 2))), Y)
    assert torch.count_nonzero(Y) == 0
    E = np.asfortranarray(np.random.default_rng(2).random((S.N, 2)))
    B = empty(S.N, 2)
    M.solve_radiosity(dev(E), dev(np.zeros(S.N)), B, iters=10, tol=1e-14)
    assert np.array_equal(host(B), E)
    T = empty(S.N, 2)
    M.solve_thermal(dev(np.zeros((S.N, 2))), dev(np.full(S.N, .1)), dev(np.full(S.N, .9)), T, iters=10, tol=1e-12)
    assert torch.count_nonzero(T) == 0


# ---------------------------------------------- full size: BASELINE configs[1]

@pytest.fixture(scope="module")
def cfg2():
    V, F = sg.cfg2_mesh()
    S = oracle.Scene(V, F)
    M = vf.ViewFactorMatrix.build(V, F, 1e-5)
    return V, F, S, M


def test_cfg2_sampled_rows_vs_exact_F(cfg2):
    V, F, S, M = cfg2
    k = 64
    X = sg.random_rhs(S.N, k)
    Y = empty(S.N, k)
    M.matvec(dev(X), Y)
    Yh = host(Y)
    crater = np.flatnonzero(S.x[:, 2] < -1e-9)
    rng = np.random.default_rng(7)
    rows = np.concatenate([rng.choice(crater, 300, replace=False), rng.choice(S.N, 300, replace=False)])
    csr = S.F_csr_rows(rows)
    Yex = oracle.apply_csr(csr, X)
    assert rel(Yh[rows], Yex) <= 10 * 1e-5


def test_cfg2_bench_configuration_thermal(cfg2):
    """The bench's launch configuration: 64 suns at 5 deg elevation, f64."""
    V, F, S, M = cfg2
    suns = sg.sun_dirs(5.0, 64)
    Q = M.insolation(suns, 1365.0)
    Q0 = S.insolation(suns, 1365.0)
    assert np.array_equal(Q > 0, Q0 > 0) and np.max(np.abs(Q - Q0)) <= 1e-12 * 1365
    csr = S.F_csr_rows()
    alb, emi = np.full(S.N, 0.12), np.full(S.N, 0.95)
    ref = oracle.thermal(lambda X: oracle.apply_csr(csr, X), Q0, alb, emi, 1e-10, 100)
    T = empty(S.N, 64)
    M.solve_thermal(dev(Q), dev(alb), dev(emi), T, iters=100, tol=1e-10)
    assert rel(host(T), ref["T"]) <= 10 * 1e-5
    sh = (Q0 == 0) & (S.x[:, 2:3] < -1e-9)
    assert rel(host(T)[sh], ref["T"][sh]) <= 10 * 1e-5


@pytest.mark.parametrize("mesh", ["cfg1", "rough"])
def test_device_evaluator_equals_host_evaluator_bitwise(mesh, tmp_path):
    """The device evaluator of Alg. 1 (vf_build_gpu.cu) repeats the host
    predicate and F_ij operation for operation (reading R-VIS): both builds
    must store byte-identical F-hat containers."""
    V, F = sg.cfg1_mesh() if mesh == "cfg1" else sg.rough_small_mesh(24, amp=0.05)
    paths = []
    for ev in (vf.VF_EVAL_HOST, vf.VF_EVAL_DEVICE):
        M = vf.ViewFactorMatrix.build(V, F, 1e-5, device=0, evaluator=ev)
        p = str(tmp_path / f"e{ev}.hvfm")
        M.save(p)
        paths.append(p)
    assert open(paths[0], "rb").read() == open(paths[1], "rb").read()


@pytest.fixture(scope="module")
def cfg2_small():
    V, F = sg.cfg2_mesh(n_side=40)               # the configs[1] scene at ~3k facets
    S = oracle.Scene(V, F)
    return V, F, S, S.F_dense()


@pytest.mark.parametrize("split", ["1", "0"])
@pytest.mark.parametrize("k", [16, 64, 130])
def test_resident_and_streaming_batched_paths(cfg2_small, rough, tmp_path_factory, k, split, monkeypatch):
    """nrhs >= 9 runs the shared-memory-resident kernel (res_kernel) when the
    layout fits; VF_NO_RESIDENT forces the streaming grouped kernel.  Both must
    match the oracle's Alg. 5 on the same blocks (matvec) and its Jacobi solve
    (identical iteration counts).  split = 1: long groups are split over
    cluster pairs (DSMEM exchange of partial tiles); 0: one CTA per group."""
    monkeypatch.setenv("VF_RES_SPLIT", split)
    for which in ("cfg2", "rough"):
        V, F, S, Fd = cfg2_small if which == "cfg2" else rough
        H = hm.compress(S.x, Fd, 1e-6, min_size=2048)
        p = str(tmp_path_factory.mktemp("res") / f"{which}{k}.hvfm")
        hm.write_hvfm(H, p)
        X = sg.random_rhs(S.N, k, seed=5)
        Yref = hm.hmatvec(H, X)
        rng = np.random.default_rng(3)
        E = np.asfortranarray(100 * rng.random((S.N, k)))
        rho = np.full(S.N, 0.5 / max(1.0, np.abs(Fd).sum(1).max()))
        B0, _, it0, _ = oracle.jacobi(lambda Z: hm.hmatvec(H, Z), E, rho, 1e-13, 200)
        for resident in (True, False):
            if resident:
                monkeypatch.delenv("VF_NO_RESIDENT", raising=False)
            else:
                monkeypatch.setenv("VF_NO_RESIDENT", "1")
            M = vf.ViewFactorMatrix.load(p, device=0)
            if which == "cfg2" or not resident:
                assert bool(M.refresh()["resident"]) == resident
            Y = empty(S.N, k)
            M.matvec(dev(X), Y)
            assert rel(host(Y), Yref) <= 1e-12
            B = empty(S.N, k)
            M.solve_radiosity(dev(E), dev(rho), B, iters=200, tol=1e-13)
            assert M.stats()["iters1"] == it0
            assert rel(host(B), B0) <= 1e-12


def test_k1_matvec_flags_equal_barrier_bitwise(rough, tmp_path_factory, monkeypatch):
    """nrhs = 1 matvec schedules.  u32 layout: the barrier-free schedule
    (per-block T flags, dynamic row queue) sums every row in the same fixed
    order as the grid-barrier static schedule, so the two agree bit for bit.
    Default (16-bit layout, X-sourced runs first in every row, phase 1 ->
    phase 2 by a finished-item counter, VF_K1_OVL): a different fixed order,
    repeatable, within 1e-13 of the barrier version (VF_K1_OVL=0, which
    keeps the u32 segment order) and within 1e-12 of the oracle."""
    V, F, S, Fd = rough
    H = hm.compress(S.x, Fd, 1e-6, min_size=2048)
    p = str(tmp_path_factory.mktemp("k1") / "r.hvfm")
    hm.write_hvfm(H, p)
    X = sg.random_rhs(S.N, 1, seed=9)
    out = []
    for mode in ("flags", "queue", "static"):     # flags+queue / queue+barrier (default) / static+barrier
        monkeypatch.delenv("VF_MV_FLAGS", raising=False)
        monkeypatch.delenv("VF_MV_STATIC", raising=False)
        if mode == "flags":
            monkeypatch.setenv("VF_MV_FLAGS", "1")
        elif mode == "static":
            monkeypatch.setenv("VF_MV_STATIC", "1")
        M = vf.ViewFactorMatrix.load(p, device=0)
        Y = empty(S.N, 1)
        for _ in range(3):                       # repeated launches reset the flags and the queue
            M.matvec(dev(X), Y)
        out.append(host(Y))
    assert np.array_equal(out[0], out[2])
    assert rel(out[1], out[0]) <= 1e-13
    for o in out:
        assert rel(o, hm.hmatvec(H, X)) <= 1e-12
    # the overlapped default vs the same 16-bit layout with the grid barrier
    monkeypatch.delenv("VF_MV_FLAGS", raising=False)
    monkeypatch.delenv("VF_MV_STATIC", raising=False)
    res = []
    for ovl in ("1", "0"):
        monkeypatch.setenv("VF_K1_OVL", ovl)
        M = vf.ViewFactorMatrix.load(p, device=0)
        Y = empty(S.N, 1)
        ys = []
        for _ in range(3):
            M.matvec(dev(X), Y)
            ys.append(host(Y))
        assert all(np.array_equal(ys[0], y) for y in ys)
        res.append(ys[0])
    assert rel(res[0], res[1]) <= 1e-13


@pytest.mark.parametrize("k", [2, 3, 8])
def test_small_batch_column_split_equals_k1_applies(rough, tmp_path_factory, monkeypatch, k):
    """2..8 columns on a large F-hat go column by column through the nrhs = 1
    kernel (VF_MV_COLSPLIT forces the rule on this small matrix): each output
    column must equal a separate nrhs = 1 apply bit for bit, host buffers
    included, and match the oracle's Alg. 5 apply."""
    V, F, S, Fd = rough
    H = hm.compress(S.x, Fd, 1e-6, min_size=2048)
    p = str(tmp_path_factory.mktemp("cs") / "r.hvfm")
    hm.write_hvfm(H, p)
    X = sg.random_rhs(S.N, k, seed=11)
    M = vf.ViewFactorMatrix.load(p, device=0)
    monkeypatch.setenv("VF_MV_COLSPLIT", "1")
    Y = empty(S.N, k)
    M.matvec(dev(X), Y)
    Yh = np.asfortranarray(np.zeros((S.N, k)))
    M.matvec(X, Yh)
    monkeypatch.setenv("VF_MV_COLSPLIT", "0")
    Yb = empty(S.N, k)
    M.matvec(dev(X), Yb)
    cols = []
    for c in range(k):
        y = empty(S.N, 1)
        M.matvec(dev(np.asfortranarray(X[:, c:c + 1])), y)
        cols.append(host(y)[:, 0])
    assert np.array_equal(host(Y), np.stack(cols, axis=1))
    assert np.array_equal(host(Y), Yh)
    Yref = hm.hmatvec(H, X)
    assert rel(host(Y), Yref) <= 1e-12
    assert rel(host(Yb), Yref) <= 1e-12


def test_wide_batch_chunks_equal_separate_applies(rough, tmp_path_factory, monkeypatch):
    """More than 64 columns on a large F-hat are applied in 64-column chunks,
    the tail in 32/16-column pieces and single columns (VF_MV_CHUNK forces
    the rule here): each piece equals a separate apply of those columns bit
    for bit, and the whole result matches the oracle's Alg. 5 apply."""
    V, F, S, Fd = rough
    H = hm.compress(S.x, Fd, 1e-6, min_size=2048)
    p = str(tmp_path_factory.mktemp("ch") / "r.hvfm")
    hm.write_hvfm(H, p)
    k, c = 150, 64
    X = sg.random_rhs(S.N, k, seed=12)
    M = vf.ViewFactorMatrix.load(p, device=0)
    monkeypatch.setenv("VF_MV_CHUNK", str(c))
    Y = empty(S.N, k)
    M.matvec(dev(X), Y)
    monkeypatch.setenv("VF_MV_CHUNK", "0")
    monkeypatch.setenv("VF_MV_COLSPLIT", "0")
    pieces, c0, piece = [], 0, c                 # libvf's piece rule: 64, 64, 16, then 6 single columns
    while c0 < k:
        n = k - c0
        if n >= piece:
            n = piece
        elif piece // 2 >= 16:
            piece //= 2
            continue
        if n <= 8:
            pieces += [1] * (k - c0)
            break
        pieces.append(n)
        c0 += n
    assert pieces == [64, 64, 16] + [1] * 6
    parts, c0 = [], 0
    for n in pieces:
        y = empty(S.N, n)
        M.matvec(dev(np.asfortranarray(X[:, c0:c0 + n])), y)
        parts.append(host(y))
        c0 += n
    assert np.array_equal(host(Y), np.concatenate(parts, axis=1))
    assert rel(host(Y), hm.hmatvec(H, X)) <= 1e-12


@pytest.mark.parametrize("k", [1, 3, 8])
def test_column_split_solves_same_blocks(cap, rough, tmp_path_factory, monkeypatch, k):
    """Column-split Jacobi (1..8 columns on a large F-hat: each column's product
    through the nrhs = 1 apply, one epilogue/decision launch per iteration;
    forced here with VF_SOLVE_COLSPLIT=1 on small meshes) against the oracle's
    Jacobi / thermal chain on the same blocks: <= 1e-12 with identical
    iteration counts (A13), and against the persistent batched solve."""
    for which in ("cap", "rough"):
        V, F, S, Fd = cap if which == "cap" else rough
        H, M = oracle_handle(S, Fd, tmp_path_factory, 1e-6, "f64", 2048, "cs" + which)
        rng = np.random.default_rng(21)
        E = np.asfortranarray(1000 * rng.random((S.N, k)))
        E[: S.N // 7, 0] = 0.0                                  # shadowed facets
        rho = (0.05 + 0.9 * rng.random(S.N)) / max(1.0, np.abs(Fd).sum(1).max())
        B0, Q0, it0, r0 = oracle.jacobi(lambda X: hm.hmatvec(H, X), E, rho, 1e-13, 200)
        res = {}
        for mode in ("1", "0"):
            monkeypatch.setenv("VF_SOLVE_COLSPLIT", mode)
            B = empty(S.N, k)
            M.solve_radiosity(dev(E), dev(rho), B, iters=200, tol=1e-13)
            res[mode] = (host(B), M.stats()["iters1"])
        assert res["1"][1] == it0 == res["0"][1]
        assert rel(res["1"][0], B0) <= 1e-12
        assert rel(res["1"][0], res["0"][0]) <= 1e-13
    V, F, S, Fd = cap
    H, M = oracle_handle(S, Fd, tmp_path_factory, 1e-5, "f64", 16384, "csth")
    Q = S.insolation(sg.sun_dirs(10.0, k, 0.1))
    alb, emi = np.full(S.N, 0.12), np.full(S.N, 0.95)
    ref = oracle.thermal(lambda X: hm.hmatvec(H, X), Q, alb, emi, 1e-12, 100)
    monkeypatch.setenv("VF_SOLVE_COLSPLIT", "1")
    T, Qv, Qi = empty(S.N, k), empty(S.N, k), empty(S.N, k)
    M.solve_thermal(dev(Q), dev(alb), dev(emi), T, Qv, Qi, iters=100, tol=1e-12)
    st = M.stats()
    assert (st["iters1"], st["iters2"]) == (ref["it1"], ref["it2"])
    for a, b in ((Qv, ref["Qvis"]), (Qi, ref["Qir"]), (T, ref["T"])):
        assert rel(host(a), b) <= 1e-12
    # no convergence within iters: ENOCONV, B holds the last iterate
    E2 = np.asfortranarray(np.random.default_rng(1).random((S.N, k)))
    B0, *_ = oracle.jacobi(lambda X: hm.hmatvec(H, X), E2, np.full(S.N, 0.9), 1e-300, 2)
    B = empty(S.N, k)
    with pytest.raises(vf.VFError) as e:
        M.solve_radiosity(dev(E2), dev(np.full(S.N, 0.9)), B, iters=2, tol=1e-300)
    assert e.value.code == vf.VF_ENOCONV
    assert rel(host(B), B0) <= 1e-12


@pytest.mark.parametrize("k", [16, 64])
def test_resident_phase2_copies(cfg2_small, tmp_path_factory, monkeypatch, k):
    """Resident layout with each phase-2 group replicated over 1, 2 or 4 CTAs
    (copy i takes the column chunks i, i + copies, ...; VF_RES_P2COPIES): every
    output element is still summed by one CTA in the same order, so the matvec
    is bitwise identical across copy counts, and the solves match the oracle
    with identical iteration counts."""
    V, F, S, Fd = cfg2_small
    H = hm.compress(S.x, Fd, 1e-6, min_size=2048)
    p = str(tmp_path_factory.mktemp("p2c") / f"c{k}.hvfm")
    hm.write_hvfm(H, p)
    X = sg.random_rhs(S.N, k, seed=6)
    rng = np.random.default_rng(4)
    E = np.asfortranarray(100 * rng.random((S.N, k)))
    rho = np.full(S.N, 0.5 / max(1.0, np.abs(Fd).sum(1).max()))
    B0, _, it0, _ = oracle.jacobi(lambda Z: hm.hmatvec(H, Z), E, rho, 1e-13, 200)
    ys = []
    for copies in ("1", "2", "4"):
        monkeypatch.setenv("VF_RES_P2COPIES", copies)
        M = vf.ViewFactorMatrix.load(p, device=0)
        assert M.refresh()["resident"] == 1
        Y = empty(S.N, k)
        M.matvec(dev(X), Y)
        ys.append(host(Y))
        B = empty(S.N, k)
        M.solve_radiosity(dev(E), dev(rho), B, iters=200, tol=1e-13)
        assert M.stats()["iters1"] == it0
        assert rel(host(B), B0) <= 1e-12
    assert np.array_equal(ys[0], ys[1]) and np.array_equal(ys[0], ys[2])
    assert rel(ys[0], hm.hmatvec(H, X)) <= 1e-12



@pytest.fixture(scope="module")
def terrain64():
    V, F = sg.cfg3_mesh(n=64, crater_D=1000.0 * 64 / 256)     # the configs[2] recipe at 64^2 cells
    S = oracle.Scene(V, F)
    M = vf.ViewFactorMatrix.build(V, F, 1e-5)
    return V, F, S, M


@pytest.mark.parametrize("k", [1, 4, 64, 128])
def test_terrain64_sampled_rows_vs_exact_F(terrain64, k):
    """configs[2]'s recipe at 64^2 cells (8,192 facets), the product's own
    device build: sampled rows of Y = F-hat X at nrhs 1 (default row kernel),
    4 (column split), 64 and 128 (streamed tiles / resident layout) against
    the same rows of the oracle's exact F (eq. FF-def): <= 10 tol."""
    V, F, S, M = terrain64
    X = sg.random_rhs(S.N, k, seed=11)
    Y = empty(S.N, k)
    M.matvec(dev(X), Y)
    rows = np.random.default_rng(9).choice(S.N, 800, replace=False)
    Yex = oracle.apply_csr(S.F_csr_rows(rows), X)
    assert rel(host(Y)[rows], Yex) <= 10 * 1e-5
