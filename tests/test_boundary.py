"""CPU tests of the C-ABI library: it loads, exports every symbol include/vf.h
declares, and its HOST logic (facet data, visibility, quadtree, Alg. 3-4
build, HVFM io, insolation) agrees with the oracle.  No compute call needs a
GPU here; apply/solve calls on a host-only handle must fail loudly
(VF_ENODEV) -- there is no CPU fallback."""
import math
import os
import re

import numpy as np
import pytest

import oracle
import oracle.hmatrix as hm
import paper_2209_07632_b200 as vf
import scenegen as sg
from tests.hvfm_io import densify, read_hvfm, block_of


def _declared_symbols():
    txt = open(vf.HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(vf_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = vf.lib()
    syms = _declared_symbols()
    assert len(syms) >= 17
    for s in syms:
        assert hasattr(L, s), s


def test_default_opts_and_errors():
    o = vf._opts()
    assert (o.dtype, o.max_depth, o.min_leaf, o.min_block, o.k0) == (vf.VF_F64, 16, 16, 16384, 8)
    with pytest.raises(vf.VFError) as e:
        vf.vf_build(np.zeros((3, 3)), np.array([[0, 1, 2]]), 1e-5, device=-1)   # zero-area face
    assert e.value.code == vf.VF_EINVAL
    with pytest.raises(vf.VFError):
        vf.vf_build(*sg.rough_small_mesh(4), 1.5, device=-1)                     # tol out of range


@pytest.fixture(scope="module")
def cap_small():
    V, F = sg.cap_mesh(300, 45)
    S = oracle.Scene(V, F)
    return V, F, S, S.F_dense()


def test_host_only_handle_has_no_cpu_fallback(cap_small, tmp_path):
    V, F, S, _ = cap_small
    M = vf.ViewFactorMatrix.build(V, F, 1e-3, device=-1)
    x = np.ones(S.N)
    for call in (lambda: M.matvec(x, np.empty(S.N)),
                 lambda: M.solve_radiosity(x, np.full(S.N, 0.1), np.empty(S.N)),
                 lambda: M.solve_thermal(x, np.full(S.N, 0.1), np.full(S.N, 0.9), np.empty(S.N))):
        with pytest.raises(vf.VFError) as e:
            call()
        assert e.value.code == vf.VF_ENODEV


def test_quadtree_permutation_matches_oracle(cap_small):
    V, F, S, _ = cap_small
    M = vf.ViewFactorMatrix.build(V, F, 1e-2, device=-1, visibility=vf.VF_VIS_CULL_ONLY)
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        M.save(os.path.join(d, "a.hvfm"))
        H = read_hvfm(os.path.join(d, "a.hvfm"))
    _, perm = hm.quadtree(S.x[:, :2], 16, 16)           # Alg. 2, same readings A1-A3
    assert np.array_equal(H["perm"], perm)


def test_insolation_matches_oracle():
    for V, F in (sg.cfg1_mesh(), sg.rough_small_mesh(12)):
        M = vf.ViewFactorMatrix.build(V, F, 1e-2, device=-1, visibility=vf.VF_VIS_CULL_ONLY)
        suns = sg.sun_dirs(10.0, 5, 0.3)
        Q = M.insolation(suns, 1365.0)
        Q0 = oracle.Scene(V, F).insolation(suns, 1365.0)
        assert np.array_equal(Q > 0, Q0 > 0)
        assert np.max(np.abs(Q - Q0)) <= 1e-12 * Q0.max()


@pytest.mark.parametrize("tol", [1e-2, 1e-5])
def test_build_matches_oracle_F_within_10tol(cap_small, tmp_path, tol):
    V, F, S, Fd = cap_small
    M = vf.ViewFactorMatrix.build(V, F, tol, device=-1, min_block=2048)
    p = str(tmp_path / "b.hvfm")
    M.save(p)
    H = read_hvfm(p)
    D = densify(H)
    assert np.linalg.norm(D - Fd) / np.linalg.norm(Fd) <= 10 * tol
    # per-SVD-block bound: || F_IJ - U S V^T ||_2 < tol * sigma_1(F_IJ)
    nsvd = 0
    for L in H["leaves"]:
        if L["kind"] == 3:
            nsvd += 1
            rows, cols = block_of(H, L)
            blk = Fd[np.ix_(rows, cols)]
            approx = np.zeros_like(blk)
            approx[np.ix_(L["urows"], L["vrows"])] = (L["U"] * L["S"]) @ L["V"].T
            s1 = np.linalg.norm(blk, 2)
            assert np.linalg.norm(blk - approx, 2) < tol * s1
    assert nsvd > 0
    # every stored visible pair is a true nonzero and vice versa (visibility parity)
    assert M.info["visible_pairs"] == np.count_nonzero(Fd)


def test_rough_mesh_visibility_parity(tmp_path):
    V, F = sg.rough_small_mesh(12)
    S = oracle.Scene(V, F, grid=0)
    Fd = S.F_dense()
    M = vf.ViewFactorMatrix.build(V, F, 1e-6, device=-1, min_block=1 << 30)   # one CSR/dense leaf per pair
    p = str(tmp_path / "r.hvfm")
    M.save(p)
    D = densify(read_hvfm(p))
    assert np.array_equal(D != 0, Fd != 0)
    assert np.max(np.abs(D - Fd)) <= 1e-15 * Fd.max()


def test_hvfm_roundtrip_and_oracle_container(cap_small, tmp_path):
    V, F, S, Fd = cap_small
    M = vf.ViewFactorMatrix.build(V, F, 1e-4, device=-1, min_block=2048)
    a, b = str(tmp_path / "a.hvfm"), str(tmp_path / "b.hvfm")
    M.save(a)
    vf.ViewFactorMatrix.load(a, device=-1).save(b)
    assert open(a, "rb").read() == open(b, "rb").read()                  # S:401 bitwise
    for dtype in ("f64", "f32"):
        H = hm.compress(S.x, Fd, 1e-5, dtype=dtype, min_size=2048)
        c, d = str(tmp_path / f"c{dtype}.hvfm"), str(tmp_path / f"d{dtype}.hvfm")
        hm.write_hvfm(H, c)
        L = vf.ViewFactorMatrix.load(c, device=-1)
        assert L.info["dtype"] == (vf.VF_F64 if dtype == "f64" else vf.VF_F32)
        L.save(d)
        assert open(c, "rb").read() == open(d, "rb").read()


def test_hvfm_rejects_corrupt_files(cap_small, tmp_path):
    V, F, S, Fd = cap_small
    H = hm.compress(S.x, Fd, 1e-3, min_size=2048)
    p = str(tmp_path / "x.hvfm")
    hm.write_hvfm(H, p)
    raw = open(p, "rb").read()
    for bad in (b"XXXX" + raw[4:], raw[: len(raw) // 2], raw[:20]):
        q = str(tmp_path / "bad.hvfm")
        open(q, "wb").write(bad)
        with pytest.raises(vf.VFError) as e:
            vf.vf_load(q, -1)
        assert e.value.code == vf.VF_EIO


def test_sphere_exact_facets_rank_one(tmp_path):
    x, n, A = sg.sphere_exact_facets(900, 1.0, cap_cos=0.3)
    M = vf.ViewFactorMatrix.build_facets(x, n, A, 1e-10, device=-1, min_block=2048)
    p = str(tmp_path / "s.hvfm")
    M.save(p)
    H = read_hvfm(p)
    qs = [L["q"] for L in H["leaves"] if L["kind"] == 3]
    assert qs and all(q == 1 for q in qs)
    Fd = oracle.F_dense_facets(x, n, A)
    assert np.linalg.norm(densify(H) - Fd) / np.linalg.norm(Fd) < 1e-12


def test_flat_plane_is_empty():
    M = vf.ViewFactorMatrix.build(*sg.flat_plane_mesh(10), 1e-5, device=-1)
    i = M.info
    assert i["n_dense"] + i["n_csr"] + i["n_svd"] == 0 and i["active_rows"] == 0


def test_set_mesh_gives_loaded_handles_insolation(tmp_path):
    """vf_set_mesh attaches the geometry of a saved F-hat so vf_insolation
     works on a loaded handle and equals the built handle's."""
    V, F = sg.rough_small_mesh(10)
    M = vf.ViewFactorMatrix.build(V, F, 1e-5, device=-1)
    p = str(tmp_path / "m.hvfm")
    M.save(p)
    L = vf.ViewFactorMatrix.load(p, device=-1)
    suns = sg.sun_dirs(20.0, 3)
    with pytest.raises(vf.VFError):
        L.insolation(suns)
    vf.vf_set_mesh(L.h, V, F)
    np.testing.assert_array_equal(L.insolation(suns), M.insolation(suns))
    with pytest.raises(vf.VFError):
        vf.vf_set_mesh(L.h, V, F[:-1])


def test_device_evaluator_needs_a_device():
    V, F = sg.rough_small_mesh(6)
    with pytest.raises(vf.VFError) as e:
        vf.vf_build(V, F, 1e-5, device=-1, evaluator=vf.VF_EVAL_DEVICE)
    assert e.value.code == vf.VF_EINVAL


def test_insolation_sum_finite_disk_equals_oracle():
    """vf_insolation_sum (finite solar disk as a sum over point sources)
    equals the oracle's insolation_disk on the same sources (cap crater, where
    the disk straddles the rim shadow for some facets)."""
    V, F = sg.cfg1_mesh()
    M = vf.ViewFactorMatrix.build(V, F, 1e-5, device=-1)
    S = oracle.Scene(V, F)
    suns = sg.sun_dirs(10.0, 2)
    dirs, w = sg.sun_disk_points(suns, radius=0.02, P=12)
    Qp = M.insolation_sum(dirs, w)
    Qo = oracle.insolation_disk(S, dirs, w)
    np.testing.assert_allclose(Qp, Qo, rtol=0, atol=1e-12)
    frac = Qp / np.maximum(M.insolation(suns), 1e-300)
    pen = (Qp > 0) & (Qp < M.insolation(suns) * 0.95)
    assert pen.sum() > 0                         # penumbra facets exist at this disk size


def test_octree_permutation_and_blocks_match_oracle(tmp_path):
    """Octree on a closed bilobed body: the product's permutation
    equals the oracle's octree (reading A1 in 3D), and its densified F-hat
    matches the oracle's exact F within 10 tol."""
    V, F = sg.bilobed_body_mesh(600)
    S = oracle.Scene(V, F, orient_up=False)
    M = vf.ViewFactorMatrix.build(V, F, 1e-5, device=-1, orient_up=0, tree=vf.VF_TREE_OCT, min_block=2048)
    p = str(tmp_path / "o.hvfm")
    M.save(p)
    H = read_hvfm(p)
    _, perm = hm.octree(S.x, 16, 16)
    assert np.array_equal(H["perm"], perm)
    Fd = S.F_dense()
    assert np.count_nonzero(Fd) > 0
    assert np.linalg.norm(densify(H) - Fd) / np.linalg.norm(Fd) <= 1e-4
