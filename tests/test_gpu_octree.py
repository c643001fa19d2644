"""GPU parity on a closed body with the octree (NEXT-3; PAPER.md P:213-214,
P:256, P:540-547 -- the 67P shape model is replaced by the synthetic bilobed
body of scenegen): same blocks vs the oracle's Alg. 5 (<= 1e-12), product
F-hat vs the oracle's exact F (<= 10 tol), thermal equilibrium vs the
oracle's chain on the exact F."""
import numpy as np
import pytest

import oracle
import oracle.hmatrix as hm
import paper_2209_07632_b200 as vf
import scenegen as sg

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64).T)).cuda().T


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.fixture(scope="module")
def body():
    V, F = sg.bilobed_body_mesh(1200)
    S = oracle.Scene(V, F, orient_up=False)
    return V, F, S, S.F_dense()


@pytest.mark.parametrize("k", [1, 4, 64])
def test_octree_same_blocks(body, tmp_path, k):
    V, F, S, Fd = body
    H = hm.compress(S.x, Fd, 1e-6, min_size=2048, tree="oct")
    p = str(tmp_path / "oct.hvfm")
    hm.write_hvfm(H, p)
    M = vf.ViewFactorMatrix.load(p, device=0)
    X = sg.random_rhs(S.N, k, seed=7)
    Y = torch.empty((k, S.N), dtype=torch.float64, device="cuda").T
    M.matvec(dev(X), Y)
    assert rel(Y.cpu().numpy(), hm.hmatvec(H, X)) <= 1e-12


def test_octree_product_build_and_thermal(body):
    V, F, S, Fd = body
    M = vf.ViewFactorMatrix.build(V, F, 1e-5, device=0, orient_up=0, tree=vf.VF_TREE_OCT, min_block=2048)
    X = sg.random_rhs(S.N, 3, seed=8)
    Y = torch.empty((3, S.N), dtype=torch.float64, device="cuda").T
    M.matvec(dev(X), Y)
    assert rel(Y.cpu().numpy(), Fd @ X) <= 1e-4
    suns = np.array([[0.3, 0.2, 0.93]])
    suns /= np.linalg.norm(suns)
    Q = S.insolation(suns)
    np.testing.assert_array_equal(M.insolation(suns), Q)
    alb, emi = np.full(S.N, 0.12), np.full(S.N, 0.95)
    ref = oracle.thermal(lambda Z: oracle.apply_dense(Fd, Z), Q, alb, emi, 1e-10, 100)
    T = np.empty((S.N, 1), order="F")
    M.solve_thermal(np.asfortranarray(Q), alb, emi, T, iters=100, tol=1e-10)
    assert rel(T, ref["T"]) <= 1e-4
