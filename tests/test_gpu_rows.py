"""GPU tests of the block-row (ROWS) mode, through
the C ABI, against the FP64 oracle on the SAME blocks (oracle/hmatrix.py's
F-hat, loaded with vf_load):

  * shards on one GPU, no communicator: each rank's vf_matvec writes exactly
    its rows of Y; the ranks' outputs sum to the oracle's Alg. 5 apply;
  * world = 1 with a real NCCL communicator: the per-iteration path (M_STEP
    launch, pack, ncclAllGather, unpack, decide) reproduces the oracle's
    Jacobi / thermal solves with identical iteration counts.

Only one GPU is available to this build, so multi-rank NCCL runs are not
exercised here; the multi-rank exchange protocol is covered by the gloo test
in tests/test_rows_shard.py."""
import numpy as np
import pytest

import oracle
import oracle.hmatrix as hm
import paper_2209_07632_b200 as vf
import scenegen as sg
from tests.test_gpu_parity import dev, empty, host, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def scenes():
    out = {}
    for name, (V, F) in {"cap": sg.cfg1_mesh(), "rough": sg.rough_small_mesh(24, amp=0.05)}.items():
        S = oracle.Scene(V, F)
        Fd = S.F_dense()
        H = hm.compress(S.x, Fd, 1e-6, min_size=2048)
        out[name] = (S, Fd, H)
    return out


def _load(H, tmp_path_factory, tag):
    p = str(tmp_path_factory.mktemp("rows") / f"{tag}.hvfm")
    hm.write_hvfm(H, p)
    return vf.ViewFactorMatrix.load(p, device=0)


@pytest.mark.parametrize("which", ["cap", "rough"])
@pytest.mark.parametrize("k", [1, 2, 64])
def test_shards_on_one_gpu_sum_to_full_apply(scenes, tmp_path_factory, which, k):
    S, Fd, H = scenes[which]
    X = sg.random_rhs(S.N, k)
    Yref = hm.hmatvec(H, X)
    world = 3
    acc = np.zeros_like(Yref)
    for g in range(world):
        M = _load(H, tmp_path_factory, f"{which}{k}_{g}")
        M.shard_rows(g, world)
        lo, hi = M.row_range()
        Y = empty(S.N, k)
        M.matvec(dev(X), Y)
        y = host(Y)
        own = np.zeros(S.N, bool)
        own[H.perm[lo:hi]] = True
        assert not np.any(y[~own])
        acc += y
    assert rel(acc, Yref) <= 1e-12


@pytest.fixture(scope="module")
def nccl_id():
    return vf.vf_get_nccl_id()


def _rows1(H, tmp_path_factory, tag):
    M = _load(H, tmp_path_factory, tag)
    M.shard_rows(0, 1)
    M.comm_init(0, 1, vf.vf_get_nccl_id())
    return M


@pytest.mark.parametrize("which", ["cap", "rough"])
@pytest.mark.parametrize("k", [1, 64])
def test_rows_world1_radiosity_and_matvec(scenes, tmp_path_factory, which, k):
    S, Fd, H = scenes[which]
    M = _rows1(H, tmp_path_factory, f"r{which}{k}")
    rng = np.random.default_rng(5)
    E = np.asfortranarray(1000 * rng.random((S.N, k)))
    rho = (0.05 + 0.9 * rng.random(S.N)) / max(1.0, np.abs(Fd).sum(1).max())
    B0, _, it0, _ = oracle.jacobi(lambda X: hm.hmatvec(H, X), E, rho, 1e-13, 200)
    B = empty(S.N, k)
    M.solve_radiosity(dev(E), dev(rho), B, iters=200, tol=1e-13)
    assert M.stats()["iters1"] == it0
    assert rel(host(B), B0) <= 1e-12
    X = sg.random_rhs(S.N, k)
    Y = empty(S.N, k)
    M.matvec(dev(X), Y)
    assert rel(host(Y), hm.hmatvec(H, X)) <= 1e-12


@pytest.mark.parametrize("k", [1, 64])
def test_rows_world1_thermal(scenes, tmp_path_factory, k):
    S, Fd, H = scenes["cap"]
    M = _rows1(H, tmp_path_factory, f"t{k}")
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


def test_rows_noconv_and_solve_needs_comm(scenes, tmp_path_factory):
    S, Fd, H = scenes["cap"]
    M = _load(H, tmp_path_factory, "nocomm")
    M.shard_rows(1, 2)
    E = np.asfortranarray(np.ones((S.N, 1)))
    with pytest.raises(vf.VFError) as e:
        M.solve_radiosity(dev(E), dev(np.full(S.N, 0.1)), empty(S.N, 1), iters=10, tol=1e-12)
    assert e.value.code == vf.VF_EINVAL
    M1 = _rows1(H, tmp_path_factory, "nc1")
    B0, *_ = oracle.jacobi(lambda X: hm.hmatvec(H, X), E, np.full(S.N, 0.9), 1e-300, 3)
    B = empty(S.N, 1)
    with pytest.raises(vf.VFError) as e:
        M1.solve_radiosity(dev(E), dev(np.full(S.N, 0.9)), B, iters=3, tol=1e-300)
    assert e.value.code == vf.VF_ENOCONV
    assert M1.stats()["iters1"] == 3
    assert rel(host(B), B0) <= 1e-12


@pytest.mark.parametrize("world,kp,k", [(2, 1, 1), (3, 2, 2), (5, 16, 13), (8, 1, 1), (8, 64, 64)])
@pytest.mark.parametrize("iter0", [0, 3])
def test_rows_exchange_kernels_at_world_above_one(world, kp, k, iter0):
    """The ROWS exchange kernels (pack, unpack, decide) at world = 2..8, all
    ranks emulated on this one GPU with the allgather done as device copies
    (vf_selftest_rows_exchange): after the exchange every rank holds every
    rank's own rows, and all ranks reach the same residuals (sum over ranks in
    rank order of each rank's CTA partials summed in CTA order, over ||E||),
    iteration count and stop flag -- the protocol of tests/test_rows_shard.py."""
    rng = np.random.default_rng(world * 100 + kp)
    N = 1000 + world * 37
    cuts = np.sort(rng.choice(np.arange(1, N), world - 1, replace=False))
    bounds = np.concatenate([[0], cuts, [N]]).astype(np.int64)
    xrank = rng.random((world, N, kp))
    nblk = 7
    part = rng.random((world, kp, nblk)) * 1e-6
    enorm2 = rng.random(k) + 0.5
    for tol in (1e-12, 1.0):
        xout, resid, it, dn = vf.vf_selftest_rows_exchange(bounds, xrank, part, enorm2, tol, 10, iter0)
        want = np.zeros((N, kp))
        for g in range(world):
            want[bounds[g]:bounds[g + 1]] = xrank[g, bounds[g]:bounds[g + 1]]
        for g in range(world):
            assert np.array_equal(xout[g], want), g
        tot = np.zeros(kp)
        for g in range(world):                       # rank order; each rank's partials in CTA order
            s = np.zeros(kp)
            for b in range(nblk):
                s = s + part[g, :, b]
            tot = tot + s
        r = np.sqrt(tot[:k]) / np.sqrt(enorm2)
        np.testing.assert_allclose(resid, r, rtol=1e-15, atol=0)
        assert np.all(it == iter0 + 1)
        assert np.all(dn == (1 if tol == 1.0 else 0))
