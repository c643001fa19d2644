"""Block-row (ROWS) sharding of F-hat: host logic on
CPU.  Alg. 5 sums Y_I = sum_J F_IJ X_J per block row, so the
shards of a partition must (1) cover the tree rows exactly once, (2) each
hold exactly the full operator's rows in their range, and (3) reproduce the
single-process Jacobi solve when every iteration ends with an allgather of
the ranks' new rows plus their residual partial sums (the exchange the
device path performs with ncclAllGather).  (3) runs as a world_size-2 gloo
job.  No GPU needed: handles are host-only (device=-1) and the shards are
applied through the independent HVFM reader in tests/hvfm_io.py."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2209_07632_b200 as vf
import scenegen as sg
from tests.hvfm_io import densify, read_hvfm


def _meshes():
    return {"cap": sg.cap_mesh(300, 45), "rough": sg.rough_small_mesh(14)}


def _dense_of(M, path):
    M.save(str(path))
    return densify(read_hvfm(str(path)))


@pytest.mark.parametrize("which", ["cap", "rough"])
@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_partition_covers_rows_and_balances_bytes(which, world):
    V, F = _meshes()[which]
    M = vf.ViewFactorMatrix.build(V, F, 1e-5, device=-1)
    b = vf.vf_row_partition(M.h, world)
    assert b[0] == 0 and b[-1] == M.N and np.all(np.diff(b) >= 0)
    # balance: shard byte totals within one row's cost of the ideal
    tot = M.info["bytes_dense"] + M.info["bytes_csr"] + M.info["bytes_svd"]
    shares = []
    for g in range(world):
        S = vf.ViewFactorMatrix.build(V, F, 1e-5, device=-1)
        S.shard_rows(g, world)
        assert S.row_range() == (b[g], b[g + 1])
        shares.append(S.info["bytes_dense"] + S.info["bytes_csr"] + S.info["bytes_svd"])
    # SVD V factors are duplicated across ranks; everything else is split
    assert sum(shares) >= tot
    if world > 1 and M.info["n_svd"] == 0:
        assert max(shares) <= 1.25 * tot / world + 8 * M.N


@pytest.mark.parametrize("which", ["cap", "rough"])
@pytest.mark.parametrize("world", [2, 3])
def test_shards_hold_exactly_their_rows(which, world, tmp_path):
    V, F = _meshes()[which]
    M = vf.ViewFactorMatrix.build(V, F, 1e-5, device=-1)
    Ffull = _dense_of(M, tmp_path / "full.hvfm")
    perm = read_hvfm(str(tmp_path / "full.hvfm"))["perm"]
    acc = np.zeros_like(Ffull)
    for g in range(world):
        S = vf.ViewFactorMatrix.build(V, F, 1e-5, device=-1)
        S.shard_rows(g, world)
        lo, hi = S.row_range()
        Fg = _dense_of(S, tmp_path / f"s{g}.hvfm")
        own = np.zeros(M.N, bool)
        own[perm[lo:hi]] = True
        assert not np.any(Fg[~own]), "a shard stores rows outside its range"
        np.testing.assert_allclose(Fg[own], Ffull[own], rtol=1e-14, atol=1e-300)
        acc += Fg
    np.testing.assert_allclose(acc, Ffull, rtol=1e-14, atol=1e-300)


def test_shard_errors():
    V, F = _meshes()["cap"]
    M = vf.ViewFactorMatrix.build(V, F, 1e-5, device=-1)
    with pytest.raises(vf.VFError):
        vf.vf_shard_rows(M.h, 2, 2)
    M.shard_rows(0, 2)
    with pytest.raises(vf.VFError):
        vf.vf_shard_rows(M.h, 1, 2)          # sharded once
    with pytest.raises(vf.VFError) as e:      # no device copy -> no communicator
        vf.vf_comm_init(M.h, 0, 2, b"\0" * 128)
    assert e.value.code == vf.VF_ENODEV


# ------------------------------------------------------------ gloo, world 2

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rows_jacobi(Fg, own, E, rho, tol, iters):
    """The device protocol in plain numpy + gloo: local rows of Q = F B,
    B' = E + rho max(Q, 0) on own rows, per-column partial sum of (B'-B)^2
    over own rows; allgather (rows, partials); r = sqrt(sum in rank order) /
    ||E||; stop as in oracle.jacobi (reading R-JAC)."""
    import torch
    world = dist.get_world_size()
    nE = np.sqrt(np.sum(E * E, axis=0))
    B = E.copy()
    it = 0
    for it in range(1, iters + 1):
        Q = np.maximum(Fg[own] @ B, 0.0)
        Bn_own = E[own] + rho[own, None] * Q
        part = np.sum((Bn_own - B[own]) ** 2, axis=0)
        msg = torch.from_numpy(np.concatenate([Bn_own.ravel(), part]))
        sizes = [None] * world
        dist.all_gather_object(sizes, (int(own.sum()), msg.numel()))
        bufs = [torch.zeros(n, dtype=torch.float64) for _, n in sizes]
        dist.all_gather(bufs, msg)
        owns = [None] * world
        dist.all_gather_object(owns, np.flatnonzero(own))
        k = E.shape[1]
        tot = np.zeros(k)
        for g in range(world):
            a = bufs[g].numpy()
            rows = owns[g]
            B[rows] = a[:rows.size * k].reshape(rows.size, k)
            tot += a[rows.size * k:]
        r = np.where(nE > 0, np.sqrt(tot) / np.where(nE > 0, nE, 1.0), 0.0)
        if np.all(r <= tol):
            break
    return B, it


def _worker(rank, world, port, tmp, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        V, F = _meshes()["rough"]
        M = vf.ViewFactorMatrix.build(V, F, 1e-5, device=-1)
        M.shard_rows(rank, world)
        lo, hi = M.row_range()
        path = os.path.join(tmp, f"r{rank}.hvfm")
        M.save(path)
        H = read_hvfm(path)
        Fg = densify(H)
        own = np.zeros(M.N, bool)
        own[H["perm"][lo:hi]] = True
        E = sg.random_rhs(M.N, 3) * 100.0
        rho = np.full(M.N, 0.1)      # spectral radius of rho F ~ 0.73 on this mesh
        B, it = _rows_jacobi(Fg, own, E, rho, 1e-12, 200)
        np.save(os.path.join(tmp, f"B{rank}.npy"), B)
        out[rank] = it
    finally:
        dist.destroy_process_group()


def test_rows_jacobi_gloo_world2_matches_single_process(tmp_path):
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, str(tmp_path), out), nprocs=world, join=True)
    V, F = _meshes()["rough"]
    M = vf.ViewFactorMatrix.build(V, F, 1e-5, device=-1)
    Ffull = _dense_of(M, tmp_path / "full.hvfm")
    E = sg.random_rhs(M.N, 3) * 100.0
    rho = np.full(M.N, 0.1)      # spectral radius of rho F ~ 0.73 on this mesh
    Bref, _, it_ref, _ = oracle.jacobi(lambda X: Ffull @ X, E, rho, 1e-12, 200)
    assert it_ref < 200 and np.all(np.isfinite(Bref))
    for g in range(world):
        B = np.load(tmp_path / f"B{g}.npy")
        assert out[g] == it_ref
        np.testing.assert_allclose(B, Bref, rtol=1e-13, atol=0)
