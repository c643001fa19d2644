"""GPU parity of the streamed-tile batched apply (bt_kernel: 16-row tiles,
[K][16] weights on the FP64 tensor cores) -- the nrhs > 8 path for an F-hat
beyond the resident shared-memory layout (configs[2]).  Forced here on small
meshes with VF_NO_RESIDENT (read at upload).  Same blocks as the oracle's
Alg. 5: relative L2 <= 1e-12; bitwise repeatable."""
import os

import numpy as np
import pytest

import oracle
import oracle.hmatrix as hm
import paper_2209_07632_b200 as vf
import scenegen as sg

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def handles(tmp_path_factory):
    out = []
    os.environ["VF_NO_RESIDENT"] = "1"
    try:
        for name, (V, F), eps, ms in (("cap", sg.cfg1_mesh(), 1e-6, 2048),
                                      ("terrain", sg.cfg3_mesh(n=24, crater_D=1000.0 * 24 / 256), 1e-5, 4096),
                                      ("rough", sg.rough_small_mesh(24, amp=0.05), 1e-5, 2048)):
            S = oracle.Scene(V, F)
            H = hm.compress(S.x, S.F_dense(), eps, min_size=ms)
            p = str(tmp_path_factory.mktemp("bt") / f"{name}.hvfm")
            hm.write_hvfm(H, p)
            M = vf.ViewFactorMatrix.load(p, device=0)
            assert M.refresh()["tiles"] > 0 and not M.refresh()["resident"]
            out.append((name, S, H, M))
    finally:
        del os.environ["VF_NO_RESIDENT"]
    return out


@pytest.mark.parametrize("k", [9, 16, 17, 32, 48, 64, 100, 128, 130, 256])
def test_tiles_same_blocks(handles, k):
    for name, S, H, M in handles:
        X = sg.random_rhs(S.N, k, seed=11 + k)
        Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().T
        Y = torch.empty((k, S.N), dtype=torch.float64, device="cuda").T
        M.matvec(Xd, Y)
        R = hm.hmatvec(H, X)
        assert np.linalg.norm(Y.cpu().numpy() - R) / np.linalg.norm(R) <= 1e-12, (name, k)
        Y2 = torch.empty_like(Y)
        M.matvec(Xd, Y2)
        assert torch.equal(Y, Y2)


@pytest.fixture(scope="module")
def handles_f32(tmp_path_factory):
    out = []
    os.environ["VF_NO_RESIDENT"] = "1"
    try:
        for name, (V, F), ms in (("cap", sg.cfg1_mesh(), 2048),
                                 ("terrain", sg.cfg3_mesh(n=24, crater_D=1000.0 * 24 / 256), 4096)):
            S = oracle.Scene(V, F)
            H = hm.compress(S.x, S.F_dense(), 1e-5, dtype="f32", min_size=ms)
            p = str(tmp_path_factory.mktemp("btf") / f"{name}.hvfm")
            hm.write_hvfm(H, p)
            M = vf.ViewFactorMatrix.load(p, device=0)
            assert M.refresh()["tiles"] > 0
            out.append((name, S, H, M))
    finally:
        del os.environ["VF_NO_RESIDENT"]
    return out


@pytest.mark.parametrize("k", [9, 64, 128, 130, 256])
def test_tiles_f32_tcgen05_3xtf32(handles_f32, k):
    """FP32 streamed tiles on the 5th-generation tensor cores (bt_tc_kernel:
    tcgen05.mma kind::tf32, TMEM accumulator, 3xTF32 split): <= 1e-5 vs the
    oracle's Alg. 5 of the same (FP32-rounded) blocks, bitwise repeatable.
    Opt-in (VF_TC=1): the default FP32 tile kernel is bt_kernel<float>."""
    os.environ["VF_TC"] = "1"
    try:
        _check_f32_tiles(handles_f32, k, seed=21 + k)
    finally:
        del os.environ["VF_TC"]


@pytest.mark.parametrize("k", [9, 16, 17, 32, 48, 64, 100, 128, 130, 256])
def test_tiles_f32_dmma(handles_f32, k):
    """FP32 streamed tiles on the FP64 tensor cores (bt_kernel<float>, the
    default FP32 wide-batch path: FP32 weights and XT rows staged in shared
    memory with the FP32 swizzles, widened to FP64 for DMMA m8n8k4, FP64
    accumulation, one rounding at the store): <= 1e-5 vs the oracle's Alg. 5
    of the same blocks (north_star FP32 tolerance), bitwise repeatable.  With
    exact products and FP64 sums the only errors are the FP32 roundings of T
    and Y, so it must also meet 1e-6."""
    _check_f32_tiles(handles_f32, k, seed=31 + k, tol=1e-6)


def _check_f32_tiles(handles_f32, k, seed, tol=1e-5):
    for name, S, H, M in handles_f32:
        X = sg.random_rhs(S.N, k, seed=seed).astype(np.float32).astype(np.float64)
        Xd = torch.from_numpy(np.ascontiguousarray(X.T.astype(np.float32))).cuda().T
        Y = torch.empty((k, S.N), dtype=torch.float32, device="cuda").T
        M.matvec(Xd, Y)
        R = hm.hmatvec(H, X)
        assert np.linalg.norm(Y.cpu().numpy().astype(np.float64) - R) / np.linalg.norm(R) <= tol, (name, k)
        Y2 = torch.empty_like(Y)
        M.matvec(Xd, Y2)
        assert torch.equal(Y, Y2)
