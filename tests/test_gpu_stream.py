"""GPU parity of the nrhs = 1 chunk-stream kernel (vf_stream.cu,
stream_k1_kernel: cp.async.bulk staging, 16-bit CSR column offsets,
phase-1 parts) against the FP64 oracle's Alg. 5 on the same blocks, and
against the row-segment kernel it replaces.  Forced layouts (env, read at
upload): VF_P1_PART (V rows per phase-1 item -> multi-part groups combined by
the last part), VF_U16_SPAN (span of a 16-bit CSR run -> many runs per row),
VF_NO_STREAM (no stream layout: the round-1 hot_kernel<T,1,1>).  The stream
kernel is opt-in (VF_K1_KERNEL=stream, read at upload): the
tests of it set that variable."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import oracle.hmatrix as hm
import paper_2209_07632_b200 as vf
import scenegen as sg

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(autouse=True)
def _stream_kernel(request, monkeypatch):
    if "row_kernel" not in request.node.name:
        monkeypatch.setenv("VF_K1_KERNEL", "stream")


def dev(a, dtype=np.float64):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=dtype).T)).cuda().T


def empty(N, k=1, dtype=torch.float64):
    return torch.empty((k, N), dtype=dtype, device="cuda").T


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.fixture(scope="module")
def meshes():
    out = {}
    for name, (V, F) in {"cap": sg.cfg1_mesh(), "rough": sg.rough_small_mesh(24, amp=0.05),
                         "terrain": sg.cfg3_mesh(n=24, crater_D=1000.0 * 24 / 256)}.items():
        S = oracle.Scene(V, F)
        out[name] = (V, F, S, S.F_dense())
    return out


def _load(H, tmp_path, tag):
    p = str(tmp_path / f"{tag}.hvfm")
    hm.write_hvfm(H, p)
    return vf.ViewFactorMatrix.load(p, device=0)


@pytest.mark.parametrize("which,eps,min_size", [("cap", 1e-5, 16384), ("cap", 1e-7, 2048),
                                                ("rough", 1e-5, 2048), ("terrain", 1e-5, 4096)])
def test_stream_same_blocks_f64(meshes, tmp_path, which, eps, min_size):
    V, F, S, Fd = meshes[which]
    H = hm.compress(S.x, Fd, eps, min_size=min_size)
    M = _load(H, tmp_path, f"{which}{eps}")
    info = M.refresh()
    assert info["stream_chunks"] > 0 and info["stream_payload_bytes"] > 0
    for seed in (3, 4):
        X = sg.random_rhs(S.N, 1, seed=seed)
        Y = empty(S.N)
        M.matvec(dev(X), Y)
        assert rel(Y.cpu().numpy(), hm.hmatvec(H, X)) <= 1e-12
    Y2 = empty(S.N)
    M.matvec(dev(X), Y2)
    assert torch.equal(Y, Y2)                    # fixed lane/part order: bitwise reproducible


def test_stream_same_blocks_f32(meshes, tmp_path):
    for which in ("cap", "rough"):
        V, F, S, Fd = meshes[which]
        H = hm.compress(S.x, Fd, 1e-5, dtype="f32", min_size=2048)
        M = _load(H, tmp_path, f"{which}f32")
        X = sg.random_rhs(S.N, 1).astype(np.float32).astype(np.float64)
        Y = empty(S.N, 1, torch.float32)
        M.matvec(dev(X, np.float32), Y)
        assert rel(Y.cpu().numpy().astype(np.float64), hm.hmatvec(H, X)) <= 1e-5


def test_stream_equals_row_segment_kernel(meshes):
    """Product-built F-hat: the stream kernel and the round-1 hot_kernel<T,1,1>
    (VF_NO_STREAM) apply the same blocks (different summation order)."""
    V, F, S, Fd = meshes["terrain"]
    M = vf.ViewFactorMatrix.build(V, F, 1e-5, device=0)
    os.environ["VF_NO_STREAM"] = "1"
    try:
        M0 = vf.ViewFactorMatrix.build(V, F, 1e-5, device=0)
    finally:
        del os.environ["VF_NO_STREAM"]
    assert M.refresh()["stream_chunks"] > 0 and M0.refresh()["stream_chunks"] == 0
    X = sg.random_rhs(S.N, 1, seed=9)
    Y, Y0 = empty(S.N), empty(S.N)
    M.matvec(dev(X), Y)
    M0.matvec(dev(X), Y0)
    assert rel(Y.cpu().numpy(), Y0.cpu().numpy()) <= 1e-13
    # and both against the exact F of the oracle within 10 tol
    assert rel(Y.cpu().numpy(), Fd @ X) <= 1e-4


_FORCED = r"""
import json, sys, numpy as np, torch
sys.path.insert(0, {root!r})
import oracle, oracle.hmatrix as hm, paper_2209_07632_b200 as vf, scenegen as sg
V, F = sg.cfg1_mesh()
S = oracle.Scene(V, F)
Fd = S.F_dense()
out = {{}}
for eps, ms in ((1e-5, 2048), (1e-7, 2048)):
    H = hm.compress(S.x, Fd, eps, min_size=ms)
    p = "/tmp/vf_forced_%g.hvfm" % eps
    hm.write_hvfm(H, p)
    M = vf.ViewFactorMatrix.load(p, device=0)
    X = sg.random_rhs(S.N, 1, seed=5)
    Y = torch.empty((1, S.N), dtype=torch.float64, device="cuda").T
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().T
    M.matvec(Xd, Y)
    Y2 = torch.empty_like(Y)
    M.matvec(Xd, Y2)
    R = hm.hmatvec(H, X)
    out[str(eps)] = dict(err=float(np.linalg.norm(Y.cpu().numpy() - R) / np.linalg.norm(R)),
                         same=bool(torch.equal(Y, Y2)), chunks=M.refresh()["stream_chunks"],
                         maxv=max(len(b.data[2]) for b in H.leaves() if b.kind == hm.SVD))
print(json.dumps(out))
"""


@pytest.mark.parametrize("env", [{"VF_P1_PART": "64"}, {"VF_U16_SPAN": "37"},
                                 {"VF_P1_PART": "32", "VF_U16_SPAN": "2"}])
def test_stream_forced_parts_and_runs(env):
    """Multi-part phase-1 groups (V columns cut into pieces of 64 or 32 rows,
    combined in part order by the last part) and CSR rows cut into many 16-bit
    runs: still <= 1e-12 vs the oracle's Alg. 5, and bitwise repeatable (the
    part counters reset themselves between launches)."""
    r = subprocess.run([sys.executable, "-c", _FORCED.format(root=ROOT)],
                       env=dict(os.environ, VF_K1_KERNEL="stream", **env),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    for eps, d in out.items():
        assert d["err"] <= 1e-12 and d["same"], (eps, d)
        assert d["chunks"] > 0
    assert any(d["maxv"] > 2 * int(env.get("VF_P1_PART", "1000000")) for d in out.values()) or "VF_P1_PART" not in env


def test_stream_column_split_bitwise(meshes, tmp_path):
    """2..8 columns on a large F-hat go column by column through the stream
    kernel (VF_MV_COLSPLIT forces the rule here): bitwise = separate applies."""
    V, F, S, Fd = meshes["rough"]
    H = hm.compress(S.x, Fd, 1e-5, min_size=2048)
    M = _load(H, tmp_path, "cs")
    X = sg.random_rhs(S.N, 4, seed=2)
    os.environ["VF_MV_COLSPLIT"] = "1"
    try:
        Y = empty(S.N, 4)
        M.matvec(dev(X), Y)
    finally:
        del os.environ["VF_MV_COLSPLIT"]
    for c in range(4):
        y = empty(S.N)
        M.matvec(dev(X[:, c:c + 1]), y)
        assert torch.equal(y[:, 0], Y[:, c])


_ROWK1 = r"""
import json, os, sys, numpy as np, torch
sys.path.insert(0, {root!r})
import oracle, oracle.hmatrix as hm, paper_2209_07632_b200 as vf, scenegen as sg
out = {{}}
for name, (V, F) in (("cap", sg.cfg1_mesh()), ("rough", sg.rough_small_mesh(24, amp=0.05))):
    S = oracle.Scene(V, F)
    H = hm.compress(S.x, S.F_dense(), 1e-6, min_size=2048)
    p = "/tmp/vf_rowk1_%s.hvfm" % name
    hm.write_hvfm(H, p)
    M = vf.ViewFactorMatrix.load(p, device=0)
    X = sg.random_rhs(S.N, 1, seed=5)
    Y = torch.empty((1, S.N), dtype=torch.float64, device="cuda").T
    M.matvec(torch.from_numpy(np.ascontiguousarray(X.T)).cuda().T, Y)
    R = hm.hmatvec(H, X)
    i = M.refresh()
    out[name] = dict(err=float(np.linalg.norm(Y.cpu().numpy() - R) / np.linalg.norm(R)),
                     k1=int(i["k1_payload_bytes"]), stream=int(i["stream_chunks"]))
print(json.dumps(out))
"""


@pytest.mark.parametrize("env", [{"VF_NO_STREAM": "1"}, {"VF_NO_STREAM": "1", "VF_U16_SPAN": "7"},
                                 {"VF_NO_STREAM": "1", "VF_K1_U32": "1"}])
def test_row_kernel_k1_u16_offsets(env):
    """The row-segment nrhs = 1 kernel (hot_kernel<T,1,1>, the stream layout
    off): 16-bit CSR offsets from per-run bases (forced short spans cut every
    merged CSR row into many runs), or 32-bit columns (VF_K1_U32): <= 1e-12
    vs the oracle's Alg. 5 on the same blocks."""
    r = subprocess.run([sys.executable, "-c", _ROWK1.format(root=ROOT)],
                       env={k: v for k, v in dict(os.environ, **env).items() if k != "VF_K1_KERNEL"},
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    for name, d in out.items():
        assert d["err"] <= 1e-12 and d["stream"] == 0, (name, d)
        assert (d["k1"] > 0) == ("VF_K1_U32" not in env), (name, d)
