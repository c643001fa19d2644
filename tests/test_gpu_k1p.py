"""GPU parity of the pipelined nrhs = 1 kernel (vf_device.cu k1p_kernel:
per-warp cp.async rings of 4-term chunks issued rounds ahead, one queue for
phase-1 part items and phase-2 rows, no grid barrier -- a row's X-sourced
runs first, its U_b runs over T rows after all phase-1 items finished)
against the FP64 oracle's Alg. 5 (oracle.hmatrix.hmatvec) on the same blocks,
and against the row-segment kernel hot_kernel<T,1,1>.

Forced layouts (env, read at upload): VF_P1_PART (V rows per phase-1 item ->
multi-part groups combined by the last part), VF_U16_SPAN (span of a 16-bit
CSR run -> many runs, rows with > 32 segments).  The kernel is selected with
VF_K1_KERNEL=pipe (or is the default when built with VF_K1_DEFAULT_PIPE)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CASE = r"""
import json, os, sys, numpy as np, torch
sys.path.insert(0, {root!r})
import oracle, oracle.hmatrix as hm, paper_2209_07632_b200 as vf, scenegen as sg
out = {{}}
meshes = (("cap", sg.cfg1_mesh(), 1e-5, 16384), ("cap7", sg.cfg1_mesh(), 1e-7, 2048),
          ("rough", sg.rough_small_mesh(24, amp=0.05), 1e-5, 2048),
          ("terrain", sg.cfg3_mesh(n=24, crater_D=1000.0 * 24 / 256), 1e-5, 4096))
for name, (V, F), eps, ms in meshes:
    S = oracle.Scene(V, F)
    for dt in ("f64", "f32"):
        if dt == "f32" and name not in ("cap", "rough"):
            continue
        H = hm.compress(S.x, S.F_dense(), eps, min_size=ms, dtype=dt)
        p = "/tmp/vf_k1p_%s_%s_%d.hvfm" % (name, dt, os.getpid())
        hm.write_hvfm(H, p)
        M = vf.ViewFactorMatrix.load(p, device=0)
        os.remove(p)
        tdt = torch.float64 if dt == "f64" else torch.float32
        errs, same = [], True
        for seed in (3, 4):
            X = sg.random_rhs(S.N, 1, seed=seed)
            if dt == "f32":
                X = X.astype(np.float32).astype(np.float64)
            Xd = torch.from_numpy(np.ascontiguousarray(X.T)).to("cuda", tdt).T
            Y = torch.empty((1, S.N), dtype=tdt, device="cuda").T
            M.matvec(Xd, Y)
            Y2 = torch.empty_like(Y)
            M.matvec(Xd, Y2)
            same = same and bool(torch.equal(Y, Y2))
            R = hm.hmatvec(H, X)
            errs.append(float(np.linalg.norm(Y.cpu().numpy().astype(np.float64) - R) / np.linalg.norm(R)))
        nsvd = sum(1 for b in H.leaves() if b.kind == hm.SVD)
        out[name + "_" + dt] = dict(err=max(errs), same=same, nsvd=nsvd, k1=int(M.refresh()["k1_payload_bytes"]))
print(json.dumps(out))
"""


def _run(env, kernel="pipe"):
    r = subprocess.run([sys.executable, "-c", _CASE.format(root=ROOT)],
                       env=dict({k: v for k, v in os.environ.items() if k != "VF_K1_KERNEL"},
                                VF_K1_KERNEL=kernel, **env),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("env", [{}, {"VF_P1_PART": "64"}, {"VF_U16_SPAN": "7"},
                                 {"VF_P1_PART": "32", "VF_U16_SPAN": "2"}])
def test_k1p_same_blocks(env):
    """<= 1e-12 (FP64) / <= 1e-5 (FP32) vs the oracle's Alg. 5 on the same
    blocks, with default and forced layouts (multi-part phase-1 groups; CSR
    rows cut into runs of span 7 or 2, i.e. rows of many more than 32
    segments, so the issuer crosses segment batches and rows mid-pipeline);
    bitwise repeatable (counters reset per launch, part counters self-reset)."""
    out = _run(env)
    assert any(d["nsvd"] > 0 for d in out.values())
    for name, d in out.items():
        bound = 1e-12 if name.endswith("f64") else 1e-5
        assert d["err"] <= bound and d["same"] and d["k1"] > 0, (name, d)


_VS_ROW = r"""
import json, os, sys, numpy as np, torch
sys.path.insert(0, {root!r})
import oracle, paper_2209_07632_b200 as vf, scenegen as sg
V, F = sg.cfg3_mesh(n=24, crater_D=1000.0 * 24 / 256)
S = oracle.Scene(V, F)
X = sg.random_rhs(S.N, 1, seed=9)
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().T
res = {{}}
for kern in ("pipe", "rows"):
    os.environ["VF_K1_KERNEL"] = kern                 # the nrhs = 1 kernel is chosen at upload
    M = vf.ViewFactorMatrix.build(V, F, 1e-5, device=0)
    assert M.refresh()["k1_kernel"] == (2 if kern == "pipe" else 0)
    Y = torch.empty((1, S.N), dtype=torch.float64, device="cuda").T
    M.matvec(Xd, Y)
    res[kern] = Y.cpu().numpy()[:, 0]
Fd = S.F_dense()
ex = Fd @ X[:, 0]
print(json.dumps(dict(d=float(np.linalg.norm(res["pipe"] - res["rows"]) / np.linalg.norm(res["rows"])),
                      ex=float(np.linalg.norm(res["pipe"] - ex) / np.linalg.norm(ex)))))
"""


def test_k1p_equals_row_kernel_on_product_build():
    """Product-built F-hat: the pipelined kernel and hot_kernel<T,1,1> apply the
    same blocks (different summation order: <= 1e-13), and both are within
    10 tol of the oracle's exact F."""
    r = subprocess.run([sys.executable, "-c", _VS_ROW.format(root=ROOT)],
                       env={k: v for k, v in os.environ.items() if k != "VF_K1_KERNEL"},
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["d"] <= 1e-13 and d["ex"] <= 1e-4, d


@pytest.mark.parametrize("env", [{}, {"VF_P1_PART": "64"}, {"VF_U16_SPAN": "7"},
                                 {"VF_P1_PART": "32", "VF_U16_SPAN": "2"}, {"VF_K1_ILV": "0"},
                                 {"VF_K1_PACK": "1"}, {"VF_K1_OVL": "1"},
                                 {"VF_K1_SMQ": "1"}, {"VF_K1_SMQ": "0"}, {"VF_K1_TL1": "0"}, {"VF_K1_TL1": "1"},
                                 {"VF_K1_SMQ": "1", "VF_K1_SMQ_NQ": "500", "VF_K1_SMQ_THR": "1e9"},
                                 {"VF_K1_SMQ": "1", "VF_K1_SMQ_NQ": "3", "VF_K1_SMQ_THR": "0.5"},
                                 {"VF_K1_SMQ": "1", "VF_K1_SMQ_THR": "1e9", "VF_K1_OVL": "1", "VF_P1_PART": "64"}])
def test_default_row_kernel_forced_layouts(env):
    """The default nrhs = 1 kernel (hot_kernel<T,1,1> with the register-prefetching
    row accumulator on the interleaved 16-bit layout) under the same forced
    layouts: multi-part phase-1 groups, CSR rows cut into runs of span 7 / 2
    (runs crossing rounds, rows of many segment batches, interleaved pieces of
    every size), the plain (non-interleaved) order, per-row packing and the
    barrier-free hand-over, and the per-SM row queues (VF_K1_SMQ: default
    queue count and pool; 500 queues with no pool, so most queues are only
    served by the end-of-kernel sweep; 3 queues with most rows in the pool, so
    most SMs own no queue; no pool with the barrier-free hand-over and
    multi-part phase 1), T-row gathers through L2 only / through L1
    (VF_K1_TL1): <= 1e-12 / 1e-5 vs the oracle's Alg. 5 on the same
    blocks, bitwise repeatable."""
    out = _run(env, kernel="rows")
    for name, d in out.items():
        bound = 1e-12 if name.endswith("f64") else 1e-5
        assert d["err"] <= bound and d["same"] and d["k1"] > 0, (name, d)


_SMQ = r"""
import json, os, sys, numpy as np, torch
sys.path.insert(0, {root!r})
import oracle, paper_2209_07632_b200 as vf, scenegen as sg
V, F = sg.cfg3_mesh(n=32, crater_D=1000.0 * 32 / 256)
S = oracle.Scene(V, F)
X = sg.random_rhs(S.N, 1, seed=11)
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().T
res = []
for env in ({{"VF_K1_SMQ": "0"}}, {{"VF_K1_SMQ": "1"}}, {{"VF_K1_SMQ": "1", "VF_K1_SMQ_NQ": "37", "VF_K1_SMQ_THR": "1.0"}},
            {{"VF_K1_SMQ": "1", "VF_K1_SMQ_NQ": "1000", "VF_K1_SMQ_THR": "1e9"}}):
    for k in ("VF_K1_SMQ", "VF_K1_SMQ_NQ", "VF_K1_SMQ_THR"):
        os.environ.pop(k, None)
    os.environ.update(env)                            # read at upload
    M = vf.ViewFactorMatrix.build(V, F, 1e-5, device=0)
    Y = torch.empty((1, S.N), dtype=torch.float64, device="cuda").T
    for _ in range(3):
        Y.zero_()
        M.matvec(Xd, Y)
    res.append(Y.cpu().numpy()[:, 0].copy())
ex = S.F_dense() @ X[:, 0]
print(json.dumps(dict(same=[bool(np.array_equal(res[0], r)) for r in res[1:]],
                      ex=float(np.linalg.norm(res[1] - ex) / np.linalg.norm(ex)))))
"""


def test_smq_bitwise_equals_global_queue():
    """Per-SM row queues change which warp sums a row and when, not how: the
    product-built configs[2]-recipe F-hat applied with the global LPT queue and
    with per-SM queues (default; 37 queues with a large pool; 1000 queues, no
    pool) gives bitwise equal Y, within 10 tol of the oracle's exact F."""
    r = subprocess.run([sys.executable, "-c", _SMQ.format(root=ROOT)],
                       env={k: v for k, v in os.environ.items() if not k.startswith("VF_K1_")},
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert all(d["same"]) and d["ex"] <= 1e-4, d
