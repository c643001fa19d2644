"""GPU parity of Alg. 6 time stepping (NEXT-1) through
the C ABI (vf_ts_create / vf_ts_step / vf_ts_get) against the oracle's
oracle/timestep.py on the same F-hat blocks (Alg. 5 apply of an oracle-built
HVFM): surface temperature of every step and the final fluxes <= 1e-10
relative (FP64), for one scenario (the nrhs = 1 stream kernel, two columns)
and for several scenarios stepped together (the batched kernels)."""
import math

import numpy as np
import pytest

import oracle
import oracle.hmatrix as hm
import oracle.timestep as ts
import paper_2209_07632_b200 as vf
import scenegen as sg

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cap(tmp_path_factory):
    V, F = sg.cfg1_mesh()
    S = oracle.Scene(V, F)
    Fd = S.F_dense()
    H = hm.compress(S.x, Fd, 1e-6, min_size=2048)
    p = str(tmp_path_factory.mktemp("ts") / "cap.hvfm")
    hm.write_hvfm(H, p)
    return S, H, p


@pytest.mark.parametrize("ns", [1, 3])
def test_alg6_matches_oracle(cap, ns):
    S, H, p = cap
    M = vf.ViewFactorMatrix.load(p, device=0)
    steps = 24
    qs = []
    for n in range(steps):                                   # sun circling at 12 deg, per-scenario phase
        suns = np.stack([sg.sun_dirs(12.0, 1, 2 * math.pi * (n / steps + 0.13 * c))[0] for c in range(ns)])
        qs.append(S.insolation(suns, 1365.0))
    alb = np.full(S.N, 0.12)
    emi = np.linspace(0.9, 0.97, S.N)
    T0 = np.full((S.N, ns), 180.0, order="F")
    kw = dict(layers=12, depth=0.3, ratio=1.2, k_th=0.008, rho_c=1.1e6, H=0.02)
    z = ts.layer_grid(kw["layers"], kw["depth"], kw["ratio"])
    dt = 1800.0
    ref = ts.simulate(lambda X: hm.hmatvec(H, X), qs, alb, emi, z, kw["k_th"], kw["rho_c"], dt, 180.0, H=kw["H"])
    st = vf.TimeStepper(M, alb, emi, np.asfortranarray(qs[0]), T0, **kw)
    Tn = np.empty((S.N, ns), order="F")
    for n in range(1, steps):
        st.step(np.asfortranarray(qs[n]), dt, Tn)
        assert np.linalg.norm(Tn - ref["T"][n]) / np.linalg.norm(ref["T"][n]) <= 1e-10, n
    Qr, Qi, Qa, Ts = (np.empty((S.N, ns), order="F") for _ in range(4))
    st.get(Qr, Qi, Qa, Ts)
    for a, b in ((Qr, ref["Qrefl"]), (Qi, ref["Qir"]), (Qa, ref["Qabs"]), (Ts, ref["T"][-1])):
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(b)
    st.close()


def test_alg6_device_buffers_and_steady_state(cap):
    """Device (torch) buffers, and a steady state: F = 0 facets in radiative
    equilibrium with constant flux keep their temperature."""
    S, H, p = cap
    M = vf.ViewFactorMatrix.load(p, device=0)
    alb, emi = np.full(S.N, 0.1), np.full(S.N, 0.95)
    Q = S.insolation(sg.sun_dirs(40.0, 1), 1365.0)
    Qd = torch.from_numpy(np.ascontiguousarray(Q.T)).cuda().T
    T0 = torch.full((1, S.N), 200.0, dtype=torch.float64, device="cuda").T
    st = vf.TimeStepper(M, alb, emi, Qd, T0, layers=8, depth=0.2)
    Tn = torch.empty((1, S.N), dtype=torch.float64, device="cuda").T
    for _ in range(5):
        st.step(Qd, 600.0, Tn)
    assert torch.isfinite(Tn).all() and (Tn > 0).all()
