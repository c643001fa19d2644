"""Pins of the oracle's time-dependent model (Alg. 6 + Crank-Nicolson column,
PAPER.md P:292-320) against things other than itself: a steady state,
exact energy conservation, the textbook periodic-flux solution of the heat
equation, an independently written explicit integrator, and the equilibrium
solver (Alg. 6's fixed point is the equilibrium of eq. 3d-equilbr).  CPU only."""
import math

import numpy as np
import pytest

import oracle
import oracle.timestep as ts
import scenegen as sg

SIG = oracle.SIGMA_SB


def test_layer_grid_geometric():
    z = ts.layer_grid(30, 2.5, 1.2)
    d = np.diff(z)
    assert z[0] == 0.0 and abs(z[-1] - 2.5) < 1e-12
    assert np.allclose(d[1:] / d[:-1], 1.2)


def test_cn_steady_state_is_kept():
    """Uniform T with eps sigma T^4 = Q_abs and no bottom flux: unchanged."""
    z = ts.layer_grid(20, 1.0)
    T = 210.0
    Q = 0.95 * SIG * T ** 4
    prof = np.full((21, 5), T)
    for _ in range(50):
        prof = ts.cn_step(prof, np.full(5, Q), 600.0, z, 0.01, 1.2e6, 0.95)
    assert np.abs(prof - T).max() < 1e-9


def test_cn_conserves_energy_without_radiation():
    """eps = 0, Q = 0, H = 0: sum_j h_j T_j is conserved (flux-conservative
    interior, zero top and bottom flux)."""
    z = ts.layer_grid(25, 1.0)
    d = np.diff(z)
    h = np.concatenate([0.5 * (d[:-1] + d[1:]), [0.5 * d[-1]]])
    rng = np.random.default_rng(1)
    prof = 200.0 + 30.0 * rng.random((26, 3))
    prof[0] = prof[1]                                   # a consistent surface node
    e0 = (h[:, None] * prof[1:]).sum(0)
    for _ in range(200):
        prof = ts.cn_step(prof, np.zeros(3), 3600.0, z, 0.02, 1.0e6, 0.0)
    assert np.allclose((h[:, None] * prof[1:]).sum(0), e0, rtol=1e-12)


def test_cn_periodic_flux_matches_textbook_amplitude_and_lag():
    """Semi-infinite solid driven by a surface flux Q0 cos(w t) (no radiation):
    T(0, t) = T_mean + Q0 / sqrt(k rho_c w) cos(w t - pi/4) (Carslaw & Jaeger)."""
    k, rc = 0.5, 1.0e6
    P = 86400.0
    w = 2 * math.pi / P
    skin = math.sqrt(2 * k / (rc * w))
    z = ts.layer_grid(80, 12 * skin, 1.05)
    dt = P / 400
    Q0 = 50.0
    prof = np.full((81, 1), 250.0)
    Ts, tt = [], []
    for n in range(1, 400 * 8 + 1):
        prof = ts.cn_step(prof, np.array([Q0 * math.cos(w * n * dt)]), dt, z, k, rc, 0.0)
        if n > 400 * 7:
            Ts.append(prof[0, 0])
            tt.append(n * dt)
    Ts, tt = np.array(Ts), np.array(tt)
    c = np.cos(w * tt - math.pi / 4)
    s_ = np.sin(w * tt - math.pi / 4)
    A = np.stack([np.ones_like(tt), c, s_], 1)
    coef, *_ = np.linalg.lstsq(A, Ts, rcond=None)
    amp = Q0 / math.sqrt(k * rc * w)
    assert abs(coef[1] - amp) < 0.01 * amp                # amplitude within 1 %
    assert abs(coef[2]) < 0.02 * amp                      # phase lag pi/4


def test_cn_matches_small_step_explicit_integrator():
    """One column from radiative equilibrium at Q = 300 W/m^2, then a flux step:
    CN at dt = 600 s (below the first layer's diffusion time) vs an explicit
    Euler of the same semi-discrete equations at a 1.5 s step with the exact
    (Newton-solved) surface balance, written here.  The linearised boundary
    lags a large jump by ~1 K at first; both agree once it has settled."""
    z = ts.layer_grid(15, 0.5, 1.2)
    d = np.diff(z)
    h = np.concatenate([0.5 * (d[:-1] + d[1:]), [0.5 * d[-1]]])
    k, rc, em = 0.01, 1.0e6, 0.95
    T00 = (300.0 / (em * SIG)) ** 0.25
    dt = 600.0
    for Qn, tol_all, tol_late in ((310.0, 0.1, 0.02), (400.0, 1.0, 0.05)):
        prof = np.full((16, 1), T00)
        cn = []
        for _ in range(100):
            prof = ts.cn_step(prof, np.array([Qn]), dt, z, k, rc, em)
            cn.append(prof[:, 0].copy())
        Te = np.full(16, T00)
        sub = 400
        hdt = dt / sub
        ex = []
        for n in range(100):
            for _ in range(sub):
                t0 = Te[0]
                for _ in range(4):
                    f = Qn - em * SIG * t0 ** 4 + k * (Te[1] - t0) / d[0]
                    t0 -= f / (-4 * em * SIG * t0 ** 3 - k / d[0])
                Te[0] = t0
                flux = k * np.diff(Te) / d
                dT = np.empty(15)
                dT[:-1] = (flux[1:] - flux[:-1]) / (rc * h[:-1])
                dT[-1] = (0.0 - flux[-1]) / (rc * h[-1])
                Te[1:] += hdt * dT
            ex.append(Te.copy())
        D = np.abs(np.array(cn) - np.array(ex))
        assert D.max() < tol_all and D[50:].max() < tol_late, (Qn, D.max(), D[50:].max())


@pytest.mark.slow
def test_alg6_constant_sun_converges_to_equilibrium():
    """Constant sun, no bottom flux: Alg. 6's fixed point is the equilibrium
    of eq. 3d-equilbr (Q_refl = F a (Q_dir + Q_refl), Q_IR = F[(1-a) Q_vis +
    Q_IR]), so the surface T approaches the equilibrium chain's T."""
    V, F = sg.cap_mesh(200, 40)
    S = oracle.Scene(V, F)
    Fd = S.F_dense()
    Q = S.insolation(sg.sun_dirs(30.0, 1), 1365.0)
    alb, emi = np.full(S.N, 0.12), np.full(S.N, 0.95)
    eq = oracle.thermal(lambda X: oracle.apply_dense(Fd, X), Q, alb, emi, 1e-12, 200)
    z = ts.layer_grid(10, 0.05, 1.2)
    out = ts.simulate(lambda X: oracle.apply_dense(Fd, X), [Q] * 400, alb, emi, z, 0.005, 1.0e5, 3600.0, 200.0)
    assert np.abs(out["T"][-1] - eq["T"]).max() < 0.5


def test_alg6_first_step_is_single_bounce():
    """Zero history: Q_refl^(1) = F diag(alpha) Q_dir^(1) and Q_IR^(1) =
    F Q_rad^(0) with Q_rad^(0) = Q_abs^(0) = (1 - alpha) Q_dir^(0)."""
    V, F = sg.cap_mesh(150, 30)
    S = oracle.Scene(V, F)
    Fd = S.F_dense()
    Q0 = S.insolation(sg.sun_dirs(20.0, 2), 1365.0)
    Q1 = S.insolation(sg.sun_dirs(25.0, 2), 1365.0)
    a = np.full(S.N, 0.3)
    z = ts.layer_grid(8, 0.1)
    out = ts.simulate(lambda X: oracle.apply_dense(Fd, X), [Q0, Q1], a, np.full(S.N, 0.9), z, 0.01, 1e6, 600.0, 200.0)
    np.testing.assert_allclose(out["Qrefl"], Fd @ (0.3 * Q1), rtol=1e-13, atol=1e-12)
    np.testing.assert_allclose(out["Qir"], Fd @ (0.7 * Q0), rtol=1e-13, atol=1e-12)
