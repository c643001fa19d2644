"""Time-dependent thermal model: Alg. 6 with a per-facet Crank-Nicolson
subsurface column (§5.2).  TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py): plain numpy, FP64, written from the paper's text.

Alg. 6, for every facet i and step n:
    Q_refl^(n+1) = F diag(alpha) [Q_dir^(n+1) + Q_refl^(n)]
    Q_IR^(n+1)   = F [Q_rad^(n) + (I - diag eps) Q_IR^(n)]
    Q_abs^(n+1)  = (I - diag alpha)(Q_dir^(n+1) + Q_refl^(n+1)) + diag(eps) Q_IR^(n+1)
    Q_rad        = eps sigma T^4
initialised with Q_abs^(0) = (I - diag alpha) Q_dir^(0) + H, Q_refl^(0) =
Q_IR^(0) = 0, Q_rad^(0) = Q_abs^(0).  Negative fluxes after each product are
clamped to 0 (reading A12, as in the solves).  H (the subsurface heat flux,
P:115) enters Q_abs^(0) and the column's lower boundary.

The subsurface column ("a Crank-Nicolson method with a linearized
upper boundary condition"; the scheme's details are deferred to Schorghofer
2017, which is not in PAPER.md -- reading A27 in DESIGN.md fixes them):
  nodes z_0 = 0 (surface, no heat capacity) and z_1 < ... < z_M with layer
  thicknesses d_j = z_j - z_{j-1} = d_1 r^(j-1) summing to the depth Dz;
  control volumes h_j = (d_j + d_{j+1})/2 (j < M), h_M = d_M / 2;
  rho_c h_j dT_j/dt = k (T_{j+1}-T_j)/d_{j+1} - k (T_j-T_{j-1})/d_j   (1 <= j < M)
  rho_c h_M dT_M/dt = H - k (T_M - T_{M-1})/d_M                        (bottom flux H)
  surface balance  0 = Q_abs - eps sigma T_0^4 + k (T_1 - T_0)/d_1,
  the interior time-centred (Crank-Nicolson, theta = 1/2), the capacity-free
  surface balance imposed at the new level with Q_abs^(n+1) and T_0^4
  linearised about T_0^(n): T^4 ~ (T^n)^4 + 4 (T^n)^3 (T - T^n) (T_0^(n),
  which enters the node-1 flux of the old level, balanced Q_abs^(n): both
  absorbed fluxes drive the step).  One (M+1) x (M+1) tridiagonal
  solve per facet per step (Thomas algorithm).
"""
from __future__ import annotations

import numpy as np

from . import SIGMA_SB


def layer_grid(M: int, depth: float, ratio: float = 1.2):
    """Node depths z_0..z_M (z_0 = 0) with geometric layer thicknesses."""
    d1 = depth * (ratio - 1.0) / (ratio ** M - 1.0) if ratio != 1.0 else depth / M
    d = d1 * ratio ** np.arange(M)
    return np.concatenate([[0.0], np.cumsum(d)])


def cn_step(T, Qnew, dt, z, k, rho_c, emiss, H=0.0):
    """One Crank-Nicolson step of the columns.  T: (M+1, ...) node
    temperatures at step n (any trailing shape: facets x scenarios); Qnew:
    absorbed flux at the surface at step n+1 (trailing shape); emiss and H
    broadcast over the trailing shape.  Returns the new (M+1, ...) array."""
    T = np.asarray(T, dtype=np.float64)
    M = T.shape[0] - 1
    d = np.diff(z)                                       # d_1..d_M
    h = np.empty(M + 1)
    h[0] = 0.0
    h[1:M] = 0.5 * (d[:-1] + d[1:])
    h[M] = 0.5 * d[-1]
    es = np.asarray(emiss, dtype=np.float64) * SIGMA_SB
    T0 = T[0]
    R = es * T0 ** 4                                     # eps sigma T0^4 at time n
    dR = 4.0 * es * T0 ** 3                              # its derivative
    # unknowns T^(n+1); rows: surface (0), interior (1..M-1), bottom (M)
    a = np.zeros_like(T)                                 # sub-diagonal (coefficient of T_{j-1})
    b = np.zeros_like(T)                                 # diagonal
    c = np.zeros_like(T)                                 # super-diagonal
    r = np.zeros_like(T)
    g1 = k / d[0]
    # surface at n+1:  0 = Qnew - R - dR (T0 - T0^n) + g1 (T1 - T0)
    b[0] = dR + g1
    c[0] = -g1
    r[0] = Qnew - R + dR * T0
    for j in range(1, M + 1):
        gm = k / d[j - 1]                                # conductance to the node above
        cap = rho_c * h[j] / dt
        if j < M:
            gp = k / d[j]
            flux_old = gp * (T[j + 1] - T[j]) - gm * (T[j] - T[j - 1])
            a[j] = -0.5 * gm
            b[j] = cap + 0.5 * (gm + gp)
            c[j] = -0.5 * gp
            r[j] = cap * T[j] + 0.5 * flux_old
        else:
            flux_old = H - gm * (T[j] - T[j - 1])
            a[j] = -0.5 * gm
            b[j] = cap + 0.5 * gm
            r[j] = cap * T[j] + 0.5 * flux_old + 0.5 * H
    # Thomas algorithm (textbook forward elimination / back substitution)
    cp = np.zeros_like(T)
    dp = np.zeros_like(T)
    cp[0] = c[0] / b[0]
    dp[0] = r[0] / b[0]
    for j in range(1, M + 1):
        den = b[j] - a[j] * cp[j - 1]
        cp[j] = c[j] / den
        dp[j] = (r[j] - a[j] * dp[j - 1]) / den
    out = np.empty_like(T)
    out[M] = dp[M]
    for j in range(M - 1, -1, -1):
        out[j] = dp[j] - cp[j] * out[j + 1]
    return out


def simulate(apply, Qdir_steps, albedo, emiss, z, k, rho_c, dt, T_init, H=0.0, clamp=True):
    """Alg. 6 over the columns of Qdir_steps (a sequence of N x s arrays, one
    per step n = 0..S-1; s independent scenarios).  apply(X) = F X.  The
    columns start from the uniform profile T_init (N x s surface-and-depth
    temperature).  Returns dict of per-step surface T (S, N, s) and the final
    fluxes."""
    a = np.asarray(albedo, dtype=np.float64).reshape(-1)[:, None]
    e = np.asarray(emiss, dtype=np.float64).reshape(-1)[:, None]
    Q0 = np.asarray(Qdir_steps[0], dtype=np.float64)
    N, s = Q0.shape
    Qabs = (1.0 - a) * Q0 + H
    Qrefl = np.zeros((N, s))
    Qir = np.zeros((N, s))
    Qrad = Qabs.copy()
    M = z.size - 1
    T = np.broadcast_to(np.asarray(T_init, dtype=np.float64), (N, s)).copy()
    prof = np.repeat(T[None], M + 1, axis=0)            # (M+1, N, s)
    Ts = [prof[0].copy()]
    for n in range(1, len(Qdir_steps)):
        Qd = np.asarray(Qdir_steps[n], dtype=np.float64)
        Y = apply(np.concatenate([a * (Qd + Qrefl), Qrad + (1.0 - e) * Qir], axis=1))
        if clamp:
            Y = np.maximum(Y, 0.0)
        Qrefl_new, Qir_new = Y[:, :s], Y[:, s:]
        Qabs_new = (1.0 - a) * (Qd + Qrefl_new) + e * Qir_new
        prof = cn_step(prof, Qabs_new, dt, z, k, rho_c, e, H)
        Qrefl, Qir, Qabs = Qrefl_new, Qir_new, Qabs_new
        Qrad = e * SIGMA_SB * prof[0] ** 4
        Ts.append(prof[0].copy())
    return dict(T=np.asarray(Ts), Qrefl=Qrefl, Qir=Qir, Qabs=Qabs, profile=prof)
