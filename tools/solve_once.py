"""Dev tool: one cfg2 thermal solve (64 suns) for profiling."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_07632_b200 as vf
import scenegen as sg
k = int(os.environ.get("K", "64"))
M = vf.ViewFactorMatrix.build(*sg.cfg2_mesh(), 1e-5)
Q = np.asfortranarray(M.insolation(sg.sun_dirs(5.0, 64), 1365.0)[:, :k])
alb, emi = np.full(M.N, 0.12), np.full(M.N, 0.95)
T = np.empty((M.N, k), order="F")
for _ in range(2):
    M.solve_thermal(Q, alb, emi, T, iters=200, tol=1e-10)
print("ok", M.stats())
