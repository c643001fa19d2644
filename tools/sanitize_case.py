"""Dev tool: a small case that launches every libvf kernel family once
(hot_kernel nrhs = 1 + batched + solve, k1p_kernel, res_kernel, bt_kernel,
bt_tc_kernel, the ROWS exchange kernels, Alg. 6 kernels) -- for compute-sanitizer runs
(one --tool per gpurun call)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2209_07632_b200 as vf  # noqa: E402
import scenegen as sg  # noqa: E402

V, F = sg.cap_mesh(250, 40)
M = vf.ViewFactorMatrix.build(V, F, 1e-5, device=0)
N = M.N
for k in (1, 2, 4, 16, 64):
    X = torch.from_numpy(np.ascontiguousarray(sg.random_rhs(N, k).T)).cuda().T
    Y = torch.empty((k, N), dtype=torch.float64, device="cuda").T
    M.matvec(X, Y)
os.environ["VF_NO_RESIDENT"] = "1"
M2 = vf.ViewFactorMatrix.build(V, F, 1e-5, device=0)
del os.environ["VF_NO_RESIDENT"]
for k in (16, 128):
    X = torch.from_numpy(np.ascontiguousarray(sg.random_rhs(N, k).T)).cuda().T
    Y = torch.empty((k, N), dtype=torch.float64, device="cuda").T
    M2.matvec(X, Y)
os.environ["VF_K1_KERNEL"] = "pipe"                  # k1p_kernel (selected at upload)
M3 = vf.ViewFactorMatrix.build(V, F, 1e-5, device=0)
del os.environ["VF_K1_KERNEL"]
X = torch.from_numpy(np.ascontiguousarray(sg.random_rhs(N, 1).T)).cuda().T
Y = torch.empty((1, N), dtype=torch.float64, device="cuda").T
M3.matvec(X, Y)
os.environ["VF_NO_RESIDENT"] = "1"                  # FP32 streamed tiles on tcgen05 (bt_tc_kernel)
M4 = vf.ViewFactorMatrix.build(V, F, 1e-5, device=0, dtype=vf.VF_F32)
del os.environ["VF_NO_RESIDENT"]
X = torch.from_numpy(np.ascontiguousarray(sg.random_rhs(N, 128).T)).cuda().float().T
Y = torch.empty((128, N), dtype=torch.float32, device="cuda").T
M4.matvec(X, Y)
Q = M.insolation(sg.sun_dirs(10.0, 3), 1365.0)
T = np.empty((N, 3), order="F")
M.solve_thermal(np.asfortranarray(Q), np.full(N, 0.12), np.full(N, 0.95), T, iters=50, tol=1e-10)
st = vf.TimeStepper(M, np.full(N, 0.12), np.full(N, 0.95), np.asfortranarray(Q[:, :1]),
                    np.full((N, 1), 200.0, order="F"), layers=8, depth=0.2)
st.step(np.asfortranarray(Q[:, :1]), 600.0)
st.close()
b = np.array([0, 300, 700, 1000], dtype=np.int64)
vf.vf_selftest_rows_exchange(b, np.random.rand(3, 1000, 2), np.random.rand(3, 2, 4), np.ones(2), 1e-9, 5, 0)
torch.cuda.synchronize()
print("sanitize case ok")
