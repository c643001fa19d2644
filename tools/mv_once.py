"""Dev tool: repeated vf_matvec on a saved/built cfg3-shaped F-hat (for ncu)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2209_07632_b200 as vf  # noqa: E402
import scenegen as sg  # noqa: E402
n, k, fhat = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
if os.path.exists(fhat):
    M = vf.ViewFactorMatrix.load(fhat, 0)
else:
    V, F = sg.cfg3_mesh(n=n, crater_D=1000.0 * n / 256)
    M = vf.ViewFactorMatrix.build(V, F, 1e-5)
    M.save(fhat)
tdt = torch.float32 if M.refresh()["dtype"] == vf.VF_F32 else torch.float64
X = torch.from_numpy(np.ascontiguousarray(sg.random_rhs(M.N, k).T)).to("cuda", tdt).T
Y = torch.empty((k, M.N), dtype=tdt, device="cuda").T
for _ in range(4):
    M.matvec(X, Y)
torch.cuda.synchronize()
print("ok")
