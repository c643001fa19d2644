"""Dev tool: radiosity solves with k = 1..8 columns on a saved configs[2] F-hat,
column-split (VF_SOLVE_COLSPLIT=1) vs the persistent batched solve (=0):
wall time per solve (host-synchronised call), iterations, agreement."""
import os, sys, time, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2209_07632_b200 as vf  # noqa: E402
M = vf.ViewFactorMatrix.load(sys.argv[1], 0)
N = M.N
rng = np.random.default_rng(5)
rho = torch.full((N,), 0.12, dtype=torch.float64, device="cuda")
out = {}
for k in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8").split(",")]:
    E = torch.from_numpy(np.ascontiguousarray((1365.0 * rng.random((N, k))).T)).cuda().T
    res = {}
    for mode in ("1", "0"):
        os.environ["VF_SOLVE_COLSPLIT"] = mode
        B = torch.empty((k, N), dtype=torch.float64, device="cuda").T
        M.solve_radiosity(E, rho, B, iters=100, tol=1e-10)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            M.solve_radiosity(E, rho, B, iters=100, tol=1e-10)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        st = M.stats()
        res[mode] = (B.cpu().numpy(), min(ts), st["iters1"])
    d = float(np.linalg.norm(res["1"][0] - res["0"][0]) / np.linalg.norm(res["0"][0]))
    out[k] = dict(cols_ms=res["1"][1] * 1e3, batched_ms=res["0"][1] * 1e3, iters_cols=res["1"][2],
                  iters_batched=res["0"][2], rel_diff=d,
                  cols_ms_per_iter=res["1"][1] * 1e3 / max(1, res["1"][2]),
                  batched_ms_per_iter=res["0"][1] * 1e3 / max(1, res["0"][2]))
    print(k, json.dumps(out[k]), flush=True)
