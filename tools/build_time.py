"""Dev tool: time the product build of a cfg3-shaped terrain (n x n cells,
crater diameter scaled with n) and print vf_info; optionally save HVFM."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_07632_b200 as vf  # noqa: E402
import scenegen as sg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("n", type=int, nargs="+")
ap.add_argument("--tol", type=float, default=1e-5)
ap.add_argument("--device", type=int, default=0)
ap.add_argument("--evaluator", type=int, default=0)
ap.add_argument("--save", default=None)
a = ap.parse_args()
for n in a.n:
    V, F = sg.cfg3_mesh(n=n, crater_D=1000.0 * n / 256)
    t = time.time()
    M = vf.ViewFactorMatrix.build(V, F, a.tol, device=a.device, evaluator=a.evaluator)
    info = M.refresh()
    keys = ["N", "alg_bytes", "nnz_csr", "n_dense", "n_csr", "n_svd", "sum_rank", "max_rank", "active_rows",
            "visible_pairs", "build_seconds", "device_bytes"]
    print(json.dumps({"n": n, "wall_s": time.time() - t, **{k: info[k] for k in keys}}), flush=True)
    if a.save:
        M.save(a.save.format(n=n))
