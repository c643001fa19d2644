"""Dev tool: run one cfg2 thermal solve with VF_TRACE_FILE and summarise the
per-CTA phase timestamps (globaltimer) of the persistent kernel."""
import os, sys, struct
import numpy as np
path = sys.argv[1] if len(sys.argv) > 1 else "/tmp/vf_trace.bin"
if "--run" in sys.argv:
    os.environ["VF_TRACE_FILE"] = path
    if os.path.exists(path):
        os.remove(path)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import paper_2209_07632_b200 as vf
    import scenegen as sg
    V, F = sg.cfg2_mesh()
    M = vf.ViewFactorMatrix.build(V, F, 1e-5)
    N = M.N
    Q = M.insolation(sg.sun_dirs(5.0, 64), 1365.0)
    k = int(os.environ.get("K", "64"))
    Q = np.asfortranarray(Q[:, :k])
    alb, emi = np.full(N, 0.12), np.full(N, 0.95)
    T = np.empty((N, k), order="F")
    for _ in range(3):
        M.solve_thermal(Q, alb, emi, T, iters=200, tol=1e-10)
buf = open(path, "rb").read()
off = 0
runs = []
while off < len(buf):
    grid, tit, kp, grouped = struct.unpack_from("<4i", buf, off)
    off += 16
    a = np.frombuffer(buf, dtype=np.uint64, count=tit * 5 * grid, offset=off).reshape(tit, 5, grid).astype(np.int64)
    off += a.nbytes
    runs.append((grid, kp, grouped, a))
grid, kp, grouped, a = runs[-1]
print(f"last launch: grid {grid} kp {kp} grouped {grouped}")
t0 = a[0, 0].min()
for it in range(a.shape[0]):
    if a[it, 0].max() == 0:
        break
    st = a[it, 0] - t0
    p1 = a[it, 1] - a[it, 0]
    b1 = a[it, 2] - a[it, 1]
    p2 = a[it, 3] - a[it, 2]
    b2 = a[it, 4] - a[it, 3]
    it_len = a[it, 4].max() - a[it, 0].min()
    red = (a[it + 1, 0] - a[it, 4]) if it + 1 < a.shape[0] and a[it + 1, 0].max() > 0 else np.zeros(1)
    print(f"it {it:2d}: iter {it_len/1e3:7.1f} us | p1 work med {np.median(p1)/1e3:6.1f} max {p1.max()/1e3:6.1f} | "
          f"bar1 med {np.median(b1)/1e3:6.1f} | p2 work med {np.median(p2)/1e3:6.1f} max {p2.max()/1e3:6.1f} | "
          f"bar2 med {np.median(b2)/1e3:6.1f} min {b2.min()/1e3:6.1f} | red max {red.max()/1e3:5.1f}")
