"""Dev tool: per-CTA phase timestamps (globaltimer) of one vf_matvec on a
cfg3-shaped terrain (--cells n) with nrhs k: phase 1 / barrier / phase 2."""
import os
import struct
import sys
import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
path = "/tmp/vf_trace_mv.bin"
os.environ["VF_TRACE_FILE"] = path
if os.path.exists(path):
    os.remove(path)
import torch  # noqa: E402
import paper_2209_07632_b200 as vf  # noqa: E402
import scenegen as sg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1
fhat = sys.argv[3] if len(sys.argv) > 3 else None
V, F = sg.cfg3_mesh(n=n, crater_D=1000.0 * n / 256)
if fhat and os.path.exists(fhat):
    M = vf.ViewFactorMatrix.load(fhat, 0)
else:
    M = vf.ViewFactorMatrix.build(V, F, 1e-5)
    if fhat:
        M.save(fhat)
N = M.N
X = torch.from_numpy(np.ascontiguousarray(sg.random_rhs(N, k).T)).cuda().T
Y = torch.empty((k, N), dtype=torch.float64, device="cuda").T
for _ in range(3):
    M.matvec(X, Y)
torch.cuda.synchronize()
buf = open(path, "rb").read()
off, runs = 0, []
while off < len(buf):
    grid, tit, kp, grouped = struct.unpack_from("<4i", buf, off)
    off += 16
    a = np.frombuffer(buf, dtype=np.uint64, count=tit * 5 * grid, offset=off).reshape(tit, 5, grid).astype(np.int64)
    off += a.nbytes
    runs.append(a)
a = runs[-1][0]
t0 = a[0].min()
p1, b1, p2 = a[1] - a[0], a[2] - a[1], a[3] - a[2]
print(f"N {N} k {k}: total {(a[3].max() - t0) / 1e3:.1f} us | p1 med {np.median(p1) / 1e3:.1f} max {p1.max() / 1e3:.1f} | "
      f"bar med {np.median(b1) / 1e3:.1f} | p2 med {np.median(p2) / 1e3:.1f} max {p2.max() / 1e3:.1f} | "
      f"p2 end spread {(a[3].max() - a[3].min()) / 1e3:.1f} us")
