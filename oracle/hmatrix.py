"""The paper's hierarchical compression and compressed MVP, step by step.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  PAPER.md = P:<line>.

  * quadtree            Alg. 2 with readings A1-A3
  * octree              its 3D analogue
  * estimate_rank       Alg. 3; numpy.linalg.svd supplies the
                        k-term truncated SVD (a library primitive); A5-A8
  * assemble            Alg. 4 dynamic programming over block
                        pairs; readings A4, A9-A11, A25
  * hmatvec             Alg. 5 recursive Y_I += F_IJ X_J
  * write_hvfm          flattens the leaves (Alg. 5 order) into the HVFM
                        container documented in include/vf.h so the GPU
                        path can apply exactly these blocks.

The source of every block is the oracle's exact F (eq. FF-def, Alg. 1
values), sliced; nothing here comes from the product library.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

ZERO, DENSE, CSR, SVD, SUB = 0, 1, 2, 3, 4
KIND_NAME = {ZERO: "zero", DENSE: "dense", CSR: "csr", SVD: "svd", SUB: "sub"}
NODE_OVERHEAD = 64   # bytes charged per Subdivided node (SPEC S:349 accounting)


# ------------------------------------------------------------------ Alg. 2

@dataclass
class Node:
    start: int                 # tree-order range [start, stop)
    stop: int
    depth: int
    children: list = field(default_factory=list)

    @property
    def size(self):
        return self.stop - self.start


def quadtree(xy: np.ndarray, max_depth: int = 16, min_leaf: int = 16):
    """Alg. 2.  Reading A1: split at x_mid, y_mid (step 3) with
    ties to the upper half; A2: one root holding all centroids; A3: stop at
    max_depth or |I| <= min_leaf.  Children in the order I1..I4 of step 4.
    Returns (root, perm) with perm[r] = original index at tree position r."""
    order = []

    def build(idx: np.ndarray, depth: int) -> Node:
        start = len(order)
        if depth >= max_depth or idx.size <= min_leaf:
            order.extend(np.sort(idx).tolist())
            return Node(start, len(order), depth)
        x, y = xy[idx, 0], xy[idx, 1]
        xmid = 0.5 * (x.min() + x.max())
        ymid = 0.5 * (y.min() + y.max())
        sets = [idx[(x < xmid) & (y < ymid)], idx[(x < xmid) & (y >= ymid)],
                idx[(x >= xmid) & (y < ymid)], idx[(x >= xmid) & (y >= ymid)]]
        node = Node(start, start, depth)
        for s in sets:
            if s.size:
                node.children.append(build(s, depth + 1))
        node.stop = len(order)
        return node

    root = build(np.arange(xy.shape[0]), 0)
    return root, np.asarray(order, dtype=np.int64)


def octree(xyz: np.ndarray, max_depth: int = 16, min_leaf: int = 16):
    """The 3D analogue of Alg. 2 ("an octree ... each internal node
    has at most 8 child nodes"; 64 first-level pairs).  Reading A1 in
    3D: split at x_mid, y_mid, z_mid, a coordinate equal to mid goes to the
    upper half; children ordered by (x, y, z) half, x slowest -- the quadtree's
    I1..I4 order with z added.  A2/A3 as for the quadtree."""
    order = []

    def build(idx: np.ndarray, depth: int) -> Node:
        start = len(order)
        if depth >= max_depth or idx.size <= min_leaf:
            order.extend(np.sort(idx).tolist())
            return Node(start, len(order), depth)
        x, y, z = xyz[idx, 0], xyz[idx, 1], xyz[idx, 2]
        xm = 0.5 * (x.min() + x.max())
        ym = 0.5 * (y.min() + y.max())
        zm = 0.5 * (z.min() + z.max())
        node = Node(start, start, depth)
        for hx in (False, True):
            for hy in (False, True):
                for hz in (False, True):
                    sel = idx[((x >= xm) == hx) & ((y >= ym) == hy) & ((z >= zm) == hz)]
                    if sel.size:
                        node.children.append(build(sel, depth + 1))
        node.stop = len(order)
        return node

    root = build(np.arange(xyz.shape[0]), 0)
    return root, np.asarray(order, dtype=np.int64)


# ------------------------------------------------------------ nbytes (A7/A8)

def nbytes_dense(m, n, w):
    return w * m * n


def nbytes_csr(m, nnz, w):
    return 8 * (m + 1) + 4 * nnz + w * nnz


def nbytes_svd(q, mu, nv, w):
    return w * q * (mu + nv) + w * q + 4 * (mu + nv)


# ------------------------------------------------------------------ Alg. 3

def estimate_rank(block: np.ndarray, eps: float, w: int, k0: int = 8):
    """Alg. 3.  Returns (q, urows, vrows, U_q, S_q, V_q) or None.

    Reading A8: U and V inherit the zero rows/columns of F_IJ;
    the SVD is taken of the block restricted to its nonzero rows/columns and
    only those rows of U/V are stored.  Reading A6: eps relative to the
    block's own sigma_1.  Reading A5: the doubling ("increase k ... jump back",
    P:230) stops only once w k (m'+n') >= nbytes(F_IJ), with m', n' the
    nonzero rows/columns that U and V store (A8) -- then no q > k can pass
    eq. nbytes-comparison -- or once the whole spectrum is in hand (k >= r)."""
    m, n = block.shape
    nnz = int(np.count_nonzero(block))
    target = nbytes_csr(m, nnz, w)                       # nbytes(F_IJ) as CSR (step 1)
    urows = np.flatnonzero(np.any(block != 0, axis=1))
    vrows = np.flatnonzero(np.any(block != 0, axis=0))
    C = block[np.ix_(urows, vrows)]
    U, s, Vt = np.linalg.svd(C, full_matrices=False)    # k-term SVD = leading k of this
    r = s.size
    k = k0
    while True:
        kk = min(k, r)
        sig = s[:kk]
        q = None
        for qq in range(1, kk + 1):                       # smallest q: sigma_{q+1}/sigma_1 < eps
            nxt = sig[qq] if qq < kk else (0.0 if kk == r else None)
            if nxt is None:
                break
            if nxt / sig[0] < eps:
                q = qq
                break
        if q is not None:
            if nbytes_svd(q, urows.size, vrows.size, w) < target:   # eq. nbytes-comparison
                return q, urows, vrows, U[:, :q].copy(), s[:q].copy(), Vt[:q, :].T.copy()
            return None
        if w * k * (urows.size + vrows.size) >= target or kk == r:
            return None
        k *= 2


# ------------------------------------------------------------------ Alg. 4

@dataclass
class Block:
    kind: int
    row0: int
    m: int
    col0: int
    n: int
    level: int
    nbytes: int
    data: object = None          # dense ndarray / (rowptr, cols, vals) / (q, urows, vrows, U, S, V)
    children: list = field(default_factory=list)


def _leaf(kind, I, J, blk, w, level):
    m, n = blk.shape
    if kind == ZERO:
        return Block(ZERO, I.start, m, J.start, n, level, 0)
    if kind == DENSE:
        return Block(DENSE, I.start, m, J.start, n, level, nbytes_dense(m, n, w), blk.copy())
    rows, cols = np.nonzero(blk)
    rowptr = np.zeros(m + 1, dtype=np.int64)
    np.add.at(rowptr, rows + 1, 1)
    rowptr = np.cumsum(rowptr)
    return Block(CSR, I.start, m, J.start, n, level, nbytes_csr(m, rows.size, w),
                 (rowptr, cols.astype(np.int64), blk[rows, cols].copy()))


def assemble(F: np.ndarray, I: Node, J: Node, eps: float, w: int, min_size: int, k0: int = 8,
             level: int = 1) -> Block:
    """Alg. 4 for the block pair (I, J) in tree order.  F is the
    tree-ordered exact matrix (its slices are Alg. 1's CSR blocks)."""
    blk = F[I.start:I.stop, J.start:J.stop]
    m, n = blk.shape
    nnz = int(np.count_nonzero(blk))
    if nnz == 0:                                            # A11: zero short-circuit
        return _leaf(ZERO, I, J, blk, w, level)
    b_csr = nbytes_csr(m, nnz, w)
    b_den = nbytes_dense(m, n, w)
    best_leaf = CSR if b_csr <= b_den else DENSE             # tie -> CSR (A25 order)
    if m * n < min_size or not I.children or not J.children:  # step 2
        return _leaf(best_leaf, I, J, blk, w, level)
    cands = [(b_csr, 1, CSR), (b_den, 2, DENSE)]
    svd = estimate_rank(blk, eps, w, k0)                     # step 3
    if svd is not None:
        q, ur, vr, U, S, V = svd
        cands.append((nbytes_svd(q, ur.size, vr.size, w), 3, SVD))
    kids = [assemble(F, Ic, Jd, eps, w, min_size, k0, level + 1)   # step 4
            for Ic in I.children for Jd in J.children]
    b_sub = sum(c.nbytes for c in kids) + NODE_OVERHEAD
    cands.append((b_sub, 4, SUB))
    _, _, kind = min(cands)                                  # step 5 (ties: A25 order)
    if kind == SVD:
        return Block(SVD, I.start, m, J.start, n, level, nbytes_svd(q, ur.size, vr.size, w),
                     (q, ur, vr, U, S, V))
    if kind in (CSR, DENSE):
        return _leaf(kind, I, J, blk, w, level)
    kinds = {c.kind for c in kids} - {ZERO}                  # step 6 (A10: Zero fits either)
    if kinds == {CSR}:
        return _leaf(CSR, I, J, blk, w, level)
    if kinds == {DENSE}:
        return _leaf(DENSE, I, J, blk, w, level)
    return Block(SUB, I.start, m, J.start, n, level, b_sub, children=kids)


@dataclass
class HMatrix:
    N: int
    perm: np.ndarray
    tops: list            # first-level Blocks in Alg. 5 order
    eps: float
    dtype: str            # "f64" | "f32"

    def leaves(self):
        out = []

        def walk(b):
            if b.kind == SUB:
                for c in b.children:
                    walk(c)
            elif b.kind != ZERO:
                out.append(b)
        for b in self.tops:
            walk(b)
        return out

    @property
    def nbytes(self):
        return sum(b.nbytes for b in self.tops)


def _round(a, dtype):
    return a.astype(np.float32).astype(np.float64) if dtype == "f32" else a


def compress(x: np.ndarray, F: np.ndarray, eps: float, dtype: str = "f64", max_depth: int = 16,
             min_leaf: int = 16, min_size: int = 16384, k0: int = 8, tree: str = "quad") -> HMatrix:
    """Quadtree (Alg. 2) or octree (tree="oct") on centroids, then
    Alg. 4 on every first-level block pair (at most 16 / 64 pairs).
    Values are rounded to the storage dtype (f32 variant: the block values a
    GPU f32 path stores)."""
    w = 8 if dtype == "f64" else 4
    root, perm = (octree(x, max_depth, min_leaf) if tree == "oct" else quadtree(x[:, :2], max_depth, min_leaf))
    Fp = F[np.ix_(perm, perm)]
    level1 = root.children if root.children else [root]
    tops = [assemble(Fp, I, J, eps, w, min_size, k0, 1) for I in level1 for J in level1]
    H = HMatrix(F.shape[0], perm, tops, eps, dtype)
    if dtype == "f32":
        for b in H.leaves():
            if b.kind == DENSE:
                b.data = _round(b.data, dtype)
            elif b.kind == CSR:
                b.data = (b.data[0], b.data[1], _round(b.data[2], dtype))
            else:
                q, ur, vr, U, S, V = b.data
                b.data = (q, ur, vr, _round(U, dtype), _round(S, dtype), _round(V, dtype))
    return H


# ------------------------------------------------------------------ Alg. 5

def _apply_leaf(b: Block, Xp: np.ndarray, Yp: np.ndarray):
    XJ = Xp[b.col0:b.col0 + b.n]
    YI = Yp[b.row0:b.row0 + b.m]
    if b.kind == DENSE:
        YI += b.data @ XJ
    elif b.kind == CSR:
        rowptr, cols, vals = b.data
        for i in range(b.m):
            s, e = rowptr[i], rowptr[i + 1]
            if e > s:
                YI[i] += vals[s:e] @ XJ[cols[s:e]]
    elif b.kind == SVD:
        q, ur, vr, U, S, V = b.data
        T = S[:, None] * (V.T @ XJ[vr])          # U (Sigma (V^T x))
        YI[ur] += U @ T


def hmatvec(H: HMatrix, X: np.ndarray) -> np.ndarray:
    """Alg. 5: Y <- 0; for each block pair, leaf -> Y_I += F_IJ X_J
    "in the obvious way", block matrix -> recurse.  X in caller order,
    column-major N x k; returns Y in caller order (FP64 accumulation)."""
    X = np.asarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X[:, None]
    Xp = X[H.perm]
    Yp = np.zeros_like(Xp)

    def walk(b):
        if b.kind == SUB:
            for c in b.children:
                walk(c)
        elif b.kind != ZERO:
            _apply_leaf(b, Xp, Yp)
    for b in H.tops:
        walk(b)
    Y = np.empty_like(Yp)
    Y[H.perm] = Yp
    return np.asfortranarray(Y)


def densify(H: HMatrix) -> np.ndarray:
    """F-hat as a dense matrix in caller order (for the 10 tol checks)."""
    Fp = np.zeros((H.N, H.N))
    for b in H.leaves():
        if b.kind == DENSE:
            Fp[b.row0:b.row0 + b.m, b.col0:b.col0 + b.n] += b.data
        elif b.kind == CSR:
            rowptr, cols, vals = b.data
            rows = np.repeat(np.arange(b.m), np.diff(rowptr))
            Fp[b.row0 + rows, b.col0 + cols] += vals
        else:
            q, ur, vr, U, S, V = b.data
            Fp[np.ix_(b.row0 + ur, b.col0 + vr)] += (U * S) @ V.T
    F = np.empty_like(Fp)
    F[np.ix_(H.perm, H.perm)] = Fp
    return F


# ------------------------------------------------------------ HVFM container

HVFM_MAGIC = b"HVFM"
HVFM_VERSION = 1


def write_hvfm(H: HMatrix, path: str):
    """Serialise F-hat in the HVFM v1 container (layout in include/vf.h):
    leaves in Alg. 5 order, tree-order ranges, values in the storage dtype."""
    dt = np.float64 if H.dtype == "f64" else np.float32
    code = 1 if H.dtype == "f64" else 2
    leaves = H.leaves()
    with open(path, "wb") as f:
        f.write(HVFM_MAGIC)
        f.write(struct.pack("<IIIqdq", HVFM_VERSION, code, 0, H.N, H.eps, len(leaves)))
        f.write(np.asarray(H.perm, dtype=np.int32).tobytes())
        for b in leaves:
            f.write(struct.pack("<iiqqqq", b.kind, b.level, b.row0, b.m, b.col0, b.n))
            if b.kind == DENSE:
                f.write(np.ascontiguousarray(b.data, dtype=dt).tobytes())
            elif b.kind == CSR:
                rowptr, cols, vals = b.data
                f.write(struct.pack("<q", cols.size))
                f.write(np.asarray(rowptr, dtype=np.int64).tobytes())
                f.write(np.asarray(cols, dtype=np.int32).tobytes())
                f.write(np.asarray(vals, dtype=dt).tobytes())
            else:
                q, ur, vr, U, S, V = b.data
                f.write(struct.pack("<qqq", q, ur.size, vr.size))
                f.write(np.asarray(ur, dtype=np.int32).tobytes())
                f.write(np.asarray(vr, dtype=np.int32).tobytes())
                f.write(np.asarray(S, dtype=dt).tobytes())
                f.write(np.ascontiguousarray(U, dtype=dt).tobytes())
                f.write(np.ascontiguousarray(V, dtype=dt).tobytes())


def stats(H: HMatrix) -> dict:
    out = {name: [0, 0] for name in ("dense", "csr", "svd")}
    for b in H.leaves():
        out[KIND_NAME[b.kind]][0] += 1
        out[KIND_NAME[b.kind]][1] += b.nbytes
    return out
