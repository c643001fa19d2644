"""Test helper: an independent reader of the HVFM v1 container (include/vf.h)
and a dense reconstruction, used to check the product's F-hat against the
oracle's exact F.  Not part of the product or of the oracle."""
import struct

import numpy as np


def read_hvfm(path):
    with open(path, "rb") as f:
        buf = f.read()
    off = 0

    def take(fmt):
        nonlocal off
        v = struct.unpack_from(fmt, buf, off)
        off += struct.calcsize(fmt)
        return v

    def arr(dt, n):
        nonlocal off
        a = np.frombuffer(buf, dtype=dt, count=n, offset=off).copy()
        off += a.nbytes
        return a

    assert buf[:4] == b"HVFM"
    off = 4
    ver, code, _ = take("<III")
    assert ver == 1
    N, tol, nl = take("<qdq")
    vt = np.float64 if code == 1 else np.float32
    perm = arr(np.int32, N)
    leaves = []
    for _ in range(nl):
        kind, level, row0, m, col0, n = take("<iiqqqq")
        L = dict(kind=kind, level=level, row0=row0, m=m, col0=col0, n=n)
        if kind == 1:
            L["D"] = arr(vt, m * n).reshape(m, n).astype(np.float64)
        elif kind == 2:
            (nnz,) = take("<q")
            L["rowptr"] = arr(np.int64, m + 1)
            L["cols"] = arr(np.int32, nnz)
            L["vals"] = arr(vt, nnz).astype(np.float64)
        elif kind == 3:
            q, mu, nv = take("<qqq")
            L["q"] = q
            L["urows"] = arr(np.int32, mu)
            L["vrows"] = arr(np.int32, nv)
            L["S"] = arr(vt, q).astype(np.float64)
            L["U"] = arr(vt, mu * q).reshape(mu, q).astype(np.float64)
            L["V"] = arr(vt, nv * q).reshape(nv, q).astype(np.float64)
        else:
            raise ValueError(kind)
        leaves.append(L)
    assert off == len(buf)
    return dict(N=N, tol=tol, dtype=code, perm=perm, leaves=leaves)


def densify(H):
    N = H["N"]
    Fp = np.zeros((N, N))
    for L in H["leaves"]:
        r0, c0 = L["row0"], L["col0"]
        if L["kind"] == 1:
            Fp[r0:r0 + L["m"], c0:c0 + L["n"]] += L["D"]
        elif L["kind"] == 2:
            rows = np.repeat(np.arange(L["m"]), np.diff(L["rowptr"]))
            Fp[r0 + rows, c0 + L["cols"]] += L["vals"]
        else:
            Fp[np.ix_(r0 + L["urows"], c0 + L["vrows"])] += (L["U"] * L["S"]) @ L["V"].T
    perm = H["perm"]
    F = np.empty_like(Fp)
    F[np.ix_(perm, perm)] = Fp
    return F


def block_of(H, L):
    """(tree-order rows, cols) of a leaf in caller order."""
    perm = H["perm"]
    return perm[L["row0"]:L["row0"] + L["m"]], perm[L["col0"]:L["col0"] + L["n"]]
