"""paper_2209_07632_b200 -- B200 (sm_100a) compressed view-factor library.

Thin Python binding over the C ABI in ``include/vf.h`` (libvf.so, built
in-tree by ``paper_2209_07632_b200.build``).  Every function here only
marshals arguments (pointers, sizes, dtypes) and maps status codes to
exceptions; every step of the apply and of the solves runs in libvf's CUDA
kernels.  There is no CPU fallback: without a B200 the apply/solve calls
raise ``VFError`` (VF_ENODEV).

Vectors are column-major N x nrhs in caller (facet) order: pass a numpy
array in Fortran order, a 1-D array (nrhs = 1), or a torch tensor of shape
(N, nrhs) with strides (1, N) -- e.g. ``t.T.contiguous().T`` -- on the
handle's device or on the host.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import build as _build

__all__ = [
    "VFError", "lib", "ViewFactorMatrix", "vf_build", "vf_build_facets", "vf_load", "vf_save", "vf_free",
    "vf_upload", "vf_set_stream", "vf_matvec", "vf_solve_radiosity", "vf_solve_thermal", "vf_insolation", "vf_insolation_sum",
    "vf_info", "vf_last_solve_stats", "vf_enable_kernel_timing", "vf_kernel_timing", "VF_F64", "VF_F32",
    "VF_VIS_RAYCAST", "VF_VIS_CULL_ONLY", "HEADER", "vf_row_partition", "vf_shard_rows", "vf_row_range",
    "vf_get_nccl_id", "vf_comm_init", "vf_set_mesh", "VF_EVAL_AUTO", "VF_EVAL_HOST", "VF_EVAL_DEVICE",
    "VF_TREE_QUAD", "VF_TREE_OCT", "vf_insolation_sum", "TimeStepper",
]

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "vf.h")

VF_OK, VF_EINVAL, VF_ENOMEM, VF_ECUDA, VF_ENOCONV, VF_EIO, VF_ENCCL, VF_EUNSUPPORTED, VF_ENODEV = \
    0, -1, -2, -3, -4, -5, -6, -7, -8
VF_F64, VF_F32 = 1, 2
VF_VIS_RAYCAST, VF_VIS_CULL_ONLY = 0, 1
VF_EVAL_AUTO, VF_EVAL_HOST, VF_EVAL_DEVICE = 0, 1, 2
VF_TREE_QUAD, VF_TREE_OCT = 0, 1
_STATUS = {0: "VF_OK", -1: "VF_EINVAL", -2: "VF_ENOMEM", -3: "VF_ECUDA", -4: "VF_ENOCONV", -5: "VF_EIO",
           -6: "VF_ENCCL", -7: "VF_EUNSUPPORTED", -8: "VF_ENODEV"}


class VFError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_STATUS.get(code, code)}: {msg}")
        self.code = code


class vf_mesh(ctypes.Structure):
    _fields_ = [("nv", ctypes.c_int64), ("nf", ctypes.c_int64),
                ("V", ctypes.c_void_p), ("F", ctypes.c_void_p)]


class vf_build_opts(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_int), ("max_depth", ctypes.c_int), ("min_leaf", ctypes.c_int),
                ("min_block", ctypes.c_int64), ("k0", ctypes.c_int), ("visibility", ctypes.c_int),
                ("orient_up", ctypes.c_int), ("device", ctypes.c_int), ("threads", ctypes.c_int),
                ("seed", ctypes.c_uint64), ("evaluator", ctypes.c_int), ("tree", ctypes.c_int)]


class vf_info_t(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int64), ("dtype", ctypes.c_int), ("tol", ctypes.c_double),
                ("n_dense", ctypes.c_int64), ("n_csr", ctypes.c_int64), ("n_svd", ctypes.c_int64),
                ("bytes_dense", ctypes.c_int64), ("bytes_csr", ctypes.c_int64), ("bytes_svd", ctypes.c_int64),
                ("nnz_csr", ctypes.c_int64), ("sum_rank", ctypes.c_int64), ("max_rank", ctypes.c_int64),
                ("active_rows", ctypes.c_int64), ("device_bytes", ctypes.c_int64), ("alg_bytes", ctypes.c_int64),
                ("alg_flops_per_col", ctypes.c_int64), ("visible_pairs", ctypes.c_int64),
                ("build_seconds", ctypes.c_double), ("device", ctypes.c_int),
                ("t_rows", ctypes.c_int64), ("p1_bytes", ctypes.c_int64), ("p2_bytes", ctypes.c_int64),
                ("p1_src_rows", ctypes.c_int64), ("p2_src_rows", ctypes.c_int64),
                ("p1_flops_per_col", ctypes.c_int64), ("p2_flops_per_col", ctypes.c_int64),
                ("groups1", ctypes.c_int64), ("groups2", ctypes.c_int64), ("resident", ctypes.c_int64),
                ("stream_payload_bytes", ctypes.c_int64), ("stream_meta_bytes", ctypes.c_int64),
                ("stream_chunks", ctypes.c_int64), ("tiles", ctypes.c_int64), ("tile_sources", ctypes.c_int64),
                ("k1_payload_bytes", ctypes.c_int64), ("k1_kernel", ctypes.c_int64)]


_lib = None


def lib():
    """Load libvf.so (building it in-tree if missing or stale)."""
    global _lib
    if _lib is None:
        path = os.environ.get("VF_LIB") or _build.build()     # VF_LIB: a prebuilt variant (experiments)
        L = ctypes.CDLL(path)
        P, I, i, d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        H = ctypes.c_void_p
        sig = {
            "vf_default_opts": ([ctypes.POINTER(vf_build_opts)], None),
            "vf_build": ([ctypes.POINTER(vf_mesh), d, ctypes.POINTER(vf_build_opts), ctypes.POINTER(H)], i),
            "vf_build_facets": ([I, P, P, P, ctypes.POINTER(vf_mesh), d, ctypes.POINTER(vf_build_opts),
                                 ctypes.POINTER(H)], i),
            "vf_load": ([ctypes.c_char_p, i, ctypes.POINTER(H)], i),
            "vf_save": ([H, ctypes.c_char_p], i),
            "vf_upload": ([H, i], i),
            "vf_free": ([H], i),
            "vf_set_stream": ([H, P], i),
            "vf_matvec": ([H, P, P, i], i),
            "vf_solve_radiosity": ([H, P, P, P, i, i, d, i], i),
            "vf_solve_thermal": ([H, P, P, P, P, P, P, i, i, d], i),
            "vf_last_solve_stats": ([H, ctypes.POINTER(i), ctypes.POINTER(d), ctypes.POINTER(i),
                                     ctypes.POINTER(d)], i),
            "vf_insolation": ([H, P, i, d, P], i),
            "vf_insolation_sum": ([H, P, P, i, i, d, P], i),
            "vf_ts_create": ([H, i, i, d, d, d, d, d, P, P, P, P, ctypes.POINTER(ctypes.c_void_p)], i),
            "vf_ts_step": ([ctypes.c_void_p, P, d, P], i),
            "vf_ts_get": ([ctypes.c_void_p, P, P, P, P], i),
            "vf_ts_free": ([ctypes.c_void_p], i),
            "vf_selftest_rows_exchange": ([i, i, i, I, P, P, P, i, P, d, i, i, P, P, P, P], i),
            "vf_info": ([H, ctypes.POINTER(vf_info_t)], i),
            "vf_enable_kernel_timing": ([H, i], i),
            "vf_kernel_timing": ([H, ctypes.POINTER(d), ctypes.POINTER(i), ctypes.POINTER(d),
                                  ctypes.POINTER(i), ctypes.POINTER(i)], i),
            "vf_row_partition": ([H, i, P], i),
            "vf_set_mesh": ([H, ctypes.POINTER(vf_mesh), i], i),
            "vf_shard_rows": ([H, i, i], i),
            "vf_row_range": ([H, ctypes.POINTER(I), ctypes.POINTER(I)], i),
            "vf_get_nccl_id": ([P], i),
            "vf_comm_init": ([H, i, i, P], i),
            "vf_last_error": ([], ctypes.c_char_p),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def _check(rc: int):
    if rc != VF_OK:
        raise VFError(rc, (lib().vf_last_error() or b"").decode())


# ------------------------------------------------------------ marshalling

def _np_dtype(dt):
    return np.float64 if dt == VF_F64 else np.float32


def _vec_ptr(a, N: int, dt: int, name: str, writable: bool = False):
    """Pointer + nrhs for a column-major N x k vector (numpy or torch)."""
    want = _np_dtype(dt)
    if a is None:
        return None, 0
    if hasattr(a, "data_ptr"):                       # torch tensor
        import torch
        tdt = torch.float64 if dt == VF_F64 else torch.float32
        if a.dtype != tdt:
            raise TypeError(f"{name}: dtype {a.dtype}, handle needs {tdt}")
        if a.dim() == 1:
            if a.shape[0] != N or a.stride(0) != 1:
                raise ValueError(f"{name}: need contiguous length-{N} vector")
            return a.data_ptr(), 1
        if a.dim() != 2 or a.shape[0] != N or (a.shape[1] > 1 and (a.stride(0) != 1 or a.stride(1) != N)):
            raise ValueError(f"{name}: need column-major ({N}, k) tensor (strides (1, {N}))")
        return a.data_ptr(), a.shape[1]
    if not isinstance(a, np.ndarray):
        raise TypeError(f"{name}: numpy array or torch tensor required")
    if a.dtype != want:
        raise TypeError(f"{name}: dtype {a.dtype}, handle needs {np.dtype(want)}")
    if a.ndim == 1:
        if a.shape[0] != N or not a.flags.c_contiguous:
            raise ValueError(f"{name}: need contiguous length-{N} vector")
        return a.ctypes.data, 1
    if a.ndim != 2 or a.shape[0] != N or not a.flags.f_contiguous:
        raise ValueError(f"{name}: need Fortran-ordered ({N}, k) array")
    if writable and not a.flags.writeable:
        raise ValueError(f"{name}: not writeable")
    return a.ctypes.data, a.shape[1]


def _opts(**kw):
    o = vf_build_opts()
    lib().vf_default_opts(ctypes.byref(o))
    for k, v in kw.items():
        if v is not None:
            setattr(o, k, v)
    return o


# ------------------------------------------------------------ C-named calls

def vf_build(V, F, tol: float, **opts):
    """vf_build(mesh, tol): host-side Alg. 1-4 build + upload.  Returns a handle."""
    V = np.ascontiguousarray(V, dtype=np.float64)
    F = np.ascontiguousarray(F, dtype=np.int32)
    m = vf_mesh(V.shape[0], F.shape[0], V.ctypes.data, F.ctypes.data)
    o = _opts(**opts)
    h = ctypes.c_void_p()
    _check(lib().vf_build(ctypes.byref(m), float(tol), ctypes.byref(o), ctypes.byref(h)))
    return h


def vf_build_facets(x, n, A, tol: float, occluders=None, **opts):
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = np.ascontiguousarray(n, dtype=np.float64)
    A = np.ascontiguousarray(A, dtype=np.float64)
    mp = None
    if occluders is not None:
        V = np.ascontiguousarray(occluders[0], dtype=np.float64)
        F = np.ascontiguousarray(occluders[1], dtype=np.int32)
        mp = ctypes.byref(vf_mesh(V.shape[0], F.shape[0], V.ctypes.data, F.ctypes.data))
    o = _opts(**opts)
    h = ctypes.c_void_p()
    _check(lib().vf_build_facets(x.shape[0], x.ctypes.data, n.ctypes.data, A.ctypes.data, mp, float(tol),
                                 ctypes.byref(o), ctypes.byref(h)))
    return h


def vf_load(path: str, device: int = 0):
    h = ctypes.c_void_p()
    _check(lib().vf_load(os.fsencode(path), int(device), ctypes.byref(h)))
    return h


def vf_save(h, path: str):
    _check(lib().vf_save(h, os.fsencode(path)))


def vf_upload(h, device: int = 0):
    _check(lib().vf_upload(h, int(device)))


def vf_free(h):
    if h:
        _DIMS.pop(h.value if hasattr(h, "value") else int(h), None)
        lib().vf_free(h)


def vf_set_stream(h, stream):
    _check(lib().vf_set_stream(h, ctypes.c_void_p(int(stream) if stream else 0)))


def vf_info(h) -> dict:
    info = vf_info_t()
    _check(lib().vf_info(h, ctypes.byref(info)))
    return {name: getattr(info, name) for name, _ in vf_info_t._fields_}


_DIMS: dict = {}


def _dims(h):
    """(N, dtype) of a handle; both are fixed for its lifetime, so they are
    cached instead of calling vf_info (a host walk over all leaves) per call."""
    key = h.value if hasattr(h, "value") else int(h)
    d = _DIMS.get(key)
    if d is None:
        info = vf_info(h)
        d = _DIMS[key] = (info["N"], info["dtype"])
    return d


def vf_set_mesh(h, V, F, orient_up: bool = True):
    V = np.ascontiguousarray(V, dtype=np.float64)
    F = np.ascontiguousarray(F, dtype=np.int32)
    m = vf_mesh(V.shape[0], F.shape[0], V.ctypes.data, F.ctypes.data)
    _check(lib().vf_set_mesh(h, ctypes.byref(m), int(bool(orient_up))))


def vf_matvec(h, X, Y, nrhs: int | None = None):
    N, dt = _dims(h)
    px, kx = _vec_ptr(X, N, dt, "X")
    py, ky = _vec_ptr(Y, N, dt, "Y", writable=True)
    k = nrhs or kx
    if kx != k or ky != k:
        raise ValueError("X/Y column counts differ")
    _check(lib().vf_matvec(h, px, py, int(k)))


def vf_solve_radiosity(h, E, rho, B, iters: int = 100, tol: float = 1e-12, clamp: bool = True):
    N, dt = _dims(h)
    pe, k = _vec_ptr(E, N, dt, "E")
    pr, _ = _vec_ptr(rho, N, dt, "rho")
    pb, kb = _vec_ptr(B, N, dt, "B", writable=True)
    if kb != k:
        raise ValueError("E/B column counts differ")
    _check(lib().vf_solve_radiosity(h, pe, pr, pb, int(k), int(iters), float(tol), int(bool(clamp))))


def vf_solve_thermal(h, Qdir, albedo, emiss, T, Qvis=None, Qir=None, iters: int = 100, tol: float = 1e-12):
    N, dt = _dims(h)
    pq, k = _vec_ptr(Qdir, N, dt, "Qdir")
    pa, _ = _vec_ptr(albedo, N, dt, "albedo")
    pe, _ = _vec_ptr(emiss, N, dt, "emiss")
    pt, kt = _vec_ptr(T, N, dt, "T", writable=True)
    pv, _ = _vec_ptr(Qvis, N, dt, "Qvis", writable=True)
    pi, _ = _vec_ptr(Qir, N, dt, "Qir", writable=True)
    if kt != k:
        raise ValueError("Qdir/T column counts differ")
    _check(lib().vf_solve_thermal(h, pq, pa, pe, pt, pv, pi, int(k), int(iters), float(tol)))


def vf_selftest_rows_exchange(bounds, xrank, part, enorm2, tol, iters, iter0):
    """Test hook: one ROWS exchange with len(bounds) - 1 ranks emulated on the
    current device (see include/vf.h).  xrank (world, N, kp), part
    (world, kp, nblk), enorm2 (k,).  Returns (xout, resid, iter_after, done_after)."""
    bounds = np.ascontiguousarray(bounds, dtype=np.int64)
    xrank = np.ascontiguousarray(xrank, dtype=np.float64)
    part = np.ascontiguousarray(part, dtype=np.float64)
    enorm2 = np.ascontiguousarray(enorm2, dtype=np.float64)
    world, N, kp = xrank.shape
    nblk = part.shape[2]
    k = enorm2.size
    xout = np.zeros_like(xrank)
    resid = np.zeros(k)
    it = np.zeros(world, dtype=np.int32)
    dn = np.zeros(world, dtype=np.int32)
    _check(lib().vf_selftest_rows_exchange(world, kp, k, N, bounds.ctypes.data, xrank.ctypes.data, part.ctypes.data,
                                           nblk, enorm2.ctypes.data, float(tol), int(iters), int(iter0),
                                           xout.ctypes.data, resid.ctypes.data, it.ctypes.data, dn.ctypes.data))
    return xout, resid, it, dn


class TimeStepper:
    """Alg. 6 on the device: vf_ts_create / vf_ts_step / vf_ts_get
    (argument marshalling only; include/vf.h documents the operation)."""

    def __init__(self, M, albedo, emiss, Qdir0, T0, layers=30, depth=0.5, ratio=1.2, k_th=0.01, rho_c=1.0e6,
                 H=0.0):
        self.h = M.h if hasattr(M, "h") else M
        N, dt = _dims(self.h)
        self.N, self.dt = N, dt
        pa, _ = _vec_ptr(albedo, N, dt, "albedo")
        pe, _ = _vec_ptr(emiss, N, dt, "emiss")
        pq, k = _vec_ptr(Qdir0, N, dt, "Qdir0")
        pt, kt = _vec_ptr(T0, N, dt, "T0")
        if kt != k:
            raise ValueError("Qdir0 / T0 column counts differ")
        self.nscen = k
        s = ctypes.c_void_p()
        _check(lib().vf_ts_create(self.h, int(k), int(layers), float(depth), float(ratio), float(k_th), float(rho_c),
                                  float(H), pa, pe, pq, pt, ctypes.byref(s)))
        self.s = s

    def step(self, Qdir, dt, Tsurf=None):
        pq, k = _vec_ptr(Qdir, self.N, self.dt, "Qdir")
        pt, _ = _vec_ptr(Tsurf, self.N, self.dt, "Tsurf", writable=True)
        if k != self.nscen:
            raise ValueError("Qdir column count differs from the state's scenarios")
        _check(lib().vf_ts_step(self.s, pq, float(dt), pt))

    def get(self, Qrefl=None, Qir=None, Qabs=None, Tsurf=None):
        ps = [_vec_ptr(a, self.N, self.dt, n, writable=True)[0] for a, n in
              ((Qrefl, "Qrefl"), (Qir, "Qir"), (Qabs, "Qabs"), (Tsurf, "Tsurf"))]
        _check(lib().vf_ts_get(self.s, *ps))

    def close(self):
        if getattr(self, "s", None) and self.s.value:
            lib().vf_ts_free(self.s)
            self.s = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def vf_last_solve_stats(h) -> dict:
    i1, i2 = ctypes.c_int(), ctypes.c_int()
    r1, r2 = ctypes.c_double(), ctypes.c_double()
    _check(lib().vf_last_solve_stats(h, ctypes.byref(i1), ctypes.byref(r1), ctypes.byref(i2), ctypes.byref(r2)))
    return dict(iters1=i1.value, resid1=r1.value, iters2=i2.value, resid2=r2.value)


def vf_insolation(h, suns, S: float = 1365.0) -> np.ndarray:
    """Host-side Q_dir: N x k column-major float64."""
    suns = np.ascontiguousarray(np.atleast_2d(suns), dtype=np.float64)
    N = _dims(h)[0]
    Q = np.empty((N, suns.shape[0]), order="F")
    _check(lib().vf_insolation(h, suns.ctypes.data, suns.shape[0], float(S), Q.ctypes.data))
    return Q


def vf_insolation_sum(h, dirs, w, S: float = 1365.0) -> np.ndarray:
    """Finite solar disk: Q[:, c] = sum_p w[p] Q_point(dirs[c*P + p]).
    dirs (k*P, 3), w (P,) -> N x k column-major float64."""
    dirs = np.ascontiguousarray(np.atleast_2d(dirs), dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64).reshape(-1)
    P = w.size
    if dirs.shape[0] % P:
        raise ValueError("dirs rows must be a multiple of len(w)")
    k = dirs.shape[0] // P
    N = _dims(h)[0]
    Q = np.empty((N, k), order="F")
    _check(lib().vf_insolation_sum(h, dirs.ctypes.data, w.ctypes.data, k, P, float(S), Q.ctypes.data))
    return Q


def vf_enable_kernel_timing(h, on: bool = True):
    _check(lib().vf_enable_kernel_timing(h, int(bool(on))))


def vf_kernel_timing(h) -> dict:
    ms2, ms1 = ctypes.c_double(), ctypes.c_double()
    l2, l1, lt = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _check(lib().vf_kernel_timing(h, ctypes.byref(ms2), ctypes.byref(l2), ctypes.byref(ms1), ctypes.byref(l1),
                                  ctypes.byref(lt)))
    return dict(ms_phase2=ms2.value, launches_phase2=l2.value, ms_phase1=ms1.value, launches_phase1=l1.value,
                launches_total=lt.value)


def vf_row_partition(h, world: int) -> np.ndarray:
    """Cut points (world + 1,) of the block-row partition (ROWS mode)."""
    b = np.zeros(world + 1, dtype=np.int64)
    _check(lib().vf_row_partition(h, int(world), b.ctypes.data))
    return b


def vf_shard_rows(h, rank: int, world: int):
    _check(lib().vf_shard_rows(h, int(rank), int(world)))


def vf_row_range(h) -> tuple[int, int]:
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().vf_row_range(h, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def vf_get_nccl_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().vf_get_nccl_id(buf))
    return buf.raw


def vf_comm_init(h, rank: int, world: int, nccl_id: bytes):
    if len(nccl_id) != 128:
        raise ValueError("nccl_id must be 128 bytes")
    buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
    _check(lib().vf_comm_init(h, int(rank), int(world), buf))


class ViewFactorMatrix:
    """Owning wrapper around a vf_handle (frees it on close / GC)."""

    def __init__(self, handle):
        self.h = handle
        self.info = vf_info(handle)
        self.N = self.info["N"]
        self.dtype = self.info["dtype"]

    @classmethod
    def build(cls, V, F, tol, **opts):
        return cls(vf_build(V, F, tol, **opts))

    @classmethod
    def build_facets(cls, x, n, A, tol, occluders=None, **opts):
        return cls(vf_build_facets(x, n, A, tol, occluders, **opts))

    @classmethod
    def load(cls, path, device=0):
        return cls(vf_load(path, device))

    def save(self, path):
        vf_save(self.h, path)

    def refresh(self):
        self.info = vf_info(self.h)
        return self.info

    def matvec(self, X, Y):
        vf_matvec(self.h, X, Y)
        return Y

    def solve_radiosity(self, E, rho, B, iters=100, tol=1e-12, clamp=True):
        vf_solve_radiosity(self.h, E, rho, B, iters, tol, clamp)
        return B

    def solve_thermal(self, Qdir, albedo, emiss, T, Qvis=None, Qir=None, iters=100, tol=1e-12):
        vf_solve_thermal(self.h, Qdir, albedo, emiss, T, Qvis, Qir, iters, tol)
        return T

    def insolation(self, suns, S=1365.0):
        return vf_insolation(self.h, suns, S)

    def insolation_sum(self, dirs, w, S=1365.0):
        return vf_insolation_sum(self.h, dirs, w, S)

    def set_stream(self, stream):
        vf_set_stream(self.h, stream)

    def stats(self):
        return vf_last_solve_stats(self.h)

    def shard_rows(self, rank, world):
        """Keep only this rank's block rows (ROWS mode)."""
        vf_shard_rows(self.h, rank, world)
        return self.refresh()

    def row_range(self):
        return vf_row_range(self.h)

    def comm_init(self, rank, world, nccl_id):
        vf_comm_init(self.h, rank, world, nccl_id)

    def init_rows(self, group=None):
        """Shard by rows over a torch.distributed process group and create the
        NCCL communicator (rank 0's unique id is broadcast through the group)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        self.shard_rows(rank, world)
        obj = [vf_get_nccl_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0, group=group)
        self.comm_init(rank, world, obj[0])

    def close(self):
        if self.h:
            vf_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
