"""ctypes binding of ``libpt_b200.so`` (declared in ``include/pt_b200.h``).

The library is built in-tree by ``paper_1510_01831_b200.build`` for sm_100a.
There is no fallback: if the shared library is missing the import of this
module fails loudly, and ``pt_create`` fails on a machine without a B200.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# PT_LIB_VARIANT=x loads libpt_b200.x.so (an in-tree experimental build) instead
LIB_PATH = os.path.join(HERE, "libpt_b200.%s.so" % os.environ["PT_LIB_VARIANT"]
                        if os.environ.get("PT_LIB_VARIANT") else "libpt_b200.so")

PT_OK = 0
PT_NOT_CONVERGED = 1
PT_INNER_NOT_CONVERGED = 2
PT_BREAKDOWN = 3
PT_BAD_ARGUMENT = 4
PT_CAPACITY = 5
PT_CUDA_ERROR = -1

EXPORTS = (
    "pt_create",
    "pt_destroy",
    "pt_set_stream",
    "pt_set_profiling",
    "pt_solve",
    "pt_solve_device",
    "pt_layer_solve",
    "pt_cell_solve",
    "pt_cell_solve_device",
    "pt_residuals_stride",
    "pt_last_error",
    "pt_version",
)

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_llp = C.POINTER(C.c_longlong)


class PtProblem(C.Structure):
    _fields_ = [
        ("nx", C.c_int), ("nz", C.c_int), ("npml", C.c_int), ("L", C.c_int), ("Lc", C.c_int),
        ("h", C.c_double), ("omega", C.c_double),
        ("layer_extents", _ip), ("cell_extents", _ip),
        ("tx", _dp), ("tz", _dp), ("m", _dp),
        ("layer_coefs", _dp), ("cell_coefs", _dp),
        ("lz", C.POINTER(_dp)), ("uz", C.POINTER(_dp)),
        ("sinv", C.POINTER(_dp)), ("green", C.POINTER(_dp)), ("gsmp", C.POINTER(_dp)),
        ("q0", C.POINTER(_dp)),
        ("inner_dense", C.POINTER(_dp)),
        ("inner_lu", C.POINTER(_dp)),
        ("assembled_boundary", C.c_int),
        ("inner_dense_count", C.c_int),
        ("hdiag", _dp),
    ]


class PtKrylov(C.Structure):
    _fields_ = [
        ("ktol", C.c_double), ("max_iter", C.c_int), ("restart", C.c_int),
        ("inner_ktol", C.c_double), ("inner_max_iter", C.c_int), ("precond", C.c_int),
        ("method", C.c_int),
    ]


class PtStats(C.Structure):
    _fields_ = [
        ("iterations", _dp), ("residuals", _dp), ("n_residuals", _ip), ("relres", _dp),
        ("converged", _ip), ("traces", _dp), ("polarized", _dp),
        ("layer_solves", _llp), ("inner_iters", _llp), ("touches", _llp),
        ("inner_hist", _ip), ("inner_hist_len", C.c_int), ("timing_ms", _dp),
        ("kernel_ms", _dp), ("k1_bytes", _dp), ("launches", _llp), ("k1_launches", _llp),
        ("class_ms", _dp), ("dense_flops", _dp), ("class_flops", _dp), ("class_bytes", _dp),
    ]


def load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1510_01831_b200.build` "
            "(the B200 path has no CPU fallback)"
        )
    lib = C.CDLL(LIB_PATH)
    lib.pt_create.argtypes = [C.POINTER(PtProblem), C.c_int, C.POINTER(C.c_void_p)]
    lib.pt_destroy.argtypes = [C.c_void_p]
    lib.pt_set_stream.argtypes = [C.c_void_p, C.c_void_p]
    lib.pt_set_profiling.argtypes = [C.c_void_p, C.c_int]
    lib.pt_solve.argtypes = [C.c_void_p, _dp, C.c_int, C.POINTER(PtKrylov), _dp, C.POINTER(PtStats)]
    lib.pt_solve_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(PtKrylov), C.c_void_p,
                                    C.POINTER(PtStats)]
    lib.pt_layer_solve.argtypes = [C.c_void_p, C.c_int, _dp, C.c_int, C.c_double, C.c_int, _dp,
                                   C.POINTER(PtStats)]
    lib.pt_cell_solve.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, C.c_int, _dp]
    lib.pt_cell_solve_device.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p]
    lib.pt_residuals_stride.argtypes = [C.POINTER(PtKrylov)]
    lib.pt_residuals_stride.restype = C.c_int
    lib.pt_last_error.restype = C.c_char_p
    lib.pt_version.restype = C.c_char_p
    for name in ("pt_create", "pt_destroy", "pt_solve", "pt_solve_device", "pt_layer_solve",
                 "pt_cell_solve", "pt_cell_solve_device", "pt_set_stream", "pt_set_profiling"):
        getattr(lib, name).restype = C.c_int
    return lib


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        _LIB = load()
    return _LIB


def dptr(a):
    return a.ctypes.data_as(_dp)


def last_error():
    return lib().pt_last_error().decode()


class Context:
    """Owns one ``pt_ctx`` (device-resident factors) and the host arrays it was built from."""

    def __init__(self, factors, device=0):
        F = factors
        self.factors = F
        keep = []

        def arr(x, dtype):
            a = np.ascontiguousarray(np.asarray(x, dtype=dtype))
            keep.append(a)
            return a

        cells = [cf for lf in F.layers for cf in lf.cells]
        nid = len(cells)
        pb = PtProblem()
        pb.nx, pb.nz, pb.npml, pb.L, pb.Lc = F.nx, F.nz, F.npml, F.L, F.Lc
        pb.h, pb.omega = F.h, F.omega
        pb.layer_extents = arr([lf.n for lf in F.layers], np.int32).ctypes.data_as(_ip)
        pb.cell_extents = arr(F.cell_extents, np.int32).ctypes.data_as(_ip)
        pb.tx = dptr(arr(np.stack(F.tx), np.complex128))
        pb.tz = dptr(arr(np.stack(F.tz), np.complex128))
        pb.m = dptr(arr(F.m, np.float64))
        pb.layer_coefs = dptr(arr(np.stack([lf.coefs for lf in F.layers]), np.complex128))
        pb.cell_coefs = dptr(arr(np.stack([cf.coefs for cf in cells]), np.complex128))
        ptr_arrays = {}
        for name in ("lz", "uz", "sinv", "green", "gsmp", "q0"):
            if name in ("green", "gsmp", "q0") and any(getattr(cf, name, None) is None for cf in cells):
                continue  # optional: the cell-solve passes produce these outputs (no green: factor-only context)
            P = (_dp * nid)()
            for i, cf in enumerate(cells):
                v = getattr(cf, name)
                if hasattr(v, "data_ptr"):  # torch tensor (host or device): pass its address
                    keep.append(v)
                    P[i] = C.cast(C.c_void_p(v.data_ptr()), _dp)
                else:
                    P[i] = dptr(arr(v, np.complex128))
            ptr_arrays[name] = P
            setattr(pb, name, C.cast(P, C.POINTER(_dp)))
        if F.Lc > 1 and all(getattr(lf, "dense", None) is not None for lf in F.layers):
            P = (_dp * F.L)()
            for i, lf in enumerate(F.layers):
                v = lf.dense
                if hasattr(v, "data_ptr"):
                    keep.append(v)
                    P[i] = C.cast(C.c_void_p(v.data_ptr()), _dp)
                else:
                    P[i] = dptr(arr(v, np.complex128))
            ptr_arrays["inner_dense"] = P
            pb.inner_dense = C.cast(P, C.POINTER(_dp))
            pb.inner_dense_count = int(F.layers[0].dense.shape[0])
        if F.Lc > 1 and all(getattr(lf, "lu_inv", None) is not None for lf in F.layers):
            P = (_dp * F.L)()
            for i, lf in enumerate(F.layers):
                v = lf.lu_inv
                if hasattr(v, "data_ptr"):
                    keep.append(v)
                    P[i] = C.cast(C.c_void_p(v.data_ptr()), _dp)
                else:
                    P[i] = dptr(arr(v, np.complex128))
            ptr_arrays["inner_lu"] = P
            pb.inner_lu = C.cast(P, C.POINTER(_dp))
        pb.assembled_boundary = int(bool(getattr(F, "assembled_boundary", False)))
        if getattr(F, "hdiag", None) is not None:  # residual of a caller-supplied global operator
            pb.hdiag = dptr(arr(F.hdiag, np.complex128))
        handle = C.c_void_p()
        rc = lib().pt_create(C.byref(pb), int(device), C.byref(handle))
        if rc != PT_OK:
            raise RuntimeError(f"pt_create failed ({rc}): {last_error()}")
        self.handle = handle
        self.device = device
        self.nI = F.L - 1
        self.shape = (F.wz, F.wx)

    def close(self):
        if getattr(self, "handle", None):
            lib().pt_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
