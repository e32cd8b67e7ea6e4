"""poisson_stencils/_gpu.py — the ctypes binding a reference maintainer adds to route
``first_step`` / ``two_step`` (pkg/src/poisson_stencils/simulator.py:166-205) through
libps.so's C-ABI (include/ps.h).  numpy + ctypes only: no torch, no part of
paper_1904_04048_b200.  INTEGRATION.md §2 shows the two-line change in simulator.py;
tests/test_gpu_integration.py loads this file as is and checks it against the golden
vectors generated from the live reference.

``PS_LIBRARY`` names the shared library (default: libps.so next to the drop-in package).
"""

import ctypes
import os

import numpy as np

_DEFAULT = os.path.join(os.path.dirname(os.path.abspath(__file__)), os.pardir,
                        "paper_1904_04048_b200", "libps.so")

H2D, D2H = 1, 2


class PsGrid(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("pitch", ctypes.c_int64),
                ("origin", ctypes.c_int64), ("ghost", ctypes.c_int64), ("row0", ctypes.c_int64),
                ("grows", ctypes.c_int64), ("ring", ctypes.c_int32), ("bc", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("arith", ctypes.c_int32)]


class PsTable(ctypes.Structure):
    _fields_ = [("ntaps", ctypes.c_int32), ("q1", ctypes.c_int32 * 32),
                ("q2", ctypes.c_int32 * 32), ("c", ctypes.c_double * 32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(os.environ.get("PS_LIBRARY") or _DEFAULT)
        G, T, vp, i64, i32 = (ctypes.POINTER(PsGrid), ctypes.POINTER(PsTable), ctypes.c_void_p,
                              ctypes.c_int64, ctypes.c_int32)
        L.ps_layout_init.argtypes = [G, i64, i64, i32, i32, i32, i32, i32]
        L.ps_level_alloc.argtypes = [G]
        L.ps_level_alloc.restype = vp
        L.ps_level_free.argtypes = [vp]
        L.ps_level_free.restype = None
        L.ps_copy_in.argtypes = [G, vp, vp, i64, i64, i64, i32, vp]
        L.ps_copy_out.argtypes = [G, vp, vp, i64, i64, i64, i32, vp]
        L.ps_fill_ghosts.argtypes = [G, vp, i32, vp]
        L.ps_two_step.argtypes = [G, vp, vp, vp, T, vp]
        L.ps_first_step.argtypes = [G, vp, vp, vp, T, T, ctypes.c_double, vp]
        L.ps_strerror.argtypes = [i32]
        L.ps_strerror.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _ok(status):
    if status:
        raise RuntimeError(lib().ps_strerror(status).decode())


def _table(pairs):
    t = PsTable()
    t.ntaps = len(pairs)
    for s, ((q1, q2), c) in enumerate(pairs):
        t.q1[s], t.q2[s], t.c[s] = q1, q2, c
    return t


class _Levels:
    """`count` device levels of an (n+1)^2 reference array's grid, freed on exit."""

    def __init__(self, like: np.ndarray, bc: str, radius: int, count: int):
        L = lib()
        self.n = like.shape[0] - 1
        rows = self.n + 1 if bc == "dirichlet" else self.n
        self.g = PsGrid()
        _ok(L.ps_layout_init(ctypes.byref(self.g), rows, rows, max(2, radius), 1,
                             int(bc == "periodic"), int(like.dtype == np.float32), 0))
        self.ptr = [ctypes.c_void_p(L.ps_level_alloc(ctypes.byref(self.g))) for _ in range(count)]
        if not all(p.value for p in self.ptr):
            self.free()
            raise MemoryError("ps_level_alloc failed")

    def put(self, k, arr, keep_alias):
        a = np.ascontiguousarray(arr)
        n1 = self.n + 1
        _ok(lib().ps_copy_in(ctypes.byref(self.g), self.ptr[k], a.ctypes.data_as(ctypes.c_void_p),
                             n1, n1, n1, H2D, None))
        _ok(lib().ps_fill_ghosts(ctypes.byref(self.g), self.ptr[k], keep_alias, None))
        return a

    def get(self, k, like):
        out = np.empty_like(like)
        n1 = self.n + 1
        # device -> pageable host on the NULL stream: complete when the call returns
        _ok(lib().ps_copy_out(ctypes.byref(self.g), self.ptr[k],
                              out.ctypes.data_as(ctypes.c_void_p), n1, n1, n1, D2H, None))
        return out

    def free(self):
        for p in self.ptr:
            if p.value:
                lib().ps_level_free(p)
        self.ptr = []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.free()


def _radius(*tables):
    return max(max(abs(q1), abs(q2)) for pairs in tables for (q1, q2), _ in pairs)


def two_step_gpu(u_k, u_km1, pairs, bc):
    """Body for simulator.two_step (simulator.py:194-205); ``pairs`` is
    ``_evaluate_table(spec.two_step, lam)`` (simulator.py:131-132), in dict order."""
    with _Levels(u_k, bc, _radius(pairs), 3) as lv:
        keep = [lv.put(0, u_k, 0), lv.put(1, u_km1.astype(u_k.dtype, copy=False), 1)]
        t = _table(pairs)
        _ok(lib().ps_two_step(ctypes.byref(lv.g), lv.ptr[0], lv.ptr[1], lv.ptr[2],
                              ctypes.byref(t), None))
        out = lv.get(2, u_k)
        del keep
        return out


def first_step_gpu(u0, v0, pairs_u, pairs_v, tau, bc):
    """Body for simulator.first_step (simulator.py:166-180)."""
    with _Levels(u0, bc, _radius(pairs_u, pairs_v), 3) as lv:
        keep = [lv.put(0, u0, 0), lv.put(1, v0.astype(u0.dtype, copy=False), 0)]
        tu, tv = _table(pairs_u), _table(pairs_v)
        _ok(lib().ps_first_step(ctypes.byref(lv.g), lv.ptr[0], lv.ptr[1], lv.ptr[2],
                                ctypes.byref(tu), ctypes.byref(tv), float(tau), None))
        out = lv.get(2, u0)
        del keep
        return out
