"""ctypes front-end of the CPU oracle (oracle/ps_oracle.c).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs as the checker.  The product package never
imports this module.

Functions take the reference's dense arrays and evaluated tables
(``[((q1, q2), coeff), ...]`` in dict order, as ``simulator._evaluate_table`` returns,
simulator.py:131-132) and mirror ``first_step`` / ``two_step`` (simulator.py:166-205);
``march`` mirrors the loop of ``run`` (simulator.py:271-274) without the error metric.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libps_oracle.so")
_lib = None

BC = {"dirichlet": 0, "periodic": 1}
ARITH = {"ref": 0, "native": 1}


def build() -> str:
    """Compile libps_oracle.so in place (Makefile beside this file)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, i32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        L.ora_two_step.argtypes = [i32, i32, i32, i32, i64, i64, i32, vp, vp, vp, vp, vp, vp,
                                   i64, i64, i32]
        L.ora_first_step.argtypes = [i32, i32, i32, i32, i64, i64, i32, vp, vp, vp, i32, vp, vp,
                                     vp, ctypes.c_double, vp, vp, vp, i32]
        L.ora_march.argtypes = [i32, i32, i32, i32, i64, i64, i32, vp, vp, vp, vp, vp, vp, i64,
                                ctypes.POINTER(ctypes.c_int), i32]
        L.ora_max_threads.argtypes = []
        for f in (L.ora_two_step, L.ora_first_step, L.ora_march, L.ora_max_threads):
            f.restype = ctypes.c_int
        _lib = L
    return _lib


def max_threads() -> int:
    return lib().ora_max_threads()


def _pack(pairs):
    q1 = np.ascontiguousarray([off[0] for off, _ in pairs], dtype=np.int32)
    q2 = np.ascontiguousarray([off[1] for off, _ in pairs], dtype=np.int32)
    c = np.ascontiguousarray([float(v) for _, v in pairs], dtype=np.float64)
    return len(pairs), q1, q2, c


def _dt(a: np.ndarray) -> int:
    if a.dtype == np.float64:
        return 0
    if a.dtype == np.float32:
        return 1
    raise TypeError(f"oracle supports float64/float32, got {a.dtype}")


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def two_step(u_k, u_km1, pairs, bc="dirichlet", ring=1, arith="ref", rows=None, threads=0):
    """Reference ``two_step`` arithmetic; ``rows=(lo, hi)`` restricts the output rows."""
    u_k = np.ascontiguousarray(u_k)
    u_km1 = np.ascontiguousarray(u_km1, dtype=u_k.dtype)
    out = np.zeros_like(u_k)
    nt, q1, q2, c = _pack(pairs)
    lo, hi = rows if rows is not None else (0, 0)
    st = lib().ora_two_step(_dt(u_k), ARITH[arith], BC[bc], ring, u_k.shape[0], u_k.shape[1],
                            nt, _p(q1), _p(q2), _p(c), _p(u_k), _p(u_km1), _p(out), lo, hi,
                            threads)
    if st:
        raise ValueError(f"oracle two_step failed with status {st}")
    return out


def first_step(u0, v0, pairs_u, pairs_v, tau, bc="dirichlet", ring=1, arith="ref", threads=0):
    u0 = np.ascontiguousarray(u0)
    v0 = np.ascontiguousarray(v0, dtype=u0.dtype)
    out = np.zeros_like(u0)
    nu, q1u, q2u, cu = _pack(pairs_u)
    nv, q1v, q2v, cv = _pack(pairs_v)
    st = lib().ora_first_step(_dt(u0), ARITH[arith], BC[bc], ring, u0.shape[0], u0.shape[1],
                              nu, _p(q1u), _p(q2u), _p(cu), nv, _p(q1v), _p(q2v), _p(cv),
                              float(tau), _p(u0), _p(v0), _p(out), threads)
    if st:
        raise ValueError(f"oracle first_step failed with status {st}")
    return out


def march(u_k, u_km1, pairs, nsteps, bc="dirichlet", ring=1, arith="ref", threads=0):
    """``nsteps`` two-step updates from (u^k, u^{k-1}); returns (newest, previous)."""
    a = np.ascontiguousarray(u_k).copy()
    b = np.zeros_like(a)
    c_ = np.ascontiguousarray(u_km1, dtype=a.dtype).copy()
    nt, q1, q2, c = _pack(pairs)
    newest = ctypes.c_int(0)
    st = lib().ora_march(_dt(a), ARITH[arith], BC[bc], ring, a.shape[0], a.shape[1], nt,
                         _p(q1), _p(q2), _p(c), _p(a), _p(b), _p(c_), int(nsteps),
                         ctypes.byref(newest), threads)
    if st:
        raise ValueError(f"oracle march failed with status {st}")
    lv = (a, b, c_)
    return lv[newest.value], lv[(newest.value + 2) % 3]


def gaussian_sum(n, centres, widths, amps, shape=None):
    """Reference-style sampling of a Gaussian sum on x = arange(n+1)/n (numpy)."""
    rows, cols = shape if shape is not None else (n + 1, n + 1)
    x1 = (np.arange(rows) / n)[:, None]
    x2 = (np.arange(cols) / n)[None, :]
    out = np.zeros((rows, cols))
    for (cx, cy), w, a in zip(centres, widths, amps):
        out += a * np.exp(-((x1 - cx) ** 2 + (x2 - cy) ** 2) / (2.0 * (w * w)))
    return out
