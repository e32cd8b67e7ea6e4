"""CPU tests of the banded host-to-host solve plan (ps_solve_plan, include/ps.h).

ps_solve_host executes exactly the op list ps_solve_plan returns: each op on its stream,
in list order per stream, after the ops it names in after0/after1.  Two checks, no GPU:

* race freedom — for every pair of ops the plan leaves unordered (no happens-before path
  through stream order and the after edges), neither writes a (level, row) the other
  reads or writes, using each kernel's real read reach (u^k rows +-R*T of a fused pass,
  u^{k-1} rows +-R*(T-1), ...).  So any interleaving the GPU picks gives the result the
  list order gives;
* semantics — replaying the list in order on the CPU oracle (each op computed from the
  levels' current contents, only its rows kept; never-written rows hold NaN) equals the
  oracle's unbanded first step + march bit for bit.
"""

from __future__ import annotations

import random

import numpy as np
import pytest

from paper_1904_04048_b200 import _native as nat
from paper_1904_04048_b200.scheme import evaluate_table, named_scheme


@pytest.fixture(scope="module")
def O():
    from oracle import oracle as O

    O.build()
    return O


def _sets(op, R, rows):
    """(reads, writes): lists of (level, lo, hi) clipped to the logical rows."""
    lo, hi, k = op["row_lo"], op["row_hi"], op["kind"]
    if hi <= lo:
        return [], []

    def clip(lv, a, b):
        return (lv, max(0, a), min(rows, b))

    if k == "load":
        return [], [clip(op["dst0"], lo, hi), clip(op["dst1"], lo, hi)]
    if k == "store":
        return [clip(op["src0"], lo, hi)], []
    if k == "first":
        # velocity half writes u1, the displacement half reads u0 +-R and u1 at own rows
        return ([clip(op["src0"], lo - R, hi + R), clip(op["src1"], lo - R, hi + R),
                 clip(op["dst1"], lo, hi)], [clip(op["dst1"], lo, hi)])
    if k == "step":
        return ([clip(op["src0"], lo - R, hi + R), clip(op["src1"], lo, hi)],
                [clip(op["dst1"], lo, hi)])
    T = op["tsteps"]
    return ([clip(op["src0"], lo - R * T, hi + R * T),
             clip(op["src1"], lo - R * (T - 1), hi + R * (T - 1))],
            [clip(op["dst0"], lo, hi), clip(op["dst1"], lo, hi)])


def _overlap(a, b):
    return any(x[0] == y[0] and max(x[1], y[1]) < min(x[2], y[2]) for x in a for y in b)


def _happens_before(ops):
    """anc[i] = bitmask of ops that complete before op i starts."""
    anc = [0] * len(ops)
    last_on_stream = {}
    for i, op in enumerate(ops):
        preds = [op["after0"], op["after1"], last_on_stream.get(op["stream"], -1)]
        m = 0
        for p in preds:
            if p >= 0:
                assert p < i, "plan edges must point backwards"
                m |= anc[p] | (1 << p)
        anc[i] = m
        last_on_stream[op["stream"]] = i
    return anc


def _race_free(ops, R, rows):
    anc = _happens_before(ops)
    sets = [_sets(op, R, rows) for op in ops]
    for i in range(len(ops)):
        ri, wi = sets[i]
        if not ri and not wi:
            continue
        for k in range(i):
            if (anc[i] >> k) & 1:
                continue
            rk, wk = sets[k]
            if _overlap(wi, rk + wk) or _overlap(wk, ri):
                return f"ops {k} and {i} race: {ops[k]} / {ops[i]}"
    return None


CASES = [(rows, R, nsteps, T, nb, ns)
         for rows, R in ((41, 1), (70, 2), (37, 1))
         for nsteps in (1, 2, 7, 14)
         for T in (1, 2, 3, 4)
         for nb in (0, 1, 2, 3, 5)
         for ns in (1, 2, 3)]


@pytest.mark.parametrize("rows,R,nsteps,T,nb,ns", CASES)
def test_solve_plan_is_race_free(rows, R, nsteps, T, nb, ns):
    ops = nat.solve_plan(rows, R, nsteps, T, nb, ns)
    assert ops, "empty plan"
    msg = _race_free(ops, R, rows)
    assert msg is None, msg


@pytest.mark.parametrize("rows,R,nsteps,T,nb", [(16385, 1, 200, 4, 0), (65536, 2, 100, 4, 0),
                                                (32768, 1, 200, 4, 16)])
def test_solve_plan_covers_every_row_once(rows, R, nsteps, T, nb):
    """Each band's launch j writes a contiguous slice; over the bands the slices of one
    launch index tile [0, rows) exactly, and so do the downloads."""
    ops = nat.solve_plan(rows, R, nsteps, T, nb, 2)
    for kind in ("load", "store"):
        spans = sorted((o["row_lo"], o["row_hi"]) for o in ops if o["kind"] == kind)
        assert spans[0][0] == 0 and spans[-1][1] == rows
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    by_band = {}
    for o in ops:
        if o["kind"] in ("first", "step", "pass"):
            by_band.setdefault(o["band"], []).append(o)
    J = len(by_band[0])
    for j in range(J):
        spans = sorted((ops_b[j]["row_lo"], ops_b[j]["row_hi"]) for ops_b in by_band.values())
        spans = [s for s in spans if s[1] > s[0]]
        assert spans[0][0] == 0 and spans[-1][1] == rows
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert sum(o["tsteps"] for o in by_band[0]) == nsteps
    if nb == 0:
        assert len(by_band) > 1


def test_solve_plan_rejects_bad_arguments():
    for args in ((0, 1, 5, 1, 0, 2), (10, 1, 0, 1, 0, 2), (10, 1, 5, 7, 0, 2),
                 (10, 1, 5, 1, -1, 2), (10, 1, 5, 1, 0, 0)):
        with pytest.raises(nat.PsStatusError):
            nat.solve_plan(*args)


def _replay(O, ops, u0, v0, pu, pv, p2, tau, ring, order):
    rows = u0.shape[0]
    lv = [np.full_like(u0, np.nan) for _ in range(4)]
    out = np.full_like(u0, np.nan)
    for i in order:
        op = ops[i]
        lo, hi = op["row_lo"], op["row_hi"]
        if hi <= lo:
            continue
        k = op["kind"]
        if k == "load":
            lv[op["dst0"]][lo:hi] = u0[lo:hi]
            lv[op["dst1"]][lo:hi] = v0[lo:hi]
        elif k == "first":
            full = O.first_step(lv[op["src0"]], lv[op["src1"]], pu, pv, tau, "dirichlet", ring)
            lv[op["dst1"]][lo:hi] = full[lo:hi]
        elif k == "step":
            full = O.two_step(lv[op["src0"]], lv[op["src1"]], p2, "dirichlet", ring)
            lv[op["dst1"]][lo:hi] = full[lo:hi]
        elif k == "pass":
            new, prev = O.march(lv[op["src0"]], lv[op["src1"]], p2, op["tsteps"], "dirichlet",
                                ring)
            lv[op["dst0"]][lo:hi] = prev[lo:hi]
            lv[op["dst1"]][lo:hi] = new[lo:hi]
        else:
            out[lo:hi] = lv[op["src0"]][lo:hi]
    assert rows == out.shape[0]
    return out


def _topo_order(ops, seed):
    """A random order consistent with stream order and the after edges."""
    rng = random.Random(seed)
    preds = []
    last = {}
    for i, op in enumerate(ops):
        p = {x for x in (op["after0"], op["after1"], last.get(op["stream"], -1)) if x >= 0}
        preds.append(p)
        last[op["stream"]] = i
    done, order = set(), []
    while len(order) < len(ops):
        ready = [i for i in range(len(ops)) if i not in done and preds[i] <= done]
        i = rng.choice(ready)
        done.add(i)
        order.append(i)
    return order


@pytest.mark.parametrize("name,n,nsteps,T,nb", [("P5", 40, 9, 4, 3), ("P9", 52, 14, 2, 4),
                                                ("P13", 63, 11, 4, 3), ("P13", 63, 6, 1, 5),
                                                ("C9", 33, 1, 4, 2), ("P9", 47, 2, 4, 0)])
def test_solve_plan_replay_equals_unbanded_march(O, name, n, nsteps, T, nb):
    spec = named_scheme(name)
    lam = 0.4
    ring = spec.radius
    rng = np.random.default_rng(7)
    u0 = rng.standard_normal((n + 1, n + 1))
    v0 = rng.standard_normal((n + 1, n + 1))
    pu = evaluate_table(spec.first_u, lam)
    pv = evaluate_table(spec.first_v, lam)
    p2 = evaluate_table(spec.two_step, lam)
    tau = lam / n
    u1 = O.first_step(u0, v0, pu, pv, tau, "dirichlet", ring)
    want = u1 if nsteps == 1 else O.march(u1, u0, p2, nsteps - 1, "dirichlet", ring)[0]
    ops = nat.solve_plan(n + 1, spec.radius, nsteps, T, nb, 2)
    for order in (range(len(ops)), _topo_order(ops, 1), _topo_order(ops, 2)):
        got = _replay(O, ops, u0, v0, pu, pv, p2, tau, ring, list(order))
        assert not np.isnan(got).any()
        assert got.tobytes() == want.tobytes()


def test_solve_host_rejects_bad_arguments_before_touching_the_gpu():
    """ps_solve_host validates everything before its first CUDA call (runs without a GPU)."""
    import ctypes

    L = nat.load_library()
    g = nat.make_grid(65, 65, 2, 1, "dirichlet", "f64")
    spec = named_scheme("P9")
    t = nat.make_table(evaluate_table(spec.two_step, 0.6))
    tu = nat.make_table(evaluate_table(spec.first_u, 0.6))
    tv = nat.make_table(evaluate_table(spec.first_v, 0.6))
    host = np.zeros((65, 65))
    hp = host.ctypes.data
    good = (ctypes.c_void_p * 4)(4096, 8192, 12288, 16384)   # never dereferenced on error

    def call(lv=good, u0=hp, out=hp, pitch=65, nsteps=5, tsteps=4, nbands=0, grid=g,
             tt=t):
        return L.ps_solve_host(ctypes.byref(grid), lv, ctypes.c_void_p(u0), None,
                               ctypes.c_void_p(out), pitch, ctypes.byref(tu), ctypes.byref(tv),
                               ctypes.byref(tt), 0.01, nsteps, tsteps, nbands, None)

    assert call(nsteps=0) == 1
    assert call(tsteps=7) == 1
    assert call(nbands=-1) == 1
    assert call(u0=0) == 1
    assert call(out=0) == 1
    assert call(pitch=10) == 1
    assert call(lv=(ctypes.c_void_p * 4)(4096, 4096, 12288, 16384)) == 1   # aliased levels
    assert call(lv=(ctypes.c_void_p * 4)(4100, 8192, 12288, 16384)) == 6   # misaligned
    wide = nat.make_table(evaluate_table(named_scheme("P13").two_step, 0.4))
    assert call(tt=wide) == 4                                              # radius > ring
    slab = nat.make_slab_grid(130, 65, 65, 65, 2, 1, "dirichlet", "f64")
    assert call(grid=slab) == 2
