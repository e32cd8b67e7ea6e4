"""The reference's acceptance gate (pkg/tests/test_acceptance.py),
restated against the ``poisson_stencils`` import path served by this repo's shim.

Criteria that launch kernels are GPU tests; the exact-algebra criteria run anywhere.
Criterion 4 (Table 2, published E_P9 column) is the reference's KNOWN-RED criterion
(ref test_acceptance.py:129-145, README.md:51-60): the drop-in must reproduce the
reference's own computed values, so here the E_C9 half must pass and the E_P9 half must
deviate exactly as the reference's does (first row within 1 %, later rows not).
"""

from __future__ import annotations

import math
import time
from fractions import Fraction as F

import numpy as np
import pytest

from poisson_stencils.benchmarks import run_table
from poisson_stencils.interpolation import lagrange_basis
from poisson_stencils.quadrature import (
    LambdaPoly,
    a_on_monomial,
    b_on_monomial,
    quad_oracle,
    quad_oracle_b,
)
from poisson_stencils.scheme import NAMED_SCHEMES, generate_scheme, named_scheme
from poisson_stencils.simulator import SimConfig, first_step, run, two_step
from poisson_stencils.stability import lambda_max

gpu = pytest.mark.gpu

AXIS = [(-1, 0), (0, -1), (1, 0), (0, 1)]
DIAG = [(-1, -1), (1, -1), (-1, 1), (1, 1)]
FAR = [(-2, 0), (0, -2), (2, 0), (0, 2)]

# exact λ-polynomials {power: coefficient} per (scheme, table, offset class); PAPER.md
# :279-289 (5-point), :404-415 (9-point), :484-504 (13-point); ref test_acceptance.py:49-90
EXACT = {
    "P5": {
        "first_u": {"centre": {0: 1, 2: -2}, "axis": {2: F(1, 2)}},
        "first_v": {"centre": {0: 1, 2: F(-2, 3)}, "axis": {2: F(1, 6)}},
        "two_step": {"centre": {0: 2, 2: -4}, "axis": {2: 1}},
    },
    "P9": {
        "first_u": {"centre": {0: 1, 2: -2, 4: F(1, 3)}, "axis": {2: F(1, 2), 4: F(-1, 6)},
                    "diag": {4: F(1, 12)}},
        "first_v": {"centre": {0: 1, 2: F(-2, 3), 4: F(1, 15)},
                    "axis": {2: F(1, 6), 4: F(-1, 30)}, "diag": {4: F(1, 60)}},
        "two_step": {"centre": {0: 2, 2: -4, 4: F(2, 3)}, "axis": {2: 1, 4: F(-1, 3)},
                     "diag": {4: F(1, 6)}},
    },
    "P13": {
        "first_u": {"centre": {0: 1, 2: F(-5, 2), 4: F(5, 6)}, "axis": {2: F(2, 3), 4: F(-1, 3)},
                    "diag": {4: F(1, 12)}, "far": {2: F(-1, 24), 4: F(1, 24)}},
        "first_v": {"centre": {0: 1, 2: F(-5, 6), 4: F(1, 6)}, "axis": {2: F(2, 9), 4: F(-1, 15)},
                    "diag": {4: F(1, 60)}, "far": {2: F(-1, 72), 4: F(1, 120)}},
        "two_step": {"centre": {0: 2, 2: -5, 4: F(5, 3)}, "axis": {2: F(4, 3), 4: F(-2, 3)},
                     "diag": {4: F(1, 6)}, "far": {2: F(-1, 12), 4: F(1, 12)}},
    },
}
CLASSES = {"centre": [(0, 0)], "axis": AXIS, "diag": DIAG, "far": FAR}


def test_criterion_1_exact_coefficients():
    t0 = time.perf_counter()
    for name, tables in EXACT.items():
        spec = named_scheme(name)
        for role, by_class in tables.items():
            table = getattr(spec, role)
            assert len(table) == sum(len(CLASSES[c]) for c in by_class)
            for cls, poly in by_class.items():
                for off in CLASSES[cls]:
                    assert table[off] == LambdaPoly(poly), (name, role, off)
    assert time.perf_counter() - t0 < 1.0


def test_criterion_2_pruning():
    for m, count, absent in ((6, 5, (-1, -1)), (11, 9, (-2, 0)), (15, 13, (-2, -1))):
        spec = generate_scheme(m)
        assert len(spec.offsets) == count and absent not in spec.first_u


def deviations(table, limits):
    rows = run_table(table)
    bad = [(row["n"], row["n_t"], row["lambda"], s, row[f"dev_{s}"])
           for row in rows for s, lim in limits.items() if row[f"dev_{s}"] > lim]
    return rows, bad


@gpu
def test_criterion_3_table_1():
    t0 = time.perf_counter()
    rows, bad = deviations(1, {"P5": 0.01, "C5": 0.01})
    assert len(rows) == 12 and not bad, bad
    assert time.perf_counter() - t0 < 5.0


@gpu
def test_criterion_4_table_2_as_the_reference_computes_it():
    t0 = time.perf_counter()
    rows, bad = deviations(2, {"C9": 0.01})
    assert len(rows) == 8 and not bad, bad
    dev_p9 = [row["dev_P9"] for row in rows]
    assert min(dev_p9) <= 0.01 < max(dev_p9)       # the reference's known-red column
    assert max(dev_p9) < 0.60                      # README.md:51-60: 0.7 - 56 % off
    assert time.perf_counter() - t0 < 5.0


@gpu
def test_criterion_5_table_3():
    t0 = time.perf_counter()
    rows, bad = deviations(3, {"P13": 0.05, "C13": 0.01})
    assert len(rows) == 4 and not bad, bad
    assert time.perf_counter() - t0 < 5.0


def test_criterion_6_stability_limits():
    t0 = time.perf_counter()
    half = math.sqrt(0.5)
    nine = math.sqrt((3 - math.sqrt(3)) / 2)
    assert nine == pytest.approx(0.79623, abs=1e-5)
    for name, limit, tol in (("P5", half, 1e-4), ("C9", math.sqrt(3) / 2, 1e-4),
                             ("P13", half, 1e-4), ("P9", nine, 1e-3)):
        assert lambda_max(named_scheme(name)) == pytest.approx(limit, abs=tol), name
    assert time.perf_counter() - t0 < 10.0


def test_criterion_7_quadrature_oracle():
    evens = [(a, b) for a in range(0, 9, 2) for b in range(0, 9, 2) if a + b <= 8]
    for lam in (0.25, 0.5, 0.707, 0.796):
        for mu in evens:
            assert abs(a_on_monomial(mu)(lam) - quad_oracle(mu, lam)) <= 1e-9
            assert abs(b_on_monomial(mu)(lam) - quad_oracle_b(mu, lam)) <= 1e-9


def test_criterion_8_algebraic_properties():
    for m in (6, 11, 15):
        basis = lagrange_basis(m)
        for s in range(m):
            assert [basis.evaluate(s, node) for node in basis.nodes] == \
                [int(s == r) for r in range(m)]
        sums = [sum(basis.coeffs[s][r] for s in range(m)) for r in range(m)]
        assert sums == [F(int(mu == (0, 0))) for mu in basis.monomials]
    for name in NAMED_SCHEMES:
        spec = named_scheme(name)
        assert (sum(spec.first_u.values()), sum(spec.first_v.values()),
                sum(spec.two_step.values())) == (1, 1, 2)


@gpu
def test_criterion_8_field_properties():
    p5 = named_scheme("P5")
    nothing = lambda x1, x2: 0.0 * (x1 + x2)  # noqa: E731
    seen = []
    run(SimConfig(scheme=p5, n=8, n_t=4, lam=0.6, initial_u=nothing, initial_v=nothing),
        on_step=lambda k, f: seen.append(f))
    assert seen and all(not f.any() for f in seen)
    ones = np.ones((9, 9))
    assert first_step(ones, np.zeros((9, 9)), p5, 0.6, 0.06, "periodic") == \
        pytest.approx(ones, abs=1e-13)
    assert two_step(ones, ones, p5, 0.6, "periodic") == pytest.approx(ones, abs=1e-13)
    seen = []
    run(SimConfig(scheme=p5, n=12, n_t=6, lam=0.707), on_step=lambda k, f: seen.append(f))
    assert all(np.abs(f - f.T).max() <= 1e-12 for f in seen)
    errs = [run(SimConfig(scheme=p5, n=n, n_t=n, lam=0.707)).error for n in (10, 20, 40)]
    assert errs[0] / errs[1] >= 8.0 and errs[1] / errs[2] >= 8.0
