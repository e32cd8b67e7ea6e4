"""numpy restatement of the reference's array algorithm (one core, ufunc by ufunc).

TEST INFRASTRUCTURE ONLY — imported by tests/ (pinned against tests/golden) and by
bench.py's ``cpu_baseline`` leg, where it stands in for the reference package itself,
which cannot travel to the GPU box.  The product package never imports this module.

The C oracle (ps_oracle.c) restates the per-point arithmetic; this module restates HOW
the reference computes it, because that is what its CPU time is made of
(poisson_stencils/simulator.py):

* ``_apply_evaluated`` (simulator.py:147-163): a zero accumulator, then for every tap in
  table order one full-size temporary ``coeff * shifted_view`` and one in-place add —
  Dirichlet taps are plain slices (:151-155), periodic taps are ``np.roll`` copies of the
  core (:156-162) followed by the alias row/column copy (``_alias_edges``, :135-138);
* ``first_step`` (:166-180): two accumulations, one scale, one add;
* ``_two_step_evaluated`` (:183-191): accumulation minus ``u_km1``, ring re-pinned.

float32 inputs behave as in the reference: the product ``python_float * float32_array``
stays float32, the accumulator is float64 (``np.zeros`` default dtype, :150/:158), the
result is cast back by assignment into ``zeros_like(values)``.

Beyond the reference: ``ring`` (Dirichlet ring width); ``ring=1`` is
the reference's code path exactly.
"""

from __future__ import annotations

import numpy as np


def apply_evaluated(pairs, values: np.ndarray, bc: str, ring: int = 1) -> np.ndarray:
    """``sum_s c_s * values[. + q_s]`` on the updated nodes; zeros elsewhere."""
    n = values.shape[0] - 1
    out = np.zeros_like(values)
    if bc == "dirichlet":
        r = ring
        acc = np.zeros((n + 1 - 2 * r, n + 1 - 2 * r))
        for (q1, q2), coeff in pairs:
            acc += coeff * values[r + q1:n + 1 - r + q1, r + q2:n + 1 - r + q2]
        out[r:n + 1 - r, r:n + 1 - r] = acc
        return out
    core = values[:n, :n]
    acc = np.zeros((n, n))
    for (q1, q2), coeff in pairs:
        acc += coeff * np.roll(core, shift=(-q1, -q2), axis=(0, 1))
    out[:n, :n] = acc
    out[n, :n] = out[0, :n]
    out[:, n] = out[:, 0]
    return out


def first_step(u0, v0, pairs_u, pairs_v, tau, bc="dirichlet", ring=1):
    out = apply_evaluated(pairs_u, u0, bc, ring)
    out += tau * apply_evaluated(pairs_v, v0, bc, ring)
    return out


def two_step(u_k, u_km1, pairs, bc="dirichlet", ring=1):
    out = apply_evaluated(pairs, u_k, bc, ring) - u_km1
    if bc == "dirichlet":
        r = ring
        out[:r, :] = 0.0
        out[-r:, :] = 0.0
        out[:, :r] = 0.0
        out[:, -r:] = 0.0
    return out


def two_step_slab(u_k, u_km1, pairs, ring: int):
    """Dirichlet ``two_step`` on a full-width slab of rows (rows x (n+1), the slab's own
    first/last ``ring`` rows acting as its ring): the reference's per-tap passes on a
    bounded sample of a grid too large to time whole (bench.py's cpu_baseline)."""
    rows, cols = u_k.shape
    r = ring
    out = np.zeros_like(u_k)
    acc = np.zeros((rows - 2 * r, cols - 2 * r))
    for (q1, q2), coeff in pairs:
        acc += coeff * u_k[r + q1:rows - r + q1, r + q2:cols - r + q2]
    out[r:rows - r, r:cols - r] = acc
    out = out - u_km1
    out[:r, :] = 0.0
    out[-r:, :] = 0.0
    out[:, :r] = 0.0
    out[:, -r:] = 0.0
    return out
