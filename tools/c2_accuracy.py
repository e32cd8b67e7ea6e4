"""BASELINE config 2 accuracy report: P9 periodic 4096^2 f64, λ=0.6, standing wave m=4,
n=6, 1000 steps.  Runs the GPU march (T=1 and the blocked T=4) and the CPU oracle for
all 1000 steps, then prints one JSON line: bitwise agreement with the oracle and the
max-norm errors against the exact solution u0·(cos ωt + sin ωt).

    python tools/c2_accuracy.py      # on a B200 (takes ~1 min, mostly the CPU oracle)
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from oracle import oracle as O
    from paper_1904_04048_b200.device import Simulation
    from paper_1904_04048_b200.scheme import evaluate_table, named_scheme

    n, lam, steps = 4096, 0.6, 1000
    out = {"config": "C2: P9 periodic 4096^2 f64, lambda=0.6, m=4, n=6, 1000 steps"}
    fields = {}
    for T in (1, 4):
        sim = Simulation("P9", n, lam, bc="periodic", tsteps=T)
        omega = sim.standing_wave_initial(4, 6)
        if T == 1:
            u0, v0 = sim.initial_fields()
        sim.first_step()
        sim.march(steps - 1)
        fields[T] = sim.field()
        tau = sim.tau
        del sim
    spec = named_scheme("P9")

    def p(role):
        return evaluate_table(getattr(spec, role), lam)

    t0 = time.perf_counter()
    u1 = O.first_step(u0, v0, p("first_u"), p("first_v"), tau, "periodic", 0)
    want, _ = O.march(u1, u0, p("two_step"), steps - 1, "periodic", 0)
    out["oracle_seconds"] = round(time.perf_counter() - t0, 1)
    out["oracle_threads"] = O.max_threads()
    out["bitwise_T1_vs_oracle"] = fields[1].tobytes() == want.tobytes()
    out["bitwise_T4_vs_oracle"] = fields[4].tobytes() == want.tobytes()
    out["max_abs_diff_vs_oracle"] = float(np.abs(fields[4] - want).max())
    coords = np.arange(n + 1) / n
    x1, x2 = np.meshgrid(coords, coords, indexing="ij")
    t = steps * tau
    exact = np.sin(2 * np.pi * 4 * x1) * np.sin(2 * np.pi * 6 * x2) * (np.cos(omega * t) +
                                                                       np.sin(omega * t))
    err = np.abs(fields[4] - exact).max()
    out["max_norm_error_vs_exact"] = float(err)
    out["relative_max_norm_error_vs_exact"] = float(err / np.abs(exact).max())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
