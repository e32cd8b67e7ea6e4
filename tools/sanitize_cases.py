"""Small runs of every kernel family for compute-sanitizer (TMA/mbarrier
rings, the setmaxnreg warpgroup split and the peer-store halo path are the risk):

    compute-sanitizer --tool memcheck  python tools/sanitize_cases.py
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
    compute-sanitizer --tool synccheck python tools/sanitize_cases.py

(one tool per gpurun call; tools/sanitize.sh wraps them and keeps the summaries).  Each case
is also compared with the CPU oracle, so a sanitizer-clean run is a correct run.
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pairs(spec, role, lam):
    from paper_1904_04048_b200.scheme import evaluate_table

    return evaluate_table(getattr(spec, role), lam)


def initial(n, dtype, bc, seed=1):
    rng = np.random.default_rng(seed)
    npdt = np.float64 if dtype == "f64" else np.float32
    u0 = rng.normal(size=(n + 1, n + 1)).astype(npdt)
    v0 = rng.normal(size=(n + 1, n + 1)).astype(npdt)
    if bc == "periodic":
        for a in (u0, v0):
            a[:-1, -1] = a[:-1, 0]
            a[-1, :] = a[0, :]
    return u0, v0


def oracle_march(spec, n, lam, steps, u0, v0, bc, ring, arith):
    from oracle import oracle as O

    r = ring if bc == "dirichlet" else 0
    u1 = O.first_step(u0, v0, pairs(spec, "first_u", lam), pairs(spec, "first_v", lam), lam / n,
                      bc, r, arith)
    return O.march(u1, u0, pairs(spec, "two_step", lam), steps, bc, r, arith)[0]


def case_march(name, n, bc, dtype, arith, tsteps, steps):
    from paper_1904_04048_b200.device import Simulation

    lam = 0.4 if name == "P13" else 0.6
    sim = Simulation(name, n, lam, bc=bc, dtype=dtype, arith=arith, tsteps=tsteps)
    u0, v0 = initial(n, dtype, bc)
    sim.load_initial(u0, v0)
    sim.first_step()
    sim.march(steps)
    want = oracle_march(sim.spec, n, lam, steps, u0, v0, bc, sim.ring, arith)
    assert sim.field().tobytes() == want.tobytes(), (name, n, bc, dtype, arith, tsteps)


def case_slabs(name, n, dtype, arith, tsteps, transport, bc="dirichlet"):
    from paper_1904_04048_b200.slab import VirtualSlabs

    lam = 0.4 if name == "P13" else 0.6
    vs = VirtualSlabs(name, n, lam, 3, dtype=dtype, arith=arith, transport=transport,
                      tsteps=tsteps, bc=bc)
    u0, v0 = initial(n, dtype, bc)
    vs.load_initial(u0, v0)
    vs.first_step()
    steps = 2 * tsteps
    vs.march(steps)
    want = oracle_march(vs.spec, n, lam, steps, u0, v0, bc, vs.ring, arith)
    assert vs.field().tobytes() == want.tobytes(), (name, transport, tsteps, bc)


def case_solve_host(n, tsteps):
    from paper_1904_04048_b200.device import Simulation

    sim = Simulation("P9", n, 0.6, bc="dirichlet", tsteps=tsteps)
    u0, v0 = initial(n, "f64", "dirichlet")
    got = sim.solve_host(u0, v0, 9, nbands=3)
    want = oracle_march(sim.spec, n, 0.6, 8, u0, v0, "dirichlet", 1, "ref")
    assert got.tobytes() == want.tobytes()


def case_run_and_tables():
    import paper_1904_04048_b200 as ps
    from paper_1904_04048_b200.benchmarks import run_table

    rep = ps.run(ps.SimConfig(scheme=ps.named_scheme("P5"), n=40, n_t=12, lam=0.707))
    assert 1e-7 < rep.error < 1e-4
    assert len(run_table(3)) == 4          # batched tiny-grid kernel (one CTA per run)


def main():
    import torch

    from paper_1904_04048_b200 import _native as nat

    torch.cuda.set_device(0)
    before = nat.launch_count()
    # streaming kernel (T=1): every shape family, both BCs, ragged widths, two strips
    case_march("P9", 300, "dirichlet", "f64", "ref", 1, 3)
    case_march("P13", 1100, "periodic", "f64", "ref", 1, 2)
    case_march("P5", 257, "periodic", "f32", "ref", 1, 3)
    case_march("P13", 300, "dirichlet", "f32", "native", 1, 3)
    # fused kernels: shared-product warpgroup-specialised (f64 radius 1), two-vector fallback
    # shapes, f32 narrow windows with setmaxnreg, periodic images, depth 3 on 8 warps
    case_march("P9", 1300, "dirichlet", "f64", "ref", 4, 9)
    case_march("C9", 300, "dirichlet", "f64", "ref", 2, 5)
    case_march("P13", 700, "dirichlet", "f64", "ref", 3, 7)
    case_march("P13", 600, "dirichlet", "f32", "native", 4, 9)
    case_march("P9", 400, "periodic", "f64", "ref", 4, 9)
    case_march("P13", 300, "periodic", "f32", "ref", 2, 5)
    # row slabs: halo copies, in-kernel halo stores (T=1 and fused), periodic ring
    case_slabs("P9", 400, "f64", "ref", 1, "kernel")
    case_slabs("P13", 500, "f64", "ref", 2, "kernel")
    case_slabs("P9", 400, "f64", "ref", 4, "copy")
    case_slabs("P9", 300, "f64", "ref", 2, "copy", bc="periodic")
    # banded host-to-host solve (four streams, skewed wavefront), run() with the fused
    # error sums, batched paper table
    case_solve_host(700, 2)
    case_run_and_tables()
    torch.cuda.synchronize()
    print(f"sanitize cases ok: {nat.launch_count() - before} libps kernel launches, all "
          "bitwise equal to the oracle")


if __name__ == "__main__":
    main()
