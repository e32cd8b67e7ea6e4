"""Full-length parity of the BASELINE configs against the CPU oracle, on a B200 box:

    python tools/full_parity.py C4 C3 C3f32ref native     # any subset; ~5 min of CPU each

For each config the GPU march runs at the temporal-blocking depth bench.py uses (C4: T=4,
C3 f64: the bench's depth, C3 f32 reference contract: T=2) from the device-generated seeded
initial data; the SAME u0/v0 bytes are downloaded and marched by the oracle
(oracle/ps_oracle.c: the reference's arithmetic, simulator.py:147-205, OpenMP over rows) on
the host for the full step count.  Writes profiles/r02_parity_<config>.json with the
bitwise flag and the relative max-norm max|u_gpu - u_ref| / max|u_ref| on both live levels
(north_star: fp64 <= 1e-12 after N steps).

`native` measures what the f32 native contract (one fma per tap, f32 accumulator — the
GPU's own contract, not a reference path) costs in accuracy: relative max-norm of the f32
native run against the f64 run on the same seed, C3 after 500 steps and C5 after 100 —
the figures tests/test_gpu_parity.py's stated tolerance is set from.

TEST/EVIDENCE TOOL: it calls the oracle, so it is not part of the product.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = {
    # name: (scheme, n, lam, dtype, arith, (K, wmin, wmax, v_zero), steps, tsteps)
    "C4": ("P9", 32767, 0.6, "f64", "ref", (64, 0.01, 0.05, True), 200, None),
    "C3": ("P13", 16383, 0.4, "f64", "ref", (32, 0.01, 0.05, False), 500, None),
    "C3f32ref": ("P13", 16383, 0.4, "f32", "ref", (32, 0.01, 0.05, False), 500, 2),
}


def bench_depth(name):
    import bench

    return bench.CONFIGS[name].get("tb", 1)


def run_case(name, quick=False):
    import torch

    from oracle import oracle as O
    from paper_1904_04048_b200.device import Simulation
    from paper_1904_04048_b200.scheme import evaluate_table

    scheme, n, lam, dtype, arith, gauss, steps, T = CASES[name]
    if T is None:
        T = bench_depth(name)
    if quick:
        steps = 12
    sim = Simulation(scheme, n, lam, bc="dirichlet", dtype=dtype, arith=arith, tsteps=T)
    K, wmin, wmax, vzero = gauss
    sim.gaussian_initial(K, wmin, wmax, seed=0, v_zero=vzero)
    u0, v0 = sim.initial_fields()
    t0 = time.perf_counter()
    sim.first_step()
    sim.march(steps - 1)
    torch.cuda.synchronize()
    gpu_s = time.perf_counter() - t0
    got, got_prev = sim.field(), sim.field("previous")
    ring = sim.ring
    tau = sim.tau
    spec = sim.spec
    del sim
    torch.cuda.empty_cache()
    p = lambda role: evaluate_table(getattr(spec, role), lam)  # noqa: E731
    t0 = time.perf_counter()
    u1 = O.first_step(u0, v0, p("first_u"), p("first_v"), tau, "dirichlet", ring, arith)
    want, want_prev = O.march(u1, u0, p("two_step"), steps - 1, "dirichlet", ring, arith)
    cpu_s = time.perf_counter() - t0
    del u0, v0, u1

    def rel(a, b):
        scale = float(np.abs(b).max())
        worst = 0.0
        for r0 in range(0, a.shape[0], 2048):      # chunked: no full-size temporaries
            worst = max(worst, float(np.abs(a[r0:r0 + 2048].astype(np.float64)
                                            - b[r0:r0 + 2048].astype(np.float64)).max()))
        return worst / scale, scale

    r_new, scale = rel(got, want)
    r_prev, _ = rel(got_prev, want_prev)
    inner = n + 1 - 2 * ring
    out = {
        "config": name, "scheme": scheme, "nodes": n + 1, "dtype": dtype, "arith": arith,
        "lambda": lam, "ring": ring, "steps": steps, "temporal_blocking": T,
        "bitwise_newest": got.tobytes() == want.tobytes(),
        "bitwise_previous": got_prev.tobytes() == want_prev.tobytes(),
        "rel_max_norm_newest": r_new, "rel_max_norm_previous": r_prev,
        "max_abs_reference": scale,
        "gpu_seconds": gpu_s, "oracle_seconds": cpu_s, "oracle_threads": O.max_threads(),
        "oracle_glups": inner * inner * steps / cpu_s / 1e9,
        "initial_data": f"seeded {K}-Gaussian sums (seed 0), generated on the device; the "
                        "oracle marches the same downloaded bytes",
        "oracle": "oracle/ps_oracle.c (reference arithmetic restated in C, pinned to the "
                  "reference's golden vectors by tests/test_host.py)",
    }
    return out


def native_error(quick=False):
    """f32 native vs f64 on the same seed (both on the GPU): C3 after 500, C5 after 100."""
    import torch

    from paper_1904_04048_b200.device import Simulation

    out = {}
    for name, n, gauss, steps in (("C3", 16383, (32, 0.01, 0.05), 500),
                                  ("C5", 65535, (128, 0.002, 0.01), 100)):
        if quick:
            steps = 12
        sim = Simulation("P13", n, 0.4, bc="dirichlet", dtype="f64", tsteps=1)
        sim.gaussian_initial(*gauss, seed=0)
        sim.first_step()
        sim.march(steps - 1)
        ref = sim.levels[sim.newest].view().clone()
        del sim
        torch.cuda.empty_cache()
        sim = Simulation("P13", n, 0.4, bc="dirichlet", dtype="f32", arith="native", tsteps=4)
        sim.gaussian_initial(*gauss, seed=0)
        sim.first_step()
        sim.march(steps - 1)
        got = sim.levels[sim.newest].view()
        scale = ref.abs().max().item()
        diff = 0.0
        for r0 in range(0, ref.shape[0], 4096):
            diff = max(diff, (got[r0:r0 + 4096].to(torch.float64)
                              - ref[r0:r0 + 4096]).abs().max().item())
        out[name] = {"nodes": n + 1, "steps": steps, "rel_max_norm_f32native_vs_f64": diff / scale,
                     "max_abs_f64": scale,
                     "old_bound_2nt2_2^-24": 2.0 * steps * steps * 2.0**-24}
        del sim, ref, got
        torch.cuda.empty_cache()
    return out


def main():
    quick = "--quick" in sys.argv
    names = [a for a in sys.argv[1:] if not a.startswith("--")] or ["C4", "C3", "C3f32ref", "native"]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    for name in names:
        res = native_error(quick) if name == "native" else run_case(name, quick)
        tag = "f32native" if name == "native" else name
        path = os.path.join(ROOT, "profiles", f"r02_parity_{tag}{'_quick' if quick else ''}.json")
        with open(path, "w") as f:
            json.dump(res, f, indent=1)
        # gpurun brings back gpurun_out/ only
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", os.path.basename(path)), "w") as f:
            json.dump(res, f, indent=1)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
