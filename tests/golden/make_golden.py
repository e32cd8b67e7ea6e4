"""Generate the golden fixtures in tests/golden/ from the LIVE reference.

Run in the build container, where the read-only reference exists:

    python tests/golden/make_golden.py [/root/reference/pkg/src]

The reference package (poisson-stencils 0.1.0, pure Python + numpy) is imported under
an alias straight from its source tree; nothing is copied.  Outputs (committed):

  tables.json   every named scheme's tables evaluated at the config Courant numbers,
                floats as float.hex() (bit-exact), plus serialize_tables() text.
  fields.npz    inputs and outputs of reference first_step / two_step calls on small
                grids: all 6 schemes x {dirichlet (radius 1), periodic} x {f64, f32},
                random fields (nonzero Dirichlet ring, inconsistent periodic alias) and
                smooth fields, plus multi-step marches (run()'s loop) with fields.
  runs.json     run() reports (error, per-step errors) for the paper tables
                (benchmarks.py:27-61 rows) and a few extra configs.

The oracle pin tests (tests/test_host.py) and the GPU parity tests
(tests/test_gpu_parity.py, tests/test_gpu_integration.py) read these files; none of
them touches /root/reference.
"""

from __future__ import annotations

import importlib
import importlib.util
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LAMS = (0.3, 0.4, 0.5, 0.6, 0.707, 0.796)


def load_reference(src):
    pkg = os.path.join(src, "poisson_stencils")
    spec = importlib.util.spec_from_file_location(
        "ref_poisson_stencils", os.path.join(pkg, "__init__.py"),
        submodule_search_locations=[pkg])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["ref_poisson_stencils"] = mod
    spec.loader.exec_module(mod)
    return mod


def main(src="/root/reference/pkg/src"):
    ref = load_reference(src)

    # ---- tables -----------------------------------------------------------------
    tables = {}
    for name in ref.NAMED_SCHEMES:
        spec = ref.named_scheme(name)
        entry = {"radius": spec.radius, "serialized": ref.serialize_tables(spec), "at": {}}
        for lam in LAMS:
            entry["at"][repr(lam)] = {
                role: [[list(off), float(poly(lam)).hex()] for off, poly in getattr(spec, role).items()]
                for role in ("first_u", "first_v", "two_step")
            }
        tables[name] = entry
    with open(os.path.join(HERE, "tables.json"), "w") as f:
        json.dump(tables, f, indent=1, sort_keys=True)

    # ---- single calls -------------------------------------------------------------
    arrays = {}
    cases = []
    rng = np.random.default_rng(20260419)
    for name in ref.NAMED_SCHEMES:
        spec = ref.named_scheme(name)
        for bc in ("dirichlet", "periodic"):
            if bc == "dirichlet" and spec.radius > 1:
                continue
            for dt in ("f64", "f32"):
                for n, kind_in in ((6, "random"), (23, "random"), (40, "smooth")):
                    lam = float(rng.choice([0.4, 0.6, 0.707]))
                    tau = lam / n
                    if kind_in == "random":
                        a = rng.normal(size=(n + 1, n + 1))
                        b = rng.normal(size=(n + 1, n + 1))
                    else:
                        x = np.arange(n + 1) / n
                        x1, x2 = np.meshgrid(x, x, indexing="ij")
                        a = np.sin(2 * np.pi * x1) * np.cos(4 * np.pi * x2) + 0.25
                        b = np.cos(2 * np.pi * x1 + 0.3) * np.sin(2 * np.pi * x2)
                    if dt == "f32":
                        a, b = a.astype(np.float32), b.astype(np.float32)
                    key = f"{name}_{bc}_{dt}_{n}"
                    arrays[key + "_a"] = a
                    arrays[key + "_b"] = b
                    arrays[key + "_two"] = ref.two_step(a, b, spec, lam, bc)
                    arrays[key + "_first"] = ref.first_step(a, b, spec, lam, tau, bc)
                    cases.append({"key": key, "scheme": name, "bc": bc, "dtype": dt, "n": n,
                                  "lam": lam, "tau": tau, "inputs": kind_in})

    # ---- marches: run()'s own loop, fields captured through on_step ---------------------
    marches = []
    for name, bc, n, nt, lam in (("P5", "dirichlet", 24, 30, 0.5), ("C9", "dirichlet", 17, 25, 0.6),
                                 ("P9", "periodic", 32, 40, 0.6), ("P13", "periodic", 20, 30, 0.4),
                                 ("C13", "periodic", 15, 12, 0.707), ("P9", "dirichlet", 31, 50, 0.6)):
        spec = ref.named_scheme(name)
        captured = []
        cfg = ref.SimConfig(scheme=spec, n=n, n_t=nt, lam=lam, bc=bc)
        rep = ref.run(cfg, on_step=lambda k, f: captured.append(f))
        key = f"march_{name}_{bc}_{n}_{nt}"
        arrays[key + "_last"] = captured[-1]
        arrays[key + "_mid"] = captured[len(captured) // 2]
        marches.append({"key": key, "scheme": name, "bc": bc, "n": n, "n_t": nt, "lam": lam,
                        "error": rep.error.hex(),
                        "per_step": [e.hex() for e in rep.per_step_errors],
                        "mid_index": len(captured) // 2})
    np.savez_compressed(os.path.join(HERE, "fields.npz"), **arrays)

    # ---- run() reports for the paper tables ------------------------------------------
    bench = importlib.import_module("ref_poisson_stencils.benchmarks")
    runs = {"cases": cases, "marches": marches, "tables": {}}
    for t in (1, 2, 3):
        runs["tables"][str(t)] = [
            {k: (v.hex() if isinstance(v, float) and k.startswith("E_") else v) for k, v in row.items()}
            for row in bench.run_table(t)
        ]
    with open(os.path.join(HERE, "runs.json"), "w") as f:
        json.dump(runs, f, indent=1, sort_keys=True)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main(*sys.argv[1:])
