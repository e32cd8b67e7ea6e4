"""The reference-side binding of INTEGRATION.md §2 (integration/_gpu.py: numpy + ctypes
over include/ps.h, nothing from paper_1904_04048_b200), exercised on the GPU against the
golden vectors generated from the live reference — and the ``poisson_stencils`` import
path (the shim package) resolving to the GPU implementation."""

from __future__ import annotations

import importlib.util
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def binding():
    spec = importlib.util.spec_from_file_location("ref_side_gpu",
                                                  os.path.join(ROOT, "integration", "_gpu.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_reference_side_binding_matches_golden_calls(binding):
    from paper_1904_04048_b200.scheme import evaluate_table, named_scheme

    with open(os.path.join(GOLD, "runs.json")) as f:
        runs = json.load(f)
    fields = np.load(os.path.join(GOLD, "fields.npz"))
    checked = 0
    for case in runs["cases"]:
        spec = named_scheme(case["scheme"])
        key, bc, lam = case["key"], case["bc"], case["lam"]
        a, b = fields[key + "_a"], fields[key + "_b"]
        two = binding.two_step_gpu(a, b, evaluate_table(spec.two_step, lam), bc)
        first = binding.first_step_gpu(a, b, evaluate_table(spec.first_u, lam),
                                       evaluate_table(spec.first_v, lam), case["tau"], bc)
        assert two.dtype == a.dtype and two.tobytes() == fields[key + "_two"].tobytes(), key
        assert first.tobytes() == fields[key + "_first"].tobytes(), key
        checked += 1
    assert checked >= 60


def test_poisson_stencils_import_path_runs_on_the_gpu():
    import poisson_stencils
    from paper_1904_04048_b200 import _native as nat
    from poisson_stencils.scheme import named_scheme
    from poisson_stencils.simulator import SimConfig, run, two_step

    import paper_1904_04048_b200.simulator as impl

    assert poisson_stencils.simulator is impl and run is impl.run
    before = nat.launch_count()
    rng = np.random.default_rng(0)
    out = two_step(rng.normal(size=(33, 33)), rng.normal(size=(33, 33)), named_scheme("P9"), 0.6)
    report = run(SimConfig(scheme=named_scheme("P5"), n=20, n_t=20, lam=0.707))
    assert out.shape == (33, 33) and report.error == pytest.approx(5.68e-5, rel=1e-2)
    assert nat.launch_count() > before
