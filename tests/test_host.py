"""CPU tests: host tables, oracle pinned to the reference's golden vectors, C-ABI exports.

None of these need a GPU.  Golden files come from tests/golden/make_golden.py, which
ran the live reference (poisson-stencils 0.1.0) in the build container.
"""

from __future__ import annotations

import ctypes
import json
import math
import os
import re
from fractions import Fraction

import numpy as np
import pytest

import paper_1904_04048_b200 as ps
from paper_1904_04048_b200 import _native as nat
from paper_1904_04048_b200.scheme import evaluate_table

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def tables():
    with open(os.path.join(GOLD, "tables.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def runs():
    with open(os.path.join(GOLD, "runs.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def fields():
    return np.load(os.path.join(GOLD, "fields.npz"))


@pytest.fixture(scope="module")
def oracle():
    from oracle import oracle as O

    O.build()
    return O


# ---------------------------------------------------------------- host tables (§8a A1/A2)
@pytest.mark.parametrize("name", ps.NAMED_SCHEMES)
def test_tables_bit_exact_against_reference(name, tables):
    spec = ps.named_scheme(name)
    gold = tables[name]
    assert spec.radius == gold["radius"]
    assert ps.serialize_tables(spec) == gold["serialized"]
    for lam_s, roles in gold["at"].items():
        lam = float(lam_s)
        for role, entries in roles.items():
            mine = evaluate_table(getattr(spec, role), lam)
            assert [list(off) for off, _ in mine] == [e[0] for e in entries], (name, role)
            assert [float(v).hex() for _, v in mine] == [e[1] for e in entries], (name, role, lam)


def test_scheme_properties():
    for name in ps.NAMED_SCHEMES:
        spec = ps.named_scheme(name)
        assert sum(spec.first_u.values()) == 1
        assert sum(spec.first_v.values()) == 1
        assert sum(spec.two_step.values()) == 2
    for m in (6, 11, 15):
        b = ps.lagrange_basis(m)
        for s in range(m):
            for r, node in enumerate(b.nodes):
                assert b.evaluate(s, node) == int(s == r)
    assert ps.lagrange_basis(6).det != 0
    with pytest.raises(ps.UnknownSchemeError):
        ps.named_scheme("P7")


def test_quadrature_oracle_agrees_with_exact_operators():
    for lam in (0.25, 0.707):
        for mu in ((0, 0), (2, 0), (2, 2), (4, 0), (0, 6)):
            assert abs(ps.a_on_monomial(mu)(lam) - ps.quad_oracle(mu, lam)) <= 1e-9
            assert abs(ps.b_on_monomial(mu)(lam) - ps.quad_oracle_b(mu, lam)) <= 1e-9
    assert ps.double_factorial(7) == 105 and ps.double_factorial(-1) == 1
    p = ps.LambdaPoly({0: 1, 2: Fraction(-1, 2)})
    assert p(0.5) == float(sum(float(c) * 0.5**k for k, c in sorted({0: 1, 2: -0.5}.items())))


@pytest.mark.parametrize("name,expected,tol", [
    ("P5", math.sqrt(0.5), 1e-4), ("C9", math.sqrt(3) / 2, 1e-4),
    ("P13", math.sqrt(0.5), 1e-4), ("P9", math.sqrt((3 - math.sqrt(3)) / 2), 1e-3)])
def test_lambda_max(name, expected, tol):
    assert ps.lambda_max(ps.named_scheme(name)) == pytest.approx(expected, abs=tol)


def test_symbol_values():
    p5 = ps.named_scheme("P5")
    assert ps.symbol(p5, 1 / math.sqrt(2), math.pi, math.pi) == pytest.approx(-1.0, abs=1e-12)
    env = ps.envelope(p5, 0.9, grid=128)
    assert not env.stable


# ---------------------------------------------------------------- oracle pin (§8c)
def _pairs(spec, role, lam):
    return evaluate_table(getattr(spec, role), lam)


def test_oracle_matches_reference_golden_calls(runs, fields, oracle):
    """Every golden first_step / two_step call, bitwise (incl. f32 and alias edges)."""
    assert len(runs["cases"]) >= 60
    for case in runs["cases"]:
        spec = ps.named_scheme(case["scheme"])
        key, bc, lam = case["key"], case["bc"], case["lam"]
        a, b = fields[key + "_a"], fields[key + "_b"]
        two = oracle.two_step(a, b, _pairs(spec, "two_step", lam), bc, 1)
        first = oracle.first_step(a, b, _pairs(spec, "first_u", lam), _pairs(spec, "first_v", lam),
                                  case["tau"], bc, 1)
        assert two.dtype == fields[key + "_two"].dtype
        assert two.tobytes() == fields[key + "_two"].tobytes(), key
        assert first.tobytes() == fields[key + "_first"].tobytes(), key


def test_oracle_matches_reference_golden_marches(runs, fields, oracle):
    """run()'s loop (first step + two-steps) reproduced bit for bit by the oracle."""
    for m in runs["marches"]:
        spec = ps.named_scheme(m["scheme"])
        n, lam, bc = m["n"], m["lam"], m["bc"]
        tau = lam * (1.0 / n)
        coords = np.arange(n + 1) / n
        x1, x2 = np.meshgrid(coords, coords, indexing="ij")
        u0 = np.zeros((n + 1, n + 1))
        v0 = ps.standing_wave_initial_v(x1, x2)
        if bc == "periodic":
            v0[:-1, -1] = v0[:-1, 0]
            v0[-1, :] = v0[0, :]
        u1 = oracle.first_step(u0, v0, _pairs(spec, "first_u", lam), _pairs(spec, "first_v", lam),
                               tau, bc, 1)
        mid_k = m["mid_index"] + 1
        if mid_k == 1:
            mid = u1
        else:
            mid, _ = oracle.march(u1, u0, _pairs(spec, "two_step", lam), mid_k - 1, bc, 1)
        last, _ = oracle.march(u1, u0, _pairs(spec, "two_step", lam), m["n_t"] - 1, bc, 1)
        assert mid.tobytes() == fields[m["key"] + "_mid"].tobytes(), m["key"]
        assert last.tobytes() == fields[m["key"] + "_last"].tobytes(), m["key"]


def test_numpy_restatement_matches_reference_golden_calls(runs, fields, oracle):
    """oracle/numpy_ref.py (the reference's array algorithm, bench.py's 1-core CPU leg) is
    bitwise equal to every golden call, and its slab form to the C oracle's row range."""
    from oracle import numpy_ref as N

    for case in runs["cases"]:
        spec = ps.named_scheme(case["scheme"])
        key, bc, lam = case["key"], case["bc"], case["lam"]
        a, b = fields[key + "_a"], fields[key + "_b"]
        two = N.two_step(a, b, _pairs(spec, "two_step", lam), bc, 1)
        first = N.first_step(a, b, _pairs(spec, "first_u", lam), _pairs(spec, "first_v", lam),
                             case["tau"], bc, 1)
        assert two.dtype == fields[key + "_two"].dtype
        assert two.tobytes() == fields[key + "_two"].tobytes(), key
        assert first.tobytes() == fields[key + "_first"].tobytes(), key
    rng = np.random.default_rng(5)
    for name, ring, dt in (("P9", 1, np.float64), ("P13", 2, np.float64), ("P13", 2, np.float32)):
        pairs = _pairs(ps.named_scheme(name), "two_step", 0.4)
        a = rng.standard_normal((37, 53)).astype(dt)
        b = rng.standard_normal((37, 53)).astype(dt)
        assert N.two_step_slab(a, b, pairs, ring).tobytes() == \
            oracle.two_step(a, b, pairs, "dirichlet", ring).tobytes()


def test_oracle_ring_generalisation_reduces_to_reference(fields, runs, oracle):
    """Ring width r=2 for radius-1 tables: ring of zeros two wide, interior unchanged
    except rows/cols 1 and n-1 (now pinned) — i.e. exactly the r=1 result restricted."""
    case = next(c for c in runs["cases"] if c["scheme"] == "P9" and c["bc"] == "dirichlet"
                and c["dtype"] == "f64" and c["n"] == 23)
    spec = ps.named_scheme("P9")
    a, b = fields[case["key"] + "_a"], fields[case["key"] + "_b"]
    r1 = oracle.two_step(a, b, _pairs(spec, "two_step", case["lam"]), "dirichlet", 1)
    r2 = oracle.two_step(a, b, _pairs(spec, "two_step", case["lam"]), "dirichlet", 2)
    assert np.array_equal(r2[2:-2, 2:-2], r1[2:-2, 2:-2])
    assert not r2[:2].any() and not r2[-2:].any() and not r2[:, :2].any() and not r2[:, -2:].any()


def test_oracle_rejects_narrow_ring(oracle):
    spec = ps.named_scheme("P13")
    z = np.zeros((12, 12))
    with pytest.raises(ValueError):
        oracle.two_step(z, z, _pairs(spec, "two_step", 0.4), "dirichlet", 1)


def test_oracle_thread_count_invariant(oracle):
    rng = np.random.default_rng(1)
    a, b = rng.normal(size=(301, 301)), rng.normal(size=(301, 301))
    pairs = _pairs(ps.named_scheme("P13"), "two_step", 0.4)
    r1 = oracle.two_step(a, b, pairs, "dirichlet", 2, threads=1)
    r4 = oracle.two_step(a, b, pairs, "dirichlet", 2, threads=4)
    assert r1.tobytes() == r4.tobytes()


# ---------------------------------------------------------------- C-ABI boundary (§8b)
def _declared_symbols():
    with open(os.path.join(ROOT, "include", "ps.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(ps_[a-z0-9_]+)\s*\(", text)))


def test_libps_exports_every_declared_symbol():
    lib = nat.load_library()
    declared = _declared_symbols()
    assert len(declared) >= 15
    for sym in declared:
        assert hasattr(lib, sym), sym
    assert set(declared) == set(nat.EXPORTS)
    assert b"sm_100a" in lib.ps_version()


def test_layout_is_aligned_and_padded():
    for dtype, esz in (("f64", 8), ("f32", 4)):
        for rows in (3, 11, 512, 4097, 32768):
            g = nat.make_grid(rows, rows, 2, 1, "dirichlet", dtype)
            assert (g.pitch * esz) % 128 == 0
            assert (g.origin * esz) % 128 == 0
            assert g.pitch >= rows + 2 * (16 // esz) + g.origin % g.pitch
            assert g.row0 == 0 and g.grows == rows
            nbytes = nat.load_library().ps_level_bytes(ctypes.byref(g))
            assert nbytes == (rows + 2 * g.ghost) * g.pitch * esz


def test_layout_and_call_errors_are_distinct():
    lib = nat.load_library()
    g = nat.PsGrid()
    assert lib.ps_layout_init(ctypes.byref(g), 0, 10, 2, 1, 0, 0, 0) == 2   # PS_ERR_SHAPE
    assert lib.ps_layout_init(ctypes.byref(g), 10, 10, 2, 1, 7, 0, 0) == 1  # PS_ERR_ARG
    g = nat.make_grid(10, 10, 2, 1, "dirichlet", "f64")
    t = nat.make_table(_pairs(ps.named_scheme("P13"), "two_step", 0.4))
    fake = ctypes.c_void_p(4096)
    # radius-2 table on a ring-1 Dirichlet grid -> PS_ERR_RADIUS (cli.py:24's code 4)
    assert lib.ps_two_step(ctypes.byref(g), fake, fake, ctypes.c_void_p(8192), ctypes.byref(t),
                           None) == 4
    assert lib.ps_two_step(ctypes.byref(g), fake, fake, fake, ctypes.byref(t), None) == 1
    assert lib.ps_strerror(4) == b"Dirichlet ring narrower than the stencil radius"
    s = nat.make_slab_grid(100, 64, 40, 20, 2, 1, "dirichlet", "f64")
    assert (s.rows, s.row0, s.grows) == (20, 40, 100)
    with pytest.raises(nat.PsStatusError):
        nat.make_slab_grid(100, 64, 90, 20, 2, 1, "dirichlet", "f64")


# ---------------------------------------------------------------- drop-in host behaviour
def test_dropin_validation_without_gpu():
    p5, p13 = ps.named_scheme("P5"), ps.named_scheme("P13")
    with pytest.raises(ValueError):
        ps.SimConfig(scheme=p5, n=1, n_t=1, lam=0.5)
    with pytest.raises(ps.RadiusUnsupportedError):
        ps.SimConfig(scheme=p13, n=10, n_t=1, lam=0.7)
    with pytest.raises(ps.RadiusUnsupportedError):
        ps.two_step(np.zeros((5, 5)), np.zeros((5, 5)), p13, 0.5, "dirichlet")
    with pytest.raises(ValueError):
        ps.two_step(np.zeros((5, 5)), np.zeros((6, 6)), p5, 0.5, "dirichlet")
    assert ps.SimConfig(scheme=p5, n=10, n_t=1, lam=0.5).tau == pytest.approx(0.05)


def test_dropin_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(nat.NativeUnavailableError):
        ps.two_step(np.zeros((5, 5)), np.zeros((5, 5)), ps.named_scheme("P5"), 0.5)


def test_relative_l2_error_host():
    n, tau = 8, 0.05
    coords = np.arange(n + 1) / n
    x1, x2 = np.meshgrid(coords, coords, indexing="ij")
    fields = [2.0 * ps.exact_standing_wave(x1, x2, k * tau) for k in range(1, 4)]
    assert ps.relative_l2_error(fields, ps.exact_standing_wave, tau) == pytest.approx(1.0)
    with pytest.raises(ps.DegenerateNormError):
        ps.relative_l2_error([np.ones((5, 5))], lambda a, b, t: 0.0 * (a + b), 0.1)


def test_csv_writer_matches_numpy_savetxt(tmp_path):
    """F3: libps.so's %.17g writer produces np.savetxt's bytes (dump_grid_csv)."""
    rng = np.random.default_rng(0)
    for dt in (np.float64, np.float32):
        a = (rng.standard_normal((7, 9)) * 10.0 ** rng.integers(-30, 30, (7, 9))).astype(dt)
        a[0, 0], a[1, 1], a[2, 2], a[3, 3] = 0.0, -0.0, np.inf, np.nan
        a[4, 4] = 1e-310 if dt == np.float64 else 1e-40
        p1, p2 = tmp_path / "np.csv", tmp_path / "ps.csv"
        np.savetxt(p1, a, delimiter=",", fmt="%.17g")
        ps.dump_grid_csv(a, p2)
        assert p1.read_bytes() == p2.read_bytes()
    loaded = np.loadtxt(p2, delimiter=",")
    assert loaded.shape == (7, 9)


def test_bench_reference_arm_prints_the_gpu_arms_config():
    """`bench.py --impl reference` runs without a GPU and reports the GPU arm's own `config`
    object (same workload, same keys), its own threading under `cpu_baseline`."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                          "--config", "C1", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    sys.path.insert(0, root)
    try:
        import bench
    finally:
        sys.path.pop(0)
    cfg = bench.CONFIGS["C1"]
    assert line["config"] == bench.single_config(cfg, 1, cfg.get("tile", 0))
    assert line["impl"] == "reference" and line["gpu_launches"] == 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
