"""Tile-resident march (ps_march_tile, csrc/ps_tile.cuh) against the CPU oracle and the
streaming march, bit for bit (reference: run()'s loop of two_step calls,
simulator.py:271-274, per-point arithmetic simulator.py:147-160, 183-191)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _oracle_march(sim, u0, v0, nsteps):
    from oracle import oracle as O
    from paper_1904_04048_b200.scheme import evaluate_table

    spec, lam = sim.spec, sim.lam
    tu = evaluate_table(spec.first_u, lam)
    tv = evaluate_table(spec.first_v, lam)
    t2 = evaluate_table(spec.two_step, lam)
    prev = u0
    cur = O.first_step(u0, v0, tu, tv, sim.tau, "dirichlet", ring=sim.ring)
    for _ in range(nsteps):
        prev, cur = cur, O.two_step(cur, prev, t2, "dirichlet", ring=sim.ring)
    return cur, prev


def _fields(n, seed):
    rng = np.random.default_rng(seed)
    u0 = rng.standard_normal((n + 1, n + 1))
    v0 = rng.standard_normal((n + 1, n + 1))
    return u0, v0


@pytest.mark.parametrize("scheme,ring", [("P5", 1), ("P9", 1), ("C9", 1), ("P13", 2)])
@pytest.mark.parametrize("n,tile,nsteps", [(64, 1, 5), (97, 3, 10), (200, 4, 13), (512, 8, 40),
                                           (333, 16, 35)])
def test_tile_march_equals_oracle(scheme, ring, n, tile, nsteps):
    from paper_1904_04048_b200 import _native as nat
    from paper_1904_04048_b200.device import Simulation

    sim = Simulation(scheme, n, 0.5 if scheme != "P13" else 0.4, bc="dirichlet", ring=ring, tile=tile)
    u0, v0 = _fields(n, seed=n + tile)
    for a in (u0, v0):   # the oracle zeroes nothing itself: start from a pinned ring
        a[:ring, :] = a[-ring:, :] = 0.0
        a[:, :ring] = a[:, -ring:] = 0.0
    sim.load_initial(u0, v0)
    sim.first_step()
    if not nat.tile_supported(sim.grid, sim.t_two, tile):
        pytest.skip("no tiling of this grid fits at this depth")
    sim.march(nsteps)
    cur, prev = _oracle_march(sim, u0, v0, nsteps)
    got_cur = sim.levels[sim.newest].download()
    got_prev = sim.levels[sim.previous].download()
    assert got_cur.tobytes() == cur.tobytes()
    assert got_prev.tobytes() == prev.tobytes()


def test_tile_march_equals_streaming_march_c1():
    """BASELINE config 1 (P5, 512^2, 200 steps): tile-resident = CUDA-graph march, bitwise;
    a second call continues from the rotated levels."""
    from paper_1904_04048_b200.device import Simulation

    a = Simulation("P5", 512, 0.5, tile=8)
    b = Simulation("P5", 512, 0.5)
    for s in (a, b):
        s.gaussian_initial(1, 0.05, 0.05, seed=3)
        s.first_step()
    a.march(120)
    a.march(79)
    b.march(199)
    assert a.levels[a.newest].download().tobytes() == b.levels[b.newest].download().tobytes()
    assert a.levels[a.previous].download().tobytes() == b.levels[b.previous].download().tobytes()


@pytest.mark.parametrize("scheme", ["P5", "P9", "P13"])
@pytest.mark.parametrize("n,tile,nsteps", [(96, 4, 17), (250, 8, 30), (512, 12, 50), (61, 16, 33)])
def test_tile_march_periodic_equals_streaming_march(scheme, n, tile, nsteps):
    """Periodic grids: tiles form a ring, halos wrap around the core; the tile-resident
    march equals the streaming march (itself pinned to the oracle and the reference's golden
    calls by tests/test_gpu_parity.py) on both live levels, alias row/column included."""
    from paper_1904_04048_b200 import _native as nat
    from paper_1904_04048_b200.device import Simulation

    lam = 0.4 if scheme == "P13" else 0.6
    a = Simulation(scheme, n, lam, bc="periodic", tile=tile)
    b = Simulation(scheme, n, lam, bc="periodic")
    for s in (a, b):
        s.standing_wave_initial(2, 3)
        s.first_step()
    if not nat.tile_supported(a.grid, a.t_two, tile):
        pytest.skip("no tiling of this grid fits at this depth")
    a.march(nsteps)
    b.march(nsteps)
    assert a._tile_ok is True
    n1 = n + 1
    for la, lb in ((a.newest, b.newest), (a.previous, b.previous)):
        assert a.levels[la].download(n1, n1).tobytes() == b.levels[lb].download(n1, n1).tobytes()
    # and the images are live again: one more streaming update on top of the tile march
    a.newest, a.previous = nat.march_tb(a.grid, a.levels, 3, a.t_two, 1, a.newest, a.previous)
    b.march(3)
    assert a.levels[a.newest].download(n1, n1).tobytes() == b.levels[b.newest].download(n1, n1).tobytes()


def test_tile_march_periodic_equals_oracle():
    from oracle import oracle as O
    from paper_1904_04048_b200.device import Simulation
    from paper_1904_04048_b200.scheme import evaluate_table

    n, nsteps = 128, 21
    sim = Simulation("P9", n, 0.6, bc="periodic", tile=6)
    rng = np.random.default_rng(5)
    u0 = rng.standard_normal((n + 1, n + 1))
    v0 = rng.standard_normal((n + 1, n + 1))
    for f in (u0, v0):
        f[:-1, -1] = f[:-1, 0]
        f[-1, :] = f[0, :]
    sim.load_initial(u0, v0)
    sim.first_step()
    sim.march(nsteps)
    tu = evaluate_table(sim.spec.first_u, sim.lam)
    tv = evaluate_table(sim.spec.first_v, sim.lam)
    t2 = evaluate_table(sim.spec.two_step, sim.lam)
    prev, cur = u0, O.first_step(u0, v0, tu, tv, sim.tau, "periodic")
    for _ in range(nsteps):
        prev, cur = cur, O.two_step(cur, prev, t2, "periodic")
    assert sim._tile_ok is True
    assert sim.levels[sim.newest].download(n + 1, n + 1).tobytes() == cur.tobytes()


def test_tile_march_falls_back_when_unsupported():
    """f32 grids do not qualify: march() takes the streaming path and still matches."""
    from paper_1904_04048_b200.device import Simulation

    a = Simulation("P9", 96, 0.5, bc="periodic", dtype="f32", arith="native", tile=4)
    b = Simulation("P9", 96, 0.5, bc="periodic", dtype="f32", arith="native")
    for s in (a, b):
        s.standing_wave_initial(1, 2)
        s.first_step()
        s.march(17)
    assert a._tile_ok is False
    assert a.levels[a.newest].download().tobytes() == b.levels[b.newest].download().tobytes()
