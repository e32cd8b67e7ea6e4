"""Multi-process (gloo, CPU) tests of the row-slab decomposition host logic.

The GPU path exchanges halo rows over NCCL; here the same DistributedSlabs code runs
over gloo with CPU tensors laid out exactly like device levels (ps_layout via
libps.so's host-only layout call), and a host update built on the oracle stands in
for the kernels.  The result after several steps must equal the single-grid oracle
bit for bit for every world size — which checks partitioning, neighbour choice, ghost
row offsets and the send/recv pairing.
"""

from __future__ import annotations

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1904_04048_b200 import _native as nat
from paper_1904_04048_b200.scheme import evaluate_table, named_scheme
from paper_1904_04048_b200.slab import SlabPlan, partition


class HostLevel:
    """CPU stand-in for nat.Level with the identical padded layout."""

    def __init__(self, grid):
        import ctypes

        self.grid = grid
        nbytes = nat.load_library().ps_level_bytes(ctypes.byref(grid))
        self.buf = torch.zeros(nbytes, dtype=torch.uint8)

    def view(self):
        tdt = torch.float64 if self.grid.dtype == 0 else torch.float32
        return self.buf.view(tdt).as_strided((self.grid.rows, self.grid.cols),
                                             (self.grid.pitch, 1), self.grid.origin)

    def padded(self):
        g = self.grid
        tdt = torch.float64 if g.dtype == 0 else torch.float32
        cpad = g.origin - g.ghost * g.pitch
        full = self.buf.view(tdt).view(g.rows + 2 * g.ghost, g.pitch)
        return full[:, cpad:cpad + g.cols]

    def upload(self, host):
        host = torch.from_numpy(np.ascontiguousarray(host))
        g = self.grid
        tdt = torch.float64 if g.dtype == 0 else torch.float32
        # (periodic callers may pass one alias row / column beyond the logical block)
        self.buf.view(tdt).as_strided(tuple(host.shape), (g.pitch, 1), g.origin).copy_(host)

    def fill_ghosts(self, keep_alias=False, stream=None):
        """Column images: OracleCompute wraps columns by index on the core, so the host
        stand-in has nothing to refresh (row halos come from the exchange)."""

    def download(self):
        return self.view().numpy().copy()


class OracleCompute:
    """Host update of a slab with global-index semantics, via the oracle (test only)."""

    is_cuda = False

    def __init__(self, spec, lam, tau, ring, bc="dirichlet"):
        self.two = evaluate_table(spec.two_step, lam)
        self.fu = evaluate_table(spec.first_u, lam)
        self.fv = evaluate_table(spec.first_v, lam)
        self.tau, self.ring, self.bc = tau, ring, bc

    @staticmethod
    def _tall(level):
        """Periodic slab: own rows plus all ghost rows (core columns) as a reference-layout
        array with one alias row/column appended.  The oracle wraps columns exactly and
        rows wrongly, but a wrong row wrap only reaches rows within R*steps of the top and
        bottom, i.e. ghost rows that are never taken."""
        loc = level.padded().numpy()
        out = np.zeros((loc.shape[0] + 1, loc.shape[1] + 1), dtype=loc.dtype)
        out[:-1, :-1] = loc
        return out

    def _periodic(self, fn, grid, out_levels, lo, hi):
        G = grid.ghost
        results = fn()
        for lvl, full in zip(out_levels, results):
            lvl.view()[lo:hi].copy_(torch.from_numpy(full[G + lo:G + hi, :grid.cols].copy()))

    def errsum_plan(self, rows_h, cols_h):
        return (rows_h, cols_h)

    def errsum(self, plan, grid, level, S, st, out2):
        """numpy's own pairwise sums over this slab's rows of the reference array (what the
        device plan reproduces bit for bit)."""
        rows_h, cols_h = plan
        g = grid
        tdt = torch.float64

        def block(lv):
            return lv.buf.view(tdt).as_strided((rows_h, cols_h), (g.pitch, 1), g.origin).numpy()

        u = block(level).copy()
        if self.bc == "periodic":            # alias column n = image of column 0
            u[:, cols_h - 1] = u[:, 0]
        ref = block(S) * st
        out2[0] = float(np.sum((u - ref) ** 2))
        out2[1] = float(np.sum(ref ** 2))

    @staticmethod
    def _embed(level):
        g = level.grid
        G = g.ghost
        out = np.zeros((g.grows, g.cols), dtype=np.float64 if g.dtype == 0 else np.float32)
        loc = level.padded().numpy()
        lo, hi = max(0, g.row0 - G), min(g.grows, g.row0 + g.rows + G)
        out[lo:hi] = loc[lo - (g.row0 - G):hi - (g.row0 - G)]
        return out

    def first_step(self, grid, u0, v0, out):
        from oracle import oracle as O

        if self.bc == "periodic":
            self._periodic(lambda: [O.first_step(self._tall(u0), self._tall(v0), self.fu, self.fv,
                                                 self.tau, "periodic", 0)],
                           grid, [out], 0, grid.rows)
            return
        full = O.first_step(self._embed(u0), self._embed(v0), self.fu, self.fv, self.tau,
                            "dirichlet", self.ring)
        out.view().copy_(torch.from_numpy(full[grid.row0:grid.row0 + grid.rows]))

    def two_step_rows(self, grid, uk, ukm1, out, lo, hi):
        from oracle import oracle as O

        if hi <= lo:
            return
        if self.bc == "periodic":
            self._periodic(lambda: [O.two_step(self._tall(uk), self._tall(ukm1), self.two,
                                               "periodic", 0)], grid, [out], lo, hi)
            return
        full = O.two_step(self._embed(uk), self._embed(ukm1), self.two, "dirichlet", self.ring,
                          rows=(grid.row0 + lo, grid.row0 + hi))
        out.view()[lo:hi].copy_(torch.from_numpy(full[grid.row0 + lo:grid.row0 + hi]))

    def tb_rows(self, grid, uk, ukm1, out_prev, out_last, T, lo, hi):
        """T fused updates of rows [lo, hi): T oracle steps on the embedded slab (its
        ghost rows hold the neighbours' R*T / R*(T-1) halo rows)."""
        from oracle import oracle as O

        if hi <= lo:
            return
        if self.bc == "periodic":
            self._periodic(lambda: O.march(self._tall(uk), self._tall(ukm1), self.two, T,
                                           "periodic", 0)[::-1],
                           grid, [out_prev, out_last], lo, hi)
            return
        last, prev = O.march(self._embed(uk), self._embed(ukm1), self.two, T, "dirichlet",
                             self.ring)
        a, b = grid.row0 + lo, grid.row0 + hi
        out_last.view()[lo:hi].copy_(torch.from_numpy(last[a:b]))
        out_prev.view()[lo:hi].copy_(torch.from_numpy(prev[a:b]))


def _initial(n, dtype, bc):
    rng = np.random.default_rng(42)
    npdt = np.float64 if dtype == "f64" else np.float32
    u0 = rng.normal(size=(n + 1, n + 1)).astype(npdt)
    v0 = rng.normal(size=(n + 1, n + 1)).astype(npdt)
    if bc == "periodic":
        for a in (u0, v0):
            a[:-1, -1] = a[:-1, 0]
            a[-1, :] = a[0, :]
    return u0, v0


def _shape_S(n):
    x = np.arange(n + 1) / n
    x1, x2 = np.meshgrid(x, x, indexing="ij")
    return np.sin(2.0 * np.pi * x1) * np.sin(2.0 * np.pi * x2)


def _worker(rank, world, port, scheme, n, lam, ring, steps, dtype, outdir, tsteps=1,
            bc="dirichlet", errsum=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1904_04048_b200.slab import DistributedSlabs

        spec = named_scheme(scheme)
        tau = lam / n
        slab = DistributedSlabs(spec, n, lam, ring=ring, dtype=dtype,
                                compute=OracleCompute(spec, lam, tau, ring, bc),
                                level_factory=HostLevel, tsteps=tsteps, bc=bc)
        u0, v0 = _initial(n, dtype, bc)
        p = slab.plan
        cols = n if bc == "periodic" else n + 1
        slab.load_initial(u0[p.row0:p.row0 + p.rows, :cols], v0[p.row0:p.row0 + p.rows, :cols])
        slab.first_step()
        if errsum:
            slab.load_reference_shape(_shape_S(n)[p.row0:p.row0 + slab.err_rows()])
            sums = slab.march_errsum(np.sin(0.3 * np.arange(1, steps + 1)))
            np.save(os.path.join(outdir, f"sums{rank}.npy"), sums)
        else:
            slab.march(steps)
        np.save(os.path.join(outdir, f"rank{rank}.npy"), slab.own_rows())
        np.save(os.path.join(outdir, f"prev{rank}.npy"), slab.own_rows("previous"))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,scheme,ring,dtype,tsteps", [
    (2, "P13", 2, "f64", 1), (3, "P9", 1, "f64", 1), (2, "P5", 1, "f32", 1),
    (2, "P13", 2, "f64", 2), (3, "P9", 1, "f64", 4)])
def test_distributed_slabs_gloo_bitwise(world, scheme, ring, dtype, tsteps):
    from oracle import oracle as O

    n, lam = 40, 0.4 if scheme == "P13" else 0.6
    steps = 5 if tsteps == 1 else 2 * tsteps
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(world, _free_port(), scheme, n, lam, ring, steps, dtype, tmp,
                                tsteps), nprocs=world, join=True)
        got = np.concatenate([np.load(os.path.join(tmp, f"rank{r}.npy")) for r in range(world)])
        got_prev = np.concatenate([np.load(os.path.join(tmp, f"prev{r}.npy"))
                                   for r in range(world)])
    spec = named_scheme(scheme)
    rng = np.random.default_rng(42)
    npdt = np.float64 if dtype == "f64" else np.float32
    u0 = rng.normal(size=(n + 1, n + 1)).astype(npdt)
    v0 = rng.normal(size=(n + 1, n + 1)).astype(npdt)
    u1 = O.first_step(u0, v0, evaluate_table(spec.first_u, lam), evaluate_table(spec.first_v, lam),
                      lam / n, "dirichlet", ring)
    want, want_prev = O.march(u1, u0, evaluate_table(spec.two_step, lam), steps, "dirichlet", ring)
    assert got.tobytes() == want.tobytes()
    assert got_prev.tobytes() == want_prev.tobytes()


def _reference_march(scheme, n, lam, steps, dtype, bc, ring):
    from oracle import oracle as O

    spec = named_scheme(scheme)
    u0, v0 = _initial(n, dtype, bc)
    r = ring if bc == "dirichlet" else 0
    u1 = O.first_step(u0, v0, evaluate_table(spec.first_u, lam), evaluate_table(spec.first_v, lam),
                      lam / n, bc, r)
    return u0, u1, evaluate_table(spec.two_step, lam), r


@pytest.mark.parametrize("world,scheme,dtype,tsteps", [
    (2, "P9", "f64", 1), (3, "P13", "f64", 1), (4, "P5", "f32", 1), (2, "P13", "f64", 2),
    (3, "P9", "f64", 3)])
def test_periodic_ring_slabs_gloo_bitwise(world, scheme, dtype, tsteps):
    """Periodic grids as a ring of slabs (rank 0 <-> rank P-1, columns wrap locally); a
    ring of two slabs has up == down, so the message pairing by tag/order is exercised."""
    from oracle import oracle as O

    n, lam = 36, 0.4 if scheme == "P13" else 0.6
    steps = 5 if tsteps == 1 else 2 * tsteps
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(world, _free_port(), scheme, n, lam, 0, steps, dtype, tmp, tsteps,
                                "periodic"), nprocs=world, join=True)
        got = np.concatenate([np.load(os.path.join(tmp, f"rank{r}.npy")) for r in range(world)])
        got_prev = np.concatenate([np.load(os.path.join(tmp, f"prev{r}.npy"))
                                   for r in range(world)])
    u0, u1, two, _ = _reference_march(scheme, n, lam, steps, dtype, "periodic", 0)
    want, want_prev = O.march(u1, u0, two, steps, "periodic", 0)
    assert got.tobytes() == want[:n, :n].tobytes()
    assert got_prev.tobytes() == want_prev[:n, :n].tobytes()


@pytest.mark.parametrize("world,bc", [(2, "dirichlet"), (3, "dirichlet"), (2, "periodic"),
                                      (3, "periodic")])
def test_distributed_error_sums_gloo(world, bc):
    """run()'s per-step error sums across slabs: every rank returns the same array, equal
    to the per-slab numpy sums added in rank order (bitwise), and to the whole-grid numpy
    sums within rounding."""
    from oracle import oracle as O

    scheme, n, lam, steps = "P9", 30, 0.6, 4
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(world, _free_port(), scheme, n, lam, 1, steps, "f64", tmp, 1, bc,
                                True), nprocs=world, join=True)
        sums = [np.load(os.path.join(tmp, f"sums{r}.npy")) for r in range(world)]
    for other in sums[1:]:
        assert other.tobytes() == sums[0].tobytes()
    u0, u1, two, ring = _reference_march(scheme, n, lam, steps, "f64", bc, 1)
    S = _shape_S(n)
    cur, prev = u1, u0
    parts = partition(n if bc == "periodic" else n + 1, world)
    for k in range(steps):
        cur, prev = O.two_step(cur, prev, two, bc, ring), cur
        ref = S * np.sin(0.3 * (k + 1))
        whole = np.array([np.sum((cur - ref) ** 2), np.sum(ref ** 2)])
        acc = None
        for p, (row0, rows) in enumerate(parts):
            hi = row0 + rows + (1 if bc == "periodic" and p == world - 1 else 0)
            part = np.array([np.sum((cur[row0:hi] - ref[row0:hi]) ** 2), np.sum(ref[row0:hi] ** 2)])
            acc = part if acc is None else acc + part
        assert sums[0][k].tobytes() == acc.tobytes()
        assert sums[0][k] == pytest.approx(whole, rel=1e-13)


def test_partition_and_plans():
    assert partition(10, 3) == [(0, 4), (4, 3), (7, 3)]
    assert sum(r for _, r in partition(32768, 8)) == 32768
    with pytest.raises(ValueError):
        partition(3, 4)
    plans = [SlabPlan.build(100, 4, r, 2, periodic=False) for r in range(4)]
    assert plans[0].up is None and plans[-1].down is None
    # every send pairs with exactly one recv of the same size on the peer
    for pl in plans:
        for msg in pl.sends:
            other = plans[msg.peer]
            assert (pl.rank, msg.rows, msg.tag) in [(m.peer, m.rows, m.tag) for m in other.recvs]
    ring = [SlabPlan.build(100, 4, r, 1, periodic=True) for r in range(4)]
    assert ring[0].up == 3 and ring[3].down == 0
    # a ring of two: both neighbours are the same rank; the k-th send to it pairs with its
    # k-th recv from me (same tag, opposite sides)
    two = [SlabPlan.build(10, 2, r, 2, periodic=True) for r in range(2)]
    for me, other in ((two[0], two[1]), (two[1], two[0])):
        assert me.up == me.down == other.rank
        assert [m.tag for m in me.sends] == [m.tag for m in other.recvs]
        for snd, rcv in zip(me.sends, other.recvs):
            assert snd.side != rcv.side
            assert me.send_rows(snd, 2) == (0 if snd.side == "up" else me.rows - 2)
            assert other.recv_rows(rcv, 2) == (-2 if rcv.side == "up" else other.rows)
    with pytest.raises(ValueError):
        SlabPlan.build(10, 8, 7, 2, periodic=False)
