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
        self.view().copy_(torch.from_numpy(np.ascontiguousarray(host)))

    def download(self):
        return self.view().numpy().copy()


class OracleCompute:
    """Host update of a slab with global-index semantics, via the oracle (test only)."""

    is_cuda = False

    def __init__(self, spec, lam, tau, ring):
        self.two = evaluate_table(spec.two_step, lam)
        self.fu = evaluate_table(spec.first_u, lam)
        self.fv = evaluate_table(spec.first_v, lam)
        self.tau, self.ring = tau, ring

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

        full = O.first_step(self._embed(u0), self._embed(v0), self.fu, self.fv, self.tau,
                            "dirichlet", self.ring)
        out.view().copy_(torch.from_numpy(full[grid.row0:grid.row0 + grid.rows]))

    def two_step_rows(self, grid, uk, ukm1, out, lo, hi):
        from oracle import oracle as O

        if hi <= lo:
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
        last, prev = O.march(self._embed(uk), self._embed(ukm1), self.two, T, "dirichlet",
                             self.ring)
        a, b = grid.row0 + lo, grid.row0 + hi
        out_last.view()[lo:hi].copy_(torch.from_numpy(last[a:b]))
        out_prev.view()[lo:hi].copy_(torch.from_numpy(prev[a:b]))


def _worker(rank, world, port, scheme, n, lam, ring, steps, dtype, outdir, tsteps=1):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1904_04048_b200.slab import DistributedSlabs

        spec = named_scheme(scheme)
        tau = lam / n
        slab = DistributedSlabs(spec, n, lam, ring=ring, dtype=dtype,
                                compute=OracleCompute(spec, lam, tau, ring),
                                level_factory=HostLevel, tsteps=tsteps)
        rng = np.random.default_rng(42)
        npdt = np.float64 if dtype == "f64" else np.float32
        u0 = rng.normal(size=(n + 1, n + 1)).astype(npdt)
        v0 = rng.normal(size=(n + 1, n + 1)).astype(npdt)
        p = slab.plan
        slab.load_initial(u0[p.row0:p.row0 + p.rows], v0[p.row0:p.row0 + p.rows])
        slab.first_step()
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


def test_partition_and_plans():
    assert partition(10, 3) == [(0, 4), (4, 3), (7, 3)]
    assert sum(r for _, r in partition(32768, 8)) == 32768
    with pytest.raises(ValueError):
        partition(3, 4)
    plans = [SlabPlan.build(100, 4, r, 2, periodic=False) for r in range(4)]
    assert plans[0].up is None and plans[-1].down is None
    # every send pairs with exactly one recv of the same size on the peer
    for pl in plans:
        for peer, first, count in pl.sends:
            other = plans[peer]
            assert (pl.rank, count) in [(q, c) for q, _, c in other.recvs]
    ring = [SlabPlan.build(100, 4, r, 1, periodic=True) for r in range(4)]
    assert ring[0].up == 3 and ring[3].down == 0
    with pytest.raises(ValueError):
        SlabPlan.build(10, 8, 7, 2, periodic=False)
