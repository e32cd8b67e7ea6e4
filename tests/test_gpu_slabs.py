"""GPU tests of the row-slab decomposition driving the real kernels.

* periodic ring slabs and the distributed error sums with P virtual slabs on one device;
* TWO PROCESSES sharing cuda:0 under a gloo group: ``DistributedSlabs`` with libps.so's
  kernels and a real cross-process transport — halo rows through send/recv (host-staged
  under gloo; NCCL cannot place two ranks on one device), or stored into the neighbour
  process's ghost rows by the update kernel through CUDA IPC, ordered by host tokens.
  No kernel ever waits on another process's kernel (the hosts wait), so this is safe on one
  GPU; on a multi-GPU box the same code runs over NCCL / NVLink;
* one distributed pass captured in a CUDA graph and replayed (NCCL group of one rank).

Everything is compared bit for bit with the CPU oracle.
"""

from __future__ import annotations

import os
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def pairs(spec, role, lam):
    from paper_1904_04048_b200.scheme import evaluate_table

    return evaluate_table(getattr(spec, role), lam)


def same_bits(a, b):
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes() == b.tobytes()


def initial(n, dtype, bc, seed=42):
    rng = np.random.default_rng(seed)
    npdt = np.float64 if dtype == "f64" else np.float32
    u0 = rng.normal(size=(n + 1, n + 1)).astype(npdt)
    v0 = rng.normal(size=(n + 1, n + 1)).astype(npdt)
    if bc == "periodic":
        for a in (u0, v0):
            a[:-1, -1] = a[:-1, 0]
            a[-1, :] = a[0, :]
    return u0, v0


def oracle_march(scheme, n, lam, steps, dtype, bc, ring, arith="ref"):
    from oracle import oracle as O
    from paper_1904_04048_b200.scheme import named_scheme

    spec = named_scheme(scheme)
    u0, v0 = initial(n, dtype, bc)
    r = ring if bc == "dirichlet" else 0
    u1 = O.first_step(u0, v0, pairs(spec, "first_u", lam), pairs(spec, "first_v", lam), lam / n,
                      bc, r, arith)
    if steps == 0:
        return u1, u0
    return O.march(u1, u0, pairs(spec, "two_step", lam), steps, bc, r, arith)


def shape_S(n):
    x = np.arange(n + 1) / n
    x1, x2 = np.meshgrid(x, x, indexing="ij")
    return np.sin(2.0 * np.pi * x1) * np.sin(2.0 * np.pi * x2)


# ---------------------------------------------------------------- virtual slabs, one process
@pytest.mark.parametrize("scheme,dtype,arith", [("P9", "f64", "ref"), ("P13", "f64", "ref"),
                                                ("P13", "f32", "native"), ("P5", "f32", "ref")])
@pytest.mark.parametrize("tsteps", [1, 2, 3, 4])
def test_periodic_ring_virtual_slabs_bitwise(scheme, dtype, arith, tsteps):
    """Periodic grids as a ring of P slabs (rank 0 <-> P-1 halos, columns wrap locally):
    bitwise equal to the oracle's periodic march for P in {1,2,3,4}."""
    from paper_1904_04048_b200.slab import VirtualSlabs

    n = 600
    lam = 0.4 if scheme == "P13" else 0.6
    steps = 5 if tsteps == 1 else 3 * tsteps
    u0, v0 = initial(n, dtype, "periodic")
    want, _ = oracle_march(scheme, n, lam, steps, dtype, "periodic", 0, arith)
    for P in (1, 2, 3, 4):
        vs = VirtualSlabs(scheme, n, lam, P, dtype=dtype, arith=arith, tsteps=tsteps,
                          bc="periodic")
        vs.load_initial(u0, v0)
        vs.first_step()
        vs.march(steps)
        assert same_bits(vs.field(), want), P


@pytest.mark.parametrize("bc", ["dirichlet", "periodic"])
def test_virtual_slab_error_sums(bc):
    """Per-step error sums across slabs: P = 1 gives run()'s device sums (numpy's pairwise
    order over the whole array, bit for bit); P > 1 equals the per-slab numpy sums added in
    slab order (bitwise) and the whole-grid sums within rounding."""
    from oracle import oracle as O
    from paper_1904_04048_b200.scheme import named_scheme
    from paper_1904_04048_b200.slab import VirtualSlabs, partition

    scheme, n, lam, steps = "P9", 301, 0.6, 5
    spec = named_scheme(scheme)
    u0, v0 = initial(n, "f64", bc)
    S = shape_S(n)
    st = np.sin(0.3 * np.arange(1, steps + 1))
    u1, _ = oracle_march(scheme, n, lam, 0, "f64", bc, 1)
    fields = []
    cur, prev = u1, u0
    ring = 1 if bc == "dirichlet" else 0
    for _ in range(steps):
        cur, prev = O.two_step(cur, prev, pairs(spec, "two_step", lam), bc, ring), cur
        fields.append(cur)
    for P in (1, 2, 3, 4):
        vs = VirtualSlabs(scheme, n, lam, P, ring=1, bc=bc)
        vs.load_initial(u0, v0)
        vs.first_step()
        vs.load_reference_shape(S)
        got = vs.march_errsum(st)
        parts = partition(n if bc == "periodic" else n + 1, P)
        for k in range(steps):
            ref = S * st[k]
            acc = None
            for p, (row0, rows) in enumerate(parts):
                hi = row0 + rows + (1 if bc == "periodic" and p == P - 1 else 0)
                part = np.array([np.sum((fields[k][row0:hi] - ref[row0:hi]) ** 2),
                                 np.sum(ref[row0:hi] ** 2)])
                acc = part if acc is None else acc + part
            whole = np.array([np.sum((fields[k] - ref) ** 2), np.sum(ref ** 2)])
            assert got[k].tobytes() == acc.tobytes(), (P, k)
            assert got[k] == pytest.approx(whole, rel=1e-13)
            if P == 1:
                assert got[k].tobytes() == whole.tobytes()


# ---------------------------------------------------------------- two processes, one GPU
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, scheme, n, lam, ring, steps, dtype, arith, tsteps, bc, transport,
          errsum, outdir):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1904_04048_b200 import _native as nat
        from paper_1904_04048_b200.slab import DistributedSlabs

        before = nat.launch_count()
        slab = DistributedSlabs(scheme, n, lam, ring=ring, dtype=dtype, arith=arith,
                                transport=transport, tsteps=tsteps, bc=bc)
        u0, v0 = initial(n, dtype, bc)
        p = slab.plan
        cols = n if bc == "periodic" else n + 1
        slab.load_initial(u0[p.row0:p.row0 + p.rows, :cols], v0[p.row0:p.row0 + p.rows, :cols])
        slab.first_step()
        if errsum:
            slab.load_reference_shape(shape_S(n)[p.row0:p.row0 + slab.err_rows()])
            sums = slab.march_errsum(np.sin(0.3 * np.arange(1, steps + 1)))
            np.save(os.path.join(outdir, f"sums{rank}.npy"), sums)
        else:
            slab.march(steps)
        torch.cuda.synchronize()
        dist.barrier()          # neighbours' last in-kernel halo stores have landed
        np.save(os.path.join(outdir, f"rank{rank}.npy"), slab.own_rows())
        np.save(os.path.join(outdir, f"prev{rank}.npy"), slab.own_rows("previous"))
        np.save(os.path.join(outdir, f"launches{rank}.npy"),
                np.array([nat.launch_count() - before]))
        slab.close()
    finally:
        dist.destroy_process_group()


def _spawn(world, *args):
    import torch.multiprocessing as mp

    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_rank, args=(world, _free_port(), *args, tmp), nprocs=world, join=True)
        load = lambda name: [np.load(os.path.join(tmp, f"{name}{r}.npy"))  # noqa: E731
                             for r in range(world) if os.path.exists(os.path.join(tmp, f"{name}{r}.npy"))]
        return load("rank"), load("prev"), load("sums"), load("launches")


@pytest.mark.parametrize("world,scheme,dtype,arith,tsteps,bc,transport", [
    (2, "P9", "f64", "ref", 1, "dirichlet", "nccl"),
    (2, "P9", "f64", "ref", 1, "dirichlet", "p2p"),
    (2, "P13", "f64", "ref", 2, "dirichlet", "p2p"),
    (3, "P13", "f32", "native", 4, "dirichlet", "p2p"),
    (2, "P9", "f64", "ref", 4, "dirichlet", "nccl"),
    (2, "P9", "f64", "ref", 5, "dirichlet", "p2p"),
    (3, "P13", "f64", "ref", 1, "periodic", "nccl"),
    (2, "P9", "f64", "ref", 2, "periodic", "nccl"),
])
def test_two_processes_one_gpu_real_kernels(world, scheme, dtype, arith, tsteps, bc, transport):
    """DistributedSlabs with libps.so's kernels across processes: overlapped boundary /
    exchange / interior passes, both transports, bitwise equal to the single-grid oracle."""
    n = 700
    lam = 0.4 if scheme == "P13" else 0.6
    ring = 2 if scheme == "P13" else 1
    steps = 6 if tsteps == 1 else 3 * tsteps
    own, prev, _, launches = _spawn(world, scheme, n, lam, ring, steps, dtype, arith, tsteps, bc,
                                    transport, False)
    want, want_prev = oracle_march(scheme, n, lam, steps, dtype, bc, ring, arith)
    if bc == "periodic":
        want, want_prev = want[:n, :n], want_prev[:n, :n]
    assert same_bits(np.concatenate(own), np.ascontiguousarray(want))
    assert same_bits(np.concatenate(prev), np.ascontiguousarray(want_prev))
    assert all(int(x[0]) > 0 for x in launches)     # the kernels ran in every process


def test_two_processes_distributed_error_sums():
    from oracle import oracle as O
    from paper_1904_04048_b200.scheme import named_scheme
    from paper_1904_04048_b200.slab import partition

    scheme, n, lam, steps, world = "P9", 400, 0.6, 4, 2
    _, _, sums, _ = _spawn(world, scheme, n, lam, 1, steps, "f64", "ref", 1, "dirichlet", "nccl",
                           True)
    assert sums[0].tobytes() == sums[1].tobytes()
    spec = named_scheme(scheme)
    u0, _ = initial(n, "f64", "dirichlet")
    u1, _ = oracle_march(scheme, n, lam, 0, "f64", "dirichlet", 1)
    S = shape_S(n)
    cur, prev = u1, u0
    for k in range(steps):
        cur, prev = O.two_step(cur, prev, pairs(spec, "two_step", lam), "dirichlet", 1), cur
        ref = S * np.sin(0.3 * (k + 1))
        acc = None
        for row0, rows in partition(n + 1, world):
            part = np.array([np.sum((cur[row0:row0 + rows] - ref[row0:row0 + rows]) ** 2),
                             np.sum(ref[row0:row0 + rows] ** 2)])
            acc = part if acc is None else acc + part
        assert sums[0][k].tobytes() == acc.tobytes(), k


# ---------------------------------------------------------------- CUDA-graph replay of a pass
@pytest.mark.parametrize("tsteps", [1, 4])
def test_distributed_pass_cuda_graph_replay(tsteps):
    """One distributed pass captured per rotation phase and replayed (NCCL group of one
    rank: the pass holds the kernels; with neighbours it also holds the send/recv and the
    cross-stream events): same bits as the eager march."""
    import torch
    import torch.distributed as dist

    from paper_1904_04048_b200.slab import DistributedSlabs

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    try:
        n, lam, steps = 900, 0.6, 12
        u0, v0 = initial(n, "f64", "dirichlet")
        res = {}
        for graph in (False, True):
            slab = DistributedSlabs("P9", n, lam, ring=1, tsteps=tsteps, graph=graph)
            slab.load_initial(u0, v0)
            slab.first_step()
            slab.march(steps)
            res[graph] = (slab.own_rows(), slab.own_rows("previous"))
            assert slab.graphed == graph, slab.graph_error
        assert same_bits(res[True][0], res[False][0])
        assert same_bits(res[True][1], res[False][1])
        want, _ = oracle_march("P9", n, lam, steps, "f64", "dirichlet", 1)
        assert same_bits(res[True][0], want)
    finally:
        dist.destroy_process_group()
