"""Row-slab domain decomposition.

The two-step update reads only an r-neighbourhood, so the global grid splits into P
contiguous row slabs with one halo exchange per step: each slab sends its first r rows
of the newest level to the slab above and its last r rows to the slab below, where
they land in the ghost padding rows (-r..-1 / rows..rows+r-1) the kernels already read.
Per-point arithmetic is unchanged, so results are bitwise independent of P.

* :func:`partition`, :class:`SlabPlan` — pure host logic (who owns which rows, which
  rows go where), shared by every transport.
* :class:`VirtualSlabs` — P slabs on ONE device, halo rows moved by device copies.
  Tests the decomposition bit for bit without more GPUs.
* :class:`DistributedSlabs` — one slab per rank (torchrun, one process per GPU),
  halo rows exchanged with NCCL send/recv on a communication stream while the
  interior rows update (boundary rows first, then exchange || interior).

The reference has no parallel path; its spec permits row partitioning that is
bitwise deterministic for a fixed partition count.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .scheme import SchemeSpec, evaluate_table, named_scheme


def partition(grows: int, P: int) -> list[tuple[int, int]]:
    """P contiguous (row0, rows) slabs covering [0, grows), sizes differing by <= 1."""
    if P < 1 or P > grows:
        raise ValueError(f"cannot split {grows} rows into {P} slabs")
    base, extra = divmod(grows, P)
    out, row0 = [], 0
    for p in range(P):
        rows = base + (1 if p < extra else 0)
        out.append((row0, rows))
        row0 += rows
    return out


@dataclass(frozen=True)
class SlabPlan:
    """Halo traffic of one slab: ``sends``/``recvs`` are (peer, first_local_row, nrows).

    A send of local rows [a, a+r) to ``peer`` pairs with that peer's recv into its
    ghost rows.  Dirichlet grids are a line (no wrap); periodic grids are a ring."""

    rank: int
    P: int
    row0: int
    rows: int
    halo: int
    up: int | None
    down: int | None
    sends: tuple[tuple[int, int, int], ...]
    recvs: tuple[tuple[int, int, int], ...]

    @staticmethod
    def build(grows: int, P: int, rank: int, halo: int, periodic: bool) -> "SlabPlan":
        parts = partition(grows, P)
        row0, rows = parts[rank]
        if rows < halo:
            raise ValueError(f"slab of {rows} rows is thinner than the halo {halo}")
        up = rank - 1 if rank > 0 else (P - 1 if periodic and P > 1 else None)
        down = rank + 1 if rank < P - 1 else (0 if periodic and P > 1 else None)
        sends, recvs = [], []
        if up is not None:
            sends.append((up, 0, halo))              # my top rows -> up's bottom ghosts
            recvs.append((up, -halo, halo))          # up's bottom rows -> my top ghosts
        if down is not None:
            sends.append((down, rows - halo, halo))  # my bottom rows -> down's top ghosts
            recvs.append((down, rows, halo))         # down's top rows -> my bottom ghosts
        return SlabPlan(rank, P, row0, rows, halo, up, down, tuple(sends), tuple(recvs))


def rows_view(level: nat.Level, first: int, count: int):
    """Flat torch view of ``count`` full-pitch rows starting at logical row ``first``
    (may be negative: ghost rows).  Rows are contiguous in the padded layout."""
    g = level.grid
    flat = level.buf.view(level.view().dtype)
    start = (g.ghost + first) * g.pitch
    return flat[start:start + count * g.pitch]


class VirtualSlabs:
    """P Dirichlet row slabs of one (n+1)^2 grid on one device (test vehicle).

    ``transport="copy"`` moves halo rows with device copies after each step;
    ``transport="kernel"`` has each slab's update kernel store its boundary rows straight
    into the neighbours' ghost rows (``ps_two_step_halo``) — the same code path the
    multi-GPU p2p transport drives with peer-mapped pointers."""

    def __init__(self, scheme, n: int, lam: float, P: int, ring: int | None = None,
                 dtype: str = "f64", arith: str = "ref", c: float = 1.0,
                 transport: str = "copy", tsteps: int = 1):
        if transport not in ("copy", "kernel"):
            raise ValueError(f"transport must be 'copy' or 'kernel', got {transport!r}")
        if tsteps not in (1, 2, 4):
            raise ValueError(f"tsteps must be 1, 2 or 4, got {tsteps}")
        self.transport = transport
        self.T = int(tsteps)
        self.spec: SchemeSpec = named_scheme(scheme) if isinstance(scheme, str) else scheme
        self.n, self.lam, self.P = int(n), float(lam), int(P)
        self.tau = self.lam / self.n / c
        R = self.spec.radius
        self.R = R
        self.ring = R if ring is None else int(ring)
        grows = self.n + 1
        H = R * self.T
        self.plans = [SlabPlan.build(grows, P, p, H, periodic=False) for p in range(P)]
        self.grids = [nat.make_slab_grid(grows, grows, pl.row0, pl.rows, max(2, H), self.ring,
                                         "dirichlet", dtype, arith) for pl in self.plans]
        self.levels = [[nat.Level(g) for _ in range(3 if self.T == 1 else 4)]
                       for g in self.grids]
        self.previous = None
        self.t_u = nat.make_table(evaluate_table(self.spec.first_u, self.lam))
        self.t_v = nat.make_table(evaluate_table(self.spec.first_v, self.lam))
        self.t_two = nat.make_table(evaluate_table(self.spec.two_step, self.lam))
        self.newest = None

    def _exchange(self, idx: int, count: int | None = None):
        for p, pl in enumerate(self.plans):
            for peer, first, halo in pl.sends:
                k = halo if count is None else count
                src_first = 0 if first == 0 else pl.rows - k
                dst_first = -k if peer > p else self.plans[peer].rows
                rows_view(self.levels[peer][idx], dst_first, k).copy_(
                    rows_view(self.levels[p][idx], src_first, k))

    def load_initial(self, u0: np.ndarray, v0: np.ndarray):
        for pl, lv in zip(self.plans, self.levels):
            lv[1].upload(u0[pl.row0:pl.row0 + pl.rows])
            lv[0].upload(v0[pl.row0:pl.row0 + pl.rows])
        self._exchange(1)
        self._exchange(0)

    def first_step(self):
        for g, lv in zip(self.grids, self.levels):
            nat.first_step(g, lv[1], lv[0], lv[2], self.t_u, self.t_v, self.tau)
        self._exchange(2)
        self.newest, self.previous = 2, 1

    def _march_blocked(self, nsteps: int):
        """Fused passes of T updates; halos of both output levels by device copies or by
        the fused kernel's own stores into the neighbours' ghost rows."""
        if nsteps % self.T:
            raise ValueError(f"nsteps={nsteps} must be a multiple of tsteps={self.T}")
        T, R = self.T, self.R
        for _ in range(nsteps // T):
            cur, prev = self.newest, self.previous
            f1, f2 = [x for x in range(4) if x not in (cur, prev)]
            for p, (g, lv) in enumerate(zip(self.grids, self.levels)):
                if self.transport == "copy":
                    nat.two_step_tb_rows(g, lv[cur], lv[prev], lv[f1], lv[f2], self.t_two, T, 0,
                                         g.rows)
                    continue
                up = ((self.levels[p - 1][f1].ptr.value, self.levels[p - 1][f2].ptr.value)
                      if p > 0 else None)
                dn = ((self.levels[p + 1][f1].ptr.value, self.levels[p + 1][f2].ptr.value)
                      if p + 1 < self.P else None)
                up_rows = self.plans[p - 1].rows if p > 0 else 0
                nat.two_step_tb_halo(g, lv[cur], lv[prev], lv[f1], lv[f2], self.t_two, T, 0,
                                     g.rows, up, up_rows, dn)
            if self.transport == "copy":
                self._exchange(f2, R * T)
                self._exchange(f1, R * (T - 1))
            self.newest, self.previous = f2, f1

    def march(self, nsteps: int):
        if self.T > 1:
            self._march_blocked(nsteps)
            return
        for _ in range(nsteps):
            cur = self.newest
            nxt, prev = (cur + 1) % 3, (cur + 2) % 3
            R = self.R
            for p, (g, lv) in enumerate(zip(self.grids, self.levels)):
                if self.transport == "copy":
                    nat.two_step(g, lv[cur], lv[prev], lv[nxt], self.t_two)
                    continue
                up = self.levels[p - 1][nxt].ptr.value if p > 0 else None
                dn = self.levels[p + 1][nxt].ptr.value if p + 1 < self.P else None
                up_rows = self.plans[p - 1].rows if p > 0 else 0
                nat.two_step_halo(g, lv[cur], lv[prev], lv[nxt], self.t_two, 0, g.rows, up,
                                  up_rows, dn)
            if self.transport == "copy":
                self._exchange(nxt, R)
            self.newest, self.previous = nxt, cur

    def field(self) -> np.ndarray:
        return np.concatenate([lv[self.newest].download() for lv in self.levels], axis=0)


class DistributedSlabs:
    """This rank's Dirichlet row slab of an (n+1)^2 grid; halo exchange over
    ``torch.distributed`` (NCCL on GPUs) overlapped with the interior update.

    ``compute`` supplies the per-slab updates (``first_step(grid, u0, v0, out)`` and
    ``two_step_rows(grid, uk, ukm1, out, lo, hi)``); the default is libps.so's kernels.
    The multi-process CPU tests substitute a host implementation to check the
    exchange logic under gloo."""

    def __init__(self, scheme, n: int, lam: float, ring: int | None = None, dtype: str = "f64",
                 arith: str = "ref", c: float = 1.0, group=None, device=None, compute=None,
                 level_factory=None, transport: str = "nccl", tsteps: int = 1):
        import torch.distributed as dist

        if transport not in ("nccl", "p2p"):
            raise ValueError(f"transport must be 'nccl' or 'p2p', got {transport!r}")
        if tsteps not in (1, 2, 4):
            raise ValueError(f"tsteps must be 1, 2 or 4, got {tsteps}")
        self.transport = transport
        # Temporal blocking depth T: one pass advances T steps, so the halo is R*T rows of
        # the newest level and R*(T-1) rows of the one before.
        self.T = int(tsteps)
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.P = dist.get_world_size(group)
        self.spec: SchemeSpec = named_scheme(scheme) if isinstance(scheme, str) else scheme
        self.n, self.lam = int(n), float(lam)
        self.tau = self.lam / self.n / c
        R = self.spec.radius
        self.R = R
        self.ring = R if ring is None else int(ring)
        grows = self.n + 1
        self.grows = grows
        self.plan = SlabPlan.build(grows, self.P, self.rank, R * self.T, periodic=False)
        self.grid = nat.make_slab_grid(grows, grows, self.plan.row0, self.plan.rows,
                                       max(2, R * self.T), self.ring, "dirichlet", dtype, arith)
        make = level_factory or (lambda g: nat.Level(g, device=device))
        self.levels = [make(self.grid) for _ in range(3 if self.T == 1 else 4)]
        self.previous = None
        self.compute = compute or _KernelCompute(self.spec, self.lam, self.tau)
        self.newest = None
        self._streams = None
        self._peer = None
        if transport == "p2p":
            self._open_peers()

    # -- p2p transport: neighbours' levels mapped through CUDA IPC ------------------------
    def _open_peers(self):
        """Exchange IPC handles of the levels; map the up/down neighbours' levels."""
        mine = [nat.ipc_handle(lv.ptr.value) for lv in self.levels]
        allh = [None] * self.P
        self.dist.all_gather_object(allh, (self.plan.rows, mine), group=self.group)
        peer = {"up": None, "dn": None, "up_rows": 0, "opened": []}
        for side, r in (("up", self.plan.up), ("dn", self.plan.down)):
            if r is None:
                continue
            rows, handles = allh[r]
            ptrs = []
            for h, off in handles:
                base = nat.ipc_open(h)
                peer["opened"].append(base)
                ptrs.append(base + off)
            peer[side] = ptrs
            if side == "up":
                peer["up_rows"] = rows
        self._peer = peer
        import torch

        self._tok = torch.zeros(4, dtype=torch.int32, device=self.levels[0].buf.device)

    def _token_exchange(self):
        """Tiny send/recv with each neighbour: orders my next step after their boundary
        kernels (whose stores into my ghost rows then have landed)."""
        ops = []
        t = self._tok
        for i, (peer, _, _) in enumerate(self.plan.recvs):
            ops.append(self.dist.P2POp(self.dist.irecv, t[i:i + 1], peer, self.group))
        for i, (peer, _, _) in enumerate(self.plan.sends):
            ops.append(self.dist.P2POp(self.dist.isend, t[2 + i:3 + i], peer, self.group))
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()

    def close(self):
        if self._peer:
            for base in self._peer["opened"]:
                try:
                    nat.ipc_close(base)
                except Exception:
                    pass
            self._peer = None

    # -- transport ---------------------------------------------------------------------
    def _p2p_ops(self, idx: int, count: int):
        """Send my first/last ``count`` rows of level ``idx`` up/down; receive the
        neighbours' into my ghost rows."""
        ops = []
        lv = self.levels[idx]
        rows = self.plan.rows
        for peer, first, _ in self.plan.recvs:
            dst = -count if first < 0 else rows
            ops.append(self.dist.P2POp(self.dist.irecv, rows_view(lv, dst, count), peer,
                                       self.group))
        for peer, first, _ in self.plan.sends:
            src = 0 if first == 0 else rows - count
            ops.append(self.dist.P2POp(self.dist.isend, rows_view(lv, src, count), peer,
                                       self.group))
        return ops

    def exchange(self, idx: int, count: int | None = None, idx2: int | None = None,
                 count2: int = 0):
        """Blocking (w.r.t. the current stream) halo exchange of level ``idx`` (``count``
        rows; default the full halo) and optionally ``count2`` rows of level ``idx2``."""
        ops = self._p2p_ops(idx, self.plan.halo if count is None else count)
        if idx2 is not None and count2 > 0:
            ops += self._p2p_ops(idx2, count2)
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()

    # -- time stepping -------------------------------------------------------------------
    def load_initial(self, u0_rows: np.ndarray, v0_rows: np.ndarray):
        """Upload this slab's own rows of u0 / v0, then exchange their halos."""
        self.levels[1].upload(u0_rows)
        self.levels[0].upload(v0_rows)
        self.exchange(1)
        self.exchange(0)

    def first_step(self):
        self.compute.first_step(self.grid, self.levels[1], self.levels[0], self.levels[2])
        self.exchange(2)
        self.newest, self.previous = 2, 1

    def step(self, overlap: bool = True):
        """One two-step update: boundary rows, then halo exchange on the communication
        stream concurrently with the interior rows."""
        if self.T > 1:
            raise RuntimeError("temporally blocked slabs advance with step_block()/march()")
        cur = self.newest
        nxt, prev = (cur + 1) % 3, (cur + 2) % 3
        lv = self.levels
        rows, R = self.plan.rows, self.R
        c = self.compute
        if self.P == 1 or rows < 3 * R or not overlap or not c.is_cuda:
            c.two_step_rows(self.grid, lv[cur], lv[prev], lv[nxt], 0, rows)
            self.exchange(nxt)
        else:
            import torch

            if self._streams is None:
                self._streams = (torch.cuda.Stream(), torch.cuda.Event(), torch.cuda.Event())
            comm, ev_edge, ev_comm = self._streams
            main = torch.cuda.current_stream()
            if self.transport == "p2p":
                # boundary rows land in the neighbours' ghost rows from inside the kernel
                pr = self._peer
                up = pr["up"][nxt] if pr["up"] else None
                dn = pr["dn"][nxt] if pr["dn"] else None
                c.two_step_halo(self.grid, lv[cur], lv[prev], lv[nxt], 0, R, up, pr["up_rows"],
                                dn)
                c.two_step_halo(self.grid, lv[cur], lv[prev], lv[nxt], rows - R, rows, up,
                                pr["up_rows"], dn)
            else:
                c.two_step_rows(self.grid, lv[cur], lv[prev], lv[nxt], 0, R)
                c.two_step_rows(self.grid, lv[cur], lv[prev], lv[nxt], rows - R, rows)
            ev_edge.record(main)
            with torch.cuda.stream(comm):
                comm.wait_event(ev_edge)
                if self.transport == "p2p":
                    self._token_exchange()
                else:
                    self.exchange(nxt)
                ev_comm.record(comm)
            c.two_step_rows(self.grid, lv[cur], lv[prev], lv[nxt], R, rows - R)
            main.wait_event(ev_comm)
        self.newest, self.previous = nxt, cur

    def step_block(self, overlap: bool = True):
        """One temporally blocked pass: T updates.  Boundary rows (R*T each side) first,
        then their halo rows of the two newest levels go to the neighbours on the
        communication stream while the interior rows update."""
        T, R, rows = self.T, self.R, self.plan.rows
        cur, prev = self.newest, self.previous
        f1, f2 = [x for x in range(4) if x not in (cur, prev)]
        lv, c = self.levels, self.compute
        H = R * T
        if self.P == 1 or rows < 3 * H or not overlap or not c.is_cuda:
            c.tb_rows(self.grid, lv[cur], lv[prev], lv[f1], lv[f2], T, 0, rows)
            self.exchange(f2, H, f1, R * (T - 1))   # (p2p slabs too: plain copy here)
        else:
            import torch

            if self._streams is None:
                self._streams = (torch.cuda.Stream(), torch.cuda.Event(), torch.cuda.Event())
            comm, ev_edge, ev_comm = self._streams
            main = torch.cuda.current_stream()
            if self.transport == "p2p":
                # the boundary passes store their rows of both output levels straight into
                # the neighbours' ghost rows (peer memory); a token orders the next pass
                pr = self._peer
                up = (pr["up"][f1], pr["up"][f2]) if pr["up"] else None
                dn = (pr["dn"][f1], pr["dn"][f2]) if pr["dn"] else None
                c.tb_halo(self.grid, lv[cur], lv[prev], lv[f1], lv[f2], T, 0, H, up,
                          pr["up_rows"], dn)
                c.tb_halo(self.grid, lv[cur], lv[prev], lv[f1], lv[f2], T, rows - H, rows, up,
                          pr["up_rows"], dn)
            else:
                c.tb_rows(self.grid, lv[cur], lv[prev], lv[f1], lv[f2], T, 0, H)
                c.tb_rows(self.grid, lv[cur], lv[prev], lv[f1], lv[f2], T, rows - H, rows)
            ev_edge.record(main)
            with torch.cuda.stream(comm):
                comm.wait_event(ev_edge)
                if self.transport == "p2p":
                    self._token_exchange()
                else:
                    self.exchange(f2, H, f1, R * (T - 1))
                ev_comm.record(comm)
            c.tb_rows(self.grid, lv[cur], lv[prev], lv[f1], lv[f2], T, H, rows - H)
            main.wait_event(ev_comm)
        self.newest, self.previous = f2, f1

    def march(self, nsteps: int, overlap: bool = True):
        if self.T == 1:
            for _ in range(nsteps):
                self.step(overlap)
            return
        if nsteps % self.T:
            raise ValueError(f"nsteps={nsteps} must be a multiple of tsteps={self.T}")
        for _ in range(nsteps // self.T):
            self.step_block(overlap)

    def own_rows(self, which: str = "newest") -> np.ndarray:
        idx = self.newest if which == "newest" else self.previous
        return self.levels[idx].download()


class _KernelCompute:
    """libps.so updates for a slab (the product path)."""

    is_cuda = True

    def __init__(self, spec, lam, tau):
        self.t_u = nat.make_table(evaluate_table(spec.first_u, lam))
        self.t_v = nat.make_table(evaluate_table(spec.first_v, lam))
        self.t_two = nat.make_table(evaluate_table(spec.two_step, lam))
        self.tau = tau

    def first_step(self, grid, u0, v0, out):
        nat.first_step(grid, u0, v0, out, self.t_u, self.t_v, self.tau)

    def two_step_rows(self, grid, uk, ukm1, out, lo, hi):
        if hi > lo:
            nat.two_step_rows(grid, uk, ukm1, out, self.t_two, lo, hi)

    def two_step_halo(self, grid, uk, ukm1, out, lo, hi, up_ptr, up_rows, dn_ptr):
        if hi > lo:
            nat.two_step_halo(grid, uk, ukm1, out, self.t_two, lo, hi, up_ptr, up_rows, dn_ptr)

    def tb_rows(self, grid, uk, ukm1, out_prev, out_last, T, lo, hi):
        if hi > lo:
            nat.two_step_tb_rows(grid, uk, ukm1, out_prev, out_last, self.t_two, T, lo, hi)

    def tb_halo(self, grid, uk, ukm1, out_prev, out_last, T, lo, hi, up, up_rows, dn):
        if hi > lo:
            nat.two_step_tb_halo(grid, uk, ukm1, out_prev, out_last, self.t_two, T, lo, hi, up,
                                 up_rows, dn)
