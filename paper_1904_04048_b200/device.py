"""Device-resident simulation: the march the BASELINE configs and bench.py run.

The reference's ``run`` (simulator.py:231-290) allocates fresh numpy grids every step
and always scores against an ``exact`` callable; it is fp64-only and supports only a
ring of width 1.  :class:`Simulation` keeps three ps_grid levels resident in HBM,
rotates them in place (``ps_march``), and adds what the BASELINE configs need:
float32 fields, a Dirichlet zero ring as wide as the stencil radius,
device-side seeded Gaussian-sum initial data and standing-wave data.
Every update still goes through the same sm_100a kernels and arithmetic contract as
the drop-in ``first_step`` / ``two_step``.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .scheme import SchemeSpec, evaluate_table, named_scheme


def gaussian_params(rng: np.random.Generator, K: int, wmin: float, wmax: float):
    """One field's Gaussian-sum parameters, drawn in the recipe's order
    (SURVEY.md §8d D1): centres U[0.1,0.9]^2, widths U[wmin,wmax], amplitudes U[-1,1]."""
    centres = rng.uniform(0.1, 0.9, size=(K, 2))
    widths = rng.uniform(wmin, wmax, size=K)
    amps = rng.uniform(-1.0, 1.0, size=K)
    return centres, widths, amps


class Simulation:
    """One grid on one GPU: ``n`` intervals per axis, three resident levels.

    Dirichlet grids hold (n+1)^2 nodes with a pinned zero ring of width ``ring``
    (default: the scheme radius); periodic grids hold n^2 independent nodes."""

    def __init__(self, scheme, n: int, lam: float, bc: str = "dirichlet", ring: int | None = None,
                 dtype: str = "f64", arith: str = "ref", c: float = 1.0, tsteps: int = 1,
                 tile: int = 0):
        self.spec: SchemeSpec = named_scheme(scheme) if isinstance(scheme, str) else scheme
        if bc not in nat.BC:
            raise ValueError(f"bc must be one of {tuple(nat.BC)}, got {bc!r}")
        if dtype not in nat.DTYPE:
            raise ValueError(f"dtype must be one of {tuple(nat.DTYPE)}, got {dtype!r}")
        self.n, self.lam, self.bc, self.dtype, self.c = int(n), float(lam), bc, dtype, float(c)
        self.tau = self.lam * (1.0 / self.n) / self.c
        radius = self.spec.radius
        self.ring = (radius if ring is None else int(ring)) if bc == "dirichlet" else 0
        self.rows = self.n + 1 if bc == "dirichlet" else self.n
        if tsteps not in (1, 2, 3, 4, 5, 6):
            raise ValueError(f"tsteps must be 1..6, got {tsteps}")
        self.tsteps = int(tsteps)
        # tile > 0: march() runs small Dirichlet f64 grids tile-resident (ps_march_tile: one
        # cooperative launch, `tile` updates per shared-memory pass) when the grid qualifies
        if not 0 <= int(tile) <= 16:
            raise ValueError(f"tile must be 0..16, got {tile}")
        self.tile = int(tile)
        self._tile_ok = None
        # periodic blocked passes read wrap-around images R*T deep
        ghost = max(2, radius * tsteps) if bc == "periodic" else max(2, radius)
        self.grid = nat.make_grid(self.rows, self.rows, ghost, self.ring, bc, dtype, arith)
        # temporal blocking writes two new levels while both inputs are still read: 4 levels
        self.levels = [nat.Level(self.grid) for _ in range(3 if tsteps == 1 and not tile else 4)]
        self.previous = None
        self.t_first_u = nat.make_table(evaluate_table(self.spec.first_u, self.lam))
        self.t_first_v = nat.make_table(evaluate_table(self.spec.first_v, self.lam))
        self.t_two = nat.make_table(evaluate_table(self.spec.two_step, self.lam))
        self.newest = None  # index of the level holding the latest time level
        self.step = 0       # time level held by levels[newest]

    # ---- sizes --------------------------------------------------------------------
    @property
    def updated_nodes(self) -> int:
        """Nodes one step updates (ring excluded) — the LUP count of one step."""
        inner = self.rows - 2 * self.ring
        return inner * inner

    @property
    def level_bytes(self) -> int:
        return self.levels[0].buf.numel()

    @property
    def itemsize(self) -> int:
        return 8 if self.dtype == "f64" else 4

    # ---- initial data -----------------------------------------------------------------
    def load_initial(self, u0: np.ndarray, v0: np.ndarray | None = None):
        """Upload u0 (and v0; None = zero) as (n+1)^2 reference-layout arrays."""
        self.levels[1].upload(u0)
        if v0 is None:
            self.levels[0].buf.zero_()
        else:
            self.levels[0].upload(v0)
        if self.bc == "periodic":
            self.levels[1].fill_ghosts()
            self.levels[0].fill_ghosts()
        self.newest, self.step = None, 0

    def gaussian_initial(self, K: int, wmin: float, wmax: float, seed: int = 0,
                         v_zero: bool = False):
        """Seeded Gaussian-sum u0 (and v0) generated on the device (ps_gaussian_sum)."""
        rng = np.random.default_rng(seed)
        pu = gaussian_params(rng, K, wmin, wmax)
        nat.gaussian_sum(self.grid, self.levels[1], pu[0], pu[1], pu[2], self.n)
        pv = None
        if v_zero:
            self.levels[0].buf.zero_()
        else:
            pv = gaussian_params(rng, K, wmin, wmax)
            nat.gaussian_sum(self.grid, self.levels[0], pv[0], pv[1], pv[2], self.n)
        self.newest, self.step = None, 0
        return pu, pv

    def standing_wave_initial(self, m: int, k: int, omega: float | None = None):
        """u0 = sin(2πm x1) sin(2πk x2), v0 = ω u0 (BASELINE config 2), sampled on the
        host exactly like the reference's ``_sample`` (simulator.py:141-144)."""
        coords = np.arange(self.n + 1) / self.n
        x1, x2 = np.meshgrid(coords, coords, indexing="ij")
        u0 = np.sin(2.0 * np.pi * m * x1) * np.sin(2.0 * np.pi * k * x2)
        if omega is None:
            omega = 2.0 * np.pi * self.c * np.sqrt(m * m + k * k)
        self.load_initial(u0, omega * u0)
        return omega

    # ---- time stepping ----------------------------------------------------------------
    def first_step(self, stream=None):
        """u^1 from (u^0 = levels[1], v0 = levels[0]) into levels[2]."""
        nat.first_step(self.grid, self.levels[1], self.levels[0], self.levels[2], self.t_first_u,
                       self.t_first_v, self.tau, stream)
        self.newest, self.previous, self.step = 2, 1, 1

    def march(self, nsteps: int, stream=None):
        """``nsteps`` two-step updates, rotating the three levels in place."""
        if self.newest is None:
            raise RuntimeError("call first_step() before march()")
        if self.tile and self._tile_ok is None:
            self._tile_ok = nat.tile_supported(self.grid, self.t_two, self.tile)
        if self.tile and self._tile_ok:
            self.newest, self.previous = nat.march_tile(self.grid, self.levels[:4], nsteps,
                                                        self.t_two, self.tile, self.newest,
                                                        self.previous, stream)
        elif self.tsteps == 1 and not self.tile:
            self.newest = nat.march(self.grid, self.levels, nsteps, self.t_two, self.newest, stream)
            self.previous = (self.newest + 2) % 3
        else:
            self.newest, self.previous = nat.march_tb(self.grid, self.levels, nsteps, self.t_two,
                                                      self.tsteps, self.newest, self.previous,
                                                      stream)
        self.step += int(nsteps)

    # ---- host-to-host solve ---------------------------------------------------------
    def solve_host(self, u0, v0, nsteps: int, out=None, nbands: int = 0, stream=None):
        """u^nsteps from HOST u0 / v0 (None = zero velocity) into a HOST array, with the
        uploads, the march and the downloads overlapped band by band (ps_solve_host).

        Arrays are the reference's (n+1)^2 layout as numpy arrays or (preferably pinned)
        CPU torch tensors of this simulation's dtype.  Blocks until ``out`` is valid and
        returns it.  The four device levels are scratch: the resident state is reset."""
        import torch

        if int(nsteps) < 1:
            raise ValueError("nsteps must be >= 1 (1 = the first step only)")
        n1 = self.n + 1
        tdt = torch.float64 if self.dtype == "f64" else torch.float32

        def host(x):
            t = torch.from_numpy(np.ascontiguousarray(x)) if isinstance(x, np.ndarray) else x
            if t.dtype != tdt or tuple(t.shape) != (n1, n1) or t.is_cuda:
                raise ValueError(f"host arrays must be ({n1}, {n1}) {tdt} on the CPU")
            return t.contiguous()

        u = host(u0)
        v = None if v0 is None else host(v0)
        dst = torch.empty((n1, n1), dtype=tdt, pin_memory=True) if out is None else host(out)
        while len(self.levels) < 4:
            self.levels.append(nat.Level(self.grid))
        st = stream or nat.current_stream()
        nat.solve_host(self.grid, self.levels[:4], u.data_ptr(), None if v is None else v.data_ptr(),
                       dst.data_ptr(), n1, self.t_first_u, self.t_first_v, self.t_two, self.tau,
                       int(nsteps), self.tsteps, nbands, st)
        torch.cuda.synchronize()
        self.newest = self.previous = None
        self.step = 0
        if out is None:
            return dst.numpy()
        return out

    # ---- read-back ----------------------------------------------------------------
    def field(self, which: str = "newest") -> np.ndarray:
        """Latest (or previous) level as the reference's (n+1)^2 array."""
        idx = self.newest if which == "newest" else self.previous
        return self.levels[idx].download(self.n + 1, self.n + 1)

    # ---- snapshots and checkpoints -------------------------------
    def snapshot(self, path, which: str = "newest"):
        """Asynchronous CSV dump of a level (dump_grid_csv's format) that does not stall
        the march: a device-to-device copy into a staging level (stream-ordered, ~3 ms for
        8.6 GB), then the device-to-host copy on a side stream and the CSV writer on a
        host thread.  Returns a ``threading.Thread``; ``join()`` it before reading."""
        import threading

        import torch

        idx = self.newest if which == "newest" else self.previous
        if getattr(self, "_stage", None) is None:
            self._stage = nat.Level(self.grid)
            self._side = torch.cuda.Stream()
            self._stage_free = None
        if self._stage_free is not None:
            # the staging level is still the source of the previous snapshot's D2H copy
            torch.cuda.current_stream().wait_event(self._stage_free)
        self._stage.buf.copy_(self.levels[idx].buf)
        ready = torch.cuda.Event()
        ready.record()
        host = torch.empty((self.n + 1, self.n + 1),
                           dtype=torch.float64 if self.dtype == "f64" else torch.float32,
                           pin_memory=True)
        with torch.cuda.stream(self._side):
            self._side.wait_event(ready)
            nat.check(nat.load_library().ps_copy_out(
                ctypes.byref(self.grid), self._stage.ptr,
                ctypes.c_void_p(host.data_ptr()), self.n + 1, self.n + 1, self.n + 1,
                nat.D2H, ctypes.c_void_p(self._side.cuda_stream)), "ps_copy_out")
            done = torch.cuda.Event()
            done.record(self._side)
        self._stage_free = done

        def write():
            done.synchronize()
            nat.write_csv(path, host.numpy())

        th = threading.Thread(target=write, daemon=True)
        th.start()
        return th

    def save_checkpoint(self, path):
        """Persist what a restart needs: both live levels (u^k, u^{k-1}) and k."""
        if self.newest is None or self.previous is None:
            raise RuntimeError("nothing to checkpoint: call first_step() first (a restart "
                               "needs two live levels)")
        np.savez(path, newest=self.field("newest"), previous=self.field("previous"),
                 step=self.step, n=self.n, lam=self.lam, bc=self.bc, dtype=self.dtype,
                 scheme=self.spec.name)

    def load_checkpoint(self, path):
        """Resume from :meth:`save_checkpoint` (same scheme, grid and dtype)."""
        ck = np.load(path)
        if int(ck["n"]) != self.n or str(ck["bc"]) != self.bc or str(ck["dtype"]) != self.dtype:
            raise ValueError("checkpoint does not match this simulation's grid")
        if str(ck["scheme"]) != self.spec.name or float(ck["lam"]) != self.lam:
            raise ValueError(f"checkpoint was written by scheme {ck['scheme']} at lambda "
                             f"{float(ck['lam'])!r}, this simulation runs {self.spec.name} at "
                             f"{self.lam!r}")
        self.levels[2].upload(ck["newest"])
        self.levels[1].upload(ck["previous"])
        if self.bc == "periodic":
            self.levels[2].fill_ghosts()
            self.levels[1].fill_ghosts()
        self.newest, self.previous, self.step = 2, 1, int(ck["step"])

    def initial_fields(self):
        """(u0, v0) as uploaded / generated (before the first step overwrites nothing)."""
        return (self.levels[1].download(self.n + 1, self.n + 1),
                self.levels[0].download(self.n + 1, self.n + 1))
