"""ctypes binding of libps.so (the C-ABI in include/ps.h) plus device-level plumbing.

Device memory and streams come from PyTorch (plumbing only); every byte of stencil
arithmetic runs in libps.so's sm_100a kernels.  There is no CPU fallback: if the
library is missing or no CUDA device is visible, every entry point raises
:class:`NativeUnavailableError`.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PS_LIBRARY points at an alternative build (tuning variants); default: the in-tree .so
LIB_PATH = os.environ.get("PS_LIBRARY") or os.path.join(_HERE, "libps.so")

PS_MAX_TAPS = 32
BC = {"dirichlet": 0, "periodic": 1}
DTYPE = {"f64": 0, "f32": 1}
ARITH = {"ref": 0, "native": 1}
NP_DTYPE = {"f64": np.float64, "f32": np.float32}
H2D, D2H, D2D = 1, 2, 3


class NativeUnavailableError(RuntimeError):
    """libps.so is not built or no CUDA device is available; there is no fallback."""


class PsStatusError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {strerror(status)} (ps_status {status})")
        self.status = status


class PsGrid(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("pitch", ctypes.c_int64),
                ("origin", ctypes.c_int64), ("ghost", ctypes.c_int64), ("row0", ctypes.c_int64),
                ("grows", ctypes.c_int64), ("ring", ctypes.c_int32),
                ("bc", ctypes.c_int32), ("dtype", ctypes.c_int32), ("arith", ctypes.c_int32)]


class PsTable(ctypes.Structure):
    _fields_ = [("ntaps", ctypes.c_int32), ("q1", ctypes.c_int32 * PS_MAX_TAPS),
                ("q2", ctypes.c_int32 * PS_MAX_TAPS), ("c", ctypes.c_double * PS_MAX_TAPS)]


class PsBatchSim(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("n_t", ctypes.c_int32), ("bc", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("tau", ctypes.c_double), ("first_u", PsTable),
                ("first_v", PsTable), ("two_step", PsTable), ("off_field", ctypes.c_int64),
                ("off_st", ctypes.c_int64), ("off_out", ctypes.c_int64)]


PS_BATCH_MAX_N = 90


class PsSolveOp(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("band", ctypes.c_int32), ("tsteps", ctypes.c_int32),
                ("stream", ctypes.c_int32), ("src0", ctypes.c_int32), ("src1", ctypes.c_int32),
                ("dst0", ctypes.c_int32), ("dst1", ctypes.c_int32), ("row_lo", ctypes.c_int64),
                ("row_hi", ctypes.c_int64), ("after0", ctypes.c_int64), ("after1", ctypes.c_int64)]


SOLVE_KINDS = ("load", "first", "step", "pass", "store")


EXPORTS = ("ps_layout_init", "ps_slab_layout_init", "ps_level_bytes", "ps_level_alloc", "ps_level_free", "ps_copy_in",
           "ps_copy_out", "ps_fill_ghosts", "ps_first_step", "ps_two_step", "ps_two_step_rows",
           "ps_march", "ps_two_step_tb", "ps_two_step_tb_rows", "ps_march_tb", "ps_march_tile",
           "ps_tile_supported", "ps_two_step_halo",
           "ps_two_step_tb_halo",
           "ps_ipc_get_handle",
           "ps_ipc_open", "ps_ipc_close",
           "ps_gaussian_sum", "ps_errsum_create", "ps_errsum_step", "ps_errsum_destroy",
           "ps_write_csv", "ps_march_errsum", "ps_batch_desc_bytes", "ps_batch_pack",
           "ps_batch_run", "ps_solve_plan", "ps_solve_host",
           "ps_launch_count", "ps_strerror", "ps_version")

_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load libps.so and declare its signatures (no GPU needed to load)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailableError(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(path)
        i64, i32, vp, dbl = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_double
        G, T = ctypes.POINTER(PsGrid), ctypes.POINTER(PsTable)
        sig = {
            "ps_layout_init": (i32, [G, i64, i64, i32, i32, i32, i32, i32]),
            "ps_slab_layout_init": (i32, [G, i64, i64, i64, i64, i32, i32, i32, i32, i32]),
            "ps_level_bytes": (ctypes.c_size_t, [G]),
            "ps_level_alloc": (vp, [G]),
            "ps_level_free": (None, [vp]),
            "ps_copy_in": (i32, [G, vp, vp, i64, i64, i64, i32, vp]),
            "ps_copy_out": (i32, [G, vp, vp, i64, i64, i64, i32, vp]),
            "ps_fill_ghosts": (i32, [G, vp, i32, vp]),
            "ps_first_step": (i32, [G, vp, vp, vp, T, T, dbl, vp]),
            "ps_two_step": (i32, [G, vp, vp, vp, T, vp]),
            "ps_two_step_rows": (i32, [G, vp, vp, vp, T, i64, i64, vp]),
            "ps_march": (i32, [G, ctypes.POINTER(vp), i64, T, ctypes.POINTER(i32), vp]),
            "ps_two_step_tb": (i32, [G, vp, vp, vp, vp, T, i32, vp]),
            "ps_two_step_halo": (i32, [G, vp, vp, vp, T, i64, i64, vp, i64, vp, vp]),
            "ps_two_step_tb_rows": (i32, [G, vp, vp, vp, vp, T, i32, i64, i64, vp]),
            "ps_two_step_tb_halo": (i32, [G, vp, vp, vp, vp, T, i32, i64, i64, vp, vp, i64, vp,
                                          vp, vp]),
            "ps_ipc_get_handle": (i32, [vp, vp, ctypes.POINTER(i64)]),
            "ps_ipc_open": (i32, [vp, ctypes.POINTER(vp)]),
            "ps_ipc_close": (i32, [vp]),
            "ps_march_tb": (i32, [G, ctypes.POINTER(vp), i64, T, i32, ctypes.POINTER(i32),
                                  ctypes.POINTER(i32), vp]),
            "ps_march_tile": (i32, [G, ctypes.POINTER(vp), i64, T, i32, ctypes.POINTER(i32),
                                    ctypes.POINTER(i32), vp]),
            "ps_tile_supported": (i32, [G, T, i32]),
            "ps_gaussian_sum": (i32, [G, vp, i32, vp, vp, vp, vp, i64, vp]),
            "ps_errsum_create": (vp, [i64, i64]),
            "ps_errsum_step": (i32, [vp, G, vp, vp, dbl, vp, vp]),
            "ps_errsum_destroy": (None, [vp]),
            "ps_write_csv": (i32, [ctypes.c_char_p, vp, i64, i64, i64, i32]),
            "ps_march_errsum": (i32, [G, ctypes.POINTER(vp), i64, T, vp, vp, vp, vp,
                                      ctypes.POINTER(i32), vp]),
            "ps_batch_desc_bytes": (ctypes.c_size_t, []),
            "ps_batch_pack": (i32, [ctypes.POINTER(PsBatchSim), vp]),
            "ps_batch_run": (i32, [i32, i32, vp, vp, vp, vp, vp, vp, vp]),
            "ps_solve_plan": (i64, [i64, i32, i64, i32, i32, i32, ctypes.POINTER(PsSolveOp), i64]),
            "ps_solve_host": (i32, [G, ctypes.POINTER(vp), vp, vp, vp, i64, T, T, T, dbl, i64, i32,
                                    i32, vp]),
            "ps_launch_count": (i64, []),
            "ps_strerror": (ctypes.c_char_p, [i32]),
            "ps_version": (ctypes.c_char_p, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        return L


def strerror(status: int) -> str:
    try:
        return load_library().ps_strerror(status).decode()
    except NativeUnavailableError:
        return f"status {status}"


def check(status: int, what: str):
    if status != 0:
        raise PsStatusError(status, what)


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailableError(
            "no CUDA device visible: the poisson_stencils GPU path has no CPU fallback")
    return torch


def current_stream():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def sync_stream(stream):
    """Block until the work queued on ``stream`` (a ``c_void_p`` handle) has finished."""
    torch = _torch()
    handle = getattr(stream, "value", stream) or 0
    if handle == torch.cuda.current_stream().cuda_stream:
        torch.cuda.current_stream().synchronize()
    elif handle == 0:
        torch.cuda.default_stream().synchronize()
    else:
        torch.cuda.ExternalStream(handle).synchronize()


def make_table(pairs) -> PsTable:
    """Pack ``[((q1, q2), coeff), ...]`` (dict order) into a ``ps_table``."""
    pairs = list(pairs)
    if not 1 <= len(pairs) <= PS_MAX_TAPS:
        raise ValueError(f"tables must hold 1..{PS_MAX_TAPS} taps, got {len(pairs)}")
    t = PsTable()
    t.ntaps = len(pairs)
    for s, ((q1, q2), c) in enumerate(pairs):
        t.q1[s], t.q2[s], t.c[s] = int(q1), int(q2), float(c)
    return t


def make_slab_grid(grows, cols, row0, rows, ghost, ring, bc, dtype, arith="ref") -> PsGrid:
    g = PsGrid()
    check(load_library().ps_slab_layout_init(ctypes.byref(g), int(grows), int(cols), int(row0),
                                             int(rows), int(ghost), int(ring), BC[bc],
                                             DTYPE[dtype], ARITH[arith]), "ps_slab_layout_init")
    return g


def make_grid(rows, cols, ghost, ring, bc, dtype, arith="ref") -> PsGrid:
    g = PsGrid()
    check(load_library().ps_layout_init(ctypes.byref(g), int(rows), int(cols), int(ghost),
                                        int(ring), BC[bc], DTYPE[dtype], ARITH[arith]),
          "ps_layout_init")
    return g


class Level:
    """One device level laid out by ``ps_layout_init`` (torch owns the bytes)."""

    def __init__(self, grid: PsGrid, device=None):
        torch = _torch()
        self.grid = grid
        nbytes = load_library().ps_level_bytes(ctypes.byref(grid))
        self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=device or "cuda")
        self.ptr = ctypes.c_void_p(self.buf.data_ptr())

    @property
    def np_dtype(self):
        return np.float64 if self.grid.dtype == 0 else np.float32

    def view(self):
        """torch view of the logical rows x cols block (strided, zero-copy)."""
        torch = _torch()
        tdt = torch.float64 if self.grid.dtype == 0 else torch.float32
        flat = self.buf.view(tdt)
        return flat.as_strided((self.grid.rows, self.grid.cols), (self.grid.pitch, 1),
                               self.grid.origin)

    def upload(self, host: np.ndarray, stream=None):
        host = np.ascontiguousarray(host, dtype=self.np_dtype)
        check(load_library().ps_copy_in(ctypes.byref(self.grid), self.ptr,
                                        host.ctypes.data_as(ctypes.c_void_p), host.shape[0],
                                        host.shape[1], host.shape[1], H2D,
                                        stream or current_stream()), "ps_copy_in")
        # pageable source: the copy has been staged before return; keep `host` alive anyway
        self._keep = host

    def download(self, rows=None, cols=None, stream=None) -> np.ndarray:
        rows = self.grid.rows if rows is None else rows
        cols = self.grid.cols if cols is None else cols
        out = np.empty((rows, cols), dtype=self.np_dtype)
        st = stream or current_stream()
        check(load_library().ps_copy_out(ctypes.byref(self.grid), self.ptr,
                                         out.ctypes.data_as(ctypes.c_void_p), rows, cols, cols,
                                         D2H, st), "ps_copy_out")
        sync_stream(st)     # the stream the copy ran on, not necessarily the current one
        return out

    def fill_ghosts(self, keep_alias=False, stream=None):
        check(load_library().ps_fill_ghosts(ctypes.byref(self.grid), self.ptr, int(keep_alias),
                                            stream or current_stream()), "ps_fill_ghosts")


def first_step(grid, u0: Level, v0: Level, out: Level, tu: PsTable, tv: PsTable, tau, stream=None):
    check(load_library().ps_first_step(ctypes.byref(grid), u0.ptr, v0.ptr, out.ptr,
                                       ctypes.byref(tu), ctypes.byref(tv), float(tau),
                                       stream or current_stream()), "ps_first_step")


def two_step(grid, uk: Level, ukm1: Level, out: Level, t: PsTable, stream=None):
    check(load_library().ps_two_step(ctypes.byref(grid), uk.ptr, ukm1.ptr, out.ptr,
                                     ctypes.byref(t), stream or current_stream()), "ps_two_step")


def two_step_rows(grid, uk: Level, ukm1: Level, out: Level, t: PsTable, lo: int, hi: int,
                  stream=None):
    check(load_library().ps_two_step_rows(ctypes.byref(grid), uk.ptr, ukm1.ptr, out.ptr,
                                          ctypes.byref(t), int(lo), int(hi),
                                          stream or current_stream()), "ps_two_step_rows")


def two_step_halo(grid, uk: Level, ukm1: Level, out: Level, t: PsTable, lo: int, hi: int,
                  up_ptr: int | None, up_rows: int, dn_ptr: int | None, stream=None):
    """Slab update that also stores its first/last R rows into the neighbours' ghost rows
    (``up_ptr`` / ``dn_ptr``: allocation base pointers of their u^{k+1} levels)."""
    check(load_library().ps_two_step_halo(ctypes.byref(grid), uk.ptr, ukm1.ptr, out.ptr,
                                          ctypes.byref(t), int(lo), int(hi),
                                          ctypes.c_void_p(up_ptr or 0), int(up_rows),
                                          ctypes.c_void_p(dn_ptr or 0),
                                          stream or current_stream()), "ps_two_step_halo")


def ipc_handle(ptr: int) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of the allocation holding ``ptr``, byte offset of ptr)."""
    buf = ctypes.create_string_buffer(64)
    off = ctypes.c_int64(0)
    check(load_library().ps_ipc_get_handle(ctypes.c_void_p(ptr), buf, ctypes.byref(off)),
          "ps_ipc_get_handle")
    return buf.raw, off.value


def ipc_open(handle: bytes) -> int:
    out = ctypes.c_void_p(0)
    check(load_library().ps_ipc_open(ctypes.create_string_buffer(handle, 64), ctypes.byref(out)),
          "ps_ipc_open")
    return out.value


def ipc_close(ptr: int):
    check(load_library().ps_ipc_close(ctypes.c_void_p(ptr)), "ps_ipc_close")


def march(grid, levels, nsteps: int, t: PsTable, newest: int, stream=None) -> int:
    arr = (ctypes.c_void_p * 3)(*[lv.ptr.value for lv in levels[:3]])
    nw = ctypes.c_int32(newest)
    check(load_library().ps_march(ctypes.byref(grid), arr, int(nsteps), ctypes.byref(t),
                                  ctypes.byref(nw), stream or current_stream()), "ps_march")
    return nw.value


def two_step_tb(grid, uk: Level, ukm1: Level, out_prev: Level, out_last: Level, t: PsTable,
                tsteps: int, stream=None):
    check(load_library().ps_two_step_tb(ctypes.byref(grid), uk.ptr, ukm1.ptr, out_prev.ptr,
                                        out_last.ptr, ctypes.byref(t), int(tsteps),
                                        stream or current_stream()), "ps_two_step_tb")


def two_step_tb_rows(grid, uk: Level, ukm1: Level, out_prev: Level, out_last: Level,
                     t: PsTable, tsteps: int, lo: int, hi: int, stream=None):
    check(load_library().ps_two_step_tb_rows(ctypes.byref(grid), uk.ptr, ukm1.ptr, out_prev.ptr,
                                             out_last.ptr, ctypes.byref(t), int(tsteps), int(lo),
                                             int(hi), stream or current_stream()),
          "ps_two_step_tb_rows")


def two_step_tb_halo(grid, uk: Level, ukm1: Level, out_prev: Level, out_last: Level,
                     t: PsTable, tsteps: int, lo: int, hi: int, up: tuple | None, up_rows: int,
                     dn: tuple | None, stream=None):
    """Fused pass over rows [lo, hi) that also stores its boundary rows of both output
    levels into the neighbours' ghost rows (``up`` / ``dn``: (out_prev, out_last)
    allocation base pointers of the neighbour slab, or None)."""
    vp = ctypes.c_void_p
    u = up or (0, 0)
    d = dn or (0, 0)
    check(load_library().ps_two_step_tb_halo(ctypes.byref(grid), uk.ptr, ukm1.ptr, out_prev.ptr,
                                             out_last.ptr, ctypes.byref(t), int(tsteps), int(lo),
                                             int(hi), vp(u[0]), vp(u[1]), int(up_rows), vp(d[0]),
                                             vp(d[1]), stream or current_stream()),
          "ps_two_step_tb_halo")


def march_tb(grid, levels, nsteps: int, t: PsTable, tsteps: int, newest: int, previous: int,
             stream=None) -> tuple[int, int]:
    arr = (ctypes.c_void_p * 4)(*[lv.ptr.value for lv in levels])
    nw, pv = ctypes.c_int32(newest), ctypes.c_int32(previous)
    check(load_library().ps_march_tb(ctypes.byref(grid), arr, int(nsteps), ctypes.byref(t),
                                     int(tsteps), ctypes.byref(nw), ctypes.byref(pv),
                                     stream or current_stream()), "ps_march_tb")
    return nw.value, pv.value


def tile_supported(grid, t: PsTable, tsteps: int) -> bool:
    """True when ps_march_tile can run this grid / table / depth (needs a GPU to ask)."""
    return bool(load_library().ps_tile_supported(ctypes.byref(grid), ctypes.byref(t), int(tsteps)))


def march_tile(grid, levels, nsteps: int, t: PsTable, tsteps: int, newest: int, previous: int,
               stream=None) -> tuple[int, int]:
    """ps_march_tile: all ``nsteps`` updates in one cooperative launch (small grids)."""
    arr = (ctypes.c_void_p * 4)(*[lv.ptr.value for lv in levels])
    nw, pv = ctypes.c_int32(newest), ctypes.c_int32(previous)
    check(load_library().ps_march_tile(ctypes.byref(grid), arr, int(nsteps), ctypes.byref(t),
                                       int(tsteps), ctypes.byref(nw), ctypes.byref(pv),
                                       stream or current_stream()), "ps_march_tile")
    return nw.value, pv.value


def solve_plan(rows: int, radius: int, nsteps: int, tsteps: int, nbands: int = 0,
               nstreams: int = 2) -> list[dict]:
    """ps_solve_plan as a list of dicts (host-only: works without a GPU)."""
    L = load_library()
    n = L.ps_solve_plan(int(rows), int(radius), int(nsteps), int(tsteps), int(nbands),
                        int(nstreams), None, 0)
    if n < 0:
        raise PsStatusError(int(-n), "ps_solve_plan")
    ops = (PsSolveOp * n)()
    L.ps_solve_plan(int(rows), int(radius), int(nsteps), int(tsteps), int(nbands), int(nstreams),
                    ops, n)
    return [{f: (SOLVE_KINDS[getattr(o, f)] if f == "kind" else getattr(o, f))
             for f, _ in PsSolveOp._fields_} for o in ops]


def solve_host(grid, levels, u0_host, v0_host, out_host, host_pitch: int, tu: PsTable,
               tv: PsTable, t: PsTable, tau: float, nsteps: int, tsteps: int, nbands: int = 0,
               stream=None):
    """ps_solve_host on raw HOST pointers (ints; v0_host may be None = zero velocity)."""
    arr = (ctypes.c_void_p * 4)(*[lv.ptr.value for lv in levels])
    check(load_library().ps_solve_host(ctypes.byref(grid), arr, ctypes.c_void_p(u0_host),
                                       ctypes.c_void_p(v0_host) if v0_host else None,
                                       ctypes.c_void_p(out_host), int(host_pitch), ctypes.byref(tu),
                                       ctypes.byref(tv), ctypes.byref(t), float(tau), int(nsteps),
                                       int(tsteps), int(nbands), stream or current_stream()),
          "ps_solve_host")


def gaussian_sum(grid, level: Level, centres, widths, amps, n: int, stream=None):
    cx = np.ascontiguousarray([c[0] for c in centres], dtype=np.float64)
    cy = np.ascontiguousarray([c[1] for c in centres], dtype=np.float64)
    w = np.ascontiguousarray(widths, dtype=np.float64)
    a = np.ascontiguousarray(amps, dtype=np.float64)
    p = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    check(load_library().ps_gaussian_sum(ctypes.byref(grid), level.ptr, len(a), p(cx), p(cy),
                                         p(w), p(a), int(n), stream or current_stream()),
          "ps_gaussian_sum")


class ErrSum:
    """Device plan for run()'s per-step error sums in numpy's pairwise order (F1)."""

    def __init__(self, rows_h: int, cols_h: int):
        _torch()
        self._lib = load_library()
        self.handle = self._lib.ps_errsum_create(int(rows_h), int(cols_h))
        if not self.handle:
            raise PsStatusError(5, "ps_errsum_create")

    def step(self, grid, level: Level, S: Level, st: float, out_ptr: int, stream=None):
        check(self._lib.ps_errsum_step(ctypes.c_void_p(self.handle), ctypes.byref(grid),
                                       level.ptr, S.ptr, float(st), ctypes.c_void_p(out_ptr),
                                       stream or current_stream()), "ps_errsum_step")

    def march(self, grid, levels, nsteps: int, t: PsTable, S: Level, st: np.ndarray,
              out_ptr: int, newest: int, stream=None) -> int:
        """``nsteps`` updates, each followed by its error sums (ps_march_errsum)."""
        arr = (ctypes.c_void_p * 3)(*[lv.ptr.value for lv in levels])
        st = np.ascontiguousarray(st, dtype=np.float64)
        nw = ctypes.c_int32(newest)
        check(self._lib.ps_march_errsum(ctypes.byref(grid), arr, int(nsteps), ctypes.byref(t),
                                        ctypes.c_void_p(self.handle), S.ptr,
                                        st.ctypes.data_as(ctypes.c_void_p),
                                        ctypes.c_void_p(out_ptr), ctypes.byref(nw),
                                        stream or current_stream()), "ps_march_errsum")
        return nw.value

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h:
            try:
                self._lib.ps_errsum_destroy(ctypes.c_void_p(h))
            except Exception:
                pass


def write_csv(path, values: np.ndarray):
    """``%.17g`` CSV of a 2-D float64/float32 host array (dump_grid_csv's format)."""
    arr = np.ascontiguousarray(values)
    if arr.dtype not in (np.float64, np.float32) or arr.ndim != 2:
        raise TypeError("write_csv takes a 2-D float64 or float32 array")
    check(load_library().ps_write_csv(os.fsencode(str(path)),
                                      arr.ctypes.data_as(ctypes.c_void_p), arr.shape[0],
                                      arr.shape[1], arr.shape[1],
                                      DTYPE["f64" if arr.dtype == np.float64 else "f32"]),
          "ps_write_csv")


def batch_run(sims, u0s, v0s, Ss, sts) -> np.ndarray:
    """Run the packed simulations in one launch; returns the concatenated per-step sums.

    ``sims``: list of PsBatchSim (offsets filled in); the float64 host arrays are the
    concatenations the offsets refer to."""
    torch = _torch()
    lib = load_library()
    dbytes = lib.ps_batch_desc_bytes()
    desc = np.zeros(len(sims) * dbytes, dtype=np.uint8)
    for k, sim in enumerate(sims):
        check(lib.ps_batch_pack(ctypes.byref(sim), desc[k * dbytes:].ctypes.data_as(ctypes.c_void_p)),
              "ps_batch_pack")
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to("cuda")  # noqa: E731
    d_desc, d_u0, d_v0, d_S, d_st = dev(desc), dev(u0s), dev(v0s), dev(Ss), dev(sts)
    nout = sum(2 * sim.n_t for sim in sims)
    d_out = torch.empty(nout, dtype=torch.float64, device="cuda")
    p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    check(lib.ps_batch_run(len(sims), max(sim.n for sim in sims), p(d_desc), p(d_u0), p(d_v0),
                           p(d_S), p(d_st), p(d_out), current_stream()), "ps_batch_run")
    return d_out.cpu().numpy()


def launch_count() -> int:
    return int(load_library().ps_launch_count())
