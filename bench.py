#!/usr/bin/env python
"""bench.py — lattice updates per second of the two-step march on B200.

Default workload (N=1): BASELINE config 4 — P9 nine-point scheme, 32768^2 f64 grid,
Dirichlet zero ring of width 1, λ=0.6, seeded 64-Gaussian u0 and v0=0 (the
largest single-GPU configuration the metric's 1/2/4/8-GPU numbers are quoted on;
see DESIGN.md §Measurement).  One "step" = one two-step update of the whole grid.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C1..C5|C3f32]
  python bench.py --impl reference ...   # the reference's CPU path (oracle port)

For N>1: one process per GPU, row slabs, halo rows over NCCL or in-kernel peer stores
(``scaling: strong`` — the grid is fixed).  Under torchrun the ranks come from the
environment; a plain ``python bench.py --gpus N`` re-executes itself under
``torch.distributed.run`` with N ranks (and fails loudly when fewer GPUs are visible).
Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grid-point updates/sec (GLUP/s) and fraction of HBM roofline, 1/2/4/8 B200"

CONFIGS = {
    "C1": dict(scheme="P5", n=511, bc="dirichlet", ring=1, dtype="f64", arith="ref", lam=0.5,
               steps=200, ic="gauss-centre", tile=12,
               desc="C1: P5 5-point, 512^2 f64, Dirichlet ring 1, lambda=0.5, 200 steps"),
    "C2": dict(scheme="P9", n=4096, bc="periodic", ring=0, dtype="f64", arith="ref", lam=0.6,
               steps=1000, ic="standing", tb=4,
               desc="C2: P9 9-point, 4096^2 f64 periodic, lambda=0.6, standing wave m=4 n=6, 1000 steps"),
    "C3": dict(scheme="P13", n=16383, bc="dirichlet", ring=2, dtype="f64", arith="ref", lam=0.4,
               steps=500, ic=(32, 0.01, 0.05, False), tb=3,
               desc="C3: P13 13-point, 16384^2 f64, Dirichlet ring 2, lambda=0.4, 500 steps"),
    "C3f32": dict(scheme="P13", n=16383, bc="dirichlet", ring=2, dtype="f32", arith="native",
                  lam=0.4, steps=500, ic=(32, 0.01, 0.05, False), tb=4,
                  desc="C3: P13 13-point, 16384^2 f32, Dirichlet ring 2, lambda=0.4, 500 steps"),
    "C4": dict(scheme="P9", n=32767, bc="dirichlet", ring=1, dtype="f64", arith="ref", lam=0.6,
               steps=200, ic=(64, 0.01, 0.05, True), tb=5,
               desc="C4: P9 9-point, 32768^2 f64, Dirichlet ring 1, lambda=0.6, 200 steps"),
    "C5": dict(scheme="P13", n=65535, bc="dirichlet", ring=2, dtype="f32", arith="native",
               lam=0.4, steps=100, ic=(128, 0.002, 0.01, False), tb=4,
               desc="C5: P13 13-point, 65536^2 f32, Dirichlet ring 2, lambda=0.4, 100 steps"),
}

REASONS = ("sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")


def load_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def compute_roofline(cfg, value_glups, T=1):
    """Arithmetic roofline of the fused kernel (temporal blocking makes it instruction-bound,
    not HBM-bound): FP-pipe instructions per update under the config's contract times the
    update rate, against the DADD (f64) / FFMA (f32) throughput tools/fp64_probe.cu measures
    on this GPU in this run.  None if the probe binary is absent."""
    import subprocess

    from paper_1904_04048_b200.scheme import named_scheme

    probe = os.path.join(ROOT, "build", "fp64_probe")
    if not os.path.exists(probe) or cfg["arith"] == "ref" and cfg["dtype"] == "f32":
        return None
    try:
        out = subprocess.run([probe], capture_output=True, text=True, timeout=60, check=True)
        rates = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception:
        return None
    spec = named_scheme(cfg["scheme"])
    ntaps = len(spec.two_step)
    shared = None
    if cfg["dtype"] == "f64":
        # reference sequence: one DMUL + one DADD per tap, one DSUB.  The shared-product
        # kernels (f64 Dirichlet; radius 2 up to depth 3) multiply once per input element
        # and coefficient class instead of once per tap: classes + taps + 1 instructions
        ipl, peak, pipe = 2 * ntaps + 1, rates["dadd_rate_32warps_per_sm_Gops"], "fp64"
        if cfg["bc"] == "dirichlet" and T > 1 and (spec.radius == 1 or T <= 3):
            classes = len({(abs(q1) + abs(q2), max(abs(q1), abs(q2))) for q1, q2 in spec.two_step})
            shared = classes + ntaps + 1
    else:                       # native f32: one FFMA per tap, one FADD
        ipl, peak, pipe = ntaps + 1, rates["ffma_rate_Gops"], "fp32"
    executed = shared or ipl
    achieved = value_glups * executed
    return {"bound": f"{pipe} pipe", "achieved": achieved, "peak": peak,
            "unit": "G thread-instructions/s", "frac": achieved / peak,
            "instr_per_lup": executed, "reference_sequence_instr_per_lup": ipl,
            **({"shared_products": "one rounded product per input element and coefficient "
                                   "class feeds every sum that reads it (same bits, "
                                   f"{ipl - shared} fewer multiplies per update)"}
               if shared else {}),
            "peak_source": "measured in this run: tools/fp64_probe.cu "
                           f"({'DADD' if pipe == 'fp64' else 'FFMA'} throughput, all SMs)",
            "note": "algorithmic instructions only (no recomputed halo columns/rows); the "
                    "reference's order fixes a dependent add chain per update"}


def load_traffic(cfg_name, T=1):
    path = os.path.join(ROOT, "profiles", f"ncu_{cfg_name}" + (f"_T{T}" if T > 1 else "") + ".json")
    try:
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """SM clock and clock-event reasons sampled through NVML every ~4 ms on a host thread
    during the timed region (``nvidia-smi -lms`` bottoms out near 100 ms, longer than a
    20-step region); falls back to ``nvidia-smi -lms 20`` when NVML cannot be loaded."""

    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40}

    def __init__(self, gpu: str, period_s: float | None = None):
        if period_s is None:
            period_s = float(os.environ.get("PS_BENCH_CLOCK_PERIOD_MS", "4")) * 1e-3
        self.gpu, self.period = gpu, period_s
        self.sm, self.mx, self.reasons = [], [], set()
        self.stop = threading.Event()
        self.thread = self.proc = None
        self.source = None

    def _nvml_loop(self, nv, h):
        reasons_fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        try:
            mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        except Exception:
            mx = None
        while True:
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                if mx:
                    self.mx.append(mx)
                bits = int(reasons_fn(h))
                for name, bit in self.BITS.items():
                    if bits & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            if self.stop.wait(self.period):
                return

    def _smi_pump(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 2 + len(REASONS):
                continue
            try:
                self.sm.append(float(parts[0]))
                self.mx.append(float(parts[1]))
            except ValueError:
                continue
            for r, v in zip(REASONS, parts[2:]):
                if v.lower() == "active":
                    self.reasons.add(r)

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = (nv.nvmlDeviceGetHandleByUUID(self.gpu) if self.gpu.startswith("GPU-")
                 else nv.nvmlDeviceGetHandleByIndex(int(self.gpu)))
            self.thread = threading.Thread(target=self._nvml_loop, args=(nv, h), daemon=True)
            self.source = f"NVML, {self.period * 1e3:.0f} ms period"
            self.thread.start()
            return self
        except Exception:
            self.thread = None
        q = "clocks.sm,clocks.max.sm," + ",".join(f"clocks_event_reasons.{r}" for r in REASONS)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "20",
                 "-i", self.gpu], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._smi_pump, daemon=True)
            self.source = "nvidia-smi -lms 20"
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.proc is not None:
            time.sleep(0.05)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "source": self.source}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": self.source}


def gpu_id(local: int) -> str:
    """nvidia-smi -i accepts the GPU UUID, which survives CUDA_VISIBLE_DEVICES remapping."""
    try:
        import torch

        uuid = str(torch.cuda.get_device_properties(local).uuid)
        return uuid if uuid.startswith("GPU-") else f"GPU-{uuid}"
    except Exception:
        return str(local)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------------------ CPU legs
def cpu_sample(cfg, seconds: float, threads: int = 0, rows_hint: int | None = None):
    """Time the oracle (the reference's arithmetic restated in C, OpenMP over rows) on a
    full-width row slab of the config's grid.  Returns (LUP/s, rows, steps, secs)."""
    import numpy as np

    from oracle import oracle as O
    from paper_1904_04048_b200.scheme import evaluate_table, named_scheme

    spec = named_scheme(cfg["scheme"])
    pairs = evaluate_table(spec.two_step, cfg["lam"])
    width = cfg["n"] + 1
    ring = cfg["ring"] if cfg["bc"] == "dirichlet" else 0
    npdt = np.float64 if cfg["dtype"] == "f64" else np.float32
    arith = cfg["arith"]

    def run(rows, steps):
        rng = np.random.default_rng(0)
        a = rng.standard_normal((rows + 2 * max(ring, 1), width)).astype(npdt)
        b = rng.standard_normal(a.shape).astype(npdt)
        bc = cfg["bc"]
        t0 = time.perf_counter()
        O.march(a, b, pairs, steps, bc, max(ring, 1) if bc == "dirichlet" else 0, arith, threads)
        dt = time.perf_counter() - t0
        inner = rows * (width - 2 * ring)
        return inner * steps / dt, dt

    rows = rows_hint or 32
    rate, dt = run(rows, 1)
    # size the slab so one step takes ~seconds/4, then run 4 steps
    per_row = dt / rows
    rows = int(max(16, min(width, (seconds / 4.0) / max(per_row, 1e-9))))
    rate, dt = run(rows, 4)
    return rate, rows, 4, dt


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.lower().startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def numpy_sample(cfg, seconds: float):
    """Time oracle/numpy_ref.py — the reference's own array algorithm (one temporary and
    one add pass per tap, np.roll per tap when periodic; simulator.py:147-191), which is
    single-threaded — on a bounded full-width slab.  Returns (LUP/s, rows, steps, secs)."""
    import numpy as np

    from oracle import numpy_ref as N
    from paper_1904_04048_b200.scheme import evaluate_table, named_scheme

    pairs = evaluate_table(named_scheme(cfg["scheme"]).two_step, cfg["lam"])
    npdt = np.float64 if cfg["dtype"] == "f64" else np.float32
    width = cfg["n"] + 1
    rng = np.random.default_rng(0)
    if cfg["bc"] == "periodic":
        # np.roll wraps both axes, so the periodic call is timed on a square grid of the
        # same algorithm: the whole config when small, else the largest square within budget
        def run(n, steps):
            a = rng.standard_normal((n + 1, n + 1)).astype(npdt)
            b = rng.standard_normal(a.shape).astype(npdt)
            t0 = time.perf_counter()
            for _ in range(steps):
                a, b = N.two_step(a, b, pairs, "periodic"), a
            return n * n * steps / (time.perf_counter() - t0), time.perf_counter() - t0

        n = min(cfg["n"], 1024)
        rate, dt = run(n, 1)
        n = int(min(cfg["n"], max(256, (seconds / 3.0 * rate) ** 0.5)))
        rate, dt = run(n, 3)
        return rate, n, 3, dt, f"{n}^2 periodic grid"
    ring = max(cfg["ring"], 1)

    def run(rows, steps):
        a = rng.standard_normal((rows + 2 * ring, width)).astype(npdt)
        b = rng.standard_normal(a.shape).astype(npdt)
        t0 = time.perf_counter()
        for _ in range(steps):
            a, b = N.two_step_slab(a, b, pairs, ring), a
        dt = time.perf_counter() - t0
        return rows * (width - 2 * ring) * steps / dt, dt

    rows = max(8, min(width - 2 * ring, 4_000_000 // width))
    rate, dt = run(rows, 1)
    rows = int(max(8, min(width - 2 * ring, seconds / 3.0 * rate / width)))
    rate, dt = run(rows, 3)
    return rate, rows, 3, dt, f"{rows} full-width rows x {width} cols"


def cpu_baseline(args, cfg):
    """The reference's CPU path on this box's host cores, beside the GPU number: the C
    port on all cores (`value`) and the reference's numpy algorithm on its one core."""
    from oracle import oracle as O

    rate, rows, steps, secs = cpu_sample(cfg, args.cpu_seconds)
    out = {"value": rate / 1e9, "unit": "GLUP/s", "cores": O.max_threads(), "kind": "port",
           "cpu_model": cpu_model(), "host_cores": os.cpu_count(),
           "sample": f"{rows} full-width rows x {cfg['n'] + 1} cols, {steps} two-step updates "
                     f"({secs:.1f} s) through oracle/ps_oracle.c (reference arithmetic, OpenMP)"}
    try:
        nrate, _, nsteps, nsecs, what = numpy_sample(cfg, min(args.cpu_seconds, 8.0))
        out["numpy_reference_algorithm"] = {
            "value": nrate / 1e9, "unit": "GLUP/s", "cores": 1,
            "cores_note": f"1 core of {os.cpu_count()} (numpy ufuncs are single-threaded)",
            "kind": "port",
            "sample": f"{what}, {nsteps} two-step updates ({nsecs:.1f} s) through "
                      "oracle/numpy_ref.py (the reference's per-tap slice/roll passes, "
                      "simulator.py:147-191; the package itself cannot travel to this box)"}
    except MemoryError:
        out["numpy_reference_algorithm"] = None
    return out


def single_config(cfg, T, tile_depth):
    """`config` of the single-GPU arm; `--impl reference` prints the same object (it runs on
    this arm's config; its own threading is in `cpu_baseline`)."""
    width = cfg["n"] + 1 if cfg["bc"] == "dirichlet" else cfg["n"]
    level = width * width * (8 if cfg["dtype"] == "f64" else 4)
    return {"workload": cfg["desc"], "scheme": cfg["scheme"], "nodes": cfg["n"] + 1,
            "lambda": cfg["lam"], "bc": cfg["bc"], "arith": cfg["arith"],
            "parallelism": "single GPU", "temporal_blocking": T,
            "tile_resident_depth": tile_depth,
            "l2": f"inputs larger than L2: {level / 1e9:.2f} GB per level, "
                  "streamed from HBM every launch" if level > 126e6 else
                  "grid fits in L2 (latency-bound correctness config)"}


def dist_config(cfg, T, world, halo_rows, transport, graphed):
    """`config` of the row-slab arm (one rank per GPU); shared with `--impl reference`."""
    return {"workload": cfg["desc"], "scheme": cfg["scheme"], "nodes": cfg["n"] + 1,
            "lambda": cfg["lam"], "bc": cfg["bc"], "arith": cfg["arith"],
            "temporal_blocking": T,
            "parallelism": f"row slabs x{world}, {halo_rows}-row halo "
                           + ("over NCCL send/recv" if transport == "nccl" else
                              "stored into peer ghost rows by the fused kernel "
                              "(CUDA IPC over NVLink)")
                           + ", overlapped with the interior update",
            "cuda_graph": graphed,
            "l2": "inputs larger than L2"}


def reference_arm(args, cfg, cfg_name):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O

    threads = O.max_threads()
    rate0, rows, _, _ = cpu_sample(cfg, 2.0)
    # per step: a full-width slab sized for ~0.25 s so K + W steps stay within minutes
    import numpy as np

    from paper_1904_04048_b200.scheme import evaluate_table, named_scheme

    spec = named_scheme(cfg["scheme"])
    pairs = evaluate_table(spec.two_step, cfg["lam"])
    width = cfg["n"] + 1
    ring = max(cfg["ring"], 1) if cfg["bc"] == "dirichlet" else 0
    lup_row = width - 2 * (cfg["ring"] if cfg["bc"] == "dirichlet" else 0)
    srows = int(max(8, min(width, 0.25 * rate0 / lup_row)))
    npdt = np.float64 if cfg["dtype"] == "f64" else np.float32
    rng = np.random.default_rng(0)
    a = rng.standard_normal((srows + 2 * max(ring, 1), width)).astype(npdt)
    b = rng.standard_normal(a.shape).astype(npdt)
    for _ in range(args.warmup):
        b = O.two_step(a, b, pairs, cfg["bc"], ring, cfg["arith"])
        a, b = b, a
    t0 = time.perf_counter()
    for _ in range(args.steps):
        b = O.two_step(a, b, pairs, cfg["bc"], ring, cfg["arith"])
        a, b = b, a
    dt = time.perf_counter() - t0
    lup = srows * lup_row * args.steps
    value = lup / dt / 1e9
    sample = (f"{srows} full-width rows x {width} cols per step (of {cfg['n'] + 1} rows), "
              f"{args.steps} steps")
    # the config object of the GPU arm launched with the same flags
    T = args.tsteps if args.tsteps > 0 else cfg.get("tb", 1)
    if world > 1 or args.force_dist:
        from paper_1904_04048_b200.scheme import named_scheme as _ns
        arm_cfg = dist_config(cfg, T, world, _ns(cfg["scheme"]).radius * T, args.transport,
                              not args.no_graph)
    else:
        tile = args.tile if args.tile >= 0 else (cfg.get("tile", 0) if T == 1 else 0)
        arm_cfg = single_config(cfg, T, tile)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GLUP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic",
        "config": arm_cfg,
        "config_note": "the GPU arm's config (the workload both arms run); this arm itself is "
                       "the reference arithmetic on the host cores, see cpu_baseline",
        "cpu_baseline": {"value": value, "unit": "GLUP/s", "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(), "host_cores": os.cpu_count(),
                         "sample": sample + "; oracle/ps_oracle.c (reference arithmetic, "
                                   "OpenMP over rows)"},
        "e2e": {"value": value, "unit": "GLUP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ GPU arm
def make_sim(cfg, tsteps=1, tile=0):
    from paper_1904_04048_b200.device import Simulation

    sim = Simulation(cfg["scheme"], cfg["n"], cfg["lam"], bc=cfg["bc"],
                     ring=cfg["ring"] if cfg["bc"] == "dirichlet" else None,
                     dtype=cfg["dtype"], arith=cfg["arith"], tsteps=tsteps, tile=tile)
    ic = cfg["ic"]
    if ic == "standing":
        sim.standing_wave_initial(4, 6)
    elif ic == "gauss-centre":
        import numpy as np

        n = cfg["n"]
        x = np.arange(n + 1) / n
        x1, x2 = np.meshgrid(x, x, indexing="ij")
        sim.load_initial(np.exp(-((x1 - 0.5) ** 2 + (x2 - 0.5) ** 2) / (2 * 0.05**2)), None)
    else:
        K, wmin, wmax, vzero = ic
        sim.gaussian_initial(K, wmin, wmax, seed=0, v_zero=vzero)
    return sim


def measure_march(args, cfg, T, tile=0):
    """Build the config's grid, first step, warm up, then time K march steps at temporal
    blocking depth T with CUDA events on the launching stream.  The K-step region is
    repeated (``--reps``; auto: 3 while one region takes under 2 s) and the MEDIAN region is
    reported, with the clock sampler running across all repetitions."""
    import torch

    from paper_1904_04048_b200 import _native as nat

    sim = make_sim(cfg, T, tile)
    sim.first_step()
    stream = torch.cuda.current_stream()
    K = args.steps
    warm = args.warmup
    if warm:
        sim.march(warm)
    # ps_march_tile: ONE launch runs all K updates
    tiled = bool(sim.tile) and nat.tile_supported(sim.grid, sim.t_two, sim.tile)
    extra = None
    if T == 1 and K >= 12 and not tiled:
        # ps_march replays a CUDA graph for calls of >= 12 steps; instantiate it outside
        # the timed region with one extra 12-step call (reported, not hidden in `warmup`)
        sim.march(12)
        extra = {"steps": 12, "why": "one untimed 12-step ps_march call instantiates the "
                                      "CUDA graph the timed call replays"}
    torch.cuda.synchronize()
    regions, launches = [], 0
    reps = args.reps if args.reps > 0 else 3
    with ClockSampler(gpu_id(0)) as clk:
        for rep in range(reps):
            t_begin, t_end = (torch.cuda.Event(enable_timing=True),
                              torch.cuda.Event(enable_timing=True))
            launches0 = nat.launch_count()
            torch.cuda.synchronize()
            t_begin.record(stream)
            sim.march(K)      # K updates: back-to-back hot-kernel launches on one stream
            t_end.record(stream)
            torch.cuda.synchronize()
            launches = nat.launch_count() - launches0
            regions.append(t_begin.elapsed_time(t_end))
            if args.reps <= 0 and regions[0] > 2000.0:
                break
    total_ms = statistics.median(regions)
    lup_step = sim.updated_nodes
    avg_launch_ms = total_ms / K * T      # K/T launches of T fused updates each
    if tiled:
        T = K                             # accounting below: one launch of K updates
        avg_launch_ms = total_ms
    peak, peak_src = load_peak()
    # algorithmic traffic = 3 words per update (read u^k, u^{k-1}, write
    # u^{k+1}); a launch of depth T performs T * lup_step updates
    bytes_launch = 3.0 * T * sim.itemsize * lup_step
    achieved = bytes_launch / (avg_launch_ms * 1e-3) / 1e9
    # what the launch must move through DRAM: a fused pass of depth T reads two levels
    # and writes two for T updates (4/T words per update); T = 1 moves the 3 words
    dram_words = 3.0 if T == 1 else 4.0 / T
    dram_model = dram_words * T * sim.itemsize * lup_step
    return {"sim": sim, "T": T, "K": K, "warmup": warm, "warmup_extra": extra, "tiled": tiled,
            "total_ms": total_ms, "regions_ms": regions,
            "value": lup_step * K / (total_ms * 1e-3) / 1e9, "launches": launches,
            "clocks": clk.summary(), "lup_step": lup_step, "bytes_launch": bytes_launch,
            "avg_launch_ms": avg_launch_ms, "peak": peak, "peak_src": peak_src,
            "achieved": achieved, "dram_words": dram_words, "dram_model": dram_model,
            "dram_achieved": dram_model / (avg_launch_ms * 1e-3) / 1e9}


def roofline_block(m, cfg_name):
    """The `roofline` object (prompt ④ / SURVEY.md §8d D2) plus the DRAM-side view."""
    T = m["T"]
    traffic = load_traffic(cfg_name, T)
    roof = {"bound": "hbm", "achieved": m["achieved"], "peak": m["peak"], "unit": "GB/s",
            "frac": m["achieved"] / m["peak"], "traffic": traffic,
            "peak_source": m["peak_src"],
            "algorithmic_bytes_per_launch": m["bytes_launch"],
            "bytes_per_lup": 3 * m["sim"].itemsize,
            "lup_per_launch": m["lup_step"] * T,
            "kernel_ms_per_launch": m["avg_launch_ms"],
            "definition": "SURVEY.md §8(d): 3 words per update x updates per launch / mean "
                          "launch duration (CUDA events over the timed region), over the "
                          "measured HBM copy peak"}
    if T > 1:
        roof["note"] = (f"temporal blocking T={T} fuses {T} updates per pass, so a launch does "
                        f"{T}x the single-update algorithmic bytes while moving 4/T words per "
                        "update through DRAM: frac > 1 is expected (SURVEY.md §8d); `dram` "
                        "below is the memory-side fraction, `compute_roofline` the binding one")
    dram = {"model_words_per_lup": m["dram_words"], "model_bytes_per_launch": m["dram_model"],
            "achieved_gbs": m["dram_achieved"], "frac_of_peak": m["dram_achieved"] / m["peak"],
            "ncu_bytes_per_launch": traffic,
            "ncu_over_model": (traffic / m["dram_model"]) if traffic else None,
            "note": "bytes a launch must move through DRAM (T=1: 3 words/update; depth T: 2 "
                    "levels read + 2 written per T updates) / launch duration; ncu figure = "
                    "dram__bytes_read.sum + dram__bytes_write.sum of one launch "
                    "(profiles/ncu_<config>[_T<depth>].json)"}
    return roof, dram


def gpu_arm_single(args, cfg, cfg_name):
    import torch

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device visible (there is no CPU fallback; "
                         "`--impl reference` times the CPU path)")
    torch.cuda.set_device(torch.device("cuda", 0))
    # auto: the fastest measured depth per config, 1 where blocking is n/a
    T = args.tsteps if args.tsteps > 0 else cfg.get("tb", 1)
    companion = None
    if T > 1 and args.tsteps == 0:
        # also time the unblocked march (one update per launch) for the roofline story
        c1 = measure_march(args, cfg, 1)
        r1, d1 = roofline_block(c1, cfg_name)
        companion = {"temporal_blocking": 1, "value": c1["value"], "unit": "GLUP/s",
                     "ms_per_step": c1["total_ms"] / c1["K"],
                     "roofline_frac": r1["frac"], "achieved_gbs": c1["achieved"],
                     "traffic": r1["traffic"], "regions_ms": c1["regions_ms"],
                     "warmup_extra": c1["warmup_extra"], "clocks": c1["clocks"]}
        del c1
        torch.cuda.empty_cache()
    tile = args.tile if args.tile >= 0 else (cfg.get("tile", 0) if T == 1 else 0)
    if tile and args.tile < 0:
        # also time the streaming march (one CUDA-graph-replayed launch per update)
        c1 = measure_march(args, cfg, 1)
        r1, d1 = roofline_block(c1, cfg_name)
        companion = {"what": "streaming march: one launch per update, CUDA-graph replay + PDL",
                     "value": c1["value"], "unit": "GLUP/s",
                     "ms_per_step": c1["total_ms"] / c1["K"], "roofline_frac": r1["frac"],
                     "regions_ms": c1["regions_ms"], "warmup_extra": c1["warmup_extra"],
                     "clocks": c1["clocks"]}
        del c1
        torch.cuda.empty_cache()
    m = measure_march(args, cfg, T, tile)
    sim = m["sim"]
    roof, dram = roofline_block(m, cfg_name)
    if m["tiled"]:
        note = ("tile-resident march (ps_march_tile): ONE cooperative launch runs all the "
                f"region's updates, {tile} per shared-memory pass; levels stay in L2 / shared "
                "memory, so the 3-words-per-update figure is algorithmic, not DRAM traffic")
        roof["note"] = note
        roof["traffic"] = load_traffic(cfg_name + "_tile")
        dram = {"note": "L2-resident grid: no DRAM-side model (see roofline.note)",
                "ncu_bytes_per_launch": roof["traffic"]}
    line = {
        "metric": METRIC, "value": m["value"], "unit": "GLUP/s", "n_gpus": 1, "steps": m["K"],
        "warmup": m["warmup"], "ms_per_step": m["total_ms"] / m["K"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": cfg["dtype"],
        "data": "synthetic (seeded initial data per SURVEY.md §8d D1, generated on the device)",
        "config": single_config(cfg, T, tile if m["tiled"] else 0),
        "timing": {"regions_ms": m["regions_ms"], "reported": "median region",
                   "what": f"{len(m['regions_ms'])} back-to-back regions of exactly "
                           f"{m['K']} steps, each between CUDA events on the launching stream"},
        "roofline": roof,
        "dram": dram,
        "clocks": m["clocks"],
        "gpu_launches": m["launches"],
    }
    if m["warmup_extra"]:
        line["warmup_extra"] = m["warmup_extra"]
    if cfg["dtype"] == "f32":
        line["config"]["arith_note"] = (
            "native = the GPU's own f32 contract (one fma per tap, f32 accumulator), narrower "
            "than the reference's float32 path (f32 products summed in f64); the reference "
            "contract (--arith ref, bitwise = numpy) is conversion-bound, see DESIGN.md §9"
            if cfg["arith"] == "native" else
            "ref = the reference's float32 sequence (f32 products, f64 accumulator), bitwise")
    if T > 1:
        line["compute_roofline"] = compute_roofline(cfg, m["value"], T)
    if companion:
        line["unblocked_companion"] = companion
    if not args.no_e2e:
        line["e2e"] = e2e_single(args, cfg, sim)
    del m, sim
    torch.cuda.empty_cache()
    if not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args, cfg)
    print(json.dumps(line), flush=True)


def e2e_single(args, cfg, sim):
    """Same metric through the public C-ABI with host buffers: ps_solve_host takes the
    pinned host u0 (v0), returns u^K in a pinned host array, and overlaps the uploads and
    downloads with the march band by band (Dirichlet; periodic grids run it unbanded).
    The companion `sequential` leg times the plain order (ps_copy_in, ps_first_step,
    ps_march_tb, ps_copy_out) for comparison."""
    import ctypes

    import torch

    from paper_1904_04048_b200 import _native as nat

    n1 = cfg["n"] + 1
    u0_host, v0_host = sim.initial_fields()
    npdt = u0_host.dtype
    tdt = torch.float64 if npdt.itemsize == 8 else torch.float32
    pin_u = torch.from_numpy(u0_host).pin_memory()
    vzero = isinstance(cfg["ic"], tuple) and cfg["ic"][3]
    pin_v = None if vzero else torch.from_numpy(v0_host).pin_memory()
    del u0_host, v0_host
    out = torch.empty((n1, n1), dtype=tdt).pin_memory()
    st = nat.current_stream()
    lib = nat.load_library()
    g = sim.grid
    K = args.steps
    h2d = pin_u.numel() * pin_u.element_size() * (1 if pin_v is None else 2)
    d2h = out.numel() * out.element_size()

    while len(sim.levels) < 4:          # ps_solve_host wants four scratch levels
        sim.levels.append(nat.Level(sim.grid))

    def solve():
        nat.solve_host(g, sim.levels[:4], pin_u.data_ptr(),
                       None if pin_v is None else pin_v.data_ptr(), out.data_ptr(), n1,
                       sim.t_first_u, sim.t_first_v, sim.t_two, sim.tau, K, sim.tsteps,
                       args.bands, st)

    def sequential():
        nat.check(lib.ps_copy_in(ctypes.byref(g), sim.levels[1].ptr,
                                 ctypes.c_void_p(pin_u.data_ptr()), n1, n1, n1, nat.H2D, st),
                  "ps_copy_in")
        if pin_v is None:
            sim.levels[0].buf.zero_()
        else:
            nat.check(lib.ps_copy_in(ctypes.byref(g), sim.levels[0].ptr,
                                     ctypes.c_void_p(pin_v.data_ptr()), n1, n1, n1, nat.H2D, st),
                      "ps_copy_in")
        if cfg["bc"] == "periodic":
            sim.levels[1].fill_ghosts()
            sim.levels[0].fill_ghosts()
        sim.first_step()
        sim.march(K - 1)
        nat.check(lib.ps_copy_out(ctypes.byref(g), sim.levels[sim.newest].ptr,
                                  ctypes.c_void_p(out.data_ptr()), n1, n1, n1, nat.D2H, st),
                  "ps_copy_out")

    def timed(fn):
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launches0 = nat.launch_count()
        with ClockSampler(gpu_id(0)) as clk:
            t0.record()
            fn()
            t1.record()
            torch.cuda.synchronize()
        return t0.elapsed_time(t1), nat.launch_count() - launches0, clk.summary()

    ms_seq, _, _ = timed(sequential)
    ms, launches, clocks = timed(solve)
    return {"value": sim.updated_nodes * K / (ms * 1e-3) / 1e9, "unit": "GLUP/s",
            "h2d_bytes_per_step": h2d / K, "d2h_bytes_per_step": d2h / K,
            "steps": K, "ms_total": ms, "gpu_launches": launches, "clocks": clocks,
            "pcie_gbs": (h2d + d2h) / (ms * 1e-3) / 1e9,
            "note": f"one solve of {K} steps: {h2d / 1e9:.2f} GB in + {d2h / 1e9:.2f} GB out cross "
                    "PCIe once per solve, so short solves are copy-bound and the figure grows "
                    "with the step count (BASELINE step counts: --steps unset)",
            "what": "ps_solve_host: pinned host u0[,v0] in, u^K out to pinned host; row bands "
                    "marched as a skewed wavefront so the PCIe copies overlap the march "
                    "(one CUDA-event-timed region on the caller's stream)",
            "sequential": {"value": sim.updated_nodes * K / (ms_seq * 1e-3) / 1e9,
                           "ms_total": ms_seq,
                           "what": "ps_copy_in + ps_first_step + ps_march_tb + ps_copy_out, "
                                   "no overlap"}}


def dist_measure(args, cfg, T, keep_ics):
    """One row-slab march on this rank's slab at temporal-blocking depth T: seeded ICs on
    the device, halo exchange, first step, warm-up, then K steps between barriers and CUDA
    events; the reported time is the max over ranks."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1904_04048_b200 import _native as nat
    from paper_1904_04048_b200.device import gaussian_params
    from paper_1904_04048_b200.slab import DistributedSlabs

    _, _, local = dist_env()
    K = args.steps
    slab = DistributedSlabs(cfg["scheme"], cfg["n"], cfg["lam"], ring=cfg["ring"],
                            dtype=cfg["dtype"], arith=cfg["arith"], transport=args.transport,
                            tsteps=T, graph=not args.no_graph)
    K0, wmin, wmax, vzero = cfg["ic"]
    rng = np.random.default_rng(0)
    pu = gaussian_params(rng, K0, wmin, wmax)
    nat.gaussian_sum(slab.grid, slab.levels[1], pu[0], pu[1], pu[2], cfg["n"])
    if vzero:
        slab.levels[0].buf.zero_()
    else:
        pv = gaussian_params(rng, K0, wmin, wmax)
        nat.gaussian_sum(slab.grid, slab.levels[0], pv[0], pv[1], pv[2], cfg["n"])
    slab.exchange(1)
    slab.exchange(0)
    ics = None
    if keep_ics:  # keep this rank's rows of u0 / v0 for the end-to-end leg
        ics = (torch.from_numpy(slab.levels[1].download()).pin_memory(),
               None if vzero else torch.from_numpy(slab.levels[0].download()).pin_memory())
    slab.first_step()
    warm = (args.warmup + T - 1) // T * T      # whole passes (rounded up, reported)
    if warm:
        slab.march(warm)
    torch.cuda.synchronize()
    dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = nat.launch_count() + slab.launch_correction
    with ClockSampler(gpu_id(local)) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        t0.record()
        slab.march(K)
        t1.record()
        torch.cuda.synchronize()
        dist.barrier()
    launches = nat.launch_count() + slab.launch_correction - launches0
    ms = torch.tensor([t0.elapsed_time(t1)], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    total_ms = float(ms.item())
    inner = cfg["n"] + 1 - 2 * cfg["ring"]
    return {"slab": slab, "ics": ics, "T": T, "K": K, "warmup": warm, "total_ms": total_ms,
            "value": inner * inner * K / (total_ms * 1e-3) / 1e9, "launches": launches,
            "clocks": clk.summary(), "lup_step": inner * inner, "graphed": slab.graphed}


def gpu_arm_dist(args, cfg, cfg_name):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if not torch.cuda.is_available() or torch.cuda.device_count() <= local:
        raise SystemExit(f"bench.py: rank {rank} needs CUDA device {local}; "
                         f"{torch.cuda.device_count()} visible (no CPU fallback)")
    # the driver's rank check reads NCCL's own init lines
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if cfg["bc"] != "dirichlet" or not isinstance(cfg["ic"], tuple):
        raise SystemExit("multi-GPU bench supports the Dirichlet Gaussian configs (C3-C5)")
    K = args.steps
    T = args.tsteps if args.tsteps > 0 else cfg.get("tb", 1)
    while T > 1 and K % T:      # the timed region must hold whole blocked passes
        T -= 1
    companion = None
    if T > 1 and args.tsteps == 0:
        # the literal config ("per-step halo exchange of R rows per neighbour"): T = 1
        c1 = dist_measure(args, cfg, 1, False)
        companion = {"temporal_blocking": 1, "value": c1["value"], "unit": "GLUP/s",
                     "ms_per_step": c1["total_ms"] / K, "gpu_launches": c1["launches"],
                     "halo": f"{c1['slab'].R} row(s) per neighbour per step",
                     "cuda_graph": c1["graphed"], "clocks": c1["clocks"]}
        c1["slab"].close()
        del c1
        torch.cuda.empty_cache()
    m = dist_measure(args, cfg, T, not args.no_e2e)
    slab, total_ms = m["slab"], m["total_ms"]
    e2e = None if args.no_e2e else e2e_dist(args, cfg, slab, dist, m["ics"])
    lup_step = m["lup_step"]
    itemsize = 8 if cfg["dtype"] == "f64" else 4
    peak, peak_src = load_peak()
    # per GPU: 3 words per update x this GPU's share of the updates / step time (incl. exchange)
    achieved = 3.0 * itemsize * lup_step / world / (total_ms / K * 1e-3) / 1e9
    dram_words = 3.0 if T == 1 else 4.0 / T
    if rank == 0:
        line = {
            "metric": METRIC, "value": m["value"], "unit": "GLUP/s", "n_gpus": world, "steps": K,
            "warmup": m["warmup"], "ms_per_step": total_ms / K, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": cfg["dtype"],
            "data": "synthetic (seeded initial data per SURVEY.md §8d D1, generated on the device)",
            "config": dist_config(cfg, T, world, slab.R * T, args.transport, m["graphed"]),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": load_traffic(cfg_name, T),
                         "peak_source": peak_src + " (per GPU; whole-step time incl. exchange)",
                         "definition": "SURVEY.md §8(d): 3 words per update x this GPU's "
                                       "updates per step / step time, over the measured peak"},
            "dram": {"model_words_per_lup": dram_words,
                     "achieved_gbs": achieved * dram_words / 3.0,
                     "frac_of_peak": achieved * dram_words / 3.0 / peak},
            "clocks": m["clocks"],
            "gpu_launches": m["launches"],
            "e2e": e2e,
        }
        if companion:
            line["unblocked_companion"] = companion
        print(json.dumps(line), flush=True)
    slab.close()
    dist.destroy_process_group()


def e2e_dist(args, cfg, slab, dist, ics):
    """Per rank: own rows of u0 (and v0) from pinned host -> device, halo exchange, first
    step, K-1 steps, own rows of u^K -> pinned host; time = max over ranks."""
    import torch

    import ctypes

    from paper_1904_04048_b200 import _native as nat

    u_host, v_host = ics
    out = torch.empty_like(u_host).pin_memory()
    K = args.steps
    lib, g, st = nat.load_library(), slab.grid, nat.current_stream()
    rows, cols = u_host.shape

    def copy_in(level, host):   # cudaMemcpy2DAsync into the padded layout (pinned source)
        nat.check(lib.ps_copy_in(ctypes.byref(g), level.ptr, ctypes.c_void_p(host.data_ptr()),
                                 rows, cols, cols, nat.H2D, st), "ps_copy_in")

    torch.cuda.synchronize()
    dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    copy_in(slab.levels[1], u_host)
    if v_host is None:
        slab.levels[0].buf.zero_()
    else:
        copy_in(slab.levels[0], v_host)
    slab.exchange(1)
    slab.exchange(0)
    slab.first_step()
    more = (K - 1) // slab.T * slab.T          # whole blocked passes after the first step
    slab.march(more)
    nat.check(lib.ps_copy_out(ctypes.byref(g), slab.levels[slab.newest].ptr,
                              ctypes.c_void_p(out.data_ptr()), rows, cols, cols, nat.D2H, st),
              "ps_copy_out")
    t1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([t0.elapsed_time(t1)], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    inner = cfg["n"] + 1 - 2 * cfg["ring"]
    h2d = u_host.numel() * u_host.element_size() * (1 if v_host is None else 2)
    K = 1 + more
    return {"value": inner * inner * K / (float(ms.item()) * 1e-3) / 1e9, "unit": "GLUP/s",
            "h2d_bytes_per_step": h2d / K, "d2h_bytes_per_step": out.numel() * out.element_size() / K,
            "what": "per rank: own rows of u0[,v0] pinned host->device, halo exchange, first "
                    "step, K-1 steps, own rows of u^K -> pinned host; max over ranks "
                    "(bytes per rank)"}


def spawn_ranks(n: int) -> int:
    """`python bench.py --gpus N` without torchrun: check that N GPUs are visible, then
    re-execute this command line under torch.distributed.run with one rank per GPU."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < n:
        print(f"bench.py: --gpus {n} needs {n} visible CUDA devices, found {have}; refusing to "
              "report a smaller run as an N-GPU number", file=sys.stderr)
        return 2
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="C4")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--bands", type=int, default=0,
                    help="row bands of the e2e solve (0 = auto, ~1024 rows each)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--arith", choices=("ref", "native"), default=None,
                    help="f32 arithmetic contract override (ref: the reference's numpy "
                         "sequence with a float64 accumulator; native: one fma per tap)")
    ap.add_argument("--transport", choices=("nccl", "p2p"), default="nccl",
                    help="multi-GPU halo transport")
    ap.add_argument("--no-graph", action="store_true",
                    help="multi-GPU: launch each pass eagerly instead of replaying one "
                         "captured CUDA graph per pass")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the torch.distributed row-slab path even at world size 1 "
                         "(exercises the multi-GPU code on one GPU)")
    ap.add_argument("--reps", type=int, default=0,
                    help="repetitions of the K-step timed region (median reported); 0 = auto: "
                         "3 while a region takes under 2 s, else 1")
    ap.add_argument("--tile", type=int, default=-1,
                    help="tile-resident march depth for small Dirichlet f64 grids (ps_march_tile); "
                         "-1 = the config's default (C1: 12, with a streaming companion), 0 = off")
    ap.add_argument("--tsteps", type=int, default=0, choices=(0, 1, 2, 3, 4, 5, 6),
                    help="temporal blocking depth; 0 = the config's measured best (C4: 5; C2, C5 "
                         "and C3 f32: 4; C3 f64: 3; with an unblocked companion measurement; "
                         "C1: 1)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.arith and cfg["dtype"] == "f32":
        cfg["arith"] = args.arith
        if args.arith == "ref":
            # the f32 reference contract (f32 products widened into an f64 sum) is bound by
            # the F2F.F64.F32 conversion rate, not by HBM: blocking only adds recomputed halo
            # columns (C5 T=1 287 vs T=4 253 GLUP/s, C3 f32 266 vs 209)
            cfg["tb"] = 1
    if args.steps is None:
        args.steps = cfg["steps"]
    args.warmup = max(args.warmup, 0)
    world, rank, _ = dist_env()
    if args.impl == "reference":
        reference_arm(args, cfg, args.config)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if world > 1 or args.force_dist:
        if "WORLD_SIZE" not in os.environ:
            # --force-dist without torchrun: a world of one on the loopback rendezvous
            import socket
            with socket.socket() as sock:
                sock.bind(("127.0.0.1", 0))
                port = sock.getsockname()[1]
            for k, v in (("RANK", "0"), ("LOCAL_RANK", "0"), ("WORLD_SIZE", "1"),
                         ("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", str(port))):
                os.environ.setdefault(k, v)
        gpu_arm_dist(args, cfg, args.config)
    else:
        gpu_arm_single(args, cfg, args.config)


if __name__ == "__main__":
    main()
