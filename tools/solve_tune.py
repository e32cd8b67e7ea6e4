"""Sweep ps_solve_host's band count, compute streams and fused-pass tile height on one
config (default C4) and print one JSON line per setting (CUDA-event time of the whole
host-to-host solve; the sequential copy-in / march / copy-out order first)."""

from __future__ import annotations

import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import argparse

    import torch

    import bench
    from paper_1904_04048_b200 import _native as nat

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--bands", default="4,8,16,32")
    ap.add_argument("--streams", default="1,2,3")
    ap.add_argument("--rc", default="128,256,512")
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    T = cfg.get("tb", 1)
    sim = bench.make_sim(cfg, T)
    n1 = cfg["n"] + 1
    u0, v0 = sim.initial_fields()
    vzero = isinstance(cfg["ic"], tuple) and cfg["ic"][3]
    pu = torch.from_numpy(u0).pin_memory()
    pv = None if vzero else torch.from_numpy(v0).pin_memory()
    del u0, v0
    out = torch.empty_like(pu).pin_memory()
    st = nat.current_stream()

    def run(bands):
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        nat.solve_host(sim.grid, sim.levels[:4], pu.data_ptr(), None if pv is None else pv.data_ptr(),
                       out.data_ptr(), n1, sim.t_first_u, sim.t_first_v, sim.t_two, sim.tau,
                       a.steps, T, bands, st)
        t1.record()
        torch.cuda.synchronize()
        return t0.elapsed_time(t1)

    run(1)  # warm-up
    ref = out.clone()
    for b, s, rc in itertools.product(*(map(int, x.split(",")) for x in (a.bands, a.streams, a.rc))):
        os.environ["PS_SOLVE_STREAMS"] = str(s)
        os.environ["PS_SOLVE_RC"] = str(rc)
        ms = min(run(b) for _ in range(2))
        same = torch.equal(out.view(torch.int64 if out.dtype == torch.float64 else torch.int32),
                           ref.view(torch.int64 if ref.dtype == torch.float64 else torch.int32))
        glups = sim.updated_nodes * a.steps / (ms * 1e-3) / 1e9
        print(json.dumps({"config": a.config, "bands": b, "streams": s, "rc": rc, "ms": ms,
                          "glups": glups, "bitwise_same_as_1band": same}), flush=True)


if __name__ == "__main__":
    main()
