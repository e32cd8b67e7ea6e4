"""Per-pass cost of the row-slab march at world size 1 against the resident march (same
grid, same fused kernel): isolates host/launch overhead of DistributedSlabs.  Run under
torchrun --nproc-per-node 1."""

from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps=3):
    import torch

    best = 1e30
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    import torch
    import torch.distributed as dist

    import bench
    from paper_1904_04048_b200 import _native as nat
    from paper_1904_04048_b200.slab import DistributedSlabs

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    cfg = bench.CONFIGS["C4"]
    K = 40
    res = {}
    sim = bench.make_sim(cfg, 4)
    sim.first_step()
    sim.march(12)
    res["simulation_march_tb"] = timed(lambda: sim.march(K))
    lv = sim.levels

    def rows_loop():
        cur, prev = sim.newest, sim.previous
        for _ in range(K // 4):
            f1, f2 = [x for x in range(4) if x not in (cur, prev)]
            nat.two_step_tb_rows(sim.grid, lv[cur], lv[prev], lv[f1], lv[f2], sim.t_two, 4, 0,
                                 sim.grid.rows)
            prev, cur = f1, f2
        sim.newest, sim.previous = cur, prev

    res["tb_rows_loop_same_grid"] = timed(rows_loop)
    del sim, lv
    torch.cuda.empty_cache()
    slab = DistributedSlabs(cfg["scheme"], cfg["n"], cfg["lam"], ring=cfg["ring"], tsteps=4)
    slab.levels[1].buf.zero_()
    slab.first_step()
    slab.march(12)
    res["slab_march"] = timed(lambda: slab.march(K))
    res["slab_grid_ghost"] = int(slab.grid.ghost)
    for k in list(res):
        if isinstance(res[k], float):
            res[k + "_glups"] = 1073610756 * K / (res[k] * 1e-3) / 1e9
    print(json.dumps(res))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
