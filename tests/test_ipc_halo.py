"""Cross-process halo delivery through CUDA IPC on one device (the p2p transport's
plumbing: ps_ipc_get_handle / ps_ipc_open / ps_two_step_halo into a peer's ghost rows).

Two processes share cuda:0.  The "upper" process owns a slab level and publishes its IPC
handle; the "lower" process maps it and runs ps_two_step_halo, whose boundary CTAs store
the lower slab's first rows straight into the upper slab's ghost rows.  No kernel waits
on another process (the parent sequences the two through pipes), so this is safe on one
GPU; on a multi-GPU box the same calls map a neighbour GPU's memory over NVLink.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _upper(conn, n, rows_up):
    import torch

    from paper_1904_04048_b200 import _native as nat

    torch.cuda.set_device(0)
    g = nat.make_slab_grid(n + 1, n + 1, 0, rows_up, 2, 1, "dirichlet", "f64")
    lv = nat.Level(g)
    lv.buf.fill_(0)
    torch.cuda.synchronize()
    conn.send(nat.ipc_handle(lv.ptr.value))
    conn.recv()                                   # lower slab's kernel has finished
    g_full = lv.buf.view(torch.float64)
    start = (g.ghost + rows_up) * g.pitch + (g.origin - g.ghost * g.pitch)
    conn.send(g_full[start:start + n + 1].cpu().numpy()[None, :])
    conn.close()


def _lower(conn, n, rows_up, uk, ukm1, pairs):
    import torch

    from paper_1904_04048_b200 import _native as nat

    torch.cuda.set_device(0)
    handle, off = conn.recv()
    peer = nat.ipc_open(handle)
    rows = n + 1 - rows_up
    g = nat.make_slab_grid(n + 1, n + 1, rows_up, rows, 2, 1, "dirichlet", "f64")
    a, b, out = nat.Level(g), nat.Level(g), nat.Level(g)
    a.upload(uk[rows_up:])            # own rows of u^k
    b.upload(ukm1[rows_up:])
    # ghost row above (the upper slab's last row): global row rows_up-1
    flat = a.buf.view(torch.float64)
    gstart = (g.ghost - 1) * g.pitch + (g.origin - g.ghost * g.pitch)
    flat[gstart:gstart + n + 1].copy_(torch.from_numpy(uk[rows_up - 1]))
    t = nat.make_table(pairs)
    nat.two_step_halo(g, a, b, out, t, 0, g.rows, peer + off, rows_up, None)
    torch.cuda.synchronize()
    mine = out.download()
    nat.ipc_close(peer)
    conn.send(mine)
    conn.close()


def test_ipc_halo_store_into_peer_ghost_rows(tmp_path):
    import torch.multiprocessing as mp

    from oracle import oracle as O
    from paper_1904_04048_b200.scheme import evaluate_table, named_scheme

    n, rows_up = 300, 140
    spec = named_scheme("P9")
    pairs = evaluate_table(spec.two_step, 0.6)
    rng = np.random.default_rng(4)
    uk, ukm1 = rng.normal(size=(n + 1, n + 1)), rng.normal(size=(n + 1, n + 1))
    ctx = mp.get_context("spawn")
    up_parent, up_child = ctx.Pipe()
    lo_parent, lo_child = ctx.Pipe()
    pu = ctx.Process(target=_upper, args=(up_child, n, rows_up))
    pl = ctx.Process(target=_lower, args=(lo_child, n, rows_up, uk, ukm1, pairs))
    pu.start()
    pl.start()
    try:
        lo_parent.send(up_parent.recv())          # hand the IPC handle to the lower slab
        mine = lo_parent.recv()                   # lower slab updated, halo stored
        up_parent.send("done")
        ghost = up_parent.recv()
    finally:
        pl.join(60)
        pu.join(60)
    assert pu.exitcode == 0 and pl.exitcode == 0
    want = O.two_step(uk, ukm1, pairs, "dirichlet", 1)
    # the lower slab's own rows, and its first row delivered into the upper's ghost row
    assert mine.tobytes() == want[rows_up:].tobytes()
    assert ghost[0].tobytes() == want[rows_up].tobytes()
