"""Host logic of the row-partitioned path on CPU: the partition
plans of all ranks agree (what rank r sends to q per colour is exactly what q
expects as ghosts from r), ghosts are whole nodes, owned rows cover the
system; plus a world-size-2 gloo run where each rank plans only from its own
rows and the counts are checked across processes."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from paper_2207_02543_b200 import problems as PR
from paper_2207_02543_b200.partition import local_rows, node_colors, plan, row_bounds


def _system(dim):
    if dim == 2:
        m = PR.Mesh(2, 12, 6, 1, 2.0, 1.0, 1.0)
    else:
        m = PR.Mesh(3, 4, 4, 4, 1.0, 1.0, 1.0)
    rp, ci = m.pattern()
    return m, rp, ci


@pytest.mark.parametrize("dim,world", [(2, 1), (2, 2), (2, 3), (3, 2), (3, 4)])
def test_partition_plans_are_consistent(dim, world):
    m, rp, ci = _system(dim)
    n, bs = m.n, m.block_size
    colors = node_colors(rp, ci, bs)
    bounds = row_bounds(n, world, bs)
    plans = []
    for r in range(world):
        rpl, cil, _ = local_rows(rp, ci, int(bounds[r]), int(bounds[r + 1]))
        plans.append(plan(r, world, bounds, n, rpl, cil, bs, colors))
    assert sum(p["n_own"] for p in plans) == n
    assert sum(p["nnz"] for p in plans) == int(rp[-1])
    for r, p in enumerate(plans):
        r0, r1 = int(bounds[r]), int(bounds[r + 1])
        lo, hi = int(rp[r0]), int(rp[r1])
        outside = {int(c) for c in ci[lo:hi] if not r0 <= c < r1}
        whole = {c - c % bs + q for c in outside for q in range(bs)}
        assert set(p["ghosts"].tolist()) == whole
        for q in range(world):
            # r sends to q per colour exactly what q receives from r
            assert np.array_equal(p["send"][:, q], plans[q]["recv"][:, r])
        assert p["send"][:, r].sum() == 0 and p["recv"][:, r].sum() == 0


def test_partition_rejects_bad_input():
    m, rp, ci = _system(2)
    colors = node_colors(rp, ci, 2)
    bounds = row_bounds(m.n, 2, 2)
    rpl, cil, _ = local_rows(rp, ci, 0, int(bounds[1]))
    with pytest.raises(ValueError):
        plan(0, 2, np.array([0, 3, m.n]), m.n, rpl, cil, 2, colors)  # not node aligned
    with pytest.raises(ValueError):
        plan(2, 2, bounds, m.n, rpl, cil, 2, colors)  # bad rank


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, rp, ci = _system(3)
    colors = node_colors(rp, ci, 3)
    bounds = row_bounds(m.n, world, 3)
    rpl, cil, _ = local_rows(rp, ci, int(bounds[rank]), int(bounds[rank + 1]))
    p = plan(rank, world, bounds, m.n, rpl, cil, 3, colors)
    send = torch.from_numpy(p["send"].copy())
    recv = torch.from_numpy(p["recv"].copy())
    sends = [torch.zeros_like(send) for _ in range(world)]
    recvs = [torch.zeros_like(recv) for _ in range(world)]
    dist.all_gather(sends, send)
    dist.all_gather(recvs, recv)
    ok = all(torch.equal(sends[r][:, s], recvs[s][:, r]) for r in range(world) for s in range(world))
    if rank == 0:
        q.put(ok)
    dist.destroy_process_group()


def test_partition_plans_agree_across_gloo_ranks():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok
