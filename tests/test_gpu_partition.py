"""GPU tests of the row-partitioned single-system path:
`world` partitions hosted in one process on one GPU (exchange = device copies)
must reproduce the single-handle solve -- same global colour-major sweep
order, so only the cross-partition reductions differ in association."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2207_02543_b200 import _lib as L
from paper_2207_02543_b200 import problems as PR
from paper_2207_02543_b200.partition import setup_partitioned
from paper_2207_02543_b200.solver import BatchSolver
from tests.helpers import random_load_basis, to_scipy

pytestmark = pytest.mark.gpu


def _problem(dim, B):
    if dim == 2:
        m = PR.Mesh(2, 48, 24, 1, 2.0, 1.0, 1.0)
    else:
        m = PR.Mesh(3, 8, 8, 8, 1.0, 1.0, 1.0)
    rp, ci = m.pattern()
    f = m.rhs()
    E, _ = m.kl_field(np.arange(B, dtype=np.uint64) + np.uint64(31), 20 if dim == 2 else 30)
    V = m.assemble(E)
    phi = random_load_basis(to_scipy(rp, ci, V[0], m.n), 8, 3)
    return m, rp, ci, f, V, phi


@pytest.mark.parametrize("dim,B,world", [(2, 1, 1), (2, 1, 2), (2, 1, 3), (2, 8, 2), (2, 40, 3),
                                         (3, 1, 2), (3, 8, 4)])
@pytest.mark.parametrize("kp", [L.KP_RECURRENCE, L.KP_SPMV])
def test_partitioned_matches_single_handle(gpu, dim, B, world, kp):
    m, rp, ci, f, V, phi = _problem(dim, B)
    F = np.broadcast_to(f, (B, m.n)).copy()
    s = BatchSolver(0)
    s.set_pattern(rp, ci, m.block_size)
    s.set_values(V)
    s.set_basis(phi)
    s.setup(kp_update=kp)
    x1, it1, c1, st1, h1 = s.solve(F, None, 1e-8, 3000, x0_mode=L.X0_REDUCED)
    s.close()
    P, bounds, bs, st = setup_partitioned(rp, ci, V, f, phi, world, m.block_size, kp_update=kp)
    assert np.all(st == 0)
    xs, it2, c2, st2, h2 = P.solve(bs, 1e-8, 3000, L.X0_REDUCED)
    P.close()
    x2 = np.concatenate([xs[r] for r in range(world)], axis=1)
    assert np.all(st2 == 0) and np.all(c2) and np.all(c1)
    assert np.all(np.abs(it1 - it2) <= 1), (it1, it2)
    for b in range(B):
        k = min(int(it1[b]), int(it2[b])) + 1
        np.testing.assert_allclose(h2[b, :k], h1[b, :k], rtol=1e-8)
        if it1[b] == it2[b]:
            assert np.linalg.norm(x2[b] - x1[b]) <= 1e-9 * np.linalg.norm(x1[b])
    if world == 1:  # one partition = the single handle exactly (same reductions? no: same kernels)
        assert np.array_equal(it1, it2)


def test_nccl_transport_single_rank(gpu):
    """The NCCL transport (send/recv + allreduce through libnccl) with one
    rank must reproduce the in-process partition exactly."""
    from paper_2207_02543_b200.partition import (PartitionedSolver, local_rows, node_colors,
                                                 row_bounds)
    m, rp, ci, f, V, phi = _problem(2, 4)
    colors = node_colors(rp, ci, m.block_size)
    bounds = row_bounds(m.n, 1, m.block_size)
    out = []
    for uid in (None, PartitionedSolver.unique_id()):
        P = PartitionedSolver(1, 0, rank=0, nccl_uid=uid)
        rpl, cil, _ = local_rows(rp, ci, 0, m.n)
        P.set_pattern(0, m.n, bounds, rpl, cil, m.block_size, colors)
        P.set_values(0, V)
        P.set_basis(0, phi, np.zeros((0, phi.shape[1])))
        assert np.all(P.setup() == 0)
        xs, it, conv, st, h = P.solve({0: np.broadcast_to(f, (4, m.n))}, 1e-8, 3000)
        out.append((xs[0], it))
        P.close()
    assert np.array_equal(out[0][1], out[1][1]) and np.array_equal(out[0][0], out[1][0])


def test_c5_driver_end_to_end_small(gpu):
    """paper_2207_02543_b200/c5.py on a small hex8 config: distributed offline
    stage (bootstrap-coarse snapshot solves, Gram partials and Phi rows on the
    tensor cores, summed over partitions) and the row-partitioned query solve;
    1 vs 2 partitions agree (same global colouring, D11 association only)."""
    from paper_2207_02543_b200 import c5
    PR.CONFIGS["c98"] = PR.Config("c98", 3, 12, 6, 6, (2.0, 1.0, 1.0), 6, 8, 1, 30)
    try:
        res1, x1 = c5.run("c98", world=1, n_snapshots=8, snap_batch=4, log=lambda *a: None)
        res2, x2 = c5.run("c98", world=2, n_snapshots=8, snap_batch=4, log=lambda *a: None)
    finally:
        PR.CONFIGS.pop("c98")
    assert res1["converged"] and res2["converged"]
    assert abs(res1["iterations"] - res2["iterations"]) <= 1
    u1 = x1[0][0]
    u2 = np.concatenate([x2[0][0], x2[1][0]])
    assert np.linalg.norm(u1 - u2) <= 1e-7 * np.linalg.norm(u1)


@pytest.mark.parametrize("world", [1, 3])
def test_partitioned_graph_loop_equals_eager_loop(gpu, monkeypatch, world):
    """The captured partitioned loop (conditional-WHILE graph, device-side
    stopping) runs the same kernels in the same order as the eager host loop:
    bit-identical solutions and equal iteration counts; launch accounting."""
    m, rp, ci, f, V, phi = _problem(3, 2)
    out = []
    for eager in (False, True):
        if eager:
            monkeypatch.setenv("P2G_PART_EAGER", "1")
        P, bounds, bs, st = setup_partitioned(rp, ci, V, f, phi, world, m.block_size)
        xs, it, conv, status, hist = P.solve(bs, 1e-8, 3000, L.X0_REDUCED)
        per, total, mode = P.launch_counts()
        assert mode == (0 if eager else 1)
        assert per > 0 or eager
        out.append((np.concatenate([xs[r] for r in range(world)], axis=1), it, hist))
        P.close()
    (x1, it1, h1), (x0, it0, h0) = out
    assert np.array_equal(it1, it0)
    assert np.array_equal(x1, x0)
    k = int(it1.max()) + 1
    assert np.array_equal(h1[:, :k], h0[:, :k])


def test_partitioned_profile_single_partition(gpu):
    """p2g_part_profile_iteration: per-class times and algorithmic bytes of one
    hosted partition's iteration (the c5 bench roofline)."""
    m, rp, ci, f, V, phi = _problem(3, 1)
    P, bounds, bs, st = setup_partitioned(rp, ci, V, f, phi, 1, m.block_size)
    P.solve(bs, 1e-8, 3000, L.X0_REDUCED)
    prof = P.profile_iteration(2)
    P.close()
    assert prof["gs_backward"][0] > 0 and prof["gs_backward"][1] > 0
    assert prof["restrict"][1] > 0 and prof["prolong"][1] > 0
    assert set(prof) >= {"halo_allreduce", "residual", "spmv_dot"}
