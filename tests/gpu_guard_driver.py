"""Run by tests/test_gpu_guard.py in a subprocess with P2G_GUARD=1: every
kernel family at every lane shape (solve, setup, x0, spmv, preconditioner,
sweeps, pod2g_solve, profile, prefetch, partitioned path), then the guard
bands of every live buffer are checked.  Prints 'guard <n>' and exits 0."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_02543_b200 import _lib as L  # noqa: E402
from paper_2207_02543_b200 import problems as PR  # noqa: E402
from paper_2207_02543_b200.partition import setup_partitioned  # noqa: E402
from paper_2207_02543_b200.solver import BatchSolver  # noqa: E402

assert os.environ.get("P2G_GUARD") == "1"
live = []
rng = np.random.default_rng(0)
for dims, B, k in [((2, 24, 12, 1), 1, 10), ((2, 24, 12, 1), 8, 10), ((2, 24, 12, 1), 40, 20),
                   ((2, 24, 12, 1), 70, 30), ((2, 16, 8, 1), 256, 30), ((3, 5, 5, 5), 1, 40),
                   ((3, 5, 5, 5), 8, 8), ((3, 5, 5, 5), 33, 30), ((3, 5, 5, 5), 64, 64)]:
    dim, nx, ny, nz = dims
    m = PR.Mesh(dim, nx, ny, nz, 2.0 if dim == 2 else 1.0, 1.0, 1.0)
    rp, ci = m.pattern()
    E, _ = m.kl_field(np.arange(B, dtype=np.uint64) + np.uint64(3), 20 if dim == 2 else 30)
    V = m.assemble(E)
    phi = np.ascontiguousarray(np.linalg.qr(rng.standard_normal((m.n, k)))[0])
    s = BatchSolver(0)
    s.set_pattern(rp, ci, m.block_size)
    s.set_values(V)
    s.prefetch_values(V)
    s.set_values(V)
    s.set_basis(phi)
    s.setup()
    F = np.broadcast_to(m.rhs(), (B, m.n)).copy()
    s.solve(F, None, 1e-8, 300, x0_mode=L.X0_REDUCED)
    s.profile_iteration(1)
    s.spmv(F)
    s.precond_apply(F)
    s.smooth(0, F, F)
    s.smooth(1, F, F)
    s.initial_guess(F)
    s.pod2g_solve(F, None, 1e-8, 50, x0_mode=L.X0_REDUCED)
    s.solve(F[:, :], None, 1e-8, 20, x0_mode=L.X0_ZERO, hist_cap=5)
    live.append(s)
    print("ok", dims, B, k, flush=True)
m = PR.Mesh(3, 6, 6, 6, 1.0, 1.0, 1.0)
rp, ci = m.pattern()
V = m.assemble(m.kl_field(np.arange(2, dtype=np.uint64), 30)[0])
phi = np.ascontiguousarray(np.linalg.qr(rng.standard_normal((m.n, 8)))[0])
P, bounds, bs, st = setup_partitioned(rp, ci, V, m.rhs(), phi, 3, m.block_size)
P.solve(bs, 1e-8, 300, L.X0_REDUCED)
print("guard", L.lib().p2g_debug_guard_check(), flush=True)
P.close()
for s in live:
    s.close()
