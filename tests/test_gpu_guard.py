"""Out-of-bounds device writes and run-to-run determinism, in place of
compute-sanitizer (closed on the GPU pool this repo is measured on):

* guard bands (P2G_GUARD=1): every handle buffer is bracketed by bands of a
  fixed byte pattern; after every kernel family ran at every lane shape
  (tests/gpu_guard_driver.py), no band may have changed;
* races: the colour-phase sweeps update s in place, the reductions go through
  DSMEM cluster partials and an atomic ticket -- a race would show up as
  run-to-run differences, so repeated solves must be bit-identical."""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_no_out_of_bounds_writes_guard_bands(gpu):
    env = dict(os.environ, P2G_GUARD="1")
    r = subprocess.run([sys.executable, os.path.join(HERE, "gpu_guard_driver.py")],
                       capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("guard ")]
    assert lines and lines[-1] == "guard 0", r.stdout[-3000:]


@pytest.mark.parametrize("dims,B", [((2, 32, 16, 1), 64), ((2, 16, 8, 1), 256),
                                    ((3, 8, 8, 8), 64), ((3, 8, 8, 8), 1), ((2, 32, 16, 1), 1)])
def test_repeated_solves_are_bit_identical(gpu, dims, B):
    from paper_2207_02543_b200 import _lib as L
    from paper_2207_02543_b200 import problems as PR
    from paper_2207_02543_b200.solver import BatchSolver
    dim, nx, ny, nz = dims
    m = PR.Mesh(dim, nx, ny, nz, 2.0 if dim == 2 else 1.0, 1.0, 1.0)
    rp, ci = m.pattern()
    V = m.assemble(m.kl_field(np.arange(B, dtype=np.uint64) + np.uint64(11), 20 if dim == 2 else 30)[0])
    phi = np.ascontiguousarray(np.linalg.qr(np.random.default_rng(1).standard_normal((m.n, 12)))[0])
    F = np.broadcast_to(m.rhs(), (B, m.n)).copy()
    out = []
    for rep in range(3):
        s = BatchSolver(0)
        s.set_pattern(rp, ci, m.block_size)
        s.set_values(V)
        s.set_basis(phi)
        s.setup()
        x, it, conv, st, hist = s.solve(F, None, 1e-8, 3000, x0_mode=L.X0_REDUCED)
        S = s.precond_apply(F)
        out.append((x, it, hist, S))
        s.close()
    for o in out[1:]:
        for a, b in zip(out[0], o):
            assert np.array_equal(a, b, equal_nan=True)
