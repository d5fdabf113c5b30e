"""Per-kernel-class profile of a single-instance (B = 1) solve: 2D c1 and a 3D hex8 cube."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2207_02543_b200 import problems as PR, _lib as L
from paper_2207_02543_b200.solver import BatchSolver

CASES = [(2, 64, 32, 1, 2.0), (3, 80, 80, 80, 1.0), (3, 128, 128, 128, 1.0)]
if len(sys.argv) > 1:  # e.g. "3,80": one case
    d, m_ = map(int, sys.argv[1].split(","))
    CASES = [c for c in CASES if c[0] == d and c[1] == m_]
for dims in CASES:
    dim, nx, ny, nz, Lx = dims
    m = PR.Mesh(dim, nx, ny, nz, Lx, 1.0, 1.0)
    rp, ci = m.pattern()
    f = m.rhs()
    E, _ = m.kl_field(np.array([7], dtype=np.uint64), 20 if dim == 2 else 30)
    rng = np.random.default_rng(0)
    k = 10 if dim == 2 else 30
    phi = np.ascontiguousarray(np.linalg.qr(rng.standard_normal((m.n, k)))[0])
    s = BatchSolver(0)
    s.set_pattern(rp, ci, m.block_size)
    s.assemble(m, E)
    s.set_basis(phi)
    s.setup()
    x, it, conv, st, h = s.solve(f[None, :], None, 1e-8, 30, x0_mode=L.X0_REDUCED, hist_cap=0)
    ms = s.last_solve_ms()
    prof = s.profile_iteration(3)
    tot = sum(v[0] for v in prof.values())
    print(f"dim {dim} n={m.n} nnz={m.nnz}: graph loop {ms[1]/max(int(it[0]),1):.3f} ms/iter ({int(it[0])} it); eager profile {tot:.3f} ms/iter")
    for kname, (t, by) in prof.items():
        if t > 0:
            print(f"   {kname:18s} {t*1e3:9.1f} us {by/1e6:9.1f} MB {by/(t*1e-3)/1e9:8.0f} GB/s")
    s.close()
