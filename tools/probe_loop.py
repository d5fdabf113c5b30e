"""Fixed-length PCG loop timing (no instance converges: tol = 0): ms per
iteration of the captured WHILE graph, every instance active throughout.
Usage: python tools/probe_loop.py [c2] [iters]"""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2207_02543_b200 import problems as PR, _lib as L
from paper_2207_02543_b200.solver import BatchSolver

name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = PR.CONFIGS[name]
m = PR.Mesh.for_config(cfg)
rp, ci = m.pattern()
f = m.rhs()
V = m.assemble(m.kl_field(PR.query_seeds(cfg), cfg.kl_terms)[0])
rng = np.random.default_rng(0)
phi, _ = np.linalg.qr(rng.standard_normal((m.n, cfg.k)))
s = BatchSolver(0)
s.set_pattern(rp, ci, m.block_size)
s.set_values(V)
s.set_basis(np.ascontiguousarray(phi))
s.setup()
F = np.broadcast_to(f, (cfg.batch, m.n)).copy()
for rep in range(3):
    x, it, conv, status, hist = s.solve(F, None, 0.0, iters, x0_mode=L.X0_REDUCED)
    ms = s.last_solve_ms()
    print(f'rep {rep}: iters {it.min()}..{it.max()} loop {ms[1]:.2f} ms -> {ms[1] / it.max() * 1e3:.1f} us/iteration', flush=True)
