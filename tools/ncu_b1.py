"""Profiling target for the single-instance (B = 1) hex8 kernels (c5's
shapes) on a smaller cube: a few PCG iterations, then eager iterations of
p2g_profile_iteration (every kernel launched outside the graph, so ncu lists
each one).  usage: python tools/ncu_b1.py [edge=128] [k=40] [reps=1]"""
import sys

import numpy as np

sys.path.insert(0, '.')
from paper_2207_02543_b200 import _lib as L  # noqa: E402
from paper_2207_02543_b200 import problems as PR  # noqa: E402
from paper_2207_02543_b200.solver import BatchSolver  # noqa: E402

edge = int(sys.argv[1]) if len(sys.argv) > 1 else 128
k = int(sys.argv[2]) if len(sys.argv) > 2 else 40
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
m = PR.Mesh(3, edge, edge, edge, 1.0, 1.0, 1.0)
rp, ci = m.pattern()
f = m.rhs()
E, _ = m.kl_field(np.array([7], dtype=np.uint64), 30)
phi = np.ascontiguousarray(np.linalg.qr(np.random.default_rng(0).standard_normal((m.n, k)))[0])
s = BatchSolver(0)
s.set_pattern(rp, ci, m.block_size)
s.assemble(m, E)
s.set_basis(phi)
s.setup()
s.solve(f[None, :], None, 1e-8, 5, x0_mode=L.X0_REDUCED, hist_cap=0)
try:  # NVTX range "profile" around the profiled iterations (ncu --nvtx-include profile/)
    import torch
    torch.cuda.nvtx.range_push("profile")
except Exception:
    torch = None
prof = s.profile_iteration(reps)
if torch is not None:
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
tot = sum(v[0] for v in prof.values())
pk = 6451.8
for kname, (ms_, by) in prof.items():
    if ms_ > 0:
        print(f'  {kname:18s} {ms_*1e3:9.1f} us  {by/1e6:9.1f} MB  {by/(ms_*1e-3)/1e9:8.1f} GB/s  '
              f'{by/(ms_*1e-3)/1e9/pk:5.2f}')
print(f'  total {tot:.3f} ms/iter (n = {m.n}, nnz = {m.nnz})')
