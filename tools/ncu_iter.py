"""Profiling target: one config's batched solve state, then eager iterations
(p2g_profile_iteration) -- keep the launch count small for ncu.
Usage: python tools/ncu_iter.py [c2] [reps]"""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2207_02543_b200 import problems as PR, _lib as L
from paper_2207_02543_b200.solver import BatchSolver

name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
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
import os
if not os.environ.get('NO_SOLVE'):
    s.solve(F, None, 1e-8, 3, x0_mode=L.X0_REDUCED)
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
for kname, (ms_, by) in prof.items():
    gbs = by / (ms_ * 1e-3) / 1e9 if ms_ > 0 else 0
    print(f'  {kname:18s} {ms_*1e3:9.1f} us  {by/1e6:9.1f} MB  {gbs:8.1f} GB/s  share {ms_/tot*100:5.1f}%')
print(f'  total {tot:.3f} ms/iter')
