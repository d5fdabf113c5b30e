"""Quick end-to-end probe: config c2 (or argv[1]) basis + batched solve timing."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from paper_2207_02543_b200 import problems as PR, _lib as L
from paper_2207_02543_b200.solver import BatchSolver

name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
cfg = PR.CONFIGS[name]
t = time.time()
prob = PR.build_problem(cfg)
print(f'{name}: n={prob.mesh.n} nnz={prob.mesh.nnz} k={prob.phi.shape[1]} build {time.time()-t:.2f}s '
      f'snapshot iters {prob.snapshot_iters.min()}..{prob.snapshot_iters.max()}', flush=True)
t = time.time()
V = prob.values(PR.query_seeds(cfg))
print(f'values {V.shape} {time.time()-t:.2f}s', flush=True)
s = BatchSolver(0)
s.set_pattern(prob.rp, prob.ci, prob.mesh.block_size)
for rep in range(3):
    t = time.time()
    s.set_values(V); s.set_basis(prob.phi); st = s.setup()
    F = np.broadcast_to(prob.f, (cfg.batch, prob.mesh.n)).copy()
    x, it, conv, status, hist = s.solve(F, None, cfg.tol, 20000, x0_mode=L.X0_REDUCED)
    wall = time.time() - t
    ms = s.last_solve_ms()
    print(f'rep {rep}: iters {it.min()}..{it.max()} mean {it.mean():.1f} conv {conv.all()} status {set(status.tolist())} '
          f'wall {wall*1e3:.1f} ms device {ms[0]:.2f} ms loop {ms[1]:.2f} ms -> {cfg.batch/(ms[0]/1e3):.1f} solves/s', flush=True)
print('launches', s.launch_counts())
prof = s.profile_iteration(5)
tot = sum(v[0] for v in prof.values())
for kname, (ms_, by) in prof.items():
    gbs = by / (ms_ * 1e-3) / 1e9 if ms_ > 0 else 0
    print(f'  {kname:18s} {ms_*1e3:9.1f} us  {by/1e6:9.1f} MB  {gbs:8.1f} GB/s  share {ms_/tot*100:5.1f}%')
print(f'  total {tot:.3f} ms/iter')
