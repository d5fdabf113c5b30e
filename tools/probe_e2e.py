"""Break one c2 e2e step (bench.py's pipelined C-ABI path) into its calls, host wall clock."""
import sys, time, ctypes as C
import numpy as np
sys.path.insert(0, '.')
import torch
from paper_2207_02543_b200 import problems as PR, _lib as L
from paper_2207_02543_b200.solver import BatchSolver

cfg = PR.CONFIGS['c2']
prob = PR.build_problem(cfg, device=0)
B = cfg.batch
values = prob.values(PR.query_seeds(cfg))
F = np.ascontiguousarray(np.broadcast_to(prob.f, (B, prob.mesh.n)))
s = BatchSolver(0); s.set_pattern(prob.rp, prob.ci, prob.mesh.block_size); s.set_basis(prob.phi); s.B = B
vals_h = torch.from_numpy(values).pin_memory(); b_h = torch.from_numpy(F).pin_memory(); x_h = torch.empty_like(b_h).pin_memory()
lib = L.lib(); Dp = L.D
it_h = np.zeros(B, dtype=np.int64); cv_h = np.zeros(B, dtype=np.int32); st_h = np.zeros(B, dtype=np.int32)
def solve():
    return lib.p2g_solve(s._h, C.cast(b_h.data_ptr(), Dp), None, L.X0_REDUCED, cfg.tol, 100000, C.cast(x_h.data_ptr(), Dp),
                         it_h.ctypes.data_as(L.I64), cv_h.ctypes.data_as(L.I32), st_h.ctypes.data_as(L.I32), None, 0)
lib.p2g_set_values(s._h, B, C.cast(vals_h.data_ptr(), Dp)); s.setup(); solve()
for rep in range(4):
    t = [time.perf_counter()]
    lib.p2g_set_values(s._h, B, C.cast(vals_h.data_ptr(), Dp)); t.append(time.perf_counter())
    if rep < 3: lib.p2g_prefetch_values(s._h, B, C.cast(vals_h.data_ptr(), Dp))
    t.append(time.perf_counter())
    s.setup(); t.append(time.perf_counter())
    solve(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print('set_values %.2f  prefetch %.2f  setup %.2f  solve %.2f  total %.2f  dev %s' % (*d, sum(d), s.last_solve_ms()), flush=True)
s.close()
