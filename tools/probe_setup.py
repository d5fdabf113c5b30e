"""Break down one bench step (c2) into its C-ABI calls (host wall, synchronous calls)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import torch
from paper_2207_02543_b200 import problems as PR, _lib as L
from paper_2207_02543_b200.solver import BatchSolver

cfg = PR.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else 'c2']
m = PR.Mesh.for_config(cfg)
rp, ci = m.pattern(); f = m.rhs()
V = m.assemble(m.kl_field(PR.query_seeds(cfg), cfg.kl_terms)[0])
rng = np.random.default_rng(0)
phi = np.ascontiguousarray(np.linalg.qr(rng.standard_normal((m.n, cfg.k)))[0])
dev = torch.device('cuda', 0)
vd = torch.from_numpy(V).to(dev); bd = torch.from_numpy(np.broadcast_to(f, (cfg.batch, m.n)).copy()).to(dev)
xd = torch.empty_like(bd)
s = BatchSolver(0); s.set_pattern(rp, ci, m.block_size)
for rep in range(4):
    t = [time.perf_counter()]
    s.set_values_device(vd.data_ptr(), cfg.batch); torch.cuda.synchronize(); t.append(time.perf_counter())
    s.set_basis(phi); torch.cuda.synchronize(); t.append(time.perf_counter())
    s.setup(); torch.cuda.synchronize(); t.append(time.perf_counter())
    it, conv, st, _ = s.solve_device(bd.data_ptr(), xd.data_ptr(), None, L.X0_REDUCED, 1e-8, 3); torch.cuda.synchronize(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f'set_values {d[0]:.2f} ms  set_basis {d[1]:.2f}  setup {d[2]:.2f}  solve(3 it) {d[3]:.2f}  ms_dev {s.last_solve_ms()}', flush=True)
