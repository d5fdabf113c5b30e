"""Is the nvidia-smi sampler perturbing the timed region?  Step times with/without it."""
import sys, time, subprocess
import numpy as np
sys.path.insert(0, '.')
import torch
import bench
from paper_2207_02543_b200 import problems as PR, _lib as L
from paper_2207_02543_b200.solver import BatchSolver
cfg = PR.CONFIGS['c2']
prob = PR.build_problem(cfg)
B, seeds, strong = PR.shard(cfg, 1, 0)
V = prob.values(seeds)
dev = torch.device('cuda', 0)
vd = torch.from_numpy(V).to(dev); bd = torch.from_numpy(np.broadcast_to(prob.f, (B, prob.mesh.n)).copy()).to(dev)
xd = torch.empty_like(bd)
s = BatchSolver(0); s.set_pattern(prob.rp, prob.ci, prob.mesh.block_size)
st = torch.cuda.ExternalStream(s.stream(), device=dev)
def step():
    s.set_values_device(vd.data_ptr(), B); s.set_basis(prob.phi); s.setup()
    return s.solve_device(bd.data_ptr(), xd.data_ptr(), None, L.X0_REDUCED, 1e-8, 100000)
for _ in range(2): step()
for mode in ['plain', 'clocks', 'plain']:
    ctx = bench.Clocks(0) if mode == 'clocks' else None
    if ctx: ctx.__enter__()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(st)
    per = []
    for _ in range(4):
        a = time.perf_counter(); it, conv, status, _ = step(); per.append((time.perf_counter()-a)*1e3)
    e1.record(st); torch.cuda.synchronize()
    if ctx: ctx.__exit__(None, None, None)
    print(mode, 'event ms/step %.1f' % (e0.elapsed_time(e1)/4), 'wall per step', ['%.1f' % p for p in per], 'solve dev ms', s.last_solve_ms(), flush=True)
