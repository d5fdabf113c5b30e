"""Probe: one 64-instance handle vs two 32-instance handles solving concurrently
(two host threads, two streams) on c2 -- does overlapping two batches' colour
phases hide the per-phase latency tails?"""
import sys, threading, time
import numpy as np
sys.path.insert(0, '.')
import torch
from paper_2207_02543_b200 import problems as PR, _lib as L
from paper_2207_02543_b200.solver import BatchSolver

cfg = PR.CONFIGS['c2']
prob = PR.build_problem(cfg, device=0)
B = cfg.batch
seeds = PR.query_seeds(cfg)
values = prob.values(seeds)
F = np.ascontiguousarray(np.broadcast_to(prob.f, (B, prob.mesh.n)))
dev = torch.device('cuda', 0)

def make(lo, hi):
    s = BatchSolver(0)
    s.set_pattern(prob.rp, prob.ci, prob.mesh.block_size)
    vd = torch.from_numpy(np.ascontiguousarray(values[lo:hi])).to(dev)
    bd = torch.from_numpy(np.ascontiguousarray(F[lo:hi])).to(dev)
    xd = torch.empty_like(bd)
    s.set_basis(prob.phi)
    return s, vd, bd, xd, hi - lo

def step(h):
    s, vd, bd, xd, n = h
    s.set_values_device(vd.data_ptr(), n)
    s.setup()
    return s.solve_device(bd.data_ptr(), xd.data_ptr(), None, L.X0_REDUCED, cfg.tol, 100000)

one = make(0, 64)
halves = [make(0, 32), make(32, 64)]
for _ in range(3):
    step(one)
    for h in halves: step(h)
torch.cuda.synchronize()
for rep in range(3):
    t = time.perf_counter(); r = step(one); torch.cuda.synchronize(); t1 = time.perf_counter() - t
    its = []
    t = time.perf_counter()
    th = [threading.Thread(target=lambda h=h: its.append(step(h)[0])) for h in halves]
    [x.start() for x in th]; [x.join() for x in th]
    torch.cuda.synchronize(); t2 = time.perf_counter() - t
    print(f'one 64-batch {t1*1e3:.1f} ms (max it {int(r[0].max())}); two 32-batches concurrent {t2*1e3:.1f} ms (max it {[int(i.max()) for i in its]})', flush=True)
t = time.perf_counter(); step(halves[0]); torch.cuda.synchronize(); print('one 32-batch alone', (time.perf_counter()-t)*1e3, 'ms')
