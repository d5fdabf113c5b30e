"""Probe: two full 64-instance c2 batches on two handles (two streams, two
host threads) concurrently vs one after the other -- do the two batches'
colour phases fill each other's latency tails?"""
import sys, threading, time
import numpy as np
sys.path.insert(0, '.')
import torch
from paper_2207_02543_b200 import problems as PR, _lib as L
from paper_2207_02543_b200.solver import BatchSolver

cfg = PR.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else 'c2']
prob = PR.build_problem(cfg, device=0)
B = min(cfg.batch, 64)
dev = torch.device('cuda', 0)

def make(off):
    s = BatchSolver(0)
    s.set_pattern(prob.rp, prob.ci, prob.mesh.block_size)
    v = prob.values(PR.query_seeds(cfg, B, offset=off))
    vd = torch.from_numpy(v).to(dev)
    bd = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(prob.f, (B, prob.mesh.n)))).to(dev)
    xd = torch.empty_like(bd)
    s.set_basis(prob.phi)
    return s, vd, bd, xd

def step(h):
    s, vd, bd, xd = h
    s.set_values_device(vd.data_ptr(), B)
    s.setup()
    return s.solve_device(bd.data_ptr(), xd.data_ptr(), None, L.X0_REDUCED, cfg.tol, 100000)

hs = [make(0), make(B)]
for _ in range(2):
    for h in hs: step(h)
torch.cuda.synchronize()
for rep in range(3):
    t = time.perf_counter()
    for h in hs: step(h)
    torch.cuda.synchronize(); t1 = time.perf_counter() - t
    t = time.perf_counter()
    th = [threading.Thread(target=lambda h=h: step(h)) for h in hs]
    [x.start() for x in th]; [x.join() for x in th]
    torch.cuda.synchronize(); t2 = time.perf_counter() - t
    print(f'{cfg.name}: two {B}-batches sequential {t1*1e3:.1f} ms, concurrent {t2*1e3:.1f} ms '
          f'({t1/t2:.3f}x)', flush=True)
