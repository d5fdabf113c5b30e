"""Randomised A/B of the warp-specialised projections (k_restrict_ws / k_prolong_ws, forced)
against the register-fed kernels: preconditioner applications and initial guesses over random
mesh sizes (partial last tiles), POD ranks in every KMAX bucket and batch sizes (tile widths
64 / 128 / 256, several tiles).  Usage: python tools/stress_ws.py [cases] [seed]"""
import os
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2207_02543_b200 import problems as PR
from paper_2207_02543_b200.solver import BatchSolver

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
worst = 0.0
for case in range(cases):
    dim = 2 if rng.random() < 0.7 else 3
    if dim == 2:
        ny = int(rng.integers(5, 40)); nx = 2 * ny
        m = PR.Mesh(2, nx, ny, 1, 2.0, 1.0, 1.0)
    else:
        q = int(rng.integers(3, 9))
        m = PR.Mesh(3, q, q, q, 1.0, 1.0, 1.0)
    k = int(rng.choice([1, 3, 8, 9, 16, 20, 24, 30, 32, 37, 40, 41, 64]))
    k = min(k, m.n // 2)
    B = int(rng.choice([33, 40, 64, 65, 100, 128, 192, 256, 300]))
    rp, ci = m.pattern()
    E, _ = m.kl_field(rng.integers(1, 1 << 30, B).astype(np.uint64), 20 if dim == 2 else 30)
    V = m.assemble(E)
    phi = np.ascontiguousarray(np.linalg.qr(rng.standard_normal((m.n, k)))[0])
    R = rng.standard_normal((B, m.n))
    # a few inactive-looking inputs: zero right-hand sides
    R[rng.integers(0, B)] = 0.0
    out = []
    for mode in ("0", "1"):
        os.environ["P2G_RESTRICT_WS"] = mode
        os.environ["P2G_PROLONG_WS"] = mode
        s = BatchSolver(0)
        s.set_pattern(rp, ci, m.block_size)
        s.set_values(V)
        s.set_basis(phi)
        st = s.setup()
        assert np.all(st == 0)
        S = s.precond_apply(R)
        X0 = s.initial_guess(R)
        out.append((S, X0))
        s.close()
    for a, b, nm in ((out[0][0], out[1][0], "precond"), (out[0][1], out[1][1], "x0")):
        den = np.linalg.norm(a, axis=1)
        den[den == 0] = 1.0
        err = float(np.max(np.linalg.norm(a - b, axis=1) / den))
        worst = max(worst, err)
        flag = "" if err <= 1e-11 and np.all(np.isfinite(b)) else "  <-- FAIL"
        print(f"case {case}: dim {dim} n {m.n} k {k} B {B} {nm} rel diff {err:.2e}{flag}", flush=True)
        if flag:
            sys.exit(1)
print(f"ok: {cases} cases, worst relative difference {worst:.2e}")
