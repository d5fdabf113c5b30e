"""Generate the committed golden fixtures from the UNMODIFIED reference
(oracle/_ref, compiled from /root/reference by oracle/Makefile).  Run here (the
reference is not available on the GPU box):  python tests/golden/make_golden.py

its32.npz   -- the reference's own `its` problem (problems.hpp:99-177) at res 32,
               offline basis exactly as run_offline builds it (LHS seed 42, 100
               snapshots, compute_pod EnergyTarget 0.9999) and test instance 0 of
               run_pcg_benchmark's sampler (seed 7); reference pcg_solve +
               Pod2gPreconditioner iteration counts / histories / solutions at the
               five tolerances of proj/test_output.txt:41-47.
q4c1.npz    -- one BASELINE c1 instance (Q4 plane-stress 64x32 from our
               generator) with a POD basis from reference-solved snapshots
               (ref_offline_basis), and reference solves in natural order AND on
               the node-colour-permuted system the GPU smoother corresponds to.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.bindings import Reference  # noqa: E402
from paper_2207_02543_b200 import problems as PR  # noqa: E402
from paper_2207_02543_b200.solver import analyze_pattern  # noqa: E402
from tests.helpers import permute_csr  # noqa: E402

TOLS = [1e-4, 1e-5, 1e-6, 1e-7, 1e-8]


def its32(R):
    rp, ci, v, f, phi = R.its_case(32, 100, 42, 7, 0, 8)
    out = dict(rp=rp, ci=ci.astype(np.int32), v=v, f=f, phi=phi, tols=np.array(TOLS))
    iters = []
    for i, tol in enumerate(TOLS):
        res = R.pcg_pod2g(rp, ci, v, f, phi, None, tol, 100000)
        iters.append(res.iters)
        if tol == 1e-8:
            out["hist_1e-8"] = res.history
            out["u_1e-8"] = res.u
    out["iters"] = np.array(iters)
    np.savez_compressed(os.path.join(HERE, "its32.npz"), **out)
    print("its32 iterations", iters)


def q4c1(R):
    cfg = PR.CONFIGS["c1"]
    m = PR.Mesh.for_config(cfg)
    rp, ci = m.pattern()
    f = m.rhs()
    snaps = m.assemble(m.kl_field(PR.snapshot_seeds(cfg), cfg.kl_terms)[0])
    F = np.broadcast_to(f, (len(snaps), m.n))
    phi = R.offline_basis(rp.astype(np.int64), ci.astype(np.int64), snaps, F, cfg.k, 1e-10, 8)
    v = m.assemble(m.kl_field(PR.query_seeds(cfg, 1), cfg.kl_terms)[0])[0]
    x0, _ = R.reduced_solve(rp, ci, v, f, phi)
    nat = R.pcg_pod2g(rp, ci, v, f, phi, x0, 1e-8, 100000)
    perm, offs = analyze_pattern(rp, ci, m.block_size)
    prp, pci, pv = permute_csr(rp, ci, v, perm)
    px0, _ = R.reduced_solve(prp, pci, pv, f[perm], phi[perm])
    mc = R.pcg_pod2g(prp, pci, pv, f[perm], phi[perm], px0, 1e-8, 100000)
    jac = R.pcg_pod2g(rp, ci, v, f, phi, x0, 1e-8, 100000, smoother=1, omega=0.5)
    np.savez_compressed(os.path.join(HERE, "q4c1.npz"), rp=rp.astype(np.int64),
                        ci=ci.astype(np.int32), v=v, f=f, phi=phi, x0=x0, perm=perm,
                        color_offsets=offs,
                        nat_iters=nat.iters, nat_hist=nat.history, nat_u=nat.u,
                        mc_iters=mc.iters, mc_hist=mc.history, mc_u=mc.u,
                        jac_iters=jac.iters, jac_hist=jac.history, jac_u=jac.u)
    print("q4c1 iterations: natural", nat.iters, "multicolour", mc.iters, "jacobi(0.5)", jac.iters)


if __name__ == "__main__":
    R = Reference()
    its32(R)
    q4c1(R)
