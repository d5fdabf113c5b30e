"""BASELINE.json's headline configuration at FULL size (c2: 64 Q4 256x128
instances, k = 20, tol 1e-8): size-independent properties of the solve and
the preconditioner, plus oracle parity on a sample of instances (the oracle
runs P K P^T, D1; each oracle solve takes seconds at this size)."""
import numpy as np
import pytest

from oracle.bindings import Oracle
from tests.helpers import permute_csr, permute_values

pytestmark = pytest.mark.gpu

from paper_2207_02543_b200 import _lib as L  # noqa: E402
from paper_2207_02543_b200 import problems as PR  # noqa: E402
from paper_2207_02543_b200.solver import BatchSolver  # noqa: E402

ORC = Oracle()


@pytest.fixture(scope="module")
def c2(gpu):
    cfg = PR.CONFIGS["c2"]
    prob = PR.build_problem(cfg)
    m = prob.mesh
    E, _ = m.kl_field(PR.query_seeds(cfg), cfg.kl_terms)
    s = BatchSolver(0)
    s.set_pattern(prob.rp, prob.ci, m.block_size)
    s.assemble(m, E)
    s.set_basis(prob.phi)
    assert np.all(s.setup() == 0)
    yield cfg, prob, E, s
    s.close()


def test_c2_all_converge_true_residual_and_determinism(c2):
    cfg, prob, E, s = c2
    B, n = cfg.batch, prob.mesh.n
    F = np.broadcast_to(prob.f, (B, n)).copy()
    x, it, conv, st, hist = s.solve(F, None, cfg.tol, 5000, x0_mode=L.X0_REDUCED)
    assert np.all(conv) and np.all(st == 0)
    assert 200 < it.mean() < 400, it.mean()
    # the recursive residual (krylov.hpp:285) against the true residual f - Kx
    Kx = s.spmv(x)
    true_rel = np.linalg.norm(F - Kx, axis=1) / np.linalg.norm(F, axis=1)
    rec = hist[np.arange(B), it]
    assert np.all(rec <= cfg.tol)
    assert np.all(true_rel <= 5 * cfg.tol), true_rel.max()
    # bit-reproducible
    x2, it2, *_ = s.solve(F, None, cfg.tol, 5000, x0_mode=L.X0_REDUCED)
    assert np.array_equal(it, it2) and np.array_equal(x, x2)


def test_c2_preconditioner_is_linear_symmetric_positive(c2):
    cfg, prob, E, s = c2
    B, n = cfg.batch, prob.mesh.n
    rng = np.random.default_rng(11)
    r1, r2 = rng.standard_normal((B, n)), rng.standard_normal((B, n))
    s1, s2 = s.precond_apply(r1), s.precond_apply(r2)
    s12 = s.precond_apply(r1 + 2.0 * r2)
    lin = np.linalg.norm(s12 - (s1 + 2.0 * s2), axis=1) / np.linalg.norm(s12, axis=1)
    assert lin.max() <= 1e-11, lin.max()
    a = np.einsum("bi,bi->b", r1, s2)
    b = np.einsum("bi,bi->b", r2, s1)
    assert np.max(np.abs(a - b) / np.abs(a)) <= 1e-9
    assert np.all(np.einsum("bi,bi->b", r1, s1) > 0)


@pytest.mark.parametrize("inst", [0, 37])
def test_c2_instances_match_the_oracle(c2, inst):
    cfg, prob, E, s = c2
    B, n = cfg.batch, prob.mesh.n
    F = np.broadcast_to(prob.f, (B, n)).copy()
    x, it, conv, st, hist = s.solve(F, None, cfg.tol, 5000, x0_mode=L.X0_REDUCED)
    perm, _ = s.permutation()
    v = prob.mesh.assemble(E[inst:inst + 1])[0]
    prp, pci, pv = permute_csr(prob.rp, prob.ci, v, perm)
    pf, pphi = prob.f[perm], prob.phi[perm]
    x0, _, _ = ORC.reduced_solve(prp, pci, pv, pf, pphi)
    ref = ORC.pcg_pod2g(prp, pci, pv, pf, pphi, x0, cfg.tol, 5000)
    assert ref.converged and abs(int(it[inst]) - ref.iters) <= 1, (int(it[inst]), ref.iters)
    m = min(int(it[inst]), ref.iters) + 1
    np.testing.assert_allclose(hist[inst, :m], ref.history[:m], rtol=1e-6)
    ref_m = ORC.pcg_pod2g(prp, pci, pv, pf, pphi, x0, 0.0, int(it[inst]))
    err = np.linalg.norm(x[inst][perm] - ref_m.u) / np.linalg.norm(ref_m.u)
    assert err <= 1e-8, err
