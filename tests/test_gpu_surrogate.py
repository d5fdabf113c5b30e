"""GPU parity of the surrogate warm start: p2g_surrogate_predict
and x0_mode P2G_X0_SURROGATE against the oracle's predict (pinned bit-exact to
the reference's surrogate.hpp:354-357 by tests/test_surrogate.py).  The MLP
runs with separately rounded products and sums in the reference's order; the
lift uses the tensor-core prolongation (D10) and CUDA's tanh, hence 1e-12."""
import numpy as np
import pytest

from oracle.bindings import Oracle
from tests.test_gpu_parity import make_solver, perm_system, small_problem

pytestmark = pytest.mark.gpu

from paper_2207_02543_b200 import _lib as L  # noqa: E402
from paper_2207_02543_b200.surrogate import SurrogateModel  # noqa: E402

ORC = Oracle()


@pytest.mark.parametrize("B,act", [(1, "tanh"), (8, "relu"), (40, "tanh"), (64, "tanh")])
def test_surrogate_predict_matches_oracle(gpu, B, act):
    m, rp, ci, f, V, phi = small_problem(B=B, k=12)
    s = make_solver(m, rp, ci, V, phi)
    model = SurrogateModel.random([20, 32, 32, 12], act, seed=B)
    s.set_surrogate(model)
    theta = np.random.default_rng(B).standard_normal((B, 20))
    got = s.surrogate_predict(theta)
    ref = ORC.surrogate_predict(model, phi, theta)
    for b in range(B):
        assert np.linalg.norm(got[b] - ref[b]) <= 1e-12 * np.linalg.norm(ref[b]), b
    s.close()


@pytest.mark.parametrize("B", [1, 40])
def test_solve_from_surrogate_x0(gpu, B):
    m, rp, ci, f, V, phi = small_problem(B=B, k=10)
    s = make_solver(m, rp, ci, V, phi)
    model = SurrogateModel.random([20, 32, 10], "tanh", seed=7)
    s.set_surrogate(model)
    theta = np.random.default_rng(2).standard_normal((B, 20))
    s.set_theta(theta)
    F = np.broadcast_to(f, (B, m.n)).copy()
    x, it, conv, st, _ = s.solve(F, None, 1e-8, 5000, x0_mode=L.X0_SURROGATE)
    assert np.all(conv) and np.all(st == 0)
    x0 = ORC.surrogate_predict(model, phi, theta)
    perm, prp, pci, pV, pf, pphi = perm_system(s, rp, ci, V, f, phi)
    for b in range(B):
        r = ORC.pcg_pod2g(prp, pci, pV[b], pf, pphi, x0[b][perm], 1e-8, 5000)
        assert abs(int(it[b]) - r.iters) <= 1, (b, int(it[b]), r.iters)
    s.close()


def test_surrogate_errors(gpu):
    m, rp, ci, f, V, phi = small_problem(B=2, k=10)
    s = make_solver(m, rp, ci, V, phi)
    F = np.broadcast_to(f, (2, m.n)).copy()
    with pytest.raises(RuntimeError):  # no model yet
        s.solve(F, None, 1e-8, 100, x0_mode=L.X0_SURROGATE)
    s.set_surrogate(SurrogateModel.random([20, 16, 7], "tanh"))  # k mismatch (7 != 10)
    with pytest.raises(ValueError):
        s.surrogate_predict(np.zeros((2, 20)))
    s.close()
