"""Row a16: compute_pod (pod.hpp:73-148) restated in paper_2207_02543_b200.problems
(numpy eigh in place of the reference's cyclic-Jacobi dense_eigh_spd,
core/dense_solve.hpp:76-141) pinned against the reference's own compute_pod
compiled from /root/reference (oracle/_ref, ref_compute_pod) on solution
snapshots of the c1 problem: the same Gram spectrum, numerical rank, energy
fraction and -- column by column, up to sign -- the same basis."""
from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle.bindings import REF_SO, Reference
from paper_2207_02543_b200 import problems as PR
from tests.helpers import to_scipy

pytestmark = pytest.mark.skipif(not __import__("os").path.exists(REF_SO),
                                reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def c1_snapshots():
    """The c1 offline inputs (30 seeded snapshot instances), solved exactly."""
    cfg = PR.CONFIGS["c1"]
    m = PR.Mesh.for_config(cfg)
    rp, ci = m.pattern()
    f = m.rhs()
    V = m.assemble(m.kl_field(PR.snapshot_seeds(cfg), cfg.kl_terms)[0])
    return np.stack([spla.spsolve(to_scipy(rp, ci, v, m.n).tocsc(), f) for v in V])


def compare(U, phi, w, energy, ref, k):
    pr, wr, er = ref
    assert phi.shape == pr.shape == (U.shape[1], k)
    # Gram eigenvalues: both solvers are backward stable, errors ~ eps lambda_max
    assert np.max(np.abs(w - wr)) <= 1e-12 * wr[0]
    assert abs(energy - er) <= 1e-12
    C = phi.T @ pr
    assert np.max(np.abs(np.abs(np.diag(C)) - 1.0)) <= 1e-8   # same columns up to sign
    assert np.max(np.abs(C - np.diag(np.diag(C)))) <= 1e-8
    assert np.max(np.abs(phi.T @ phi - np.eye(k))) <= 1e-8


@pytest.mark.parametrize("k", [1, 4, 10, 20])
def test_compute_pod_matches_reference(c1_snapshots, k):
    U = c1_snapshots
    phi, w, energy = PR.compute_pod(U, k)
    compare(U, phi, w, energy, Reference().compute_pod(U, rank=k), k)


def test_compute_pod_rank_cutoff_matches_reference():
    """Rank-deficient snapshots: RankTarget{k} is capped at the numerical rank
    (eigenvalues > 1e-12 lambda_max, pod.hpp:91-101) on both sides."""
    rng = np.random.default_rng(5)
    base = rng.standard_normal((3, 500))
    U = np.concatenate([base, base[:2] * 2.0, base[1:] - base[:2]])  # rank 3
    phi, w, energy = PR.compute_pod(U, 6)
    pr, wr, er = Reference().compute_pod(U, rank=6)
    assert phi.shape[1] == pr.shape[1] == 3
    assert abs(energy - er) <= 1e-12
    sv = np.linalg.svd(phi.T @ pr, compute_uv=False)
    assert np.all(np.abs(sv - 1.0) <= 1e-10)
