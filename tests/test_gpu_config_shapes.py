"""Oracle parity at the lane shapes of the large BASELINE.json configs
(SURVEY 8(c) protocol: iterations within +-1, residual histories within 1e-6
relative, and at MATCHED iteration counts ||x - x_ref|| / ||x_ref|| <= 1e-8),
against the oracle run on the colour-permuted system P K P^T (D1):

  * c4 shape: hex8, B = 64 -> the ShB64 node-blocked hex8 kernels at
    2 CTAs/SM (Kp recurrence, forward/backward sweeps, upper residual),
    k = 30 -> the k <= 32 tensor-core restriction / prolongation;
  * c3 shape: Q4, B = 256 -> four 64-instance tiles (grid.y = 4) through every
    kernel, k = 30;
  * the row-partitioned path (c5's) at 2, 3 and 4 partitions directly against
    the oracle (not only against the single handle).
The full-size c5 prefix check is in test_gpu_c5_parity.py.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle.bindings import Oracle
from tests.helpers import permute_csr, permute_values, random_load_basis, to_scipy

pytestmark = pytest.mark.gpu

from paper_2207_02543_b200 import _lib as L  # noqa: E402
from paper_2207_02543_b200 import problems as PR  # noqa: E402
from paper_2207_02543_b200.solver import BatchSolver  # noqa: E402

ORC = Oracle()
HIST_RTOL = 1e-6
X_RTOL = 1e-8


def _problem(dim, nx, ny, nz, B, k, seed):
    L_ = (2.0, 1.0, 1.0) if dim == 2 else (1.0, 1.0, 1.0)
    m = PR.Mesh(dim, nx, ny, nz, *L_)
    rp, ci = m.pattern()
    f = m.rhs()
    E, _ = m.kl_field(np.arange(B, dtype=np.uint64) + np.uint64(seed), 20 if dim == 2 else 30)
    V = m.assemble(E)
    phi = random_load_basis(to_scipy(rp, ci, V[0], m.n), k, seed)
    return m, rp, ci, f, V, phi


def _solver(m, rp, ci, V, phi):
    s = BatchSolver(0)
    s.set_pattern(rp, ci, m.block_size)
    s.set_values(V)
    s.set_basis(phi)
    assert np.all(s.setup() == 0)
    return s


def _permuted(perm, rp, ci, V, f, phi):
    prp, pci, _ = permute_csr(rp, ci, V[0], perm)
    return prp, pci, permute_values(rp, ci, V, perm), f[perm], phi[perm]


def _check_against_oracle(x, it, conv, status, hist, perm, prp, pci, pv, pf, pphi, tol, max_iter):
    """One instance: the SURVEY 8(c) protocol (ii)-(iv)."""
    x0_ref, _, st = ORC.reduced_solve(prp, pci, pv, pf, pphi)
    assert st == 0
    ref = ORC.pcg_pod2g(prp, pci, pv, pf, pphi, x0_ref, tol, max_iter)
    assert ref.converged and status == 0 and conv
    assert abs(int(it) - ref.iters) <= 1, (int(it), ref.iters)
    mm = min(int(it), ref.iters) + 1
    np.testing.assert_allclose(hist[:mm], ref.history[:mm], rtol=HIST_RTOL)
    ref_m = ORC.pcg_pod2g(prp, pci, pv, pf, pphi, x0_ref, 0.0, int(it))
    err = np.linalg.norm(x[perm] - ref_m.u) / np.linalg.norm(ref_m.u)
    assert err <= X_RTOL, err
    return ref.iters


@pytest.fixture(scope="module")
def c4_shape():
    """hex8 10^3 (n = 3,630), B = 64, k = 30: the c4 lane shape on a small mesh."""
    m, rp, ci, f, V, phi = _problem(3, 10, 10, 10, 64, 30, 4100)
    s = _solver(m, rp, ci, V, phi)
    perm, _ = s.permutation()
    sysp = _permuted(perm, rp, ci, V, f, phi)
    yield m, rp, ci, f, V, phi, s, perm, sysp
    s.close()


def test_c4_shape_spmv_bit_exact_all_instances(gpu, c4_shape):
    m, rp, ci, f, V, phi, s, perm, (prp, pci, pV, pf, pphi) = c4_shape
    X = np.random.default_rng(41).standard_normal((64, m.n))
    Y = s.spmv(X)
    for b in range(64):
        assert np.array_equal(Y[b][perm], ORC.spmv(prp, pci, pV[b], X[b][perm])), b


def _oracle_apply(rp, ci, v, phi, r):
    n = phi.shape[0]
    s, _ = ORC.gauss_seidel(rp, ci, v, r, np.zeros(n), 1, backward=False)
    t = ORC.residual(rp, ci, v, r, s)
    e, _ = ORC.dense_solve(ORC.reduced_operator(rp, ci, v, phi), ORC.project(phi, t))
    s, _ = ORC.gauss_seidel(rp, ci, v, r, s + ORC.lift(phi, e), 1, backward=True)
    return s


def test_c4_shape_preconditioner_all_instances(gpu, c4_shape):
    """Every one of the 64 lanes of the hex8 ShB64 kernels (node-blocked
    forward sweep from zero, upper residual, DMMA restriction / prolongation,
    coarse LDL^T, backward sweep) against Pod2gPreconditioner::apply."""
    m, rp, ci, f, V, phi, s, perm, (prp, pci, pV, pf, pphi) = c4_shape
    R = np.random.default_rng(42).standard_normal((64, m.n))
    S = s.precond_apply(R)
    for b in range(64):
        ref = _oracle_apply(prp, pci, pV[b], pphi, R[b][perm])
        assert np.linalg.norm(S[b][perm] - ref) <= 1e-11 * np.linalg.norm(ref), b


def test_c4_shape_solves(gpu, c4_shape):
    """The batched hex8 solve (Kp recurrence at 2 CTAs/SM, conditional-WHILE
    graph) for all 64 instances; three checked against the reference pcg_solve
    on P K P^T (krylov.hpp:243-297) with the full protocol."""
    m, rp, ci, f, V, phi, s, perm, (prp, pci, pV, pf, pphi) = c4_shape
    F = np.broadcast_to(f, (64, m.n)).copy()
    x, it, conv, status, hist = s.solve(F, None, 1e-8, 3000, x0_mode=L.X0_REDUCED)
    assert np.all(conv) and np.all(status == 0)
    for b in (0, 31, 63):
        _check_against_oracle(x[b], it[b], conv[b], status[b], hist[b], perm, prp, pci, pV[b],
                              pf, pphi, 1e-8, 3000)


def test_pcg_3d_hex8_matched_iteration_solution(gpu):
    """hex8 at the B = 1 / B = 8 lane shapes with the matched-iteration x check."""
    for B in (1, 8):
        m, rp, ci, f, V, phi = _problem(3, 6, 6, 6, B, 8, 777)
        s = _solver(m, rp, ci, V, phi)
        perm, _ = s.permutation()
        prp, pci, pV, pf, pphi = _permuted(perm, rp, ci, V, f, phi)
        F = np.broadcast_to(f, (B, m.n)).copy()
        x, it, conv, status, hist = s.solve(F, None, 1e-8, 2000, x0_mode=L.X0_REDUCED)
        for b in range(B):
            _check_against_oracle(x[b], it[b], conv[b], status[b], hist[b], perm, prp, pci,
                                  pV[b], pf, pphi, 1e-8, 2000)
        s.close()


def test_c3_shape_four_tiles(gpu):
    """Q4 32x16, B = 256 (the c3 batch: grid.y = 4 instance tiles), k = 30:
    the preconditioner of all 256 instances, and solves of two instances per
    tile against the oracle."""
    B = 256
    m, rp, ci, f, V, phi = _problem(2, 32, 16, 1, B, 30, 3100)
    s = _solver(m, rp, ci, V, phi)
    perm, _ = s.permutation()
    prp, pci, pV, pf, pphi = _permuted(perm, rp, ci, V, f, phi)
    R = np.random.default_rng(43).standard_normal((B, m.n))
    S = s.precond_apply(R)
    for b in range(B):
        ref = _oracle_apply(prp, pci, pV[b], pphi, R[b][perm])
        assert np.linalg.norm(S[b][perm] - ref) <= 1e-11 * np.linalg.norm(ref), b
    F = np.broadcast_to(f, (B, m.n)).copy()
    x, it, conv, status, hist = s.solve(F, None, 1e-8, 3000, x0_mode=L.X0_REDUCED)
    assert np.all(conv) and np.all(status == 0)
    for b in (0, 63, 64, 127, 128, 191, 192, 255):
        _check_against_oracle(x[b], it[b], conv[b], status[b], hist[b], perm, prp, pci, pV[b],
                              pf, pphi, 1e-8, 3000)
    s.close()


@pytest.mark.parametrize("dim,world,B", [(2, 2, 1), (2, 3, 1), (2, 4, 8), (3, 2, 1), (3, 4, 1),
                                         (3, 3, 4)])
def test_partitioned_matches_oracle(gpu, dim, world, B):
    _partitioned_vs_oracle(dim, world, B)


def test_partitioned_with_warp_specialised_projections(gpu, monkeypatch):
    """A batched row-partitioned solve (B = 40 -> one 64-instance tile, 3
    partitions) with k_restrict_ws / k_prolong_ws forced: the prolongation
    covers the ghost rows, the restriction the owned rows only."""
    monkeypatch.setenv("P2G_RESTRICT_WS", "1")
    monkeypatch.setenv("P2G_PROLONG_WS", "1")
    _partitioned_vs_oracle(2, 3, 40)


def _partitioned_vs_oracle(dim, world, B):
    """The row-partitioned path (p2g_part_*, in-process transport) against the
    oracle directly.  All partitions share the global node colouring, so the
    partitioned sweep is natural-order GS on the globally colour-permuted
    system; only the cross-partition sums (dots, Phi^T t, A_c) are associated
    per partition (D11)."""
    from paper_2207_02543_b200.partition import setup_partitioned
    if dim == 2:
        m, rp, ci, f, V, phi = _problem(2, 48, 24, 1, B, 8, 5100 + world)
    else:
        m, rp, ci, f, V, phi = _problem(3, 8, 8, 8, B, 8, 5200 + world)
    s = BatchSolver(0)
    s.set_pattern(rp, ci, m.block_size)
    perm, _ = s.permutation()
    s.close()
    prp, pci, pV, pf, pphi = _permuted(perm, rp, ci, V, f, phi)
    P, bounds, bs, st = setup_partitioned(rp, ci, V, f, phi, world, m.block_size)
    assert np.all(st == 0)
    xs, it, conv, status, hist = P.solve(bs, 1e-8, 3000, L.X0_REDUCED)
    assert np.all(conv) and np.all(status == 0)
    for b in range(B):
        x0_ref, _, _ = ORC.reduced_solve(prp, pci, pV[b], pf, pphi)
        ref = ORC.pcg_pod2g(prp, pci, pV[b], pf, pphi, x0_ref, 1e-8, 3000)
        assert abs(int(it[b]) - ref.iters) <= 1, (int(it[b]), ref.iters)
        mm = min(int(it[b]), ref.iters) + 1
        np.testing.assert_allclose(hist[b, :mm], ref.history[:mm], rtol=HIST_RTOL)
    # matched iteration count: run the partitioned solve for exactly it[b] iterations
    xs_m, it_m, _, _, _ = P.solve(bs, 0.0, int(it.max()), L.X0_REDUCED)
    P.close()
    x = np.concatenate([xs_m[r] for r in range(world)], axis=1)
    for b in range(B):
        x0_ref, _, _ = ORC.reduced_solve(prp, pci, pV[b], pf, pphi)
        ref_m = ORC.pcg_pod2g(prp, pci, pV[b], pf, pphi, x0_ref, 0.0, int(it_m[b]))
        err = np.linalg.norm(x[b][perm] - ref_m.u) / np.linalg.norm(ref_m.u)
        assert err <= X_RTOL, err
