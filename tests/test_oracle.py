"""Pins the oracle (oracle/pod2g_oracle.c) -- CPU only.

1. Against the reference's own known answers: the PCG + POD-2G iteration
   table of proj/test_output.txt:47 (its, res 32: 28/72/84/93/101), and the
   unit-test KATs of test_sparse_core.cpp, test_smoothers.cpp,
   test_krylov.cpp and test_pod.cpp restated on the oracle.
2. Against the unmodified reference compiled from /root/reference
   (oracle/_ref): bit-for-bit equality on fixtures and on Q4 instances.
3. Against the committed golden fixtures (tests/golden/*.npz, made by
   tests/golden/make_golden.py from oracle/_ref), so the pin holds where the
   reference is not available.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle.bindings import REF_SO, SMOOTHER_GS, SMOOTHER_JACOBI, Oracle, Reference
from tests.helpers import (from_scipy, laplacian_1d, laplacian_2d, permute_csr, random_load_basis,
                           random_spd)

HERE = os.path.dirname(os.path.abspath(__file__))
ORC = Oracle()
needs_ref = pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")


def golden(name):
    return np.load(os.path.join(HERE, "golden", name))


# ---------------------------------------------------------------- known answers
def test_its32_iteration_table_matches_published_run():
    """proj/test_output.txt:47 -- pod-2g row 28/72/84/93/101 (u0 = 0)."""
    g = golden("its32.npz")
    rp, ci, v, f, phi = g["rp"], g["ci"], g["v"], g["f"], g["phi"]
    assert phi.shape[1] == 1  # rank 1 (test_output.txt:32)
    iters = []
    for tol in g["tols"]:
        res = ORC.pcg_pod2g(rp, ci, v, f, phi, None, float(tol), 100000)
        assert res.status == 0 and res.converged
        iters.append(res.iters)
        if tol == 1e-8:
            assert np.array_equal(res.history, g["hist_1e-8"])
            assert np.array_equal(res.u, g["u_1e-8"])
    assert iters == [28, 72, 84, 93, 101]
    assert list(g["iters"]) == iters


def test_q4c1_golden_natural_multicolour_and_jacobi():
    g = golden("q4c1.npz")
    rp, ci, v, f, phi, x0 = g["rp"], g["ci"], g["v"], g["f"], g["phi"], g["x0"]
    x0_o, _, st = ORC.reduced_solve(rp, ci, v, f, phi)
    assert st == 0 and np.array_equal(x0_o, x0)
    nat = ORC.pcg_pod2g(rp, ci, v, f, phi, x0, 1e-8, 100000)
    assert nat.iters == int(g["nat_iters"]) and np.array_equal(nat.history, g["nat_hist"])
    assert np.array_equal(nat.u, g["nat_u"])
    perm = g["perm"]
    prp, pci, pv = permute_csr(rp, ci, v, perm)
    px0, _, _ = ORC.reduced_solve(prp, pci, pv, f[perm], phi[perm])
    mc = ORC.pcg_pod2g(prp, pci, pv, f[perm], phi[perm], px0, 1e-8, 100000)
    assert mc.iters == int(g["mc_iters"]) and np.array_equal(mc.history, g["mc_hist"])
    assert np.array_equal(mc.u, g["mc_u"])
    jac = ORC.pcg_pod2g(rp, ci, v, f, phi, x0, 1e-8, 100000, smoother=SMOOTHER_JACOBI, omega=0.5)
    assert jac.iters == int(g["jac_iters"]) and np.array_equal(jac.u, g["jac_u"])


def test_spmv_kats():
    """test_sparse_core.cpp:22-38: identity, tridiag(-1,2,-1).1 = [1,0,1], A.0 = 0."""
    rp, ci, v = from_scipy(laplacian_1d(3))
    assert np.array_equal(ORC.spmv(rp, ci, v, np.ones(3)), [1.0, 0.0, 1.0])
    assert np.array_equal(ORC.spmv(rp, ci, v, np.zeros(3)), np.zeros(3))
    rp = np.arange(4)
    assert np.array_equal(ORC.spmv(rp, np.arange(3), np.ones(3), [1.0, 2.0, 3.0]), [1, 2, 3])


def test_spmv_linearity():
    """test_sparse_core.cpp:40-53 (1e-12)."""
    rp, ci, v = from_scipy(random_spd(40, 0.1, 3))
    rng = np.random.default_rng(0)
    x, y = rng.standard_normal(40), rng.standard_normal(40)
    lhs = ORC.spmv(rp, ci, v, 2.0 * x - 3.0 * y)
    rhs = 2.0 * ORC.spmv(rp, ci, v, x) - 3.0 * ORC.spmv(rp, ci, v, y)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.max(np.abs(lhs))


def test_dense_solve_kats():
    """test_sparse_core.cpp:171-204: identity, Hilbert residual, singular throws."""
    b = np.array([1.0, -2.0, 3.0])
    x, st = ORC.dense_solve(np.eye(3), b)
    assert st == 0 and np.array_equal(x, b)
    H = 1.0 / (np.arange(4)[:, None] + np.arange(4)[None, :] + 1.0)
    x, st = ORC.dense_solve(H, np.ones(4))
    assert np.linalg.norm(H @ x - 1.0) <= 1e-10 * (np.linalg.norm(H) * np.linalg.norm(x) + 2)
    _, st = ORC.dense_solve(np.ones((3, 3)), b)
    assert st == 4  # singular


def test_gauss_seidel_kats():
    """test_smoothers.cpp:9-51 and :145-177."""
    K = laplacian_2d(5)
    rp, ci, v = from_scipy(K)
    n = K.shape[0]
    rng = np.random.default_rng(4)
    f = rng.standard_normal(n)
    u0 = rng.standard_normal(n)
    u, st = ORC.gauss_seidel(rp, ci, v, f, u0, 0)
    assert st == 0 and np.array_equal(u, u0)  # 0 sweeps: no-op
    # diagonal matrix: one sweep is exact
    d = np.arange(1.0, n + 1)
    u, _ = ORC.gauss_seidel(np.arange(n + 1), np.arange(n), d, f, u0, 1)
    assert np.allclose(u, f / d, rtol=0, atol=1e-15)
    # zero diagonal -> error
    v0 = v.copy()
    v0[np.flatnonzero(ci[:rp[1]] == 0)[0]] = 0.0
    _, st = ORC.gauss_seidel(rp, ci, v0, f, u0, 1)
    assert st == 5
    # backward sweep = K-adjoint of the forward one: <M_f e1, e2>_K = <e1, M_b e2>_K
    Kd = K.toarray()
    e1, e2 = rng.standard_normal(n), rng.standard_normal(n)
    Mf, _ = ORC.gauss_seidel(rp, ci, v, Kd @ e1 * 0, e1, 1)   # error propagation, f = 0
    Mb, _ = ORC.gauss_seidel(rp, ci, v, np.zeros(n), e2, 1, backward=True)
    lhs = Mf @ Kd @ e2
    rhs = e1 @ Kd @ Mb
    assert abs(lhs - rhs) <= 1e-12 * max(abs(lhs), 1.0)


def test_identity_pcg_equals_cg_iterate_for_iterate():
    """test_krylov.cpp:76-90 (1e-12); needs the reference's cg_solve."""
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    R = Reference()
    rp, ci, v = from_scipy(laplacian_2d(8))
    f = np.ones(64)
    a = ORC.pcg_pod2g(rp, ci, v, f, None, None, 1e-10, 1000)
    b = R.cg_solve(rp, ci, v, f, 1e-10, 1000)
    assert a.iters == b.iters
    np.testing.assert_allclose(a.history, b.history, rtol=1e-12)


def test_pod2g_preconditioner_symmetric_spd_and_exact_cases():
    """test_pod.cpp:304-323 (symmetric 1e-10 max, SPD) and :122-181
    (complete basis: reduced_solve = full solve)."""
    K = random_spd(30, 0.2, 7)
    rp, ci, v = from_scipy(K)
    n = 30
    phi = random_load_basis(K, 4, 2)
    from oracle.bindings import _Csr  # noqa: F401
    cols = []
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        cols.append(_apply(rp, ci, v, phi, e))
    Bm = np.array(cols).T
    assert np.max(np.abs(Bm - Bm.T)) <= 1e-10 * np.max(np.abs(Bm))
    assert np.min(np.linalg.eigvalsh(0.5 * (Bm + Bm.T))) > 0
    Q, _ = np.linalg.qr(np.random.default_rng(1).standard_normal((n, n)))
    f = np.arange(1.0, n + 1)
    x0, _, st = ORC.reduced_solve(rp, ci, v, f, Q)
    assert st == 0
    np.testing.assert_allclose(x0, np.linalg.solve(K.toarray(), f), rtol=1e-10, atol=1e-12)


def _apply(rp, ci, v, phi, r):
    res = ORC.pcg_pod2g(rp, ci, v, r, phi, None, 0.0, 0)  # setup only
    assert res.status == 0
    n = len(r)
    s, _ = ORC.gauss_seidel(rp, ci, v, r, np.zeros(n), 1)
    t = ORC.residual(rp, ci, v, r, s)
    e, _ = ORC.dense_solve(ORC.reduced_operator(rp, ci, v, phi), ORC.project(phi, t))
    s = s + ORC.lift(phi, e)
    s, _ = ORC.gauss_seidel(rp, ci, v, r, s, 1, backward=True)
    return s


def test_exact_basis_converges_in_one_iteration():
    """test_krylov.cpp:92-98 analogue: a complete basis makes the coarse
    correction exact, so PCG stops after one iteration."""
    K = laplacian_2d(4)
    rp, ci, v = from_scipy(K)
    f = np.arange(16.0)
    res = ORC.pcg_pod2g(rp, ci, v, f, np.eye(16), None, 1e-10, 100)
    assert res.converged and res.iters <= 1


# ---------------------------------------------------------------- vs oracle/_ref
@needs_ref
@pytest.mark.parametrize("which", ["lap2d", "spd", "q4"])
def test_bit_exact_against_reference(which):
    R = Reference()
    if which == "lap2d":
        K = laplacian_2d(12)
        rp, ci, v = from_scipy(K)
        phi = random_load_basis(K, 5, 0)
    elif which == "spd":
        K = random_spd(200, 0.03, 11)
        rp, ci, v = from_scipy(K)
        phi = random_load_basis(K, 6, 1)
    else:
        g = golden("q4c1.npz")
        rp, ci, v, phi = g["rp"], g["ci"].astype(np.int64), g["v"], g["phi"]
    n = len(rp) - 1
    rng = np.random.default_rng(5)
    x, f = rng.standard_normal(n), rng.standard_normal(n)
    assert np.array_equal(ORC.spmv(rp, ci, v, x), R.spmv(rp, ci, v, x))
    assert np.array_equal(ORC.residual(rp, ci, v, f, x), R.residual(rp, ci, v, f, x))
    for bw in (False, True):
        assert np.array_equal(ORC.gauss_seidel(rp, ci, v, f, x, 2, bw)[0],
                              R.gauss_seidel(rp, ci, v, f, x, 2, bw))
    assert np.array_equal(ORC.jacobi_sweep(rp, ci, v, f, x, 0.5, 2)[0],
                          R.jacobi_sweep(rp, ci, v, f, x, 0.5, 2))
    assert np.array_equal(ORC.reduced_operator(rp, ci, v, phi), R.reduced_operator(rp, ci, v, phi))
    xo, uo, _ = ORC.reduced_solve(rp, ci, v, f, phi)
    xr, ur = R.reduced_solve(rp, ci, v, f, phi)
    assert np.array_equal(xo, xr) and np.array_equal(uo, ur)
    for sm in (SMOOTHER_GS, SMOOTHER_JACOBI):
        a = ORC.pcg_pod2g(rp, ci, v, f, phi, xo, 1e-9, 5000, smoother=sm, omega=0.5)
        b = R.pcg_pod2g(rp, ci, v, f, phi, xr, 1e-9, 5000, smoother=sm, omega=0.5)
        assert a.iters == b.iters and a.converged == b.converged
        assert np.array_equal(a.history, b.history) and np.array_equal(a.u, b.u)


@needs_ref
def test_reference_jacobi_two_thirds_breaks_down_on_its():
    """damped Jacobi at the reference default omega = 2/3 is not
    a safe smoother for the reference's own `its` problem (breakdown)."""
    g = golden("its32.npz")
    rp, ci, v, f, phi = g["rp"], g["ci"].astype(np.int64), g["v"], g["f"], g["phi"]
    res = ORC.pcg_pod2g(rp, ci, v, f, phi, None, 1e-8, 2000, smoother=SMOOTHER_JACOBI,
                        omega=2.0 / 3.0)
    R = Reference()
    ref = R.pcg_pod2g(rp, ci, v, f, phi, None, 1e-8, 2000, smoother=SMOOTHER_JACOBI,
                      omega=2.0 / 3.0)
    assert res.status == 2 and ref.status != 0


@needs_ref
def test_pod2g_solve_restatement_equals_reference():
    """pod.hpp:224-256 standalone two-grid iteration: the oracle's restatement is
    bit-identical to the compiled reference (cycles, history, solution)."""
    REF = Reference()
    g = golden("q4c1.npz")
    rp, ci, v, f, phi, x0 = g["rp"], g["ci"], g["v"], g["f"], g["phi"], g["x0"]
    for u0, tol in ((x0, 1e-8), (None, 1e-6)):
        a = ORC.pod2g_solve(rp, ci, v, f, phi, u0, tol, 3000)
        b = REF.pod2g_solve(rp, ci, v, f, phi, u0, tol, 3000)
        assert a.status == 0 and b.status == 0 and a.converged and b.converged
        assert a.iters == b.iters
        assert np.array_equal(a.history, b.history) and np.array_equal(a.u, b.u)


def test_fast_permutation_equals_reference_permutation():
    """oracle/csr_permute.c (used for the full-size c5 parity check) builds the
    same P K P^T as tests/helpers.permute_csr, for any thread count."""
    from oracle.bindings import permute_csr_fast
    from paper_2207_02543_b200 import problems as PR
    from tests.helpers import permute_csr
    m = PR.Mesh(3, 5, 5, 5, 1.0, 1.0, 1.0)
    rp, ci = m.pattern()
    v = m.assemble(m.kl_field(np.array([3], dtype=np.uint64), 30)[0])[0]
    perm = np.random.default_rng(0).permutation(m.n)
    ref = permute_csr(rp, ci, v, perm)
    for threads in (1, 3, 8):
        got = permute_csr_fast(rp, ci, v, perm, threads=threads)
        assert all(np.array_equal(a, b) for a, b in zip(ref, got))
    with pytest.raises(ValueError):
        permute_csr_fast(rp, ci, v, np.zeros(m.n, dtype=np.int64))
