"""compute_pod's contractions on the FP64 tensor cores:
p2g_gram (pod.hpp:81-87) and p2g_combine (pod.hpp:120-129) against numpy,
determinism, and compute_pod(device=...) against the host restatement."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2207_02543_b200 import problems as PR  # noqa: E402


@pytest.mark.parametrize("N,d", [(5, 1000), (48, 12345), (70, 4097), (130, 2000)])
def test_gram_matches_numpy_and_is_deterministic(gpu, N, d):
    U = np.random.default_rng(N).standard_normal((N, d))
    G = PR.gram_device(U)
    ref = U @ U.T
    assert np.linalg.norm(G - ref) <= 1e-13 * np.linalg.norm(ref)
    assert np.array_equal(G, G.T)
    assert np.array_equal(G, PR.gram_device(U))


@pytest.mark.parametrize("N,d,r", [(4, 777, 1), (48, 20000, 40), (60, 1001, 64), (9, 333, 10)])
def test_combine_matches_numpy(gpu, N, d, r):
    rng = np.random.default_rng(d)
    U, W = rng.standard_normal((N, d)), rng.standard_normal((N, r))
    P = PR.combine_device(U, W)
    ref = U.T @ W
    assert np.linalg.norm(P - ref) <= 1e-13 * np.linalg.norm(ref)


def test_compute_pod_on_device_spans_the_host_basis(gpu):
    rng = np.random.default_rng(3)
    # snapshots with a decaying spectrum (like solution snapshots)
    modes = np.linalg.qr(rng.standard_normal((5000, 30)))[0].T
    U = (rng.standard_normal((40, 30)) * (0.5 ** np.arange(30))[None, :]) @ modes
    ph, wh, eh = PR.compute_pod(U, 12)
    pd, wd, ed = PR.compute_pod(U, 12, device=0)
    # eigenvalue errors scale with eps * lambda_max, not with lambda itself
    assert np.max(np.abs(wd[:12] - wh[:12])) <= 1e-12 * wh[0]
    assert abs(ed - eh) <= 1e-12
    C = pd.T @ ph  # same orthonormal columns up to sign
    assert np.max(np.abs(np.abs(C) - np.eye(12))) <= 1e-8
    assert np.max(np.abs(pd.T @ pd - np.eye(12))) <= 1e-8


def test_compute_pod_on_device_matches_reference_compute_pod(gpu):
    """Row a16 on the GPU: Gram and Phi = U Psi Lambda^-1/2 on the FP64 tensor
    cores, against the reference's own compute_pod (oracle/_ref) on the c1
    solution snapshots."""
    import scipy.sparse.linalg as spla
    from oracle.bindings import Reference
    from tests.helpers import to_scipy
    from tests.test_pod_pin import compare
    cfg = PR.CONFIGS["c1"]
    m = PR.Mesh.for_config(cfg)
    rp, ci = m.pattern()
    f = m.rhs()
    V = m.assemble(m.kl_field(PR.snapshot_seeds(cfg), cfg.kl_terms)[0])
    U = np.stack([spla.spsolve(to_scipy(rp, ci, v, m.n).tocsc(), f) for v in V])
    for k in (4, 10):
        phi, w, energy = PR.compute_pod(U, k, device=0)
        compare(U, phi, w, energy, Reference().compute_pod(U, rank=k), k)
