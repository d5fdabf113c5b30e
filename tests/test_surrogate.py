"""Surrogate warm start, host side: the oracle's predict against
the UNMODIFIED reference (surrogate.hpp:354-357), and the artefact reader /
writer against the reference's own save_surrogate_model / load_surrogate_model
(surrogate.hpp:361-432, pod.hpp:280-308, core/io.hpp:92-160)."""
import numpy as np
import pytest

import os

from oracle.bindings import REF_SO, Oracle, Reference
from paper_2207_02543_b200.surrogate import SurrogateModel, fnv1a, load_pod_basis, save_pod_basis

if not os.path.exists(REF_SO):
    pytest.skip("oracle/_ref not built", allow_module_level=True)
ORC = Oracle()
REF = Reference()


def _phi(n, k, seed=1):
    q, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((n, k)))
    return np.ascontiguousarray(q)


@pytest.mark.parametrize("act", ["tanh", "relu"])
@pytest.mark.parametrize("widths", [[5, 12], [20, 32, 32, 10], [30, 64, 16, 8, 40]])
def test_oracle_predict_equals_reference(act, widths):
    m = SurrogateModel.random(widths, act, seed=len(widths))
    phi = _phi(300, widths[-1])
    theta = np.random.default_rng(5).standard_normal((4, widths[0]))
    a = ORC.surrogate_predict(m, phi, theta)
    b = REF.surrogate_predict(m, phi, theta)
    assert np.array_equal(a, b)


def test_reference_artefact_loads_unchanged(tmp_path):
    m = SurrogateModel.random([20, 32, 32, 10], "tanh", seed=3)
    phi = _phi(257, 10, 4)
    REF.save_surrogate(tmp_path, m, phi)
    got = SurrogateModel.load(tmp_path)
    assert got.widths == m.widths and got.activation == m.activation
    for x, y in zip(got.weights + got.biases, m.weights + m.biases):
        assert np.array_equal(x, y)
    for f in ("input_mean", "input_std", "latent_mean", "latent_std"):
        assert np.array_equal(getattr(got, f), getattr(m, f))
    assert np.array_equal(got.basis, phi)


def test_written_artefact_loads_in_the_reference(tmp_path):
    m = SurrogateModel.random([6, 16, 7], "relu", seed=9)
    m.basis = _phi(99, 7, 2)
    m.save(tmp_path)
    theta = np.random.default_rng(1).standard_normal((3, 6))
    assert np.array_equal(REF.load_predict(tmp_path, theta), ORC.surrogate_predict(m, m.basis, theta))
    assert np.array_equal(load_pod_basis(str(tmp_path / "basis")), m.basis)


def test_corrupt_artefacts_are_rejected(tmp_path):
    m = SurrogateModel.random([4, 8, 3], "tanh", seed=1)
    m.basis = _phi(20, 3)
    m.save(tmp_path)
    raw = (tmp_path / "weights.bin").read_bytes()
    (tmp_path / "weights.bin").write_bytes(raw[:-8])
    with pytest.raises(ValueError, match="hash mismatch"):
        SurrogateModel.load(tmp_path)
    save_pod_basis(str(tmp_path / "b2"), m.basis)
    (tmp_path / "b2.bin").write_bytes((tmp_path / "b2.bin").read_bytes()[:-8])
    with pytest.raises(ValueError, match="size mismatch"):
        load_pod_basis(str(tmp_path / "b2"))
    with pytest.raises(ValueError):
        SurrogateModel([4], "tanh", [], [], np.zeros(4), np.ones(4), np.zeros(4), np.ones(4))


def test_fnv1a_is_the_reference_definition():
    """core/io.hpp:92-99 with its offset constant 1469598103934665603."""
    def ref(b):
        h = 1469598103934665603
        for c in b:
            h = ((h ^ c) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
        return h
    rng = np.random.default_rng(0)
    for n in (0, 1, 7, 1000):
        b = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert fnv1a(b) == ref(b)
