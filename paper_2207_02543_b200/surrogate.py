"""Surrogate warm start: the reference's SurrogateModel
(surrogate.hpp:192-199) as a host-side container for BatchSolver.set_surrogate,
and a reader/writer of the reference's on-disk artefact so a model trained by
the reference loads unchanged:

  <dir>/model.json   kind "surrogate_model", widths, activation, input/latent
                     mean/std, weights_fnv1a (save_surrogate_model,
                     surrogate.hpp:361-386)
  <dir>/weights.bin  f64le: every W_l row-major (widths[l+1] x widths[l]) in
                     layer order, then every bias (load_surrogate_model,
                     surrogate.hpp:388-432)
  <dir>/basis.json + basis.bin   the POD basis as a vector batch of its k
                     columns (save_pod_basis pod.hpp:280-292, core/io.hpp:101-160)

predict itself runs on the device (p2g_surrogate_predict / X0_SURROGATE).
Training (surrogate.hpp:218-352) is out of scope.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field

import numpy as np


def fnv1a(payload: bytes) -> int:
    """fnv1a_hash (core/io.hpp:92-99), 64-bit (p2g_fnv1a64 in the host library).
    The reference's offset constant is 1469598103934665603 (not the published
    FNV offset basis 14695981039346656037); its artefacts carry that hash, so
    this reproduces the reference, not the textbook test vectors."""
    from . import _lib as L
    return int(L.lib().p2g_fnv1a64(payload, len(payload)))


@dataclass
class SurrogateModel:
    widths: list
    activation: str  # "tanh" | "relu"
    weights: list    # W_l: (widths[l+1], widths[l])
    biases: list     # b_l: (widths[l+1],)
    input_mean: np.ndarray
    input_std: np.ndarray
    latent_mean: np.ndarray
    latent_std: np.ndarray
    basis: np.ndarray | None = None  # Phi [n][k] when loaded with the artefact
    best_validation_loss: float = 0.0
    best_epoch: int = 0
    extra: dict = field(default_factory=dict)

    def __post_init__(self):
        if len(self.widths) < 2:
            raise ValueError("Mlp: at least input and output layers required")
        if self.activation not in ("tanh", "relu"):
            raise ValueError("SurrogateModel: activation must be 'tanh' or 'relu'")
        for l, (W, b) in enumerate(zip(self.weights, self.biases)):
            if np.shape(W) != (self.widths[l + 1], self.widths[l]) or np.shape(b) != (self.widths[l + 1],):
                raise ValueError(f"SurrogateModel: layer {l} shape mismatch")

    @property
    def input_dim(self) -> int:
        return int(self.widths[0])

    @property
    def output_dim(self) -> int:
        return int(self.widths[-1])

    def flat_parameters(self):
        """(weights, biases) concatenated in weights.bin order."""
        W = np.concatenate([np.asarray(w, dtype=np.float64).ravel() for w in self.weights])
        b = np.concatenate([np.asarray(x, dtype=np.float64).ravel() for x in self.biases])
        return np.ascontiguousarray(W), np.ascontiguousarray(b)

    @classmethod
    def random(cls, widths, activation="tanh", seed=0, p_scale=1.0):
        """A Glorot-normal network (the scaling of Mlp::create, surrogate.hpp:25-38,
        with numpy's generator) and arbitrary normalisers -- tests and benches."""
        rng = np.random.default_rng(seed)
        Ws, bs = [], []
        for fi, fo in zip(widths[:-1], widths[1:]):
            Ws.append(np.sqrt(2.0 / (fi + fo)) * rng.standard_normal((fo, fi)))
            bs.append(0.1 * rng.standard_normal(fo))
        p, k = widths[0], widths[-1]
        return cls(list(widths), activation, Ws, bs, p_scale * rng.standard_normal(p),
                   0.5 + rng.random(p), 0.01 * rng.standard_normal(k), 0.05 + 0.1 * rng.random(k))

    # ---- the reference's artefact ------------------------------------------
    @classmethod
    def load(cls, directory):
        """load_surrogate_model (surrogate.hpp:388-432), basis included."""
        with open(os.path.join(directory, "model.json")) as fh:
            js = json.load(fh)
        if js.get("kind", "") != "surrogate_model":
            raise ValueError("load_surrogate_model: wrong artifact")
        with open(os.path.join(directory, "weights.bin"), "rb") as fh:
            payload = fh.read()
        if fnv1a(payload) != int(js["weights_fnv1a"]):
            raise ValueError("load_surrogate_model: weight payload hash mismatch")
        widths = [int(w) for w in js["widths"]]
        vals = np.frombuffer(payload, dtype="<f8")
        need = sum(a * b for a, b in zip(widths[:-1], widths[1:])) + sum(widths[1:])
        if vals.size < need:
            raise ValueError("load_surrogate_model: truncated weights")
        if vals.size > need:
            raise ValueError("load_surrogate_model: trailing bytes in weights")
        Ws, bs, o = [], [], 0
        for fi, fo in zip(widths[:-1], widths[1:]):
            Ws.append(vals[o:o + fi * fo].reshape(fo, fi).copy())
            o += fi * fo
        for fo in widths[1:]:
            bs.append(vals[o:o + fo].copy())
            o += fo
        basis = load_pod_basis(os.path.join(directory, "basis")) \
            if os.path.exists(os.path.join(directory, "basis.json")) else None
        return cls(widths, js["activation"], Ws, bs, np.asarray(js["input_mean"], dtype=np.float64),
                   np.asarray(js["input_std"], dtype=np.float64),
                   np.asarray(js["latent_mean"], dtype=np.float64),
                   np.asarray(js["latent_std"], dtype=np.float64), basis,
                   float(js.get("best_validation_loss", 0.0)), int(js.get("best_epoch", 0)))

    def save(self, directory):
        """save_surrogate_model's layout (surrogate.hpp:361-386)."""
        os.makedirs(directory, exist_ok=True)
        W, b = self.flat_parameters()
        payload = np.concatenate([W, b]).astype("<f8").tobytes()
        with open(os.path.join(directory, "weights.bin"), "wb") as fh:
            fh.write(payload)
        js = {"kind": "surrogate_model", "widths": list(map(int, self.widths)),
              "activation": self.activation,
              "input_mean": list(map(float, self.input_mean)), "input_std": list(map(float, self.input_std)),
              "latent_mean": list(map(float, self.latent_mean)),
              "latent_std": list(map(float, self.latent_std)),
              "best_validation_loss": self.best_validation_loss, "best_epoch": self.best_epoch,
              "weights_fnv1a": fnv1a(payload)}
        with open(os.path.join(directory, "model.json"), "w") as fh:
            fh.write(json.dumps(js, indent=2) + "\n")
        if self.basis is not None:
            save_pod_basis(os.path.join(directory, "basis"), self.basis)


def load_pod_basis(stem):
    """load_pod_basis (pod.hpp:294-308) over load_vector_batch (core/io.hpp:139-160):
    returns Phi [dim][rank]."""
    with open(stem + ".json") as fh:
        header = json.load(fh)
    if header["dtype"] != "f64le":
        raise ValueError("load_vector_batch: unsupported dtype")
    if header.get("meta", {}).get("kind", "") != "pod_basis":
        raise ValueError("load_pod_basis: wrong artifact kind")
    count, dim = int(header["count"]), int(header["dim"])
    with open(stem + ".bin", "rb") as fh:
        payload = fh.read()
    if len(payload) != count * dim * 8:
        raise ValueError("load_vector_batch: payload size mismatch")
    if "payload_fnv1a" in header and fnv1a(payload) != int(header["payload_fnv1a"]):
        raise ValueError("load_vector_batch: payload hash mismatch")
    cols = np.frombuffer(payload, dtype="<f8").reshape(count, dim)
    return np.ascontiguousarray(cols.T)


def save_pod_basis(stem, phi, eigenvalues=None, energy_fraction=0.0):
    """save_pod_basis (pod.hpp:280-292): the k columns as a vector batch."""
    phi = np.asarray(phi, dtype=np.float64)
    payload = np.ascontiguousarray(phi.T).astype("<f8").tobytes()
    meta = {"kind": "pod_basis", "dim": int(phi.shape[0]), "rank": int(phi.shape[1]),
            "eigenvalues": [] if eigenvalues is None else list(map(float, eigenvalues)),
            "energy_fraction": float(energy_fraction), "snapshot_fnv1a": 0}
    header = {"count": int(phi.shape[1]), "dim": int(phi.shape[0]), "dtype": "f64le",
              "payload_fnv1a": fnv1a(payload), "meta": meta}
    with open(stem + ".bin", "wb") as fh:
        fh.write(payload)
    with open(stem + ".json", "w") as fh:
        fh.write(json.dumps(header, indent=2) + "\n")
