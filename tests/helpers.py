"""Shared test helpers: permuted systems for the oracle, small fixtures."""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def to_scipy(rp, ci, v, n):
    return sp.csr_matrix((np.asarray(v, dtype=np.float64), np.asarray(ci, dtype=np.int64),
                          np.asarray(rp, dtype=np.int64)), shape=(n, n))


def from_scipy(K):
    K = K.tocsr()
    K.sort_indices()
    return K.indptr.astype(np.int64), K.indices.astype(np.int64), K.data.astype(np.float64)


def permute_csr(rp, ci, v, perm):
    """P K P^T with new row i = old row perm[i]; columns sorted ascending.
    Returns (rp, ci, v) int64/int64/float64 with explicit zeros kept."""
    rp = np.asarray(rp, dtype=np.int64)
    ci = np.asarray(ci, dtype=np.int64)
    v = np.asarray(v, dtype=np.float64)
    n = len(rp) - 1
    iperm = np.empty(n, dtype=np.int64)
    iperm[perm] = np.arange(n)
    lens = rp[1:] - rp[:-1]
    new_lens = lens[perm]
    nrp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(new_lens, out=nrp[1:])
    nci = np.empty_like(ci)
    nv = np.empty_like(v)
    for i in range(n):
        o = perm[i]
        cols = iperm[ci[rp[o]:rp[o + 1]]]
        order = np.argsort(cols, kind="stable")
        nci[nrp[i]:nrp[i + 1]] = cols[order]
        nv[nrp[i]:nrp[i + 1]] = v[rp[o]:rp[o + 1]][order]
    return nrp, nci, nv


def permute_values(rp, ci, values_batch, perm):
    """Permute [B][nnz] value sets the same way as permute_csr (shared pattern)."""
    rp = np.asarray(rp, dtype=np.int64)
    ci = np.asarray(ci, dtype=np.int64)
    n = len(rp) - 1
    iperm = np.empty(n, dtype=np.int64)
    iperm[perm] = np.arange(n)
    idx = []
    for i in range(n):
        o = perm[i]
        cols = iperm[ci[rp[o]:rp[o + 1]]]
        order = np.argsort(cols, kind="stable")
        idx.append(np.arange(rp[o], rp[o + 1])[order])
    idx = np.concatenate(idx)
    return np.asarray(values_batch)[..., idx]


def laplacian_1d(n):
    main = 2.0 * np.ones(n)
    off = -np.ones(n - 1)
    return sp.diags([off, main, off], [-1, 0, 1], format="csr")


def laplacian_2d(m):
    T = laplacian_1d(m)
    I = sp.identity(m, format="csr")
    return (sp.kron(I, T) + sp.kron(T, I)).tocsr()


def random_spd(n, density, seed):
    rng = np.random.default_rng(seed)
    A = sp.random(n, n, density=density, random_state=rng, format="csr")
    A = A + A.T
    A = A + sp.identity(n) * (abs(A).sum(axis=1).max() + 1.0)
    A = A.tocsr()
    A.sort_indices()
    return A


def random_load_basis(K, k, seed):
    """Basis from dense solves under random loads (test_pod.cpp:17-24 style)."""
    rng = np.random.default_rng(seed)
    Kd = K.toarray()
    U = np.linalg.solve(Kd, rng.standard_normal((K.shape[0], k)))
    Q, _ = np.linalg.qr(U)
    return np.ascontiguousarray(Q)
