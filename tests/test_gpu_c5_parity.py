"""Oracle parity for config c5 ITSELF (BASELINE.json configs[4]: hex8 160^3,
12,442,080 dofs, 995 M nonzeros, k = 40), SURVEY 8(c) protocol (iv) on a
matched-iteration prefix: the GPU's row-partitioned path (2 partitions on the
device, in-process halo exchange, conditional-WHILE graph) runs exactly
N_PREFIX PCG iterations; the oracle (the reference's pcg_solve restated,
oracle/pod2g_oracle.c) runs the same N_PREFIX iterations on the globally
colour-permuted system P K P^T -- every one of its 4 x 10^9-term sweeps on one
host core.  Residual histories within 1e-6 relative, solutions within 1e-8.

Inputs: the c5 query instance (seeded KL modulus) and a k = 40 basis of
random combinations of the smooth displacement modes (any full-rank basis
defines the same preconditioner family; the POD basis itself needs the
~5-minute offline stage, exercised by bench.py --config c5).  x0 = 0 on both
sides, so the oracle builds A_c (k SpMVs + k^2 dots at n = 12.4 M) once.
"""
from __future__ import annotations

import time

import numpy as np
import pytest

from oracle.bindings import Oracle, permute_csr_fast

pytestmark = pytest.mark.gpu

from paper_2207_02543_b200 import _lib as L  # noqa: E402
from paper_2207_02543_b200 import c5 as C5  # noqa: E402
from paper_2207_02543_b200 import problems as PR  # noqa: E402
from paper_2207_02543_b200.partition import PartitionedSolver, row_bounds  # noqa: E402

N_PREFIX = 10
WORLD = 2


def test_c5_matched_iteration_prefix_against_oracle(gpu):
    t0 = time.perf_counter()
    cfg = PR.CONFIGS["c5"]
    m = PR.Mesh.for_config(cfg)
    n, bs = m.n, m.block_size
    assert n == 12_442_080
    E, _ = m.kl_field(PR.query_seeds(cfg, 1), cfg.kl_terms)
    f = m.rhs()
    colors = m.node_colors()
    # k = 40 orthonormal basis: random combinations of the degree <= 3 modes
    S = C5.smooth_space(m, np.arange(n, dtype=np.int64))
    S = S @ np.random.default_rng(40).standard_normal((S.shape[1], cfg.k))
    R = np.linalg.cholesky(S.T @ S).T
    phi = np.ascontiguousarray(S @ np.linalg.inv(R))
    del S
    # ---- GPU: row-partitioned path, values generated on the device
    bounds = row_bounds(n, WORLD, bs)
    P = PartitionedSolver(WORLD, 0)
    bvec = {}
    for r in range(WORLD):
        r0, r1 = int(bounds[r]), int(bounds[r + 1])
        rpl, cil = m.pattern_range(r0, r1)
        P.set_pattern(r, n, bounds, rpl, cil, bs, colors)
        del rpl, cil
        g = P.ghosts(r)
        P.assemble(r, m, E)
        P.set_basis(r, phi[r0:r1], phi[g])
        bvec[r] = f[r0:r1][None, :]
    assert np.all(P.setup() == 0)
    xs, it, conv, status, hist = P.solve(bvec, 0.0, N_PREFIX, L.X0_ZERO)
    P.close()
    assert int(it[0]) == N_PREFIX and status[0] == 0
    x_gpu = np.concatenate([xs[r][0] for r in range(WORLD)])
    t1 = time.perf_counter()
    # ---- oracle on P K P^T (global colour-major order of the partitions)
    nodes = np.argsort(colors, kind="stable").astype(np.int64)
    perm = (nodes[:, None] * bs + np.arange(bs, dtype=np.int64)[None, :]).ravel()
    rp, ci = m.pattern()
    v = m.assemble(E)[0]
    prp, pci, pv = permute_csr_fast(rp, ci, v, perm)
    del rp, ci, v
    ref = Oracle().pcg_pod2g(prp, pci, pv, f[perm], phi[perm], np.zeros(n), 0.0, N_PREFIX)
    t2 = time.perf_counter()
    assert ref.status == 0 and ref.iters == N_PREFIX
    np.testing.assert_allclose(hist[0, :N_PREFIX + 1], ref.history[:N_PREFIX + 1], rtol=1e-6)
    err = np.linalg.norm(x_gpu[perm] - ref.u) / np.linalg.norm(ref.u)
    print(f"c5 prefix: {N_PREFIX} iterations, rel residual {hist[0, N_PREFIX]:.3e}, "
          f"x rel diff {err:.2e}; GPU side {t1 - t0:.0f} s, oracle {t2 - t1:.0f} s")
    assert err <= 1e-8, err
