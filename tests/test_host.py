"""Host-side logic on CPU: generator, colouring/permutation, sharding, and
the C-ABI library surface (loads and exports every declared symbol without a
GPU; no compute calls)."""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2207_02543_b200 import _lib as L
from paper_2207_02543_b200 import problems as PR
from paper_2207_02543_b200.solver import analyze_node_blocking, analyze_pattern
from tests.helpers import from_scipy, laplacian_2d, to_scipy

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---------------------------------------------------------------- C-ABI surface
def declared_functions():
    names = []
    for h in ("pod2g_b200.h", "pod2g_gen.h"):
        txt = open(os.path.join(ROOT, "include", h)).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        names += re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(p2g_\w+)\s*\(", txt, flags=re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(L.LIB_PATH)
    gen = C.CDLL(L.GEN_PATH)
    names = declared_functions()
    assert len(names) >= 30
    gen_names = {n for n, _, _ in L.GEN_SIGNATURES}
    missing = [n for n in names if not hasattr(gen if n in gen_names else lib, n)]
    assert not missing, missing
    bound = {n for n, _, _ in L.SIGNATURES} | gen_names
    assert set(names) <= bound, set(names) - bound


def test_generator_library_is_cpu_only():
    """libpod2g_gen.so (the seeded inputs) carries no CUDA code or runtime, so
    the CPU reference arm never maps the CUDA library."""
    import subprocess
    out = subprocess.run(["ldd", L.GEN_PATH], capture_output=True, text=True).stdout
    assert "cuda" not in out.lower() and "pod2g_b200" not in out, out
    syms = subprocess.run(["nm", "-D", "--defined-only", L.GEN_PATH], capture_output=True,
                          text=True).stdout
    assert "cuda" not in syms.lower()


def test_abi_version_and_status_strings():
    lib = L.lib()
    assert lib.p2g_abi_version() == 2
    assert lib.p2g_status_string(L.EBREAKDOWN).decode().startswith("PCG breakdown")


def test_no_cpu_fallback_without_device():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except Exception:
        pass
    h = C.c_void_p()
    assert L.lib().p2g_create(0, C.byref(h)) == L.ECUDA
    from paper_2207_02543_b200.solver import BatchSolver
    with pytest.raises(RuntimeError):
        BatchSolver(0)


# ---------------------------------------------------------------- generator
@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_config_sizes_match_survey(name):
    """SURVEY.md 8 table / Appendix B closed forms."""
    cfg = PR.CONFIGS[name]
    m = PR.Mesh.for_config(cfg)
    if cfg.dim == 2:
        n = 2 * cfg.nx * (cfg.ny + 1)
        z = 4 * (3 * cfg.nx - 2) * (3 * (cfg.ny + 1) - 2)
    else:
        mm = cfg.nx
        n = 3 * mm * (mm + 1) ** 2
        z = 9 * (3 * mm - 2) * (3 * (mm + 1) - 2) ** 2
    assert (m.n, m.nnz) == (n, z)
    assert m.block_size == cfg.dim


def _dense_q4_assembly(nx, ny, Lx, Ly, E, Ke):
    """Independent dense assembly (test_problems.cpp:16-73 style)."""
    NX = nx + 1
    ndof = 2 * NX * (ny + 1)
    Kf = np.zeros((ndof, ndof))
    for ey in range(ny):
        for ex in range(nx):
            nodes = [ey * NX + ex, ey * NX + ex + 1, (ey + 1) * NX + ex + 1, (ey + 1) * NX + ex]
            dofs = [2 * a + c for a in nodes for c in range(2)]
            Kf[np.ix_(dofs, dofs)] += E[ey * nx + ex] * Ke
    free = [d for d in range(ndof) if (d // 2) % NX != 0]
    return Kf[np.ix_(free, free)]


def test_q4_assembly_matches_dense_oracle_and_is_spd():
    m = PR.Mesh(2, 6, 3, 1, 2.0, 1.0, 1.0)
    rp, ci = m.pattern()
    E = np.random.default_rng(0).uniform(0.5, 2.0, m.nelem)
    v = m.assemble(E)[0]
    K = to_scipy(rp, ci, v, m.n).toarray()
    Kd = _dense_q4_assembly(6, 3, 2.0, 1.0, E, m.element_stiffness())
    assert np.max(np.abs(K - Kd)) <= 1e-14 * np.max(np.abs(Kd))
    assert np.array_equal(K, K.T)
    assert np.linalg.eigvalsh(K)[0] > 0


def test_element_stiffness_rigid_modes_and_symmetry():
    for dim in (2, 3):
        m = PR.Mesh(dim, 2, 2, 2 if dim == 3 else 1, 1.0, 1.0, 1.0)
        Ke = m.element_stiffness()
        assert np.array_equal(Ke, Ke.T)
        nen = 2 ** dim
        for c in range(dim):  # translations are in the null space
            t = np.zeros(dim * nen)
            t[c::dim] = 1.0
            assert np.max(np.abs(Ke @ t)) <= 1e-13 * np.max(np.abs(Ke))
        ev = np.linalg.eigvalsh(Ke)
        nrig = 3 if dim == 2 else 6
        assert np.sum(np.abs(ev) < 1e-10 * ev.max()) == nrig


def test_hex8_small_is_spd_and_loads_sum():
    m = PR.Mesh(3, 3, 3, 3, 1.0, 1.0, 1.0)
    rp, ci = m.pattern()
    v = m.assemble(np.ones(m.nelem))[0]
    K = to_scipy(rp, ci, v, m.n).toarray()
    assert np.array_equal(K, K.T) and np.linalg.eigvalsh(K)[0] > 0
    f = m.rhs()
    assert abs(f.sum() + 1.0) < 1e-14  # unit traction on the unit face
    assert np.all(f[0::3] == 0) and np.all(f[1::3] == 0)
    f2 = PR.Mesh(2, 8, 4, 1, 2.0, 1.0, 1.0).rhs()
    assert abs(f2.sum() + 1.0) < 1e-14 and np.all(f2[0::2] == 0)


def test_kl_field_reproducible_and_lognormal():
    cfg = PR.CONFIGS["c2"]
    m = PR.Mesh.for_config(cfg)
    E1, xi1 = m.kl_field(PR.query_seeds(cfg, 3), cfg.kl_terms)
    E2, xi2 = m.kl_field(PR.query_seeds(cfg, 3), cfg.kl_terms)
    assert np.array_equal(E1, E2) and np.array_equal(xi1, xi2)
    lam = m.kl_eigenvalues(cfg.kl_terms)
    assert np.all(np.diff(lam) <= 0) and lam[0] > 0
    g = np.log(m.kl_field(PR.query_seeds(cfg, 64), cfg.kl_terms)[0])
    # pointwise variance of g ~ sigma^2 * (captured KL fraction), mean ~ 0
    assert abs(g.mean()) < 0.05
    assert 0.5 * PR.SIGMA ** 2 < g.var() < 1.2 * PR.SIGMA ** 2


def test_normal_draws_moments():
    x = PR.normal_draws(123, 200000)
    assert abs(x.mean()) < 0.01 and abs(x.std() - 1.0) < 0.01
    assert np.array_equal(x[:10], PR.normal_draws(123, 10))


def test_compute_pod_restatement():
    """pod.hpp:73-148: orthonormal, spans the snapshots, rank truncation."""
    rng = np.random.default_rng(0)
    U = rng.standard_normal((8, 100)) @ np.diag(np.linspace(1, 2, 100))
    phi, w, energy = PR.compute_pod(U, 5)
    assert phi.shape == (100, 5)
    assert np.max(np.abs(phi.T @ phi - np.eye(5))) < 1e-12
    phi8, w8, e8 = PR.compute_pod(U, 50)  # capped at the numerical rank
    assert phi8.shape[1] == 8 and abs(e8 - 1.0) < 1e-12
    resid = U.T - phi8 @ (phi8.T @ U.T)
    assert np.max(np.abs(resid)) < 1e-10 * np.max(np.abs(U))


# ---------------------------------------------------------------- colouring
@pytest.mark.parametrize("dims", [(2, 16, 8, 1), (3, 4, 4, 4)])
def test_node_colouring_is_valid_and_structured(dims):
    dim, nx, ny, nz = dims
    m = PR.Mesh(dim, nx, ny, nz, float(nx) / ny * (1 if dim == 2 else 1), 1.0, 1.0) if dim == 2 \
        else PR.Mesh(3, nx, ny, nz, 1.0, 1.0, 1.0)
    rp, ci = m.pattern()
    perm, offs = analyze_pattern(rp, ci, m.block_size)
    assert sorted(perm.tolist()) == list(range(m.n))
    assert len(offs) - 1 == 2 ** dim  # parity colouring of the node grid
    bs = m.block_size
    colour = np.empty(m.n // bs, dtype=int)
    for c in range(len(offs) - 1):
        colour[perm[offs[c]:offs[c + 1]] // bs] = c
    K = to_scipy(rp, ci, np.ones(len(ci)), m.n).tocoo()
    a, b = K.row // bs, K.col // bs
    off = a != b
    assert np.all(colour[a[off]] != colour[b[off]])  # independent sets
    # a node's dofs stay adjacent and in order
    assert np.all(perm[0::bs] % bs == 0)
    for c in range(1, bs):
        assert np.all(perm[c::bs] == perm[0::bs] + c)


def test_pattern_validation_errors():
    rp, ci, v = from_scipy(laplacian_2d(3))
    with pytest.raises(ValueError):
        analyze_pattern(rp, ci[::-1].copy(), 1)  # columns not increasing
    bad = sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 1.0]]))
    rpb, cib, _ = from_scipy(bad)
    with pytest.raises(ValueError, match="diagonal"):
        analyze_pattern(rpb, cib, 1)
    with pytest.raises(ValueError):
        analyze_pattern(rp, ci, 2)  # 9 rows not a multiple of 2
    asym = sp.csr_matrix(np.array([[1.0, 1.0], [0.0, 1.0]]))
    asym.eliminate_zeros()
    rpa, cia, _ = from_scipy(asym)
    with pytest.raises(ValueError, match="symmetric"):
        analyze_pattern(rpa, cia, 1)


# ---------------------------------------------------------------- sharding
def test_shard_weak_and_strong():
    """BASELINE's instance totals are split across ranks (c2/c4: 64, c3: 256);
    single-instance c1 runs one replica per rank with disjoint seeds."""
    c1, c2, c3, c4 = (PR.CONFIGS[c] for c in ("c1", "c2", "c3", "c4"))
    n, seeds, strong = PR.shard(c2, 1, 0)
    assert n == 64 and not strong
    for cfg, world in ((c2, 4), (c3, 8), (c4, 2), (c4, 8), (c3, 3)):
        parts = [PR.shard(cfg, world, r) for r in range(world)]
        assert all(p[2] for p in parts) and sum(p[0] for p in parts) == cfg.batch
        assert np.array_equal(np.concatenate([p[1] for p in parts]), PR.query_seeds(cfg))
    reps = [PR.shard(c1, 4, r) for r in range(4)]
    assert not any(p[2] for p in reps) and [p[0] for p in reps] == [1, 1, 1, 1]
    assert len(np.unique(np.concatenate([p[1] for p in reps]))) == 4


@pytest.mark.parametrize("dims,nmax", [((2, 16, 8, 1), 9), ((3, 4, 4, 4), 27)])
def test_node_blocking_detected_on_fem_patterns(dims, nmax):
    """FEM vector patterns are node-blocked (the node-blocked kernels run),
    with 9 (Q4) / 27 (hex8) neighbour nodes at most."""
    dim, nx, ny, nz = dims
    m = PR.Mesh(dim, nx, ny, nz, 2.0 if dim == 2 else 1.0, 1.0, 1.0)
    rp, ci = m.pattern()
    ok, nm = analyze_node_blocking(rp, ci, m.block_size)
    assert ok and nm == nmax
    # as a point pattern (block size 1) every row is its own node: Q4 rows hold
    # 18 entries (blocked), hex8 rows 81 (> 32 neighbours: row kernels)
    ok1, nm1 = analyze_node_blocking(rp, ci, 1)
    assert (ok1, nm1) == ((True, 18) if dim == 2 else (False, 0))


def test_node_blocking_rejects_unequal_node_rows():
    """A node whose rows hold different column sets falls back to the row
    kernels (the pattern is still valid)."""
    m = PR.Mesh(2, 8, 4, 1, 2.0, 1.0, 1.0)
    rp, ci = m.pattern()
    rp = rp.astype(np.int64)
    ci = ci.astype(np.int64)
    # drop the symmetric pair (row 0, col j) / (row j, col 0) for one off-node column j
    j = int(ci[rp[0]:rp[1]][-1])
    assert j // 2 != 0
    keep = np.ones(len(ci), dtype=bool)
    keep[rp[0] + np.where(ci[rp[0]:rp[1]] == j)[0][0]] = False
    keep[rp[j] + np.where(ci[rp[j]:rp[j + 1]] == 0)[0][0]] = False
    counts = np.diff(rp) - np.add.reduceat(~keep, rp[:-1])
    rp2 = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
    ci2 = ci[keep].astype(np.uint64)
    analyze_pattern(rp2, ci2, 2)  # valid, colourable
    ok, _ = analyze_node_blocking(rp2, ci2, 2)
    assert not ok
    with pytest.raises(ValueError):
        analyze_node_blocking(rp2, ci2[::-1].copy(), 2)


def test_wavefront_colouring_knob_is_valid(monkeypatch):
    """P2G_WAVE_COLOURS=C (measured and off by default): colour =
    natural-order GS level mod C; classes are independent sets and the node's
    dofs stay adjacent, like the default parity colouring."""
    m = PR.Mesh(2, 16, 8, 1, 2.0, 1.0, 1.0)
    rp, ci = m.pattern()
    monkeypatch.setenv("P2G_WAVE_COLOURS", "8")
    perm, offs = analyze_pattern(rp, ci, m.block_size)
    assert len(offs) - 1 == 8
    bs = m.block_size
    colour = np.empty(m.n // bs, dtype=int)
    for c in range(len(offs) - 1):
        colour[perm[offs[c]:offs[c + 1]] // bs] = c
    K = to_scipy(rp, ci, np.ones(len(ci)), m.n).tocoo()
    a, b = K.row // bs, K.col // bs
    off = a != b
    assert np.all(colour[a[off]] != colour[b[off]])
    assert np.all(perm[1::bs] == perm[0::bs] + 1)


@pytest.mark.parametrize("dims", [(3, 6, 4, 4, 1.5, 1.0, 1.0), (2, 14, 7, 1, 2.0, 1.0, 1.0)])
def test_range_assembly_equals_full_assembly(dims):
    """p2g_mesh_assemble_range (a partition's rows, the e2e input of the
    partitioned c5 bench) gives the full assembly's entries bit for bit."""
    m = PR.Mesh(*dims)
    rp, ci = m.pattern()
    E, _ = m.kl_field(np.arange(2, dtype=np.uint64), 20)
    V = m.assemble(E)
    d = m.block_size
    for r0, r1 in ((0, m.n), (d * 7, d * 40), (d * 3, d * 3)):
        prp, _ = m.pattern_range(r0, r1)
        W = m.assemble_rows(E, r0, r1, int(prp[-1]))
        assert np.array_equal(W, V[:, int(rp[r0]):int(rp[r1])])
