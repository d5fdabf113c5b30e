"""Seeded inputs for the BASELINE.json configs c1..c5.

The reference has no Q4 / plane-stress / cantilever / KL / pure-hex8 problem
(it ships `its` and `biot`, problems.hpp:99-344), so this module builds them
with the C++ generator of libpod2g_b200 (include/pod2g_gen.h) and produces the
offline artefacts the solve phase consumes:
  * the CSR pattern and the per-instance values (K(E) = sum_e E_e K_e^1),
  * the traction load b,
  * the POD basis Phi from GPU-solved snapshots (compute_pod, pod.hpp:73-148,
    restated below with RankTarget{k}).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L

SIGMA = 0.3      # std of the Gaussian field g
ELL = 0.2        # correlation length
NU = 0.3         # Poisson ratio (2D given; 3D unstated -> 0.3)
KL_QUAD = 128    # Nystrom points per axis
SNAP_TOL = 1e-10  # generate_snapshots tolerance (problems.hpp:489)


@dataclass(frozen=True)
class Config:
    name: str
    dim: int
    nx: int
    ny: int
    nz: int
    L: tuple
    k: int
    n_snapshots: int
    batch: int
    kl_terms: int
    tol: float = 1e-8

    @property
    def seed_base(self) -> int:
        return 1000 * int(self.name[1:])


CONFIGS = {
    "c1": Config("c1", 2, 64, 32, 1, (2.0, 1.0, 1.0), 10, 30, 1, 20),
    "c2": Config("c2", 2, 256, 128, 1, (2.0, 1.0, 1.0), 20, 50, 64, 20),
    "c3": Config("c3", 2, 1024, 512, 1, (2.0, 1.0, 1.0), 30, 60, 256, 20),
    "c4": Config("c4", 3, 64, 64, 64, (1.0, 1.0, 1.0), 30, 60, 64, 30),
    "c5": Config("c5", 3, 160, 160, 160, (1.0, 1.0, 1.0), 40, 60, 1, 30),
}


def shard(cfg: Config, world: int, rank: int):
    """Instance sharding across `world` GPUs (BASELINE.json: independent
    instances, no communication).  A config's instance total (c2/c4: 64, c3:
    256) is split contiguously across the ranks (strong scaling: the whole
    job is BASELINE's batch at every world size).  Single-instance configs
    (c1) run one replica per rank with disjoint seeds (weak scaling; c5 is
    row-partitioned instead, c5.py).  Returns (instances_on_rank, seeds, strong)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard: bad world/rank")
    strong = world > 1 and cfg.batch >= world
    if world == 1 or strong:
        base, extra = divmod(cfg.batch, world)
        count = base + (1 if rank < extra else 0)
        offset = rank * base + min(rank, extra)
    else:
        count, offset = cfg.batch, rank * cfg.batch
    return count, query_seeds(cfg, count, offset=offset), strong


def snapshot_seeds(cfg: Config, count=None):
    """Seeds of the offline snapshots: disjoint from the query seeds."""
    count = cfg.n_snapshots if count is None else count
    return np.arange(count, dtype=np.uint64) + np.uint64(10_000_000 + cfg.seed_base)


def query_seeds(cfg: Config, count=None, offset=0):
    """Instance i of config cN uses seed 20_000_000 + 1000*N + i."""
    count = cfg.batch if count is None else count
    return np.arange(offset, offset + count, dtype=np.uint64) + np.uint64(20_000_000 + cfg.seed_base)


class Mesh:
    """p2g_mesh: structured Q4 (dim 2) / hex8 (dim 3) elasticity generator."""

    def __init__(self, dim, nx, ny, nz=1, Lx=1.0, Ly=1.0, Lz=1.0, nu=NU):
        self._L = L.gen()
        h = C.c_void_p()
        st = self._L.p2g_mesh_create(dim, nx, ny, nz, Lx, Ly, Lz, nu, C.byref(h))
        if st != 0:
            raise ValueError("p2g_mesh_create: invalid mesh parameters")
        self._h = h
        n, nnz, ne = C.c_int64(), C.c_int64(), C.c_int64()
        bs = C.c_int32()
        self._L.p2g_mesh_info(h, C.byref(n), C.byref(nnz), C.byref(ne), C.byref(bs))
        self.dim, self.n, self.nnz, self.nelem, self.block_size = dim, n.value, nnz.value, ne.value, bs.value
        self.nx, self.ny, self.nz = nx, ny, nz if dim == 3 else 1
        self.h = Lx / nx

    @classmethod
    def for_config(cls, cfg: Config):
        return cls(cfg.dim, cfg.nx, cfg.ny, cfg.nz, *cfg.L)

    def close(self):
        if getattr(self, "_h", None):
            self._L.p2g_mesh_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def pattern(self):
        rp = np.empty(self.n + 1, dtype=np.uint64)
        ci = np.empty(self.nnz, dtype=np.uint64)
        self._L.p2g_mesh_pattern(self._h, rp.ctypes.data_as(L.U64), ci.ctypes.data_as(L.U64))
        return rp, ci

    def pattern_range(self, r0, r1):
        """Rows [r0, r1) with global columns (node aligned)."""
        rp = np.empty(r1 - r0 + 1, dtype=np.uint64)
        if self._L.p2g_mesh_pattern_range(self._h, r0, r1, rp.ctypes.data_as(L.U64), None) != 0:
            raise ValueError("pattern_range: bad row range")
        ci = np.empty(int(rp[-1]), dtype=np.uint64)
        self._L.p2g_mesh_pattern_range(self._h, r0, r1, rp.ctypes.data_as(L.U64),
                                       ci.ctypes.data_as(L.U64))
        return rp, ci

    def node_colors(self):
        col = np.empty(self.n // self.block_size, dtype=np.int32)
        self._L.p2g_mesh_node_colors(self._h, col.ctypes.data_as(L.I32))
        return col

    def dof_coords(self, r0=0, r1=None):
        """(x, y, z, component) of free dofs [r0, r1) (node-major numbering)."""
        r1 = self.n if r1 is None else r1
        return self.dof_coords_rows(np.arange(r0, r1, dtype=np.int64))

    def dof_coords_rows(self, g):
        """(x, y, z, component) of the free dofs with global indices g."""
        g = np.asarray(g, dtype=np.int64)
        d = self.block_size
        rn, comp = g // d, g % d
        ix = rn % self.nx + 1
        t = rn // self.nx
        iy = t % (self.ny + 1)
        iz = t // (self.ny + 1)
        return ix * self.h, iy * self.h, iz * self.h, comp

    def rhs(self):
        f = np.empty(self.n)
        self._L.p2g_mesh_rhs(self._h, f.ctypes.data_as(L.D))
        return f

    def element_stiffness(self):
        ned = self.dim * 2 ** self.dim
        Ke = np.empty((ned, ned))
        self._L.p2g_mesh_element_stiffness(self._h, Ke.ctypes.data_as(L.D))
        return Ke

    def kl_field(self, seeds, M, sigma=SIGMA, ell=ELL, quad=KL_QUAD):
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        E = np.empty((len(seeds), self.nelem))
        xi = np.empty((len(seeds), M))
        st = self._L.p2g_kl_field(self._h, M, sigma, ell, quad, len(seeds),
                                  seeds.ctypes.data_as(L.U64), E.ctypes.data_as(L.D),
                                  xi.ctypes.data_as(L.D))
        if st != 0:
            raise ValueError("p2g_kl_field failed")
        return E, xi

    def kl_eigenvalues(self, M, ell=ELL, quad=KL_QUAD):
        lam = np.empty(M)
        self._L.p2g_kl_eigenvalues(self._h, M, ell, quad, lam.ctypes.data_as(L.D))
        return lam

    def assemble(self, E, nthreads=0):
        E = np.ascontiguousarray(E, dtype=np.float64)
        if E.ndim == 1:
            E = E[None, :]
        vals = np.empty((E.shape[0], self.nnz))
        st = self._L.p2g_mesh_assemble(self._h, E.shape[0], E.ctypes.data_as(L.D),
                                       vals.ctypes.data_as(L.D), nthreads)
        if st != 0:
            raise ValueError("p2g_mesh_assemble failed")
        return vals


def _assemble_rows(self, E, r0, r1, nnz_range, nthreads=0):
    """Values of free rows [r0, r1) (node aligned): [B][nnz_range], the
    pattern_range(r0, r1) layout, bit-identical to assemble()'s entries."""
    E = np.ascontiguousarray(np.atleast_2d(E), dtype=np.float64)
    vals = np.empty((E.shape[0], nnz_range))
    st = self._L.p2g_mesh_assemble_range(self._h, E.shape[0], E.ctypes.data_as(L.D), r0, r1,
                                         vals.ctypes.data_as(L.D), nthreads)
    if st != 0:
        raise ValueError("p2g_mesh_assemble_range failed")
    return vals


Mesh.assemble_rows = _assemble_rows


def normal_draws(seed: int, count: int):
    out = np.empty(count)
    L.gen().p2g_normal_draws(np.uint64(seed), count, out.ctypes.data_as(L.D))
    return out


def gram_device(U, device=0):
    """G = U U^T on the FP64 tensor cores (p2g_gram, pod.hpp:81-87)."""
    U = np.ascontiguousarray(U, dtype=np.float64)
    N, d = U.shape
    G = np.empty((N, N))
    st = L.lib().p2g_gram(device, N, d, U.ctypes.data, 0, G.ctypes.data_as(L.D))
    if st != L.OK:
        raise RuntimeError(f"p2g_gram failed: status {st}")
    return G


def combine_device(U, W, device=0):
    """Phi = U^T W on the FP64 tensor cores (p2g_combine, pod.hpp:120-129)."""
    U = np.ascontiguousarray(U, dtype=np.float64)
    W = np.ascontiguousarray(W, dtype=np.float64)
    N, d = U.shape
    r = W.shape[1]
    Phi = np.empty((d, r))
    st = L.lib().p2g_combine(device, N, d, U.ctypes.data, 0, r, W.ctypes.data_as(L.D),
                             Phi.ctypes.data)
    if st != L.OK:
        raise RuntimeError(f"p2g_combine failed: status {st}")
    return Phi


def compute_pod(snapshots: np.ndarray, rank: int, device=None):
    """pod.hpp:73-148 with RankTarget{rank}: Gram U^T U, eigenpairs, cutoff
    1e-12 lambda_max, Phi = U Psi Lambda^{-1/2}, MGS if the orthonormality
    defect exceeds 1e-8.  snapshots: [N][d].  Returns (phi [d][r], eigenvalues,
    energy_fraction).  device: run the two contractions (Gram, Phi) on that GPU
    (SURVEY f4); the N x N eigenproblem stays on the host."""
    U = np.ascontiguousarray(snapshots, dtype=np.float64)
    N = U.shape[0]
    if N < 1:
        raise ValueError("compute_pod: no snapshots")
    if rank < 1:
        raise ValueError("compute_pod: rank target must be >= 1")
    G = U @ U.T if device is None else gram_device(U, device)
    G = 0.5 * (G + G.T)
    w, V = np.linalg.eigh(G)
    order = np.argsort(-w, kind="stable")
    w, V = w[order], V[:, order]
    if w[0] <= 0:
        raise RuntimeError("compute_pod: snapshot matrix is zero")
    numerical_rank = int(np.sum(w > 1e-12 * w[0]))
    r = min(rank, numerical_rank)
    Wr = V[:, :r] / np.sqrt(w[:r])[None, :]
    phi = U.T @ Wr if device is None or r > 64 else combine_device(U, Wr, device)
    total = float(np.sum(np.maximum(w, 0.0)))
    energy = float(np.sum(w[:r]) / total)
    defect = np.max(np.abs(phi.T @ phi - np.eye(r)))
    if defect > 1e-8:
        for j in range(r):
            for q in range(j):
                phi[:, j] -= (phi[:, q] @ phi[:, j]) * phi[:, q]
            nrm = np.linalg.norm(phi[:, j])
            if nrm <= 0:
                raise ValueError("compute_pod: re-orthonormalization collapsed a column")
            phi[:, j] /= nrm
    return np.ascontiguousarray(phi), w, energy


@dataclass
class Problem:
    """One config's shared data: pattern, load, basis (+ the mesh)."""
    cfg: Config
    mesh: Mesh
    rp: np.ndarray
    ci: np.ndarray
    f: np.ndarray
    phi: np.ndarray
    pod_eigenvalues: np.ndarray
    snapshot_iters: np.ndarray

    def values(self, seeds):
        E, _ = self.mesh.kl_field(seeds, self.cfg.kl_terms)
        return self.mesh.assemble(E)


def build_problem(cfg: Config, device: int = 0, n_snapshots=None, k=None, solver_cls=None):
    """Generate pattern, load and the POD basis (snapshots solved on the GPU
    to SNAP_TOL by symmetric-GS PCG, i.e. the solve path with k = 0)."""
    from .solver import BatchSolver
    mesh = Mesh.for_config(cfg)
    rp, ci = mesh.pattern()
    f = mesh.rhs()
    ns = cfg.n_snapshots if n_snapshots is None else n_snapshots
    kk = cfg.k if k is None else k
    E = mesh.kl_field(snapshot_seeds(cfg, ns), cfg.kl_terms)[0]
    s = (solver_cls or BatchSolver)(device)
    try:
        s.set_pattern(rp, ci, mesh.block_size)
        s.assemble(mesh, E)  # on-device generation
        s.set_basis(None)
        s.setup()
        F = np.broadcast_to(f, (ns, mesh.n)).copy()
        x, it, conv, status, _ = s.solve(F, None, SNAP_TOL, 20 * mesh.n, hist_cap=0)
        if not np.all(conv) or np.any(status != 0):
            bad = int(np.flatnonzero(~conv | (status != 0))[0])
            raise RuntimeError(f"generate_snapshots: sample {bad} failed to reach the snapshot tolerance")
    finally:
        s.close()
    phi, w, _ = compute_pod(x, kk, device=device)
    return Problem(cfg, mesh, rp, ci, f, phi, w, it)
