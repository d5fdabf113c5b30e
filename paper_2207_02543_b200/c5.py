"""Config c5 (BASELINE.json configs[4]): the 12.4M-dof hex8 system solved by
the ROW-PARTITIONED path.

Every rank only ever holds its own rows: the pattern comes from
p2g_mesh_pattern_range, values are generated on the device
(p2g_part_assemble), the node colouring is the mesh parity
colouring, and the POD stage is distributed: the Gram matrix U^T U is a sum of
per-rank products, Phi's owned rows are U_own Psi Lambda^-1/2, and its ghost
rows are the same combination of the snapshots' ghost rows (shipped from the
owning ranks).

Offline stage (outside the measured solve).  Solving 12.4M-dof snapshots to
1e-10 with symmetric-GS PCG alone needs thousands of iterations each, so the
snapshots are solved with the same PCG + two-grid preconditioner using a
generic smooth coarse space -- the polynomials of total degree <= 3 in
(x, y, z) for each displacement component (60 vectors), orthonormalised --
and the POD basis (k = 40) is built from those snapshots (compute_pod,
pod.hpp:73-148, RankTarget{k}).  Stated in DESIGN.md.

Transport: `world` partitions in one process on one GPU (device copies), or
one partition per process over NCCL when launched by torchrun.
"""
from __future__ import annotations

import itertools
import time

import numpy as np

from . import _lib as L
from . import problems as PR
from .partition import PartitionedSolver, row_bounds


class Comm:
    """Cross-rank sums / ghost-row gathers for the offline stage."""

    def __init__(self, hosted, world):
        self.hosted, self.world = hosted, world
        self.dist = None
        if len(hosted) < world:
            import torch.distributed as dist
            self.dist = dist

    def sum(self, parts):  # parts: dict rank -> array, same shape
        tot = sum(parts[r] for r in self.hosted)
        if self.dist is not None:
            import torch
            t = torch.from_numpy(np.ascontiguousarray(tot)).cuda()
            self.dist.all_reduce(t)
            tot = t.cpu().numpy()
        return tot

    def rows(self, owned, bounds, need):
        """owned: rank -> [ns][n_own] rows; need: rank -> global rows wanted.
        Returns rank -> [ns][len(need)] (the owners' values)."""
        out = {}
        if self.dist is None:
            full = np.concatenate([owned[r] for r in range(self.world)], axis=1)
            for r in self.hosted:
                out[r] = np.ascontiguousarray(full[:, need[r]])
            return out
        # one partition per process: every rank ships what each peer needs
        import torch
        me = self.hosted[0]
        reqs = [None] * self.world
        self.dist.all_gather_object(reqs, need[me])
        ns = owned[me].shape[0]
        r0 = int(bounds[me])
        sends = []
        for q in range(self.world):
            rows = np.asarray(reqs[q], dtype=np.int64)
            mine = rows[(rows >= r0) & (rows < int(bounds[me + 1]))] - r0
            sends.append(torch.from_numpy(np.ascontiguousarray(owned[me][:, mine])).cuda())
        recv = []
        for q in range(self.world):
            rows = np.asarray(need[me], dtype=np.int64)
            cnt = int(((rows >= int(bounds[q])) & (rows < int(bounds[q + 1]))).sum())
            recv.append(torch.empty((ns, cnt), dtype=torch.float64, device="cuda"))
        self.dist.all_to_all(recv, sends)
        res = np.concatenate([t.cpu().numpy() for t in recv], axis=1)
        # need[me] is ascending and owners' blocks are in rank order: res is in need order
        out[me] = res
        return out


def smooth_space(mesh, rows, deg=3):
    """Monomials x^a y^b z^c (a+b+c <= deg) per displacement component at the
    given global dof rows (unnormalised)."""
    x, y, z, comp = mesh.dof_coords_rows(rows)
    dims = mesh.dim
    exps = [e for e in itertools.product(range(deg + 1), repeat=3)
            if sum(e) <= deg and (dims == 3 or e[2] == 0)]
    cols = []
    for d in range(dims):
        for a, b, c in exps:
            cols.append(np.where(comp == d, x ** a * y ** b * z ** c, 0.0))
    return np.stack(cols, axis=1)


def _orthonormal(parts_own, parts_ghost, comm):
    G = comm.sum({r: parts_own[r].T @ parts_own[r] for r in parts_own})
    R = np.linalg.cholesky(G).T
    Ri = np.linalg.inv(R)
    return ({r: np.ascontiguousarray(v @ Ri) for r, v in parts_own.items()},
            {r: np.ascontiguousarray(v @ Ri) for r, v in parts_ghost.items()})


class C5Case:
    """The row-partitioned system after the offline stage: partition handle
    `P` (pattern, device-generated query values, POD basis installed), the
    right-hand sides of the hosted ranks, and the offline-stage record."""

    def __init__(self, **kw):
        self.__dict__.update(kw)

    def query_values(self):
        """The query instance's values on the device (p2g_part_assemble)."""
        for r in self.hosted:
            self.P.assemble(r, self.mesh, self.E)
            self.P.set_basis(r, self.phi_own[r], self.phi_gh[r])

    def host_values(self, r):
        """Rank r's rows of the query instance's values, assembled on the host
        ([1][local nnz], local rows, global columns) -- the e2e input."""
        r0, r1 = int(self.bounds[r]), int(self.bounds[r + 1])
        rp, ci = self.mesh.pattern_range(r0, r1)
        return self.mesh.assemble_rows(self.E, r0, r1, int(rp[-1]))

    def solve(self, max_iter=20000, tol=None):
        self.P.setup()
        return self.P.solve({r: self.bvec[r][None, :] for r in self.hosted},
                            self.cfg.tol if tol is None else tol, max_iter, L.X0_REDUCED)

    def close(self):
        self.P.close()


def run(cfg_name="c5", world=1, hosted=None, nccl_uid=None, n_snapshots=48, snap_batch=8,
        k=None, snap_tol=None, log=print, device=0):
    """The offline stage (prepare) and one query solve; returns (record, x)."""
    case = prepare(cfg_name, world, hosted, nccl_uid, n_snapshots, snap_batch, k, snap_tol, log,
                   device)
    t2 = time.perf_counter()
    case.query_values()
    xs, it, conv, status, hist = case.solve()
    t_solve = time.perf_counter() - t2
    P = case.P
    log(f"[c5] query: iterations {int(it[0])} converged {bool(conv[0])} status {int(status[0])} "
        f"setup+solve {t_solve * 1e3:.1f} ms (device solve {P.last_solve_ms():.1f} ms)")
    res = dict(n=case.mesh.n, nnz=case.mesh.nnz, world=world, iterations=int(it[0]),
               converged=bool(conv[0]), solve_ms=P.last_solve_ms(), setup_solve_s=t_solve,
               offline_s=case.offline_s, snapshot_iterations_mean=case.snapshot_iterations_mean,
               history=hist[0, :int(it[0]) + 1])
    case.close()
    return res, xs


def prepare(cfg_name="c5", world=1, hosted=None, nccl_uid=None, n_snapshots=48, snap_batch=8,
            k=None, snap_tol=None, log=print, device=0):
    cfg = PR.CONFIGS[cfg_name]
    k = cfg.k if k is None else k
    snap_tol = PR.SNAP_TOL if snap_tol is None else snap_tol
    hosted = list(range(world)) if hosted is None else hosted
    comm = Comm(hosted, world)
    t0 = time.perf_counter()
    mesh = PR.Mesh.for_config(cfg)
    n, bs = mesh.n, mesh.block_size
    colors = mesh.node_colors()
    bounds = row_bounds(n, world, bs)
    f = mesh.rhs()
    P = PartitionedSolver(world, device, rank=hosted[0] if nccl_uid is not None else None,
                          nccl_uid=nccl_uid)
    ghosts, own_rows = {}, {}
    for r in hosted:
        r0, r1 = int(bounds[r]), int(bounds[r + 1])
        rp, ci = mesh.pattern_range(r0, r1)
        P.set_pattern(r, n, bounds, rp, ci, bs, colors)
        ghosts[r] = P.ghosts(r)
        own_rows[r] = np.arange(r0, r1, dtype=np.int64)
    log(f"[c5] n={n} nnz={mesh.nnz} world={world} pattern {time.perf_counter() - t0:.1f}s")
    # bootstrap coarse space for the snapshot solves
    sm_own = {r: smooth_space(mesh, own_rows[r]) for r in hosted}
    sm_gh = {r: smooth_space(mesh, ghosts[r]) for r in hosted}
    sm_own, sm_gh = _orthonormal(sm_own, sm_gh, comm)
    bvec = {r: f[int(bounds[r]):int(bounds[r + 1])] for r in hosted}
    seeds = PR.snapshot_seeds(cfg, n_snapshots)
    snaps = {r: [] for r in hosted}
    it_all = []
    t1 = time.perf_counter()
    for s0 in range(0, n_snapshots, snap_batch):
        sb = seeds[s0:s0 + snap_batch]
        E, _ = mesh.kl_field(sb, cfg.kl_terms)
        for r in hosted:
            P.assemble(r, mesh, E)
            P.set_basis(r, sm_own[r], sm_gh[r])
        st = P.setup()
        xs, it, conv, status, _ = P.solve({r: np.broadcast_to(bvec[r], (len(sb), len(bvec[r])))
                                           for r in hosted}, snap_tol, 20000, L.X0_REDUCED, hist_cap=0)
        if not np.all(conv) or np.any(status != 0) or np.any(st != 0):
            raise RuntimeError("c5 snapshot solve failed")
        for r in hosted:
            snaps[r].append(xs[r])
        it_all.extend(it.tolist())
        log(f"[c5] snapshots {s0 + len(sb)}/{n_snapshots}: iterations {it.tolist()}")
    U = {r: np.concatenate(snaps[r], axis=0) for r in hosted}
    U_gh = comm.rows(U, bounds, ghosts)
    # compute_pod (pod.hpp:73-148) with RankTarget{k}, distributed Gram
    # the Gram partials and Phi's rows on the FP64 tensor cores
    G = comm.sum({r: PR.gram_device(U[r], device) for r in hosted})
    G = 0.5 * (G + G.T)
    w, V = np.linalg.eigh(G)
    order = np.argsort(-w, kind="stable")
    w, V = w[order], V[:, order]
    # numerical-rank cutoff as compute_pod (pod.hpp:92-101): eigenvalues > 1e-12 lambda_max
    r_num = int(np.count_nonzero(w > 1e-12 * w[0])) if w.size and w[0] > 0 else 0
    if r_num < 1:
        raise RuntimeError("c5 offline stage: snapshot Gram matrix has no positive eigenvalue")
    k = min(k, r_num)
    w, V = w[:k], V[:, :k]
    Wk = np.ascontiguousarray(V / np.sqrt(w))
    phi_own = {r: PR.combine_device(U[r], Wk, device) for r in hosted}
    phi_gh = {r: (PR.combine_device(U_gh[r], Wk, device) if U_gh[r].shape[1]
                  else np.zeros((0, k))) for r in hosted}
    defect = np.max(np.abs(comm.sum({r: phi_own[r].T @ phi_own[r] for r in hosted}) - np.eye(k)))
    if defect > 1e-8:
        phi_own, phi_gh = _orthonormal(phi_own, phi_gh, comm)
    t_off = time.perf_counter() - t1
    log(f"[c5] offline: {n_snapshots} snapshots in {t_off:.1f}s (mean iterations "
        f"{np.mean(it_all):.0f}), POD rank {k}, defect {defect:.1e}")
    # the measured query: one instance (query seed 0), x0 = reduced_solve, tol 1e-8
    E, _ = mesh.kl_field(PR.query_seeds(cfg, 1), cfg.kl_terms)
    return C5Case(cfg=cfg, P=P, mesh=mesh, bounds=bounds, hosted=hosted, world=world,
                  ghosts=ghosts, bvec=bvec, phi_own=phi_own, phi_gh=phi_gh, E=E, k=k,
                  offline_s=t_off, snapshot_iterations_mean=float(np.mean(it_all)),
                  n_snapshots=n_snapshots)
