"""Row-partitioned single-system solves over the
C-ABI p2g_part_* entry points.

The system is split by contiguous, node-aligned blocks of global rows; all
ranks share one global node colouring, so the partitioned multicolour sweeps
equal the single-GPU sweeps ("Multi-GPU").
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .solver import _raise, analyze_pattern


def node_colors(row_offsets, col_indices, block_size):
    """The greedy node colouring p2g_set_pattern uses, as a colour per node."""
    perm, offs = analyze_pattern(row_offsets, col_indices, block_size)
    nn = len(perm) // block_size
    col = np.empty(nn, dtype=np.int32)
    for c in range(len(offs) - 1):
        col[perm[offs[c]:offs[c + 1]:block_size] // block_size] = c
    return col


def row_bounds(n_global, world, block_size):
    """Balanced node-aligned row blocks: world+1 offsets."""
    nn = n_global // block_size
    b = [(nn * r) // world * block_size for r in range(world + 1)]
    return np.asarray(b, dtype=np.int64)


def local_rows(row_offsets, col_indices, r0, r1):
    """CSR slice of rows [r0, r1) with GLOBAL column indices."""
    rp = np.asarray(row_offsets, dtype=np.uint64)
    lo, hi = int(rp[r0]), int(rp[r1])
    return (rp[r0:r1 + 1] - np.uint64(lo)).astype(np.uint64), \
        np.ascontiguousarray(col_indices[lo:hi], dtype=np.uint64), (lo, hi)


def plan(rank, world, bounds, n_global, rp_loc, ci_loc, block_size, colors):
    """Host-only partition plan summary (no device): sizes, ghosts, counts."""
    lib = L.lib()
    bounds = np.ascontiguousarray(bounds, dtype=np.int64)
    rp_loc = np.ascontiguousarray(rp_loc, dtype=np.uint64)
    ci_loc = np.ascontiguousarray(ci_loc, dtype=np.uint64)
    colors = np.ascontiguousarray(colors, dtype=np.int32)
    ncol = int(colors.max()) + 1
    sizes = np.zeros(4, dtype=np.int64)
    sc = np.zeros((ncol, world), dtype=np.int64)
    rc = np.zeros((ncol, world), dtype=np.int64)
    err = C.create_string_buffer(256)
    st = lib.p2g_plan_partition(rank, world, bounds.ctypes.data_as(L.I64), n_global,
                                rp_loc.ctypes.data_as(L.U64), ci_loc.ctypes.data_as(L.U64),
                                block_size, colors.ctypes.data_as(L.I32),
                                sizes.ctypes.data_as(L.I64), None, sc.ctypes.data_as(L.I64),
                                rc.ctypes.data_as(L.I64), err, 256)
    if st != L.OK:
        _raise(st, err.value.decode())
    ghosts = np.empty(int(sizes[1]), dtype=np.int64)
    lib.p2g_plan_partition(rank, world, bounds.ctypes.data_as(L.I64), n_global,
                           rp_loc.ctypes.data_as(L.U64), ci_loc.ctypes.data_as(L.U64), block_size,
                           colors.ctypes.data_as(L.I32), sizes.ctypes.data_as(L.I64),
                           ghosts.ctypes.data_as(L.I64), None, None, err, 256)
    return {"n_own": int(sizes[0]), "n_ghost": int(sizes[1]), "nnz": int(sizes[2]),
            "ncolors": int(sizes[3]), "ghosts": ghosts, "send": sc, "recv": rc}


class PartitionedSolver:
    """p2g_part handle: `world` partitions in-process (local=True) or this
    process's rank over NCCL."""

    def __init__(self, world, device=0, rank=None, nccl_uid=None):
        self._L = L.lib()
        p = C.c_void_p()
        if nccl_uid is None:
            st = self._L.p2g_part_create_local(device, world, C.byref(p))
            self.ranks = list(range(world))
        else:
            buf = C.create_string_buffer(bytes(nccl_uid), 128)
            st = self._L.p2g_part_create_nccl(device, rank, world, buf, C.byref(p))
            self.ranks = [rank]
        if st != L.OK:
            raise RuntimeError(f"p2g_part_create failed: status {st}")
        self._p = p
        self.world = world
        self.B = 0
        self.n_own = {}

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        st = L.lib().p2g_nccl_unique_id(buf)
        if st != L.OK:
            raise RuntimeError("p2g_nccl_unique_id failed")
        return buf.raw

    def close(self):
        if getattr(self, "_p", None):
            self._L.p2g_part_destroy(self._p)
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st, what):
        if st != L.OK:
            _raise(st, f"{what}: {self._L.p2g_part_last_error(self._p).decode()}")

    def set_pattern(self, rank, n_global, bounds, rp_loc, ci_loc, block_size, colors):
        bounds = np.ascontiguousarray(bounds, dtype=np.int64)
        rp_loc = np.ascontiguousarray(rp_loc, dtype=np.uint64)
        ci_loc = np.ascontiguousarray(ci_loc, dtype=np.uint64)
        colors = np.ascontiguousarray(colors, dtype=np.int32)
        self._check(self._L.p2g_part_set_pattern(self._p, rank, n_global, bounds.ctypes.data_as(L.I64),
                                                 rp_loc.ctypes.data_as(L.U64),
                                                 ci_loc.ctypes.data_as(L.U64), block_size,
                                                 colors.ctypes.data_as(L.I32)), "set_pattern")
        self.n_own[rank] = len(rp_loc) - 1

    def ghosts(self, rank):
        no, ng = C.c_int64(), C.c_int64()
        self._check(self._L.p2g_part_ghosts(self._p, rank, C.byref(no), C.byref(ng), None), "ghosts")
        g = np.empty(ng.value, dtype=np.int64)
        self._check(self._L.p2g_part_ghosts(self._p, rank, None, None, g.ctypes.data_as(L.I64)),
                    "ghosts")
        return g

    def set_values(self, rank, values):
        v = np.ascontiguousarray(values, dtype=np.float64)
        if v.ndim == 1:
            v = v[None, :]
        self._check(self._L.p2g_part_set_values(self._p, rank, v.shape[0], v.ctypes.data_as(L.D)),
                    "set_values")
        self.B = v.shape[0]

    def assemble(self, rank, mesh, E):
        """Generate partition `rank`'s rows of K(E_b) on the device."""
        E = np.ascontiguousarray(np.atleast_2d(E), dtype=np.float64)
        self._check(self._L.p2g_part_assemble(self._p, rank, mesh._h, E.shape[0],
                                              E.ctypes.data_as(C.c_void_p), 0), "assemble")
        self.B = E.shape[0]

    def set_basis(self, rank, phi_own, phi_ghost):
        po = np.ascontiguousarray(phi_own, dtype=np.float64)
        pg = np.ascontiguousarray(phi_ghost, dtype=np.float64)
        self._check(self._L.p2g_part_set_basis(self._p, rank, po.shape[1], po.ctypes.data_as(L.D),
                                               pg.ctypes.data_as(L.D) if pg.size else None),
                    "set_basis")

    def setup(self, residual_form=L.RESIDUAL_UPPER, kp_update=L.KP_RECURRENCE):
        cfg = L.Config(L.SMOOTHER_GS_MULTICOLOR, 1, 1, residual_form, 0.5, kp_update, 0)
        st = np.zeros(max(self.B, 1), dtype=np.int32)
        rc = self._L.p2g_part_setup(self._p, C.byref(cfg), st.ctypes.data_as(L.I32))
        if rc in (L.EINVAL, L.ECUDA, L.ESTATE, L.ENCCL):
            self._check(rc, "setup")
        return st[: self.B]

    def solve(self, bs, tol=1e-8, max_iter=100000, x0_mode=L.X0_REDUCED, x0s=None, hist_cap=None):
        """bs / x0s: dict rank -> [B][n_own] for the hosted ranks."""
        B = self.B
        barr = [np.ascontiguousarray(np.reshape(bs[r], (B, -1)), dtype=np.float64) for r in self.ranks]
        xs = [np.empty_like(b) for b in barr]
        Dp = C.POINTER(C.c_double)
        bp = (Dp * len(barr))(*[b.ctypes.data_as(Dp) for b in barr])
        xp = (Dp * len(xs))(*[x.ctypes.data_as(Dp) for x in xs])
        x0p = None
        if x0s is not None:
            x0arr = [np.ascontiguousarray(np.reshape(x0s[r], (B, -1)), dtype=np.float64) for r in self.ranks]
            x0p = (Dp * len(x0arr))(*[x.ctypes.data_as(Dp) for x in x0arr])
        cap = int(hist_cap if hist_cap is not None else min(max_iter, 100000) + 1)
        it = np.zeros(B, dtype=np.int64)
        conv = np.zeros(B, dtype=np.int32)
        status = np.zeros(B, dtype=np.int32)
        hist = np.empty((B, max(cap, 1)))
        rc = self._L.p2g_part_solve(self._p, bp, x0p, x0_mode, tol, max_iter, xp,
                                    it.ctypes.data_as(L.I64), conv.ctypes.data_as(L.I32),
                                    status.ctypes.data_as(L.I32),
                                    hist.ctypes.data_as(L.D) if cap > 0 else None, cap)
        if rc in (L.EINVAL, L.ECUDA, L.ESTATE, L.ENCCL):
            self._check(rc, "solve")
        return dict(zip(self.ranks, xs)), it, conv.astype(bool), status, hist[:, :cap]

    def last_solve_ms(self):
        ms = C.c_double()
        self._L.p2g_part_last_solve_ms(self._p, C.byref(ms))
        return ms.value

    def stream(self) -> int:
        """cudaStream_t of the hosted partitions (time with events on it)."""
        return int(self._L.p2g_part_get_stream(self._p) or 0)

    def launch_counts(self):
        """(launches per iteration, running total, loop mode of the last solve)."""
        per, tot, mode = C.c_int64(), C.c_int64(), C.c_int32()
        self._check(self._L.p2g_part_launch_counts(self._p, C.byref(per), C.byref(tot),
                                                   C.byref(mode)), "launch_counts")
        return per.value, tot.value, mode.value

    def profile_iteration(self, reps=3):
        """{class: (ms per iteration, algorithmic bytes per iteration)} (one hosted partition)."""
        ms = np.zeros(L.NUM_KCLASS)
        by = np.zeros(L.NUM_KCLASS)
        names = (C.c_char_p * L.NUM_KCLASS)()
        self._check(self._L.p2g_part_profile_iteration(self._p, reps, ms.ctypes.data_as(L.D),
                                                       by.ctypes.data_as(L.D), names),
                    "profile_iteration")
        return {names[i].decode(): (float(ms[i]), float(by[i])) for i in range(L.NUM_KCLASS)}


def setup_partitioned(rp, ci, values, f, phi, world, block_size, device=0, colors=None,
                      **setup_kw):
    """Convenience: split a global system into `world` in-process partitions."""
    n = len(rp) - 1
    colors = node_colors(rp, ci, block_size) if colors is None else colors
    bounds = row_bounds(n, world, block_size)
    values = np.atleast_2d(values)
    S = PartitionedSolver(world, device)
    bs = {}
    for r in range(world):
        r0, r1 = int(bounds[r]), int(bounds[r + 1])
        rpl, cil, (lo, hi) = local_rows(rp, ci, r0, r1)
        S.set_pattern(r, n, bounds, rpl, cil, block_size, colors)
        S.set_values(r, values[:, lo:hi])
        g = S.ghosts(r)
        S.set_basis(r, phi[r0:r1], phi[g] if len(g) else np.zeros((0, phi.shape[1])))
        bs[r] = np.atleast_2d(f)[:, r0:r1] if np.ndim(f) == 2 else np.broadcast_to(f[r0:r1], (values.shape[0], r1 - r0))
    st = S.setup(**setup_kw)
    return S, bounds, bs, st
