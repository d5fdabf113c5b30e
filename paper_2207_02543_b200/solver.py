"""Host-side mirror of the reference's POD-2G solver interface over the C-ABI.

Reference interface (paths under /root/reference/proj/include/pod2g/):
  CsrMatrix            core/csr.hpp:14-59
  PodBasis             pod.hpp:19-58
  SolveReport          core/report.hpp:13-23
  Pod2gPreconditioner  pod.hpp:259-274  (apply(r, s), name() == "pod2g")
  pcg_solve            krylov.hpp:243-297
  reduced_solve        pod.hpp:167-179
Errors keep the reference's split: std::invalid_argument -> ValueError,
std::runtime_error -> RuntimeError.

Everything here runs on the GPU through libpod2g_b200.so; nothing computes on
the CPU.  ``BatchSolver`` is the batched handle (B instances sharing one
pattern), the B200-native shape of the reference's parallel_for over
instances (bench.hpp:290-330).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


def _d(a):
    return None if a is None else a.ctypes.data_as(L.D)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class CsrMatrix:
    """core/csr.hpp:14-59 (size_t indices -> uint64)."""
    nrows: int
    ncols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray
    symmetric_hint: bool = True

    def nnz(self) -> int:
        return int(len(self.values))


@dataclass
class PodBasis:
    """pod.hpp:19-58: phi_r is d x r row-major, orthonormal columns."""
    phi_r: np.ndarray
    eigenvalues: np.ndarray = field(default_factory=lambda: np.zeros(0))
    energy_fraction: float = 0.0

    @property
    def rank(self) -> int:
        return int(self.phi_r.shape[1])

    def dim(self) -> int:
        return int(self.phi_r.shape[0])


@dataclass
class SolveReport:
    """core/report.hpp:13-23."""
    converged: bool = False
    cycles: int = 0
    residual_history: list = field(default_factory=list)
    wall_time_s: float = 0.0

    def final_residual(self) -> float:
        return self.residual_history[-1] if self.residual_history else float("nan")


def _raise(status: int, msg: str):
    if status == L.EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


class BatchSolver:
    """One libpod2g_b200 handle: one device, one pattern, one basis, B instances."""

    def __init__(self, device: int = 0):
        self._L = L.lib()
        h = C.c_void_p()
        st = self._L.p2g_create(device, C.byref(h))
        if st != L.OK:
            raise RuntimeError(f"p2g_create(device={device}) failed: "
                               f"{self._L.p2g_status_string(st).decode()} (no CUDA device?)")
        self._h = h
        self.n = 0
        self.nnz = 0
        self.B = 0
        self.k = 0

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None):
            self._L.p2g_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, st, what=""):
        if st != L.OK:
            msg = self._L.p2g_last_error(self._h).decode()
            _raise(st, f"{what}: {msg}" if what else msg)

    # -- data
    def set_pattern(self, row_offsets, col_indices, block_size: int = 1, batch_hint: int = 0):
        """batch_hint: the number of instances the handle will be solved with (0 =
        unknown); large batches on large patterns get the wavefront colouring
        (p2g_set_batch_hint, D1)."""
        rp = np.ascontiguousarray(row_offsets, dtype=np.uint64)
        ci = np.ascontiguousarray(col_indices, dtype=np.uint64)
        n = len(rp) - 1
        self._check(self._L.p2g_set_batch_hint(self._h, int(batch_hint)), "set_batch_hint")
        self._check(self._L.p2g_set_pattern(self._h, n, rp.ctypes.data_as(L.U64),
                                            ci.ctypes.data_as(L.U64), block_size),
                    "set_pattern")
        self.n, self.nnz = n, int(rp[-1])

    def set_values(self, values):
        v = _f64(values)
        if v.ndim == 1:
            v = v[None, :]
        if v.shape[1] != self.nnz:
            raise ValueError("set_values: values must be [B][nnz]")
        self._check(self._L.p2g_set_values(self._h, v.shape[0], _d(v)), "set_values")
        self.B = v.shape[0]
        if getattr(self, "_pref_keep", None) is v:
            self._pref_keep = None  # consumed

    def prefetch_values(self, values):
        """p2g_prefetch_values: start the copy of the next batch's values; a
        later set_values with the SAME array consumes it.  Keep `values`
        alive and unchanged until then."""
        if values.dtype != np.float64 or not values.flags.c_contiguous or values.ndim != 2:
            raise ValueError("prefetch_values: C-contiguous float64 [B][nnz] required")
        self._check(self._L.p2g_prefetch_values(self._h, values.shape[0], _d(values)),
                    "prefetch_values")
        self._pref_keep = values  # the copy reads it asynchronously

    def set_values_device(self, ptr: int, batch: int):
        self._check(self._L.p2g_set_values_device(self._h, batch, C.c_void_p(ptr)),
                    "set_values_device")
        self.B = batch

    def assemble(self, mesh, E):
        """Generate the instances K(E_b) on the device (p2g_mesh_assemble_into);
        E: [B][nelem] host array.  The pattern must be mesh.pattern()."""
        E = np.ascontiguousarray(np.atleast_2d(E), dtype=np.float64)
        self._check(self._L.p2g_mesh_assemble_into(mesh._h, self._h, E.shape[0],
                                                   E.ctypes.data_as(C.c_void_p), 0), "assemble")
        self.B = E.shape[0]

    def set_basis(self, phi):
        if phi is None or (hasattr(phi, "shape") and phi.shape[1] == 0):
            self._check(self._L.p2g_set_basis(self._h, 0, None), "set_basis")
            self.k = 0
            return
        p = _f64(phi)
        if p.shape[0] != self.n:
            raise ValueError("set_basis: basis dimension mismatch")
        self._check(self._L.p2g_set_basis(self._h, p.shape[1], _d(p)), "set_basis")
        self.k = p.shape[1]

    def setup(self, smoother=L.SMOOTHER_GS_MULTICOLOR, pre_sweeps=1, post_sweeps=1,
              residual_form=L.RESIDUAL_UPPER, omega=0.5, kp_update=L.KP_RECURRENCE,
              raise_on_error=False):
        cfg = L.Config(smoother, pre_sweeps, post_sweeps, residual_form, omega, kp_update, 0)
        st_arr = np.zeros(max(self.B, 1), dtype=np.int32)
        st = self._L.p2g_setup(self._h, C.byref(cfg), st_arr.ctypes.data_as(L.I32))
        if st in (L.EINVAL, L.ECUDA, L.ESTATE) or (raise_on_error and st != L.OK):
            self._check(st, "setup")
        return st_arr[: self.B]

    # -- solve
    def initial_guess(self, b):
        b = _f64(b).reshape(self.B, self.n)
        x0 = np.empty_like(b)
        self._check(self._L.p2g_initial_guess(self._h, _d(b), _d(x0)), "initial_guess")
        return x0

    def set_surrogate(self, model):
        """The surrogate's MLP and normalisers (surrogate.SurrogateModel); its
        decoder is this handle's basis (set_basis)."""
        widths = np.ascontiguousarray(model.widths, dtype=np.int32)
        W, b = model.flat_parameters()
        norms = [_f64(a) for a in (model.input_mean, model.input_std, model.latent_mean,
                                   model.latent_std)]
        act = L.ACT_TANH if model.activation == "tanh" else L.ACT_RELU
        self._check(self._L.p2g_set_surrogate(self._h, len(widths) - 1,
                                              widths.ctypes.data_as(L.I32), act, _d(W), _d(b),
                                              *[_d(a) for a in norms]), "set_surrogate")
        self._sg_p = int(widths[0])

    def set_theta(self, theta):
        """Instance parameters [B][p] for x0_mode=X0_SURROGATE."""
        th = _f64(theta).reshape(self.B, self._sg_p)
        self._check(self._L.p2g_set_theta(self._h, _d(th)), "set_theta")

    def surrogate_predict(self, theta):
        """predict(model, theta_b) per instance (surrogate.hpp:354-357) -> [B][n]."""
        th = _f64(theta).reshape(self.B, self._sg_p)
        x = np.empty((self.B, self.n))
        self._check(self._L.p2g_surrogate_predict(self._h, _d(th), _d(x)), "surrogate_predict")
        return x

    def solve(self, b, x0=None, tol=1e-8, max_iter=100000, x0_mode=None, hist_cap=None,
              _entry="p2g_solve"):
        """Batched pcg_solve.  Returns (x[B][n], iters[B], converged[B], status[B], hist)."""
        b = _f64(b).reshape(self.B, self.n)
        if x0_mode is None:
            x0_mode = L.X0_ZERO if x0 is None else L.X0_GIVEN
        x0a = None if x0 is None else _f64(x0).reshape(self.B, self.n)
        cap = int(hist_cap if hist_cap is not None else min(max_iter, 100000) + 1)
        x = np.empty_like(b)
        it = np.zeros(self.B, dtype=np.int64)
        conv = np.zeros(self.B, dtype=np.int32)
        status = np.zeros(self.B, dtype=np.int32)
        hist = np.empty((self.B, max(cap, 1)))
        st = getattr(self._L, _entry)(self._h, _d(b), _d(x0a), x0_mode, tol, max_iter, _d(x),
                                      it.ctypes.data_as(L.I64), conv.ctypes.data_as(L.I32),
                                      status.ctypes.data_as(L.I32), _d(hist) if cap > 0 else None,
                                      cap)
        if st in (L.EINVAL, L.ECUDA, L.ESTATE):
            self._check(st, "solve")
        return x, it, conv.astype(bool), status, hist[:, :cap]

    def pod2g_solve(self, b, x0=None, tol=1e-8, max_cycles=100000, x0_mode=None, hist_cap=None):
        """Batched pod2g_solve (pod.hpp:224-256), the standalone two-grid
        iteration.  Returns (x, cycles, converged, status, hist)."""
        return self.solve(b, x0, tol, max_cycles, x0_mode, hist_cap, _entry="p2g_pod2g_solve")

    def solve_device(self, b_ptr, x_ptr, x0_ptr=None, x0_mode=L.X0_ZERO, tol=1e-8,
                     max_iter=100000, hist_cap=0):
        it = np.zeros(self.B, dtype=np.int64)
        conv = np.zeros(self.B, dtype=np.int32)
        status = np.zeros(self.B, dtype=np.int32)
        hist = np.empty((self.B, max(hist_cap, 1)))
        st = self._L.p2g_solve_device(self._h, C.c_void_p(b_ptr),
                                      C.c_void_p(x0_ptr) if x0_ptr else None, x0_mode, tol,
                                      max_iter, C.c_void_p(x_ptr), it.ctypes.data_as(L.I64),
                                      conv.ctypes.data_as(L.I32), status.ctypes.data_as(L.I32),
                                      _d(hist) if hist_cap > 0 else None, hist_cap)
        if st in (L.EINVAL, L.ECUDA, L.ESTATE):
            self._check(st, "solve_device")
        return it, conv.astype(bool), status, hist[:, :hist_cap]

    def last_solve_ms(self):
        ms = np.zeros(2)
        self._check(self._L.p2g_last_solve_ms(self._h, _d(ms)))
        return float(ms[0]), float(ms[1])

    # -- hooks
    def spmv(self, x):
        x = _f64(x).reshape(self.B, self.n)
        y = np.empty_like(x)
        self._check(self._L.p2g_spmv(self._h, _d(x), _d(y)), "spmv")
        return y

    def precond_apply(self, r):
        r = _f64(r).reshape(self.B, self.n)
        s = np.empty_like(r)
        self._check(self._L.p2g_precond_apply(self._h, _d(r), _d(s)), "precond_apply")
        return s

    def smooth(self, direction, f, u):
        f = _f64(f).reshape(self.B, self.n)
        u = _f64(u).reshape(self.B, self.n).copy()
        self._check(self._L.p2g_smooth(self._h, direction, _d(f), _d(u)), "smooth")
        return u

    def coarse_operator(self):
        Ac = np.empty((self.B, self.k, self.k))
        self._check(self._L.p2g_coarse_operator(self._h, _d(Ac)), "coarse_operator")
        return Ac

    def permutation(self):
        perm = np.empty(self.n, dtype=np.int64)
        nc = C.c_int32()
        offs = np.zeros(65, dtype=np.int64)
        self._check(self._L.p2g_get_permutation(self._h, perm.ctypes.data_as(L.I64), C.byref(nc),
                                                offs.ctypes.data_as(L.I64), 65))
        return perm, offs[: nc.value + 1]

    def profile_iteration(self, reps=5):
        ms = np.zeros(L.NUM_KCLASS)
        by = np.zeros(L.NUM_KCLASS)
        names = (C.c_char_p * L.NUM_KCLASS)()
        self._check(self._L.p2g_profile_iteration(self._h, reps, _d(ms), _d(by), names),
                    "profile_iteration")
        return {names[i].decode(): (float(ms[i]), float(by[i])) for i in range(L.NUM_KCLASS)}

    def stream(self) -> int:
        """cudaStream_t of the handle (all its kernels run there)."""
        return int(self._L.p2g_get_stream(self._h) or 0)

    def launch_counts(self):
        a, b = C.c_int64(), C.c_int64()
        self._check(self._L.p2g_launch_counts(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value


def analyze_pattern(row_offsets, col_indices, block_size=1):
    """Host-only colouring (no device): (perm new->old, colour row offsets)."""
    lib = L.lib()
    rp = np.ascontiguousarray(row_offsets, dtype=np.uint64)
    ci = np.ascontiguousarray(col_indices, dtype=np.uint64)
    n = len(rp) - 1
    perm = np.empty(n, dtype=np.int64)
    nc = C.c_int32()
    offs = np.zeros(65, dtype=np.int64)
    err = C.create_string_buffer(256)
    st = lib.p2g_analyze_pattern(n, rp.ctypes.data_as(L.U64), ci.ctypes.data_as(L.U64),
                                 block_size, perm.ctypes.data_as(L.I64), C.byref(nc),
                                 offs.ctypes.data_as(L.I64), 65, err, 256)
    if st != L.OK:
        _raise(st, err.value.decode())
    return perm, offs[: nc.value + 1]


def analyze_node_blocking(row_offsets, col_indices, block_size):
    """Host-only: (node-blocked?, most neighbour nodes of a node) -- whether
    the node-blocked kernels run for this pattern (p2g_analyze_node_blocking)."""
    lib = L.lib()
    rp = np.ascontiguousarray(row_offsets, dtype=np.uint64)
    ci = np.ascontiguousarray(col_indices, dtype=np.uint64)
    nm, bl = C.c_int32(), C.c_int32()
    st = lib.p2g_analyze_node_blocking(len(rp) - 1, rp.ctypes.data_as(L.U64),
                                       ci.ctypes.data_as(L.U64), block_size, C.byref(bl),
                                       C.byref(nm))
    if st != L.OK:
        _raise(st, "p2g_analyze_node_blocking: invalid pattern")
    return bool(bl.value), int(nm.value)


# ---------------------------------------------------------------------------
# Reference-shaped single-instance API
class Preconditioner:
    """krylov.hpp:14-19."""

    def apply(self, r):
        raise NotImplementedError

    def name(self) -> str:
        raise NotImplementedError


class Pod2gPreconditioner(Preconditioner):
    """pod.hpp:259-274 on the GPU: construction computes A_c = Phi^T K Phi and
    its factor (Pod2gOperator ctor, pod.hpp:186-189); apply is s = B r.

    Deviation (D1): the Gauss-Seidel sweeps run in node-colour order
    (block_size = dofs per node); smoother=SMOOTHER_JACOBI gives the
    reference's damped Jacobi option instead."""

    def __init__(self, K: CsrMatrix, basis: PodBasis, r1: int = 1, r2: int = 1, *,
                 block_size: int = 1, smoother: int = L.SMOOTHER_GS_MULTICOLOR,
                 omega: float = 0.5, residual_form: int = L.RESIDUAL_UPPER, device: int = 0):
        if K.nrows != K.ncols or basis.dim() != K.nrows:
            raise ValueError("Pod2gPreconditioner: dimension mismatch")
        self.K = K
        self.basis = basis
        self.solver = BatchSolver(device)
        self.solver.set_pattern(K.row_offsets, K.col_indices, block_size)
        self.solver.set_values(K.values[None, :])
        self.solver.set_basis(basis.phi_r)
        st = self.solver.setup(smoother, r1, r2, residual_form, omega)
        if st[0] == L.ESINGULAR:
            raise RuntimeError("DenseLu: matrix is singular to working precision")
        self._setup_status = int(st[0])

    def apply(self, r):
        if self._setup_status == L.EZERODIAG:
            raise RuntimeError("gauss_seidel_sweep: zero diagonal")
        return self.solver.precond_apply(np.asarray(r)[None, :])[0]

    def name(self) -> str:
        return "pod2g"


def pcg_solve(K: CsrMatrix, f, T: Pod2gPreconditioner, u0=None, delta: float = 1e-8,
              max_iter: int = 100000):
    """krylov.hpp:243-297 with T the GPU Pod2gPreconditioner; returns (u, SolveReport)."""
    f = _f64(f)
    if K.nrows != K.ncols or f.shape[0] != K.nrows:
        raise ValueError("pcg_solve: dimension mismatch")
    if u0 is not None and len(u0) == 0:
        u0 = None
    if u0 is not None and len(u0) != K.nrows:
        raise ValueError("pcg_solve: initial guess dimension mismatch")
    if not isinstance(T, Pod2gPreconditioner) or T.K is not K:
        raise ValueError("pcg_solve: the GPU path needs the Pod2gPreconditioner built on K")
    t0 = time.perf_counter()
    x, it, conv, status, hist = T.solver.solve(f[None, :], None if u0 is None else
                                               _f64(u0)[None, :], delta, max_iter)
    wall = time.perf_counter() - t0
    st = int(status[0])
    if st == L.EBREAKDOWN:
        raise RuntimeError("pcg_solve: breakdown (preconditioner or matrix not SPD)")
    if st == L.ENONFINITE:
        raise RuntimeError("pcg_solve: non-finite entries in solution")
    if st == L.ESINGULAR:
        raise RuntimeError("DenseLu: matrix is singular to working precision")
    if st == L.EZERODIAG:
        raise RuntimeError("gauss_seidel_sweep: zero diagonal")
    n_hist = int(it[0]) + 1
    rep = SolveReport(bool(conv[0]), int(it[0]), list(hist[0, :n_hist]), wall)
    return x[0], rep


def reduced_solve(K: CsrMatrix, f, basis: PodBasis, device: int = 0):
    """pod.hpp:167-179: x0 = Phi (Phi^T K Phi)^{-1} Phi^T f on the GPU."""
    s = BatchSolver(device)
    try:
        s.set_pattern(K.row_offsets, K.col_indices, 1)
        s.set_values(K.values[None, :])
        s.set_basis(basis.phi_r)
        st = s.setup()
        if st[0] == L.ESINGULAR:
            raise RuntimeError("reduced_solve: reduced operator is singular for this basis")
        return s.initial_guess(_f64(f)[None, :])[0]
    finally:
        s.close()
