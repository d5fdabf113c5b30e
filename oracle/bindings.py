"""ctypes bindings for the two CPU oracles -- TEST INFRASTRUCTURE ONLY.

* ``Oracle``    -> oracle/_build/libpod2g_oracle.so, the C restatement
                   (oracle/pod2g_oracle.c) of the reference path.
* ``Reference`` -> oracle/_ref/libpod2g_ref.so, the unmodified reference headers
                   (/root/reference/proj/include/pod2g) compiled by
                   oracle/Makefile behind oracle/ref_shim.cpp.

Both take CSR matrices with int64 indices (the reference's size_t) and
row-major n x k bases, and return numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libpod2g_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpod2g_ref.so")

_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)
_I32 = C.POINTER(C.c_int)

SMOOTHER_GS = 0
SMOOTHER_JACOBI = 1


def _d(a):
    return None if a is None else a.ctypes.data_as(_D)


def _i64(a):
    return None if a is None else a.ctypes.data_as(_I64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ix(a):
    return np.ascontiguousarray(a, dtype=np.int64)


@dataclass
class SolveResult:
    u: np.ndarray
    iters: int
    converged: bool
    history: np.ndarray
    status: int
    wall_s: float = float("nan")


class _Csr(C.Structure):
    _fields_ = [("n", C.c_int64), ("rp", _I64), ("ci", _I64), ("v", _D)]


def _surrogate_args(model, phi, theta):
    """Flatten a surrogate model (any object with the reference's fields:
    widths, activation 'tanh'/'relu', weights [W_l], biases [b_l], input_mean,
    input_std, latent_mean, latent_std) for or_/ref_surrogate_predict."""
    widths = np.ascontiguousarray(model.widths, dtype=np.int64)
    W = np.ascontiguousarray(np.concatenate([np.asarray(w, dtype=np.float64).ravel() for w in model.weights]))
    b = np.ascontiguousarray(np.concatenate([np.asarray(x, dtype=np.float64).ravel() for x in model.biases]))
    norms = [np.ascontiguousarray(a, dtype=np.float64) for a in
             (model.input_mean, model.input_std, model.latent_mean, model.latent_std)]
    phi = _f64(phi)
    theta = np.ascontiguousarray(np.atleast_2d(theta), dtype=np.float64)
    act = 0 if model.activation == "tanh" else 1
    keep = (widths, W, b, norms, phi, theta)
    args = [len(widths) - 1, _i64(widths), act, _d(W), _d(b)] + [_d(a) for a in norms] + \
        [phi.shape[0], _d(phi), theta.shape[0], _d(theta)]
    return args, keep, (theta.shape[0], phi.shape[0])


class Oracle:
    """The C restatement of krylov.hpp/pod.hpp/smoothers.hpp/csr.hpp."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle not built: {path} (run make -C oracle)")
        self.lib = L = C.CDLL(path)
        L.or_dot.restype = C.c_double
        L.or_dot.argtypes = [C.c_int64, _D, _D]
        for name in ("or_spmv",):
            getattr(L, name).argtypes = [C.POINTER(_Csr), _D, _D]
        L.or_residual.argtypes = [C.POINTER(_Csr), _D, _D, _D]
        L.or_gs_forward.argtypes = [C.POINTER(_Csr), _D, _D, C.c_int64]
        L.or_gs_backward.argtypes = [C.POINTER(_Csr), _D, _D, C.c_int64]
        L.or_jacobi_sweep.argtypes = [C.POINTER(_Csr), _D, _D, C.c_double, C.c_int64]
        L.or_project.argtypes = [C.c_int64, C.c_int64, _D, _D, _D]
        L.or_lift.argtypes = [C.c_int64, C.c_int64, _D, _D, _D]
        L.or_lu_factor.argtypes = [C.c_int64, _D, _I64]
        L.or_lu_solve.argtypes = [C.c_int64, _D, _I64, _D, _D]
        L.or_reduced_operator.argtypes = [C.POINTER(_Csr), C.c_int64, _D, _D]
        L.or_reduced_solve.argtypes = [C.POINTER(_Csr), _D, C.c_int64, _D, _D, _D]
        L.or_pcg_pod2g.argtypes = [C.POINTER(_Csr), _D, C.c_int64, _D, _D, C.c_double, C.c_int64,
                                   C.c_int, C.c_double, C.c_int64, C.c_int64, _D, _I64, _I32,
                                   _D, C.c_int64, _I64]
        L.or_pcg_pod2g_batch.argtypes = [C.c_int64, _I64, _I64, C.c_int64, _D, C.c_int64, _D,
                                         C.c_int64, _D, _D, C.c_double, C.c_int64, C.c_int,
                                         C.c_double, _D, _I64, _I32, _I32, C.c_int]
        L.or_surrogate_predict.argtypes = [C.c_int, _I64, C.c_int, _D, _D, _D, _D, _D, _D,
                                           C.c_int64, _D, C.c_int64, _D, _D]
        L.or_permute_csr.argtypes = [C.c_int64, _I64, _I64, _D, _I64, C.c_int, _I64, _I64, _D]
        L.or_pod2g_solve.argtypes = [C.POINTER(_Csr), _D, C.c_int64, _D, _D, C.c_double,
                                     C.c_int64, C.c_int64, C.c_int64, _D, _I64, _I32, _D,
                                     C.c_int64, _I64]

    @staticmethod
    def _csr(rp, ci, v):
        keep = (_ix(rp), _ix(ci), _f64(v))
        return _Csr(len(keep[0]) - 1, _i64(keep[0]), _i64(keep[1]), _d(keep[2])), keep

    def spmv(self, rp, ci, v, x):
        A, keep = self._csr(rp, ci, v)
        x = _f64(x)
        y = np.empty(A.n)
        self.lib.or_spmv(C.byref(A), _d(x), _d(y))
        return y

    def residual(self, rp, ci, v, f, u):
        A, keep = self._csr(rp, ci, v)
        f, u = _f64(f), _f64(u)
        r = np.empty(A.n)
        self.lib.or_residual(C.byref(A), _d(f), _d(u), _d(r))
        return r

    def gauss_seidel(self, rp, ci, v, f, u, sweeps=1, backward=False):
        A, keep = self._csr(rp, ci, v)
        f = _f64(f)
        u = _f64(u).copy()
        fn = self.lib.or_gs_backward if backward else self.lib.or_gs_forward
        st = fn(C.byref(A), _d(f), _d(u), sweeps)
        return u, st

    def jacobi_sweep(self, rp, ci, v, f, u, omega, sweeps=1):
        A, keep = self._csr(rp, ci, v)
        f = _f64(f)
        u = _f64(u).copy()
        st = self.lib.or_jacobi_sweep(C.byref(A), _d(f), _d(u), omega, sweeps)
        return u, st

    def project(self, phi, u):
        phi, u = _f64(phi), _f64(u)
        n, k = phi.shape
        z = np.empty(k)
        self.lib.or_project(n, k, _d(phi), _d(u), _d(z))
        return z

    def lift(self, phi, z):
        phi, z = _f64(phi), _f64(z)
        n, k = phi.shape
        u = np.empty(n)
        self.lib.or_lift(n, k, _d(phi), _d(z), _d(u))
        return u

    def surrogate_predict(self, model, phi, theta):
        """predict (surrogate.hpp:354-357) for each row of theta -> [B][n]."""
        args, keep, (B, n) = _surrogate_args(model, phi, theta)
        x = np.empty((B, n))
        if self.lib.or_surrogate_predict(*args, _d(x)) != 0:
            raise ValueError("or_surrogate_predict: bad model")
        return x

    def dense_solve(self, A, b):
        A = _f64(A).copy()
        k = A.shape[0]
        perm = np.empty(k, dtype=np.int64)
        st = self.lib.or_lu_factor(k, _d(A), _i64(perm))
        if st != 0:
            return None, st
        x = np.empty(k)
        self.lib.or_lu_solve(k, _d(A), _i64(perm), _d(_f64(b)), _d(x))
        return x, 0

    def reduced_operator(self, rp, ci, v, phi):
        A, keep = self._csr(rp, ci, v)
        phi = _f64(phi)
        k = phi.shape[1]
        Ac = np.empty((k, k))
        self.lib.or_reduced_operator(C.byref(A), k, _d(phi), _d(Ac))
        return Ac

    def reduced_solve(self, rp, ci, v, f, phi):
        A, keep = self._csr(rp, ci, v)
        phi, f = _f64(phi), _f64(f)
        k = phi.shape[1]
        x0 = np.empty(A.n)
        ur = np.empty(k)
        st = self.lib.or_reduced_solve(C.byref(A), _d(f), k, _d(phi), _d(x0), _d(ur))
        return x0, ur, st

    def pcg_pod2g(self, rp, ci, v, f, phi, u0=None, delta=1e-8, max_iter=100000,
                  smoother=SMOOTHER_GS, omega=2.0 / 3.0, r1=1, r2=1, hist_cap=None):
        A, keep = self._csr(rp, ci, v)
        f = _f64(f)
        if phi is None:
            k, phi_a = 0, np.zeros((1, 1))
        else:
            phi_a = _f64(phi)
            k = phi_a.shape[1]
        u0a = None if u0 is None else _f64(u0)
        u = np.empty(A.n)
        it = C.c_int64()
        conv = C.c_int()
        cap = int(hist_cap if hist_cap is not None else min(max_iter, 200000) + 1)
        hist = np.empty(cap)
        hl = C.c_int64()
        st = self.lib.or_pcg_pod2g(C.byref(A), _d(f), k, _d(phi_a), _d(u0a), delta, max_iter,
                                   smoother, omega, r1, r2, _d(u), C.byref(it), C.byref(conv),
                                   _d(hist), cap, C.byref(hl))
        return SolveResult(u, it.value, bool(conv.value), hist[: min(hl.value, cap)].copy(), st)

    def pod2g_solve(self, rp, ci, v, f, phi, u0=None, delta=1e-8, max_cycles=100000, r1=1, r2=1,
                    hist_cap=None):
        """pod2g_solve (pod.hpp:224-256)."""
        A, keep = self._csr(rp, ci, v)
        f, phi_a = _f64(f), _f64(phi)
        u0a = None if u0 is None else _f64(u0)
        u = np.empty(A.n)
        it = C.c_int64()
        conv = C.c_int()
        cap = int(hist_cap if hist_cap is not None else min(max_cycles, 200000) + 1)
        hist = np.empty(cap)
        hl = C.c_int64()
        st = self.lib.or_pod2g_solve(C.byref(A), _d(f), phi_a.shape[1], _d(phi_a), _d(u0a), delta,
                                     max_cycles, r1, r2, _d(u), C.byref(it), C.byref(conv),
                                     _d(hist), cap, C.byref(hl))
        return SolveResult(u, it.value, bool(conv.value), hist[: min(hl.value, cap)].copy(), st)

    def pcg_pod2g_batch(self, rp, ci, values, f, phi, u0=None, delta=1e-8, max_iter=100000,
                        smoother=SMOOTHER_GS, omega=2.0 / 3.0, nthreads=1):
        rp, ci = _ix(rp), _ix(ci)
        values = _f64(values)
        B, nnz = values.shape
        n = len(rp) - 1
        f = _f64(f)
        phi = _f64(phi)
        k = phi.shape[1]
        u0a = None if u0 is None else _f64(u0)
        u = np.empty((B, n))
        it = np.empty(B, dtype=np.int64)
        conv = np.empty(B, dtype=np.int32)
        status = np.empty(B, dtype=np.int32)
        self.lib.or_pcg_pod2g_batch(n, _i64(rp), _i64(ci), nnz, _d(values), B, _d(f), k, _d(phi),
                                    _d(u0a), delta, max_iter, smoother, omega, _d(u), _i64(it),
                                    conv.ctypes.data_as(_I32), status.ctypes.data_as(_I32),
                                    nthreads)
        return u, it, conv, status


def permute_csr_fast(rp, ci, v, perm, threads=None):
    """P K P^T as tests/helpers.permute_csr (new row i = old row perm[i],
    columns sorted ascending, explicit zeros kept), in C with threads: for the
    full-size systems.  rp / ci may be uint64 (viewed as int64, no copy)."""
    def as_i64(a):
        a = np.ascontiguousarray(a)
        return a.view(np.int64) if a.dtype == np.uint64 else np.ascontiguousarray(a, dtype=np.int64)
    rp, ci, perm = as_i64(rp), as_i64(ci), as_i64(perm)
    v = _f64(v)
    n = len(rp) - 1
    nrp = np.empty(n + 1, dtype=np.int64)
    nci = np.empty(len(ci), dtype=np.int64)
    nv = np.empty(len(v))
    L = Oracle().lib
    st = L.or_permute_csr(n, _i64(rp), _i64(ci), _d(v), _i64(perm),
                          int(threads or os.cpu_count() or 1), _i64(nrp), _i64(nci), _d(nv))
    if st != 0:
        raise ValueError("or_permute_csr: invalid permutation or arguments")
    return nrp, nci, nv


class Reference:
    """The unmodified reference, compiled from /root/reference (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"reference not built: {path} (run make -C oracle ref)")
        self.lib = L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_spmv.argtypes = [C.c_int64, _I64, _I64, _D, _D, _D]
        L.ref_residual.argtypes = [C.c_int64, _I64, _I64, _D, _D, _D, _D]
        L.ref_gauss_seidel.argtypes = [C.c_int64, _I64, _I64, _D, _D, _D, C.c_int64, C.c_int]
        L.ref_jacobi_sweep.argtypes = [C.c_int64, _I64, _I64, _D, _D, _D, C.c_double, C.c_int64]
        L.ref_reduced_operator.argtypes = [C.c_int64, _I64, _I64, _D, C.c_int64, _D, _D]
        L.ref_reduced_solve.argtypes = [C.c_int64, _I64, _I64, _D, _D, C.c_int64, _D, _D, _D]
        L.ref_dense_solve.argtypes = [C.c_int64, _D, _D, _D]
        L.ref_pod2g_apply.argtypes = [C.c_int64, _I64, _I64, _D, C.c_int64, _D, C.c_int,
                                      C.c_double, _D, _D]
        L.ref_pcg_pod2g.argtypes = [C.c_int64, _I64, _I64, _D, _D, C.c_int64, _D, _D, C.c_double,
                                    C.c_int64, C.c_int, C.c_double, _D, _I64, _I32, _D,
                                    C.c_int64, _I64, _D]
        L.ref_cg_solve.argtypes = [C.c_int64, _I64, _I64, _D, _D, C.c_double, C.c_int64, _D,
                                   _I64, _I32, _D, C.c_int64, _I64]
        L.ref_pcg_pod2g_batch.argtypes = [C.c_int64, _I64, _I64, C.c_int64, _D, C.c_int64, _D,
                                          C.c_int64, _D, C.c_int, C.c_double, C.c_int64, _D,
                                          _I64, _I32, _I32, C.c_int]
        L.ref_offline_basis.argtypes = [C.c_int64, _I64, _I64, C.c_int64, _D, C.c_int64, _D,
                                         C.c_double, C.c_int64, C.c_int, _D, _I64]
        L.ref_offline_basis_pod2g.argtypes = [C.c_int64, _I64, _I64, C.c_int64, _D, C.c_int64, _D,
                                              C.c_double, C.c_int64, C.c_int, C.c_int64, _D, _D,
                                              _I64]
        L.ref_pcg_pod2g_batch_timed.argtypes = [C.c_int64, _I64, _I64, C.c_int64, _D, C.c_int64,
                                                _D, C.c_int64, _D, C.c_double, C.c_int64, _I64,
                                                _I32, _D, _D, C.c_int]
        L.ref_compute_pod.argtypes = [C.c_int64, C.c_int64, _D, C.c_double, C.c_int64, _D,
                                      _I64, _D, _D]
        L.ref_its_case.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_uint64, C.c_int64,
                                   C.c_int64, _I64, _I64, _I64, _I64, _I64, _D, _D, _D,
                                   C.c_int64]
        L.ref_surrogate_predict.argtypes = [C.c_int, _I64, C.c_int, _D, _D, _D, _D, _D, _D,
                                            C.c_int64, _D, C.c_int64, _D, _D]
        L.ref_save_surrogate.argtypes = [C.c_char_p, C.c_int, _I64, C.c_int, _D, _D, _D, _D,
                                         _D, _D, C.c_int64, _D]
        L.ref_load_predict.argtypes = [C.c_char_p, C.c_int64, _D, _D]
        L.ref_pod2g_solve.argtypes = [C.c_int64, _I64, _I64, _D, _D, C.c_int64, _D, _D,
                                      C.c_double, C.c_int64, _D, _I64, _I32, _D, C.c_int64,
                                      _I64, _D]

    def _check(self, st):
        if st != 0:
            msg = self.lib.ref_last_error().decode()
            raise (ValueError if st == 1 else RuntimeError)(msg)

    def surrogate_predict(self, model, phi, theta):
        """pod2g::predict (surrogate.hpp:354-357) for each row of theta."""
        args, keep, (B, n) = _surrogate_args(model, phi, theta)
        x = np.empty((B, n))
        self._check(self.lib.ref_surrogate_predict(*args, _d(x)))
        return x

    def save_surrogate(self, directory, model, phi):
        """pod2g::save_surrogate_model of `model` with basis `phi`."""
        args, keep, _ = _surrogate_args(model, phi, np.zeros((1, len(model.input_mean))))
        self._check(self.lib.ref_save_surrogate(str(directory).encode(), *args[:9],
                                                args[9], args[10]))

    def load_predict(self, directory, theta):
        """pod2g::load_surrogate_model(directory) then predict per theta row."""
        theta = np.ascontiguousarray(np.atleast_2d(theta), dtype=np.float64)
        with open(os.path.join(directory, "basis.json")) as fh:
            import json
            n = int(json.load(fh)["dim"])
        x = np.empty((theta.shape[0], n))
        self._check(self.lib.ref_load_predict(str(directory).encode(), theta.shape[0], _d(theta),
                                              _d(x)))
        return x

    def spmv(self, rp, ci, v, x):
        rp, ci, v, x = _ix(rp), _ix(ci), _f64(v), _f64(x)
        y = np.empty(len(rp) - 1)
        self._check(self.lib.ref_spmv(len(rp) - 1, _i64(rp), _i64(ci), _d(v), _d(x), _d(y)))
        return y

    def residual(self, rp, ci, v, f, u):
        rp, ci, v, f, u = _ix(rp), _ix(ci), _f64(v), _f64(f), _f64(u)
        r = np.empty(len(rp) - 1)
        self._check(self.lib.ref_residual(len(rp) - 1, _i64(rp), _i64(ci), _d(v), _d(f), _d(u),
                                          _d(r)))
        return r

    def gauss_seidel(self, rp, ci, v, f, u, sweeps=1, backward=False):
        rp, ci, v, f = _ix(rp), _ix(ci), _f64(v), _f64(f)
        u = _f64(u).copy()
        self._check(self.lib.ref_gauss_seidel(len(rp) - 1, _i64(rp), _i64(ci), _d(v), _d(f),
                                              _d(u), sweeps, 1 if backward else 0))
        return u

    def jacobi_sweep(self, rp, ci, v, f, u, omega, sweeps=1):
        rp, ci, v, f = _ix(rp), _ix(ci), _f64(v), _f64(f)
        u = _f64(u).copy()
        self._check(self.lib.ref_jacobi_sweep(len(rp) - 1, _i64(rp), _i64(ci), _d(v), _d(f),
                                              _d(u), omega, sweeps))
        return u

    def reduced_operator(self, rp, ci, v, phi):
        rp, ci, v, phi = _ix(rp), _ix(ci), _f64(v), _f64(phi)
        k = phi.shape[1]
        Ac = np.empty((k, k))
        self._check(self.lib.ref_reduced_operator(len(rp) - 1, _i64(rp), _i64(ci), _d(v), k,
                                                  _d(phi), _d(Ac)))
        return Ac

    def reduced_solve(self, rp, ci, v, f, phi):
        rp, ci, v, f, phi = _ix(rp), _ix(ci), _f64(v), _f64(f), _f64(phi)
        k = phi.shape[1]
        x0 = np.empty(len(rp) - 1)
        ur = np.empty(k)
        self._check(self.lib.ref_reduced_solve(len(rp) - 1, _i64(rp), _i64(ci), _d(v), _d(f), k,
                                               _d(phi), _d(x0), _d(ur)))
        return x0, ur

    def dense_solve(self, A, b):
        A, b = _f64(A), _f64(b)
        x = np.empty(A.shape[0])
        self._check(self.lib.ref_dense_solve(A.shape[0], _d(A), _d(b), _d(x)))
        return x

    def pod2g_apply(self, rp, ci, v, phi, r, smoother=SMOOTHER_GS, omega=2.0 / 3.0):
        rp, ci, v, phi, r = _ix(rp), _ix(ci), _f64(v), _f64(phi), _f64(r)
        s = np.empty(len(rp) - 1)
        self._check(self.lib.ref_pod2g_apply(len(rp) - 1, _i64(rp), _i64(ci), _d(v),
                                             phi.shape[1], _d(phi), smoother, omega, _d(r),
                                             _d(s)))
        return s

    def pod2g_solve(self, rp, ci, v, f, phi, u0=None, delta=1e-8, max_cycles=100000,
                    hist_cap=None):
        """pod2g::pod2g_solve (pod.hpp:224-256), r1 = r2 = 1."""
        rp, ci, v, f, phi = _ix(rp), _ix(ci), _f64(v), _f64(f), _f64(phi)
        n = len(rp) - 1
        u0a = None if u0 is None else _f64(u0)
        u = np.empty(n)
        it = C.c_int64()
        conv = C.c_int()
        cap = int(hist_cap if hist_cap is not None else min(max_cycles, 200000) + 1)
        hist = np.empty(cap)
        hl = C.c_int64()
        wall = C.c_double()
        st = self.lib.ref_pod2g_solve(n, _i64(rp), _i64(ci), _d(v), _d(f), phi.shape[1], _d(phi),
                                      _d(u0a), delta, max_cycles, _d(u), C.byref(it),
                                      C.byref(conv), _d(hist), cap, C.byref(hl), C.byref(wall))
        if st != 0:
            return SolveResult(u, 0, False, np.empty(0), st)
        return SolveResult(u, it.value, bool(conv.value), hist[: min(hl.value, cap)].copy(), 0,
                           wall.value)

    def pcg_pod2g(self, rp, ci, v, f, phi, u0=None, delta=1e-8, max_iter=100000,
                  smoother=SMOOTHER_GS, omega=2.0 / 3.0, hist_cap=None):
        rp, ci, v, f = _ix(rp), _ix(ci), _f64(v), _f64(f)
        n = len(rp) - 1
        if phi is None:
            k, phi_a = 0, np.zeros((1, 1))
        else:
            phi_a = _f64(phi)
            k = phi_a.shape[1]
        u0a = None if u0 is None else _f64(u0)
        u = np.empty(n)
        it = C.c_int64()
        conv = C.c_int()
        cap = int(hist_cap if hist_cap is not None else min(max_iter, 200000) + 1)
        hist = np.empty(cap)
        hl = C.c_int64()
        wall = C.c_double()
        st = self.lib.ref_pcg_pod2g(n, _i64(rp), _i64(ci), _d(v), _d(f), k, _d(phi_a), _d(u0a),
                                    delta, max_iter, smoother, omega, _d(u), C.byref(it),
                                    C.byref(conv), _d(hist), cap, C.byref(hl), C.byref(wall))
        if st != 0:
            return SolveResult(u, 0, False, np.empty(0), st)
        return SolveResult(u, it.value, bool(conv.value), hist[: min(hl.value, cap)].copy(), 0,
                           wall.value)

    def cg_solve(self, rp, ci, v, f, delta=1e-8, max_iter=100000):
        rp, ci, v, f = _ix(rp), _ix(ci), _f64(v), _f64(f)
        n = len(rp) - 1
        u = np.empty(n)
        it = C.c_int64()
        conv = C.c_int()
        cap = max_iter + 1
        hist = np.empty(cap)
        hl = C.c_int64()
        self._check(self.lib.ref_cg_solve(n, _i64(rp), _i64(ci), _d(v), _d(f), delta, max_iter,
                                          _d(u), C.byref(it), C.byref(conv), _d(hist), cap,
                                          C.byref(hl)))
        return SolveResult(u, it.value, bool(conv.value), hist[: min(hl.value, cap)].copy(), 0)

    def pcg_pod2g_batch(self, rp, ci, values, f, phi, x0_mode=1, delta=1e-8, max_iter=100000,
                        jobs=1):
        rp, ci = _ix(rp), _ix(ci)
        values, f, phi = _f64(values), _f64(f), _f64(phi)
        B, nnz = values.shape
        n = len(rp) - 1
        u = np.empty((B, n))
        it = np.empty(B, dtype=np.int64)
        conv = np.empty(B, dtype=np.int32)
        failed = np.empty(B, dtype=np.int32)
        self._check(self.lib.ref_pcg_pod2g_batch(
            n, _i64(rp), _i64(ci), nnz, _d(values), B, _d(f), phi.shape[1], _d(phi), x0_mode,
            delta, max_iter, _d(u), _i64(it), conv.ctypes.data_as(_I32),
            failed.ctypes.data_as(_I32), jobs))
        return u, it, conv, failed

    def pcg_pod2g_batch_timed(self, rp, ci, values, f, phi, delta, max_iter, jobs=1):
        """Per instance: (iterations, setup seconds, PCG loop seconds), x0 = reduced_solve."""
        rp, ci = _ix(rp), _ix(ci)
        values, f, phi = _f64(values), _f64(f), _f64(phi)
        B, nnz = values.shape
        n = len(rp) - 1
        it = np.empty(B, dtype=np.int64)
        failed = np.empty(B, dtype=np.int32)
        su, lo = np.empty(B), np.empty(B)
        self._check(self.lib.ref_pcg_pod2g_batch_timed(
            n, _i64(rp), _i64(ci), nnz, _d(values), B, _d(f), phi.shape[1], _d(phi), delta,
            max_iter, _i64(it), failed.ctypes.data_as(_I32), _d(su), _d(lo), jobs))
        if np.any(failed):
            raise RuntimeError("reference pcg_solve failed on an instance")
        return it, su, lo

    def offline_basis(self, rp, ci, values, F, rank, tol=1e-10, jobs=1):
        """Snapshots (Jacobi-PCG ladder) + compute_pod(RankTarget{rank})."""
        rp, ci, values, F = _ix(rp), _ix(ci), _f64(values), _f64(F)
        N, nnz = values.shape
        n = len(rp) - 1
        phi = np.empty((n, rank))
        r = C.c_int64()
        self._check(self.lib.ref_offline_basis(n, _i64(rp), _i64(ci), nnz, _d(values), N, _d(F),
                                               tol, rank, jobs, _d(phi), C.byref(r)))
        return np.ascontiguousarray(phi[:, : r.value])

    def compute_pod(self, snapshots, rank=None, energy=None):
        """pod2g::compute_pod (pod.hpp:73-148), RankTarget{rank} or EnergyTarget{energy}.
        Returns (phi [d][r], Gram eigenvalues, energy fraction)."""
        U = _f64(snapshots)
        N, d = U.shape
        target = float(rank) if energy is None else -float(energy)
        phi = np.empty((d, N))
        eig = np.empty(N)
        r, en = C.c_int64(), C.c_double()
        self._check(self.lib.ref_compute_pod(N, d, _d(U), target, N, _d(phi), C.byref(r),
                                             _d(eig), C.byref(en)))
        return np.ascontiguousarray(phi.reshape(-1)[: d * r.value].reshape(d, r.value)), eig, \
            en.value

    def offline_basis_pod2g(self, rp, ci, values, F, rank, phi0, tol=1e-10, jobs=1):
        """Snapshots (pcg_solve + Pod2gPreconditioner over bootstrap basis phi0,
        generate_snapshots' tolerance ladder) + compute_pod(RankTarget{rank})."""
        rp, ci, values, F, phi0 = _ix(rp), _ix(ci), _f64(values), _f64(F), _f64(phi0)
        N, nnz = values.shape
        n = len(rp) - 1
        phi = np.empty((n, rank))
        r = C.c_int64()
        self._check(self.lib.ref_offline_basis_pod2g(n, _i64(rp), _i64(ci), nnz, _d(values), N,
                                                     _d(F), tol, rank, jobs, phi0.shape[1],
                                                     _d(phi0), _d(phi), C.byref(r)))
        return np.ascontiguousarray(phi[:, : r.value])

    def its_case(self, res=32, n_snapshots=100, offline_seed=42, bench_seed=7, inst=0, jobs=8):
        n, nnz, rank = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(self.lib.ref_its_case(res, n_snapshots, offline_seed, bench_seed, inst, jobs,
                                          C.byref(n), C.byref(nnz), C.byref(rank), None, None,
                                          None, None, None, 0))
        rp = np.empty(n.value + 1, dtype=np.int64)
        ci = np.empty(nnz.value, dtype=np.int64)
        v = np.empty(nnz.value)
        f = np.empty(n.value)
        phi = np.empty((n.value, rank.value))
        self._check(self.lib.ref_its_case(res, n_snapshots, offline_seed, bench_seed, inst, jobs,
                                          C.byref(n), C.byref(nnz), C.byref(rank), _i64(rp),
                                          _i64(ci), _d(v), _d(f), _d(phi), phi.size))
        return rp, ci, v, f, phi
