"""ctypes binding of libpod2g_b200.so (include/pod2g_b200.h, include/pod2g_gen.h).

The library is built in-tree by ``make -C paper_2207_02543_b200/csrc`` (or
``__graft_entry__.build()``).  There is no fallback: if it is missing, every
entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpod2g_b200.so")
GEN_PATH = os.path.join(HERE, "libpod2g_gen.so")

D = C.POINTER(C.c_double)
I64 = C.POINTER(C.c_int64)
U64 = C.POINTER(C.c_uint64)
I32 = C.POINTER(C.c_int32)
H = C.c_void_p

# (name, restype, argtypes) for every exported symbol of include/*.h
SIGNATURES = [
    # pod2g_b200.h
    ("p2g_config_default", None, [C.c_void_p]),
    ("p2g_abi_version", C.c_int, []),
    ("p2g_status_string", C.c_char_p, [C.c_int]),
    ("p2g_create", C.c_int, [C.c_int, C.POINTER(H)]),
    ("p2g_destroy", C.c_int, [H]),
    ("p2g_last_error", C.c_char_p, [H]),
    ("p2g_set_pattern", C.c_int, [H, C.c_int64, U64, U64, C.c_int32]),
    ("p2g_set_values", C.c_int, [H, C.c_int32, D]),
    ("p2g_set_values_device", C.c_int, [H, C.c_int32, C.c_void_p]),
    ("p2g_prefetch_values", C.c_int, [H, C.c_int32, D]),
    ("p2g_set_basis", C.c_int, [H, C.c_int32, D]),
    ("p2g_setup", C.c_int, [H, C.c_void_p, I32]),
    ("p2g_initial_guess", C.c_int, [H, D, D]),
    ("p2g_pod2g_solve", C.c_int, [H, D, D, C.c_int32, C.c_double, C.c_int64, D, I64, I32, I32, D,
                                  C.c_int64]),
    ("p2g_set_surrogate", C.c_int, [H, C.c_int32, I32, C.c_int32, D, D, D, D, D, D]),
    ("p2g_set_theta", C.c_int, [H, D]),
    ("p2g_fnv1a64", C.c_uint64, [C.c_char_p, C.c_int64]),
    ("p2g_gram", C.c_int, [C.c_int32, C.c_int64, C.c_int64, C.c_void_p, C.c_int32, D]),
    ("p2g_combine", C.c_int, [C.c_int32, C.c_int64, C.c_int64, C.c_void_p, C.c_int32, C.c_int64,
                              D, C.c_void_p]),
    ("p2g_surrogate_predict", C.c_int, [H, D, D]),
    ("p2g_solve", C.c_int, [H, D, D, C.c_int32, C.c_double, C.c_int64, D, I64, I32, I32, D,
                            C.c_int64]),
    ("p2g_solve_device", C.c_int, [H, C.c_void_p, C.c_void_p, C.c_int32, C.c_double, C.c_int64,
                                   C.c_void_p, I64, I32, I32, D, C.c_int64]),
    ("p2g_last_solve_ms", C.c_int, [H, D]),
    ("p2g_spmv", C.c_int, [H, D, D]),
    ("p2g_precond_apply", C.c_int, [H, D, D]),
    ("p2g_smooth", C.c_int, [H, C.c_int32, D, D]),
    ("p2g_coarse_operator", C.c_int, [H, D]),
    ("p2g_get_permutation", C.c_int, [H, I64, I32, I64, C.c_int32]),
    ("p2g_set_batch_hint", C.c_int, [H, C.c_int64]),
    ("p2g_analyze_node_blocking", C.c_int, [C.c_int64, U64, U64, C.c_int32, I32, I32]),
    ("p2g_analyze_pattern", C.c_int, [C.c_int64, U64, U64, C.c_int32, I64, I32, I64, C.c_int32,
                                      C.c_char_p, C.c_int32]),
    ("p2g_profile_iteration", C.c_int, [H, C.c_int32, D, D, C.POINTER(C.c_char_p)]),
    ("p2g_launch_counts", C.c_int, [H, I64, I64]),
    ("p2g_get_stream", C.c_void_p, [H]),
    ("p2g_debug_guard_check", C.c_int, []),
    ("p2g_nccl_unique_id", C.c_int, [C.c_void_p]),
    ("p2g_part_create_local", C.c_int, [C.c_int, C.c_int, C.POINTER(H)]),
    ("p2g_part_create_nccl", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(H)]),
    ("p2g_part_destroy", C.c_int, [H]),
    ("p2g_part_last_error", C.c_char_p, [H]),
    ("p2g_part_set_pattern", C.c_int, [H, C.c_int, C.c_int64, I64, U64, U64, C.c_int32, I32]),
    ("p2g_part_ghosts", C.c_int, [H, C.c_int, I64, I64, I64]),
    ("p2g_part_set_values", C.c_int, [H, C.c_int, C.c_int32, D]),
    ("p2g_part_set_basis", C.c_int, [H, C.c_int, C.c_int32, D, D]),
    ("p2g_part_setup", C.c_int, [H, C.c_void_p, I32]),
    ("p2g_part_solve", C.c_int, [H, C.POINTER(D), C.POINTER(D), C.c_int32, C.c_double, C.c_int64,
                                 C.POINTER(D), I64, I32, I32, D, C.c_int64]),
    ("p2g_part_last_solve_ms", C.c_int, [H, D]),
    ("p2g_part_launch_counts", C.c_int, [H, I64, I64, I32]),
    ("p2g_part_get_stream", C.c_void_p, [H]),
    ("p2g_part_profile_iteration", C.c_int, [H, C.c_int32, D, D, C.POINTER(C.c_char_p)]),
    ("p2g_plan_partition", C.c_int, [C.c_int, C.c_int, I64, C.c_int64, U64, U64, C.c_int32, I32,
                                     I64, I64, I64, I64, C.c_char_p, C.c_int32]),
    # pod2g_gen.h, device-side assembly (in libpod2g_b200.so)
    ("p2g_mesh_assemble_into", C.c_int, [H, H, C.c_int32, C.c_void_p, C.c_int32]),
    ("p2g_part_assemble", C.c_int, [H, C.c_int, H, C.c_int32, C.c_void_p, C.c_int32]),
]

# pod2g_gen.h host generator: libpod2g_gen.so (CPU-only, no CUDA runtime)
GEN_SIGNATURES = [
    ("p2g_mesh_create", C.c_int, [C.c_int32, C.c_int64, C.c_int64, C.c_int64, C.c_double,
                                  C.c_double, C.c_double, C.c_double, C.POINTER(H)]),
    ("p2g_mesh_destroy", None, [H]),
    ("p2g_mesh_info", C.c_int, [H, I64, I64, I64, I32]),
    ("p2g_mesh_pattern", C.c_int, [H, U64, U64]),
    ("p2g_mesh_rhs", C.c_int, [H, D]),
    ("p2g_mesh_pattern_range", C.c_int, [H, C.c_int64, C.c_int64, U64, U64]),
    ("p2g_mesh_node_colors", C.c_int, [H, I32]),
    ("p2g_mesh_element_stiffness", C.c_int, [H, D]),
    ("p2g_mesh_assemble", C.c_int, [H, C.c_int64, D, D, C.c_int32]),
    ("p2g_mesh_assemble_range", C.c_int, [H, C.c_int64, D, C.c_int64, C.c_int64, D, C.c_int32]),
    ("p2g_kl_field", C.c_int, [H, C.c_int32, C.c_double, C.c_double, C.c_int32, C.c_int64, U64,
                               D, D]),
    ("p2g_kl_eigenvalues", C.c_int, [H, C.c_int32, C.c_double, C.c_int32, D]),
    ("p2g_normal_draws", C.c_int, [C.c_uint64, C.c_int64, D]),
]

_lib = None


class P2GError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{msg} (status {status})")
        self.status = status


def lib():
    """Load libpod2g_b200.so (once).  Raises if it has not been built."""
    global _lib
    if _lib is None:
        path = os.environ.get("P2G_LIB_PATH", LIB_PATH)  # tuning experiments only
        if not os.path.exists(path):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `make -C {HERE}/csrc` "
                "(there is no CPU fallback)")
        L = C.CDLL(path)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


_gen = None


def gen():
    """Load the CPU-only generator library libpod2g_gen.so (once).  It links no
    CUDA code: the reference arm of bench.py builds its inputs with it."""
    global _gen
    if _gen is None:
        if not os.path.exists(GEN_PATH):
            raise RuntimeError(f"{GEN_PATH} is missing: build it with `make -C {HERE}/csrc`")
        G = C.CDLL(GEN_PATH)
        for name, res, args in GEN_SIGNATURES:
            fn = getattr(G, name)
            fn.restype = res
            fn.argtypes = args
        _gen = G
    return _gen


class Config(C.Structure):
    """p2g_config (include/pod2g_b200.h)."""
    _fields_ = [("smoother", C.c_int32), ("pre_sweeps", C.c_int32), ("post_sweeps", C.c_int32),
                ("residual_form", C.c_int32), ("omega", C.c_double), ("kp_update", C.c_int32),
                ("reserved", C.c_int32)]


# status codes
OK, EINVAL, EBREAKDOWN, ENONFINITE, ESINGULAR, EZERODIAG, ECUDA, ENCCL, ESTATE = range(9)
SMOOTHER_GS_MULTICOLOR, SMOOTHER_JACOBI = 0, 1
RESIDUAL_FULL, RESIDUAL_UPPER = 0, 1
KP_SPMV, KP_RECURRENCE = 0, 1
X0_ZERO, X0_GIVEN, X0_REDUCED, X0_SURROGATE = 0, 1, 2, 3
ACT_TANH, ACT_RELU = 0, 1
NUM_KCLASS = 11
