"""ctypes mirror of include/propgate_b200.h and the in-tree library loader.

The structs here are byte-for-byte the C structs of the drop-in boundary
(include/propgate_b200.h).  The product library ``libpropgate_b200.so`` is
built in-tree by ``__graft_entry__.build()``; loading fails loudly when it is
missing -- there is no CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
LIB_PATH = os.path.join(PKG_DIR, "libpropgate_b200.so")

PG_OK, PG_EINVAL, PG_ENOMEM, PG_ECUDA, PG_ENCCL, PG_ENODEV, PG_ERANGE = 0, -1, -2, -3, -4, -5, -6
PG_EPARSE = -7
PG_CONVERGED, PG_ROUNDLIMIT, PG_INFEASIBLE = 0, 1, 2
PG_MULTI_ROWS = 0
PG_WIDE64, PG_NARROW32 = 0, 1
PG_LOOP_GRAPH, PG_LOOP_HOST = 0, 1
PG_FLAG_ROWCHECK, PG_FLAG_WORKLIST, PG_FLAG_DELTA_EXCHANGE = 0x1, 0x2, 0x4

STATUS_NAMES = {PG_CONVERGED: "Converged", PG_ROUNDLIMIT: "RoundLimit", PG_INFEASIBLE: "Infeasible"}

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)
_up = C.POINTER(C.c_uint8)


class PgProblem(C.Structure):
    _fields_ = [
        ("num_rows", C.c_int32),
        ("num_cols", C.c_int32),
        ("nnz", C.c_int64),
        ("row_ptr", _ip),
        ("col_idx", _ip),
        ("values", _dp),
        ("lhs", _dp),
        ("rhs", _dp),
        ("lower", _dp),
        ("upper", _dp),
        ("integral", _up),
    ]


class PgConfig(C.Structure):
    _fields_ = [
        ("round_limit", C.c_int32),
        ("infinity_threshold", C.c_double),
        ("improvement_abs", C.c_double),
        ("improvement_rel", C.c_double),
        ("integrality_eps", C.c_double),
        ("nnz_budget", C.c_int32),
        ("vector_threshold", C.c_int32),
        ("worker_count", C.c_int32),
        ("scalar_mode", C.c_int32),
        ("device", C.c_int32),
        ("loop_mode", C.c_int32),
        ("flags", C.c_uint32),
    ]


class PgResult(C.Structure):
    _fields_ = [
        ("lower", _dp),
        ("upper", _dp),
        ("per_round_changes", _lp),
        ("per_round_capacity", C.c_int32),
        ("status", C.c_int32),
        ("rounds_executed", C.c_int32),
        ("_pad", C.c_int32),
        ("total_bound_changes", C.c_int64),
        ("constraints_processed", C.c_int64),
        ("elapsed_ns", C.c_int64),
    ]


def ptr(a: np.ndarray | None, ctype):
    if a is None:
        return C.cast(None, C.POINTER(ctype))
    assert a.flags["C_CONTIGUOUS"], "arrays crossing the C-ABI must be contiguous"
    return a.ctypes.data_as(C.POINTER(ctype))


def default_config() -> PgConfig:
    """Reference EngineConfig defaults (model.hpp:131-140) + GPU defaults."""
    c = PgConfig()
    c.round_limit = 100
    c.infinity_threshold = 1e20
    c.improvement_abs = 1e-7
    c.improvement_rel = 1e-7
    c.integrality_eps = 1e-6
    c.nnz_budget = 1024
    c.vector_threshold = 64
    c.worker_count = 0
    c.scalar_mode = PG_WIDE64
    c.device = 0
    c.loop_mode = PG_LOOP_GRAPH
    c.flags = PG_FLAG_ROWCHECK
    return c


# header prototypes: name -> (restype, argtypes)
PROTOTYPES = {
    "pg_config_default": (None, [C.POINTER(PgConfig)]),
    "pg_config_validate": (C.c_int, [C.POINTER(PgConfig)]),
    "pg_propagate": (C.c_int, [C.POINTER(PgProblem), C.POINTER(PgConfig), C.POINTER(PgResult)]),
    "pg_round": (C.c_int, [C.POINTER(PgProblem), C.POINTER(PgConfig), _dp, _dp, _dp, _dp, _ip, _ip, _lp]),
    "pg_partition_row_blocks": (C.c_int, [C.POINTER(PgProblem), C.POINTER(PgConfig), _ip, _ip, _ip]),
    "pg_session_create": (C.c_int, [C.POINTER(PgProblem), C.POINTER(PgConfig), C.POINTER(C.c_void_p)]),
    "pg_session_destroy": (None, [C.c_void_p]),
    "pg_session_propagate": (C.c_int, [C.c_void_p, _dp, _dp, C.POINTER(PgResult)]),
    "pg_session_round": (C.c_int, [C.c_void_p, _dp, _dp, _dp, _dp, _ip, _ip, _lp]),
    "pg_session_run": (C.c_int, [C.c_void_p, C.POINTER(PgResult)]),
    "pg_session_propagate_batch": (C.c_int, [C.c_void_p, C.c_int32, _dp, _dp, _dp, _dp, _ip, _ip]),
    "pg_session_time_round_kernel": (C.c_int, [C.c_void_p, C.c_int32, _dp, _dp]),
    "pg_session_info": (C.c_int, [C.c_void_p, _lp, C.c_int32]),
    "pg_session_set_root": (C.c_int, [C.c_void_p, C.POINTER(PgResult)]),
    "pg_session_propagate_nodes": (C.c_int, [C.c_void_p, C.c_int32, _ip, _ip, _dp, _dp, _ip, _ip,
                                             _dp, _dp, _lp]),
    "pg_nccl_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "pg_session_attach_comm": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8), C.c_int32, C.c_int32]),
    "pg_multi_propagate": (C.c_int, [C.POINTER(PgProblem), C.POINTER(PgConfig), C.c_int32, C.c_int32,
                                     C.POINTER(PgResult)]),
    "pg_csr_from_triplets": (C.c_int, [C.c_int32, C.c_int32, C.c_int64, _ip, _ip, _dp, C.c_int32,
                                       _ip, _ip, _dp, _lp]),
    "pg_mps_read": (C.c_int, [C.c_char_p, C.c_double, C.c_int32, C.POINTER(C.c_void_p)]),
    "pg_mps_read_buffer": (C.c_int, [C.c_char_p, C.c_int64, C.c_double, C.c_int32,
                                     C.POINTER(C.c_void_p)]),
    "pg_mps_dims": (C.c_int, [C.c_void_p, _ip, _ip, _lp]),
    "pg_mps_name": (C.c_char_p, [C.c_void_p]),
    "pg_mps_arrays": (C.c_int, [C.c_void_p] + [C.POINTER(_ip)] * 2 + [C.POINTER(_dp)] * 5 +
                      [C.POINTER(_up)]),
    "pg_mps_to_csr": (C.c_int, [C.c_void_p, C.c_int32, _ip, _ip, _dp, _lp]),
    "pg_mps_free": (None, [C.c_void_p]),
    "pg_last_error": (C.c_char_p, []),
    "pg_abi_version": (C.c_int32, []),
}


class EngineError(RuntimeError):
    pass


_lib = None


def load_library(path: str | None = None):
    """Load the product library; raises if it is absent (no fallback).
    PG_LIB overrides the path (build variants for experiments)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("PG_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise EngineError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 engine has no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class MpsError(RuntimeError):
    """propgate::MpsError (core/include/propgate/mps.hpp:12-23) / the
    reference's std::runtime_error for unreadable files."""


def check(rc: int, what: str):
    if rc != PG_OK:
        msg = load_library().pg_last_error()
        msg = msg.decode() if msg else ""
        if rc == PG_EINVAL:
            raise ValueError(f"{what}: {msg}")
        if rc == PG_ERANGE:  # std::out_of_range in the reference
            raise IndexError(f"{what}: {msg}")
        if rc == PG_EPARSE:  # MpsError / std::runtime_error in the reference
            raise MpsError(msg)
        raise EngineError(f"{what} failed ({rc}): {msg}")
