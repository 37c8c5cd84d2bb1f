"""ORACLE -- test infrastructure only.

Python binding of
  * oracle/liboracle.so            the plain-C restatement (kind "port"), and
  * oracle/_ref/libpropgate_ref.so the reference compiled from its own sources
                                   (kind "reference"; present when built).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
legs may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2009_07785_b200 import abi
from paper_2009_07785_b200.model import (PropagationResult, PropagationStatus, ProblemInstance,
                                         VariableBounds, new_c_result, result_from_c)

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libpropgate_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)
_P = C.POINTER(abi.PgProblem)
_G = C.POINTER(abi.PgConfig)
_R = C.POINTER(abi.PgResult)

SEQ, PAR = 0, 1


def _bind_common(lib, prefix):
    f = getattr(lib, prefix + "propagate")
    f.argtypes = [C.c_int, _P, _G, _dp, _dp, _R]
    f.restype = C.c_int


class _Lib:
    def __init__(self, path, kind):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.kind = kind
        self.lib = C.CDLL(path)


_orc = None
_ref = None


def oracle_lib():
    global _orc
    if _orc is None:
        lib = C.CDLL(ORACLE_LIB)
        lib.orc_propagate.argtypes = [C.c_int, _P, _G, _dp, _dp, _R]
        lib.orc_propagate.restype = C.c_int
        lib.orc_round.argtypes = [_P, _G, _dp, _dp, _dp, _dp, _ip, _ip, _lp]
        lib.orc_round.restype = C.c_int
        lib.orc_round_rows.argtypes = [_P, _G, C.c_int32, C.c_int32, _dp, _dp, _dp, _dp, _ip]
        lib.orc_round_rows.restype = C.c_int
        lib.orc_commit.argtypes = [C.c_int64, _dp, _dp, _dp, _dp, C.c_double, _ip]
        lib.orc_commit.restype = C.c_int64
        lib.orc_partition_row_blocks.argtypes = [_P, _G, _ip, _ip, _ip]
        lib.orc_partition_row_blocks.restype = C.c_int
        lib.orc_validate.argtypes = [_G]
        lib.orc_validate.restype = C.c_int
        lib.orc_row_activities.argtypes = [_ip, _dp, C.c_int64, _dp, _dp, _dp]
        lib.orc_row_activities.restype = None
        lib.orc_residual.argtypes = [_dp, C.c_double, C.c_double, C.c_double, _dp]
        lib.orc_residual.restype = None
        lib.orc_candidates.argtypes = [C.c_double] * 5 + [C.c_int32, _G, _dp]
        lib.orc_candidates.restype = None
        lib.orc_classify.argtypes = [_dp, C.c_double, C.c_double, _G]
        lib.orc_classify.restype = C.c_int32
        lib.orc_tighten.argtypes = [C.c_double] * 4 + [_G, _dp]
        lib.orc_tighten.restype = C.c_int32
        lib.orc_propcore_rows.argtypes = [C.c_int32, _ip, _dp, _dp, _dp, _dp, _G, _dp, _ip, _dp, _dp,
                                          _dp, _ip]
        lib.orc_propcore_rows.restype = None
        lib.orc_csr_from_triplets.argtypes = [C.c_int32, C.c_int32, C.c_int64, _ip, _ip, _dp, _ip,
                                              _ip, _dp, _lp]
        lib.orc_csr_from_triplets.restype = C.c_int
        _orc = lib
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def ref_lib():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_LIB)
        lib.ref_propagate.argtypes = [C.c_int, _P, _G, _dp, _dp, _R]
        lib.ref_propagate.restype = C.c_int
        lib.ref_round.argtypes = [_P, _G, _dp, _dp, _dp, _dp, _ip, _ip, _lp]
        lib.ref_round.restype = C.c_int
        lib.ref_partition.argtypes = [_P, _G, _ip, _ip, _ip]
        lib.ref_partition.restype = C.c_int
        lib.ref_gen_random.argtypes = [C.c_int32, C.c_int32, C.c_uint64, C.c_double, C.c_double,
                                       C.c_double, C.c_double, C.c_int64]
        lib.ref_gen_random.restype = C.c_void_p
        lib.ref_gen_cascade.argtypes = [C.c_int32]
        lib.ref_gen_cascade.restype = C.c_void_p
        lib.ref_parse_mps.argtypes = [C.c_char_p]
        lib.ref_parse_mps.restype = C.c_void_p
        lib.ref_permute.argtypes = [C.c_void_p, C.c_uint64, _ip]
        lib.ref_permute.restype = C.c_void_p
        lib.ref_inst_view.argtypes = [C.c_void_p, _P]
        lib.ref_inst_view.restype = None
        lib.ref_inst_free.argtypes = [C.c_void_p]
        lib.ref_inst_free.restype = None
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_hardware_concurrency.restype = C.c_int
        lib.ref_row_activities.argtypes = [_ip, _dp, C.c_int64, _dp, _dp, C.c_int32, _dp]
        lib.ref_row_activities.restype = None
        lib.ref_residual.argtypes = [_dp, C.c_double, C.c_double, C.c_double, _dp]
        lib.ref_residual.restype = None
        lib.ref_candidates.argtypes = [C.c_double] * 5 + [C.c_int32, _G, _dp]
        lib.ref_candidates.restype = None
        lib.ref_classify.argtypes = [_dp, C.c_double, C.c_double, _G]
        lib.ref_classify.restype = C.c_int32
        lib.ref_tighten.argtypes = [C.c_double] * 4 + [_G, _dp]
        lib.ref_tighten.restype = C.c_int32
        lib.ref_csr_from_triplets.argtypes = [C.c_int32, C.c_int32, C.c_int64, _ip, _ip, _dp, _ip,
                                              _ip, _dp, _lp]
        lib.ref_csr_from_triplets.restype = C.c_int
        _ref = lib
    return _ref


def _cfg(cfg):
    return cfg if isinstance(cfg, abi.PgConfig) else cfg.to_c()


def _run(fn, engine, inst: ProblemInstance, cfg, lower=None, upper=None) -> PropagationResult:
    c = _cfg(cfg)
    p = inst.to_c()
    r, lo, up, prc = new_c_result(inst.num_cols(), c.round_limit)
    lo_p = abi.ptr(np.ascontiguousarray(lower, dtype=np.float64), C.c_double) if lower is not None else None
    up_p = abi.ptr(np.ascontiguousarray(upper, dtype=np.float64), C.c_double) if upper is not None else None
    rc = fn(engine, C.byref(p), C.byref(c), lo_p, up_p, C.byref(r))
    if rc == abi.PG_EINVAL:
        raise ValueError("invalid config")
    if rc != 0:
        raise RuntimeError(f"oracle failed {rc}")
    return result_from_c(r, lo, up, prc)


def propagate_sequential(inst, cfg, lower=None, upper=None):
    """Restated cpu_seq (seq_engine.cpp:12-99)."""
    return _run(oracle_lib().orc_propagate, SEQ, inst, cfg, lower, upper)


def propagate_parallel(inst, cfg, lower=None, upper=None):
    """Restated cpu_par (par_engine.cpp:203-273), single-threaded, exact."""
    return _run(oracle_lib().orc_propagate, PAR, inst, cfg, lower, upper)


def ref_propagate_sequential(inst, cfg, lower=None, upper=None):
    return _run(ref_lib().ref_propagate, SEQ, inst, cfg, lower, upper)


def ref_propagate_parallel(inst, cfg, lower=None, upper=None):
    return _run(ref_lib().ref_propagate, PAR, inst, cfg, lower, upper)


def _round(fn, inst, cfg, lb_in, ub_in):
    c = _cfg(cfg)
    p = inst.to_c()
    n = inst.num_cols()
    lb_in = np.ascontiguousarray(lb_in, dtype=np.float64)
    ub_in = np.ascontiguousarray(ub_in, dtype=np.float64)
    lo = np.empty(n)
    up = np.empty(n)
    ch = C.c_int32()
    inf = C.c_int32()
    cnt = C.c_int64()
    rc = fn(C.byref(p), C.byref(c), abi.ptr(lb_in, C.c_double), abi.ptr(ub_in, C.c_double),
            abi.ptr(lo, C.c_double), abi.ptr(up, C.c_double), C.byref(ch), C.byref(inf),
            C.byref(cnt))
    if rc != 0:
        raise ValueError(f"round failed {rc}")
    return dict(changed=bool(ch.value), infeasible=bool(inf.value), changes=int(cnt.value),
                lower=lo, upper=up)


def propagate_round_parallel(inst, cfg, lb_in, ub_in):
    return _round(oracle_lib().orc_round, inst, cfg, lb_in, ub_in)


def ref_propagate_round_parallel(inst, cfg, lb_in, ub_in):
    return _round(ref_lib().ref_round, inst, cfg, lb_in, ub_in)


def round_rows(inst, cfg, r0, r1, lb_in, ub_in, lb_out, ub_out):
    """process_block over rows [r0, r1) merging into lb_out/ub_out in place."""
    c = _cfg(cfg)
    p = inst.to_c()
    inf = C.c_int32()
    rc = oracle_lib().orc_round_rows(C.byref(p), C.byref(c), r0, r1,
                                     abi.ptr(lb_in, C.c_double), abi.ptr(ub_in, C.c_double),
                                     abi.ptr(lb_out, C.c_double), abi.ptr(ub_out, C.c_double),
                                     C.byref(inf))
    assert rc == 0
    return bool(inf.value)


def commit(lb_in, ub_in, lb_out, ub_out, slack=1e-7):
    inf = C.c_int32(0)
    ch = oracle_lib().orc_commit(lb_in.shape[0], abi.ptr(lb_in, C.c_double),
                                 abi.ptr(ub_in, C.c_double), abi.ptr(lb_out, C.c_double),
                                 abi.ptr(ub_out, C.c_double), slack, C.byref(inf))
    return int(ch), bool(inf.value)


def _ref_inst(h, name):
    if not h:
        raise ValueError(ref_lib().ref_last_error().decode())
    lib = ref_lib()
    try:
        p = abi.PgProblem()
        lib.ref_inst_view(h, C.byref(p))
        return ProblemInstance.from_c(p, name=name)
    finally:
        lib.ref_inst_free(h)


def ref_gen_random(num_rows=100, num_cols=100, seed=0, mean_row_nnz=6.0, integral_fraction=0.3,
                   infinite_bound_fraction=0.05, infinite_side_fraction=0.25, max_nnz=0):
    h = ref_lib().ref_gen_random(num_rows, num_cols, seed, mean_row_nnz, integral_fraction,
                                 infinite_bound_fraction, infinite_side_fraction, max_nnz)
    return _ref_inst(h, f"random_r{num_rows}_c{num_cols}_s{seed}")


def ref_gen_cascade(m):
    return _ref_inst(ref_lib().ref_gen_cascade(m), f"cascade{m}")


def ref_parse_mps(path):
    return _ref_inst(ref_lib().ref_parse_mps(path.encode()), os.path.basename(path))


def canon(x: np.ndarray) -> np.ndarray:
    """Canonicalise -0.0 to +0.0 for bitwise comparisons."""
    return np.where(x == 0.0, 0.0, x)


def bounds_equal(a, b, t_abs=1e-8, t_rel=1e-5):
    """harness.cpp:17-20 bounds_equal, vectorised: |a-b| <= t_abs + t_rel*|b|,
    infinities equal only to the same infinity."""
    a = np.asarray(a)
    b = np.asarray(b)
    inf = np.isinf(a) | np.isinf(b)
    with np.errstate(invalid="ignore"):
        close = np.abs(a - b) <= t_abs + t_rel * np.abs(b)
    return np.where(inf, a == b, close)


_TRIP_MSG = {1: "triplet row index out of range", 2: "triplet column index out of range"}


def csr_from_triplets(rows, cols, values, num_rows: int, num_cols: int, impl: str = "port"):
    """csr_from_triplets (core/src/model.cpp:37-80): the C restatement ("port")
    or the reference itself ("reference").  Returns (row_ptr, col_idx, values);
    IndexError for an out-of-range triplet (std::out_of_range)."""
    r = np.ascontiguousarray(rows, dtype=np.int32)
    c = np.ascontiguousarray(cols, dtype=np.int32)
    v = np.ascontiguousarray(values, dtype=np.float64)
    cnt = r.shape[0]
    rp = np.zeros(num_rows + 1, dtype=np.int32)
    ci = np.empty(max(cnt, 1), dtype=np.int32)
    vo = np.empty(max(cnt, 1), dtype=np.float64)
    nnz = C.c_int64()
    args = (num_rows, num_cols, cnt, abi.ptr(r, C.c_int32), abi.ptr(c, C.c_int32),
            abi.ptr(v, C.c_double), abi.ptr(rp, C.c_int32), abi.ptr(ci, C.c_int32),
            abi.ptr(vo, C.c_double), C.byref(nnz))
    if impl == "reference":
        lib = ref_lib()
        rc = lib.ref_csr_from_triplets(*args)
        if rc == 1:
            raise IndexError(lib.ref_last_error().decode())
    else:
        rc = oracle_lib().orc_csr_from_triplets(*args)
        if rc in _TRIP_MSG:
            raise IndexError(_TRIP_MSG[rc])
    if rc != 0:
        raise RuntimeError(f"csr_from_triplets ({impl}) failed: {rc}")
    k = int(nnz.value)
    return rp, ci[:k].copy(), vo[:k].copy()
