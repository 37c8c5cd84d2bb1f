"""Seeded synthetic instances (test/bench input; see instances/pgen.cpp).

gen_random / gen_cascade restate the reference generators
(core/src/generators.cpp:13-168) bit-for-bit; the config generators follow
SURVEY.md 8(d):

  C1  gen_random(10k x 10k, mean 8, 50% integer), seeds 1..5
  C2  gen_powerlaw(1M x 1M, x_min 4.25, beta 1.5, cap 10k), seeds 20090778+{0..4}
  C3  gen_longrows(100k x 200k, every 100th row 100k-150k entries), seeds 3001..3003
  C4  gen_random(500k x 500k, mean 8, 50% int, seed 4) + gen_nodes(K = 8192)
  C5  gen_setpart(1M x 5M, 50 per row, f = 0.2), seeds 5001..5003
"""
from __future__ import annotations

import ctypes as C

import numpy as np

import os

from paper_2009_07785_b200 import abi
from paper_2009_07785_b200.model import ProblemInstance

GEN_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpgen.so")
_gen = None


def load_gen(path: str = GEN_PATH):
    """libpgen.so (instances/pgen.cpp), built by __graft_entry__.build()."""
    global _gen
    if _gen is not None:
        return _gen
    if not os.path.exists(path):
        raise abi.EngineError(f"{path} is missing: run __graft_entry__.build()")
    g = C.CDLL(path)
    g.pgen_view.argtypes = [C.c_void_p, C.POINTER(abi.PgProblem)]
    g.pgen_view.restype = None
    g.pgen_free.argtypes = [C.c_void_p]
    g.pgen_free.restype = None
    g.pgen_from_arrays.argtypes = [C.POINTER(abi.PgProblem)]
    g.pgen_from_arrays.restype = C.c_void_p
    g.pgen_random.argtypes = [C.c_int32, C.c_int32, C.c_uint64, C.c_double, C.c_double,
                              C.c_double, C.c_double, C.c_int64]
    g.pgen_random.restype = C.c_void_p
    g.pgen_cascade.argtypes = [C.c_int32]
    g.pgen_cascade.restype = C.c_void_p
    g.pgen_powerlaw.argtypes = [C.c_int32, C.c_int32, C.c_uint64, C.c_double, C.c_double,
                                C.c_int32, C.c_double, C.c_double, C.c_double]
    g.pgen_powerlaw.restype = C.c_void_p
    g.pgen_longrows.argtypes = [C.c_int32, C.c_int32, C.c_uint64, C.c_int32, C.c_int32,
                                C.c_int32, C.c_double, C.c_double, C.c_double, C.c_double]
    g.pgen_longrows.restype = C.c_void_p
    g.pgen_setpart.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double,
                               C.c_uint64, C.c_int32]
    g.pgen_setpart.restype = C.c_void_p
    g.pgen_nodes.argtypes = [C.POINTER(abi.PgProblem), abi._dp, abi._dp, C.c_int32, C.c_uint64, C.c_int32,
                             C.c_int32, abi._dp, abi._dp]
    g.pgen_nodes.restype = C.c_int
    g.pgen_acceptance_sizes.argtypes = [C.c_int32, abi._ip, abi._ip]
    g.pgen_acceptance_sizes.restype = None
    _gen = g
    return g



def _take(h, name) -> ProblemInstance:
    if not h:
        raise ValueError(f"{name}: invalid generator arguments")
    g = load_gen()
    try:
        p = abi.PgProblem()
        g.pgen_view(h, C.byref(p))
        return ProblemInstance.from_c(p, name=name)
    finally:
        g.pgen_free(h)


def gen_random(num_rows=100, num_cols=100, seed=0, mean_row_nnz=6.0, integral_fraction=0.3,
               infinite_bound_fraction=0.05, infinite_side_fraction=0.25, max_nnz=0):
    """RandomInstanceOptions defaults (generators.hpp:19-28)."""
    h = load_gen().pgen_random(num_rows, num_cols, seed, mean_row_nnz, integral_fraction,
                                   infinite_bound_fraction, infinite_side_fraction, max_nnz)
    return _take(h, f"random_r{num_rows}_c{num_cols}_s{seed}")


def gen_cascade(m: int):
    return _take(load_gen().pgen_cascade(m), f"cascade{m}")


def gen_powerlaw(num_rows=1_000_000, num_cols=1_000_000, seed=20090778, x_min=4.25, beta=1.5,
                 cap=10_000, integral_fraction=0.5, infinite_bound_fraction=0.05,
                 infinite_side_fraction=0.25):
    h = load_gen().pgen_powerlaw(num_rows, num_cols, seed, x_min, beta, cap, integral_fraction,
                                     infinite_bound_fraction, infinite_side_fraction)
    return _take(h, f"powerlaw_r{num_rows}_c{num_cols}_s{seed}")


def gen_longrows(num_rows=100_000, num_cols=200_000, seed=3001, long_every=100, long_min=100_000,
                 long_max=150_000, mean_short=8.0, integral_fraction=0.5,
                 infinite_bound_fraction=0.05, infinite_side_fraction=0.25):
    h = load_gen().pgen_longrows(num_rows, num_cols, seed, long_every, long_min, long_max,
                                     mean_short, integral_fraction, infinite_bound_fraction,
                                     infinite_side_fraction)
    return _take(h, f"longrows_r{num_rows}_c{num_cols}_s{seed}")


def gen_setpart(num_rows=1_000_000, num_cols=5_000_000, per_row=50, s1_fraction=0.1,
                f_fixed=0.2, seed=5001, infeasible=False):
    h = load_gen().pgen_setpart(num_rows, num_cols, per_row, s1_fraction, f_fixed, seed,
                                    1 if infeasible else 0)
    return _take(h, f"setpart_r{num_rows}_c{num_cols}_s{seed}{'_inf' if infeasible else ''}")


def gen_nodes(inst: ProblemInstance, root_lower, root_upper, K: int, seed_base=4_000_000, dmin=1,
              dmax=8):
    """K child-node bound vectors (node-major arrays [K, n])."""
    n = inst.num_cols()
    lo = np.empty((K, n), dtype=np.float64)
    up = np.empty((K, n), dtype=np.float64)
    rl = np.ascontiguousarray(root_lower, dtype=np.float64)
    ru = np.ascontiguousarray(root_upper, dtype=np.float64)
    p = inst.to_c()
    rc = load_gen().pgen_nodes(C.byref(p), abi.ptr(rl, C.c_double), abi.ptr(ru, C.c_double), K,
                                   seed_base, dmin, dmax, abi.ptr(lo, C.c_double),
                                   abi.ptr(up, C.c_double))
    if rc != 0:
        raise ValueError("gen_nodes failed")
    return lo, up


def config_instance(name: str, seed: int | None = None) -> ProblemInstance:
    """The SURVEY.md 8(d) instances by config name."""
    name = name.lower()
    if name == "c1":
        return gen_random(10_000, 10_000, seed if seed is not None else 1, mean_row_nnz=8.0,
                          integral_fraction=0.5)
    if name == "c2":
        return gen_powerlaw(seed=seed if seed is not None else 20090778)
    if name == "c3":
        return gen_longrows(seed=seed if seed is not None else 3001)
    if name == "c4":
        return gen_random(500_000, 500_000, seed if seed is not None else 4, mean_row_nnz=8.0,
                          integral_fraction=0.5)
    if name == "c5":
        return gen_setpart(seed=seed if seed is not None else 5001)
    raise ValueError(f"unknown config {name!r}")


def acceptance_suite_params(count=500):
    """(rows, cols, seed, max_nnz) of the reference acceptance suite
    (tests/acceptance.cpp:56-75)."""
    rows = np.zeros(count, dtype=np.int32)
    cols = np.zeros(count, dtype=np.int32)
    load_gen().pgen_acceptance_sizes(count, abi.ptr(rows, C.c_int32), abi.ptr(cols, C.c_int32))
    return [(int(r), int(c), 1000 + i, 50000) for i, (r, c) in enumerate(zip(rows, cols))]


def acceptance_suite(count=500):
    for r, c, seed, mx in acceptance_suite_params(count):
        yield gen_random(r, c, seed, max_nnz=mx)
