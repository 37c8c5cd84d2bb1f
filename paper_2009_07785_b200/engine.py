"""Python mirror of the reference propagator API over the CUDA C-ABI.

  propagate_gpu(instance, cfg)          ~ propagate_parallel  (par_engine.hpp:41-42)
                                          with cpu_seq verdicts when cfg.row_check
  propagate_round_gpu(instance, snap)   ~ propagate_round_parallel (par_engine.hpp:33-36)
  partition_row_blocks(matrix, cfg)     ~ partition_row_blocks (par_engine.hpp:12-13)
  csr_from_triplets_gpu(rows, cols, ...) ~ csr_from_triplets (model.cpp:37-80), built on
                                          the device (IndexError ~ std::out_of_range)
  Session(instance, cfg)                matrix resident in HBM; re-propagate new
                                        start bounds (B&B warm start) and node batches

Errors follow the reference: an invalid EngineConfig raises ValueError (the
reference throws std::invalid_argument, core/src/model.cpp:21-35);
Infeasible / RoundLimit are statuses, not exceptions.  Every call goes to the
CUDA library; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import abi
from .model import (EngineConfig, PropagationResult, ProblemInstance, SparseMatrix,
                    VariableBounds, new_c_result, result_from_c)


def _lib():
    return abi.load_library()


def validate(cfg: EngineConfig) -> None:
    c = cfg.to_c()
    abi.check(_lib().pg_config_validate(C.byref(c)), "EngineConfig.validate")


def csr_from_triplets_gpu(rows, cols, values, num_rows: int, num_cols: int,
                          device: int = 0) -> SparseMatrix:
    """csr_from_triplets (core/src/model.cpp:37-80) on the GPU: stable (row, col)
    order, duplicates summed in input order, zero sums dropped; IndexError with
    the reference's message for the first out-of-range triplet."""
    r = np.ascontiguousarray(rows, dtype=np.int32)
    c = np.ascontiguousarray(cols, dtype=np.int32)
    v = np.ascontiguousarray(values, dtype=np.float64)
    if not (r.shape == c.shape == v.shape) or r.ndim != 1:
        raise ValueError("rows, cols and values must be 1-D arrays of one length")
    cnt = r.shape[0]
    rp = np.zeros(num_rows + 1, dtype=np.int32)
    ci = np.empty(max(cnt, 1), dtype=np.int32)
    vo = np.empty(max(cnt, 1), dtype=np.float64)
    nnz = C.c_int64()
    abi.check(_lib().pg_csr_from_triplets(num_rows, num_cols, cnt, abi.ptr(r, C.c_int32),
                                          abi.ptr(c, C.c_int32), abi.ptr(v, C.c_double), device,
                                          abi.ptr(rp, C.c_int32), abi.ptr(ci, C.c_int32),
                                          abi.ptr(vo, C.c_double), C.byref(nnz)),
              "csr_from_triplets")
    k = int(nnz.value)
    return SparseMatrix(num_rows, num_cols, rp, ci[:k], vo[:k])


def propagate_multi_gpu(instance: ProblemInstance, cfg: EngineConfig | None = None,
                        ngpus: int = 1) -> PropagationResult:
    """pg_multi_propagate: one process, ngpus devices (cfg.device ..), row
    shards merged over NCCL every round; same results as propagate_gpu."""
    cfg = cfg or EngineConfig()
    c = cfg.to_c()
    p = instance.to_c()
    r, lo, up, prc = new_c_result(instance.num_cols(), cfg.round_limit)
    abi.check(_lib().pg_multi_propagate(C.byref(p), C.byref(c), ngpus, abi.PG_MULTI_ROWS,
                                        C.byref(r)), "pg_multi_propagate")
    return result_from_c(r, lo, up, prc)


def propagate_gpu(instance: ProblemInstance, cfg: EngineConfig | None = None,
                  out=None) -> PropagationResult:
    """pg_propagate.  `out` = (lower, upper): the caller's result buffers
    (float64, n each; page-locked ones download at full PCIe speed), else
    fresh arrays."""
    cfg = cfg or EngineConfig()
    c = cfg.to_c()
    p = instance.to_c()
    r, lo, up, prc = new_c_result(instance.num_cols(), cfg.round_limit, out)
    abi.check(_lib().pg_propagate(C.byref(p), C.byref(c), C.byref(r)), "pg_propagate")
    return result_from_c(r, lo, up, prc)


class MpsFile:
    """pg_mps_read: an MPS file parsed on host threads (mps_reader.h), the
    triplets still in file order.  .instance(device) builds the CSR on the
    GPU (pg_mps_to_csr)."""

    def __init__(self, path: str | None = None, text: bytes | None = None,
                 infinity_threshold: float = 1e20, threads: int = 0):
        self._h = C.c_void_p()
        if text is not None:
            abi.check(_lib().pg_mps_read_buffer(text, len(text), infinity_threshold, threads,
                                                C.byref(self._h)), "parse_mps")
        else:
            abi.check(_lib().pg_mps_read(os.fsencode(path), infinity_threshold, threads,
                                         C.byref(self._h)), "parse_mps_file")
        m, n, t = C.c_int32(), C.c_int32(), C.c_int64()
        abi.check(_lib().pg_mps_dims(self._h, C.byref(m), C.byref(n), C.byref(t)), "pg_mps_dims")
        self.m, self.n, self.ntrip = m.value, n.value, t.value
        self.name = (_lib().pg_mps_name(self._h) or b"").decode()
        ptrs = [C.POINTER(C.c_int32)(), C.POINTER(C.c_int32)()] + \
            [C.POINTER(C.c_double)() for _ in range(5)] + [C.POINTER(C.c_uint8)()]
        abi.check(_lib().pg_mps_arrays(self._h, *[C.byref(p) for p in ptrs]), "pg_mps_arrays")

        def view(p, count, dt):
            return np.ctypeslib.as_array(p, shape=(count,)).astype(dt, copy=True) if count else \
                np.zeros(0, dt)
        self.rows = view(ptrs[0], self.ntrip, np.int32)
        self.cols = view(ptrs[1], self.ntrip, np.int32)
        self.values = view(ptrs[2], self.ntrip, np.float64)
        self.lhs = view(ptrs[3], self.m, np.float64)
        self.rhs = view(ptrs[4], self.m, np.float64)
        self.lower = view(ptrs[5], self.n, np.float64)
        self.upper = view(ptrs[6], self.n, np.float64)
        self.integral = view(ptrs[7], self.n, np.uint8)

    def instance(self, device: int = 0) -> ProblemInstance:
        rp = np.zeros(self.m + 1, dtype=np.int32)
        ci = np.empty(max(self.ntrip, 1), dtype=np.int32)
        vo = np.empty(max(self.ntrip, 1), dtype=np.float64)
        nnz = C.c_int64()
        abi.check(_lib().pg_mps_to_csr(self._h, device, abi.ptr(rp, C.c_int32),
                                       abi.ptr(ci, C.c_int32), abi.ptr(vo, C.c_double),
                                       C.byref(nnz)), "pg_mps_to_csr")
        k = int(nnz.value)
        return ProblemInstance.from_arrays(rp, ci[:k], vo[:k], self.lhs, self.rhs, self.lower,
                                           self.upper, self.integral, num_cols=self.n,
                                           name=self.name)

    def close(self):
        if self._h:
            _lib().pg_mps_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def read_mps(path: str, infinity_threshold: float = 1e20, device: int = 0,
             threads: int = 0) -> ProblemInstance:
    """parse_mps_file (core/src/mps.cpp:409-420): host-parallel parse, CSR on the GPU."""
    f = MpsFile(path, infinity_threshold=infinity_threshold, threads=threads)
    try:
        return f.instance(device)
    finally:
        f.close()


@dataclass
class RoundSnapshot:
    """par_engine.hpp:18-21"""
    bounds_in: VariableBounds
    bounds_out: VariableBounds | None = None


@dataclass
class RoundOutcome:
    """par_engine.hpp:23-27"""
    changed: bool = False
    infeasible: bool = False
    changes: int = 0


def propagate_round_gpu(instance: ProblemInstance, snap: RoundSnapshot,
                        cfg: EngineConfig | None = None) -> RoundOutcome:
    cfg = cfg or EngineConfig()
    c = cfg.to_c()
    p = instance.to_c()
    n = instance.num_cols()
    lb_in = np.ascontiguousarray(snap.bounds_in.lower, dtype=np.float64)
    ub_in = np.ascontiguousarray(snap.bounds_in.upper, dtype=np.float64)
    lo = np.empty(n)
    up = np.empty(n)
    ch, inf, cnt = C.c_int32(), C.c_int32(), C.c_int64()
    abi.check(_lib().pg_round(C.byref(p), C.byref(c), abi.ptr(lb_in, C.c_double),
                              abi.ptr(ub_in, C.c_double), abi.ptr(lo, C.c_double),
                              abi.ptr(up, C.c_double), C.byref(ch), C.byref(inf), C.byref(cnt)),
              "pg_round")
    snap.bounds_out = VariableBounds(lo, up)
    return RoundOutcome(bool(ch.value), bool(inf.value), int(cnt.value))


def partition_row_blocks(instance: ProblemInstance, cfg: EngineConfig | None = None):
    cfg = cfg or EngineConfig()
    c = cfg.to_c()
    p = instance.to_c()
    m = instance.num_rows()
    starts = np.zeros(m + 1, dtype=np.int32)
    kinds = np.zeros(max(m, 1), dtype=np.int32)
    nb = C.c_int32()
    abi.check(_lib().pg_partition_row_blocks(C.byref(p), C.byref(c), abi.ptr(starts, C.c_int32),
                                             abi.ptr(kinds, C.c_int32), C.byref(nb)),
              "pg_partition_row_blocks")
    return starts[: nb.value + 1].copy(), kinds[: nb.value].copy()


class Session:
    """One problem resident on the device (pg_session_*)."""

    INFO_FIELDS = ("m", "n", "nnz", "slices", "seg_rows", "segments", "short_rows", "short_nnz",
                   "seg_nnz", "chains", "sell_elems", "split_rows", "persistent",
                   "delta_rounds", "host_syncs", "held_rounds", "shard_rounds", "delta_graphs",
                   "gather_bytes")

    def __init__(self, instance: ProblemInstance, cfg: EngineConfig | None = None):
        self.cfg = cfg or EngineConfig()
        self.instance = instance
        self._h = C.c_void_p()
        c = self.cfg.to_c()
        p = instance.to_c()
        abi.check(_lib().pg_session_create(C.byref(p), C.byref(c), C.byref(self._h)),
                  "pg_session_create")

    def close(self):
        if self._h:
            _lib().pg_session_destroy(self._h)
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def propagate(self, lower=None, upper=None, out=None) -> PropagationResult:
        n = self.instance.num_cols()
        r, lo, up, prc = new_c_result(n, self.cfg.round_limit, out)
        lp = up_ = None
        if lower is not None:
            lower = np.ascontiguousarray(lower, dtype=np.float64)
            upper = np.ascontiguousarray(upper, dtype=np.float64)
            lp, up_ = abi.ptr(lower, C.c_double), abi.ptr(upper, C.c_double)
        abi.check(_lib().pg_session_propagate(self._h, lp, up_, C.byref(r)), "pg_session_propagate")
        return result_from_c(r, lo, up, prc)

    def round(self, snap: RoundSnapshot) -> RoundOutcome:
        """propagate_round_parallel on the resident matrix (pg_session_round)."""
        n = self.instance.num_cols()
        lb_in = np.ascontiguousarray(snap.bounds_in.lower, dtype=np.float64)
        ub_in = np.ascontiguousarray(snap.bounds_in.upper, dtype=np.float64)
        lo = np.empty(n)
        up = np.empty(n)
        ch, inf, cnt = C.c_int32(), C.c_int32(), C.c_int64()
        abi.check(_lib().pg_session_round(self._h, abi.ptr(lb_in, C.c_double),
                                          abi.ptr(ub_in, C.c_double), abi.ptr(lo, C.c_double),
                                          abi.ptr(up, C.c_double), C.byref(ch), C.byref(inf),
                                          C.byref(cnt)), "pg_session_round")
        snap.bounds_out = VariableBounds(lo, up)
        return RoundOutcome(bool(ch.value), bool(inf.value), int(cnt.value))

    def run(self, download=False, out=None) -> PropagationResult:
        """Solve from the device-resident start bounds (nothing crosses PCIe
        unless download=True; `out` as for propagate_gpu)."""
        n = self.instance.num_cols()
        r, lo, up, prc = new_c_result(n, self.cfg.round_limit, out)
        if not download:
            r.lower = C.cast(None, C.POINTER(C.c_double))
            r.upper = C.cast(None, C.POINTER(C.c_double))
        abi.check(_lib().pg_session_run(self._h, C.byref(r)), "pg_session_run")
        return result_from_c(r, lo, up, prc)

    def propagate_batch(self, lower: np.ndarray, upper: np.ndarray):
        K, n = lower.shape
        lower = np.ascontiguousarray(lower, dtype=np.float64)
        upper = np.ascontiguousarray(upper, dtype=np.float64)
        lo = np.empty_like(lower)
        up = np.empty_like(upper)
        st = np.zeros(K, dtype=np.int32)
        rd = np.zeros(K, dtype=np.int32)
        abi.check(_lib().pg_session_propagate_batch(
            self._h, K, abi.ptr(lower, C.c_double), abi.ptr(upper, C.c_double),
            abi.ptr(lo, C.c_double), abi.ptr(up, C.c_double), abi.ptr(st, C.c_int32),
            abi.ptr(rd, C.c_int32)), "pg_session_propagate_batch")
        return lo, up, st, rd

    def time_round_kernel(self, reps=10):
        mean_ns, nbytes = C.c_double(), C.c_double()
        abi.check(_lib().pg_session_time_round_kernel(self._h, reps, C.byref(mean_ns),
                                                      C.byref(nbytes)), "time_round_kernel")
        return mean_ns.value, nbytes.value

    def info(self) -> dict:
        v = np.zeros(len(self.INFO_FIELDS), dtype=np.int64)
        abi.check(_lib().pg_session_info(self._h, abi.ptr(v, C.c_int64), v.shape[0]), "info")
        return dict(zip(self.INFO_FIELDS, (int(x) for x in v)))

    # ---- branch-and-bound nodes (config C4) ------------------------------------
    def set_root(self) -> PropagationResult:
        """Propagate the start bounds; a Converged result becomes the
        device-resident root for propagate_nodes."""
        n = self.instance.num_cols()
        r, lo, up, prc = new_c_result(n, self.cfg.round_limit)
        abi.check(_lib().pg_session_set_root(self._h, C.byref(r)), "pg_session_set_root")
        return result_from_c(r, lo, up, prc)

    def propagate_nodes(self, node_ptr, vars_, lo, up, want_bounds=False):
        """K child nodes of the root, node k overriding vars_[node_ptr[k]:node_ptr[k+1]]
        with [lo, up].  Returns (status[K], rounds[K], lower[K,n]|None,
        upper[K,n]|None, device_ns)."""
        node_ptr = np.ascontiguousarray(node_ptr, dtype=np.int32)
        vars_ = np.ascontiguousarray(vars_, dtype=np.int32)
        lo = np.ascontiguousarray(lo, dtype=np.float64)
        up = np.ascontiguousarray(up, dtype=np.float64)
        K = node_ptr.shape[0] - 1
        n = self.instance.num_cols()
        st = np.zeros(K, dtype=np.int32)
        rd = np.zeros(K, dtype=np.int32)
        lo_out = np.empty((K, n)) if want_bounds else None
        up_out = np.empty((K, n)) if want_bounds else None
        ns = C.c_int64()
        abi.check(_lib().pg_session_propagate_nodes(
            self._h, K, abi.ptr(node_ptr, C.c_int32), abi.ptr(vars_, C.c_int32),
            abi.ptr(lo, C.c_double), abi.ptr(up, C.c_double), abi.ptr(st, C.c_int32),
            abi.ptr(rd, C.c_int32), abi.ptr(lo_out, C.c_double), abi.ptr(up_out, C.c_double),
            C.byref(ns)), "pg_session_propagate_nodes")
        return st, rd, lo_out, up_out, ns.value


def node_overrides(root_lower, root_upper, lower, upper):
    """Sparse form of node bound vectors ([K, n]) relative to the root:
    (node_ptr, vars, lo, up)."""
    ptr, vs, ls, us = [0], [], [], []
    for k in range(lower.shape[0]):
        d = np.flatnonzero((lower[k] != root_lower) | (upper[k] != root_upper))
        vs.append(d)
        ls.append(lower[k][d])
        us.append(upper[k][d])
        ptr.append(ptr[-1] + len(d))
    cat = (lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt))
    return (np.array(ptr, dtype=np.int32), cat(vs, np.int32), cat(ls, np.float64),
            cat(us, np.float64))
