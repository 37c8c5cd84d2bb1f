"""Host-side mirror of the reference model types (core/include/propgate/model.hpp).

Same names and field meanings as the C++ reference so that parity tests read
like the reference's own tests:

  SparseMatrix        model.hpp:20-37   (int32 row_ptr/col_idx, fp64 values)
  VariableBounds      model.hpp:59-64
  ProblemInstance     model.hpp:68-79
  PropagationStatus   model.hpp:112
  PropagationResult   model.hpp:119-127
  ScalarMode          model.hpp:129
  EngineConfig        model.hpp:131-144 (+ GPU fields: device, loop_mode, row_check)

These are plain containers; all computation happens in the CUDA library
behind the C-ABI (include/propgate_b200.h).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import abi

kInf = float("inf")


class PropagationStatus(enum.IntEnum):
    Converged = abi.PG_CONVERGED
    RoundLimit = abi.PG_ROUNDLIMIT
    Infeasible = abi.PG_INFEASIBLE


class ScalarMode(enum.IntEnum):
    Wide64 = abi.PG_WIDE64
    Narrow32 = abi.PG_NARROW32


class LoopMode(enum.IntEnum):
    Graph = abi.PG_LOOP_GRAPH   # device-resident loop (CUDA graph, conditional WHILE)
    Host = abi.PG_LOOP_HOST     # one host sync per round (the paper's cpu_loop)


@dataclass
class SparseMatrix:
    num_rows: int
    num_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def nnz(self) -> int:
        return int(self.col_idx.shape[0])

    def row_nnz(self, row: int) -> int:
        return int(self.row_ptr[row + 1] - self.row_ptr[row])


@dataclass
class VariableBounds:
    lower: np.ndarray
    upper: np.ndarray

    def size(self) -> int:
        return int(self.lower.shape[0])


@dataclass
class ProblemInstance:
    matrix: SparseMatrix
    lhs: np.ndarray
    rhs: np.ndarray
    bounds: VariableBounds
    integral: np.ndarray
    name: str = ""

    def num_rows(self) -> int:
        return self.matrix.num_rows

    def num_cols(self) -> int:
        return self.matrix.num_cols

    @staticmethod
    def from_arrays(row_ptr, col_idx, values, lhs, rhs, lower, upper, integral=None, num_cols=None,
                    name=""):
        row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int32)
        col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
        values = np.ascontiguousarray(values, dtype=np.float64)
        lower = np.ascontiguousarray(lower, dtype=np.float64)
        upper = np.ascontiguousarray(upper, dtype=np.float64)
        n = int(num_cols if num_cols is not None else lower.shape[0])
        if integral is None:
            integral = np.zeros(n, dtype=np.uint8)
        m = int(row_ptr.shape[0] - 1)
        return ProblemInstance(
            SparseMatrix(m, n, row_ptr, col_idx, values),
            np.ascontiguousarray(lhs, dtype=np.float64), np.ascontiguousarray(rhs, dtype=np.float64),
            VariableBounds(lower, upper), np.ascontiguousarray(integral, dtype=np.uint8), name)

    def with_bounds(self, lower, upper) -> "ProblemInstance":
        return ProblemInstance(self.matrix, self.lhs, self.rhs,
                               VariableBounds(np.ascontiguousarray(lower, dtype=np.float64),
                                              np.ascontiguousarray(upper, dtype=np.float64)),
                               self.integral, self.name)

    def to_c(self) -> abi.PgProblem:
        """Borrowed view for the C-ABI (keep `self` alive during the call)."""
        p = abi.PgProblem()
        p.num_rows = self.matrix.num_rows
        p.num_cols = self.matrix.num_cols
        p.nnz = self.matrix.nnz()
        p.row_ptr = abi.ptr(self.matrix.row_ptr, C.c_int32)
        p.col_idx = abi.ptr(self.matrix.col_idx, C.c_int32)
        p.values = abi.ptr(self.matrix.values, C.c_double)
        p.lhs = abi.ptr(self.lhs, C.c_double)
        p.rhs = abi.ptr(self.rhs, C.c_double)
        p.lower = abi.ptr(self.bounds.lower, C.c_double)
        p.upper = abi.ptr(self.bounds.upper, C.c_double)
        p.integral = abi.ptr(self.integral, C.c_uint8)
        return p

    @staticmethod
    def from_c(p: abi.PgProblem, name="") -> "ProblemInstance":
        """Owning copy of a C view."""
        m, n, nnz = p.num_rows, p.num_cols, p.nnz

        def arr(ptr_, count, dt):
            if count == 0:
                return np.zeros(0, dtype=dt)
            return np.ctypeslib.as_array(ptr_, shape=(count,)).astype(dt, copy=True)

        return ProblemInstance.from_arrays(
            arr(p.row_ptr, m + 1, np.int32), arr(p.col_idx, nnz, np.int32),
            arr(p.values, nnz, np.float64), arr(p.lhs, m, np.float64), arr(p.rhs, m, np.float64),
            arr(p.lower, n, np.float64), arr(p.upper, n, np.float64), arr(p.integral, n, np.uint8),
            num_cols=n, name=name)


@dataclass
class EngineConfig:
    round_limit: int = 100
    infinity_threshold: float = 1e20
    improvement_abs: float = 1e-7
    improvement_rel: float = 1e-7
    integrality_eps: float = 1e-6
    nnz_budget: int = 1024
    vector_threshold: int = 64
    worker_count: int = 0
    scalar_mode: ScalarMode = ScalarMode.Wide64
    # GPU fields
    device: int = 0
    loop_mode: LoopMode = LoopMode.Graph
    row_check: bool = True
    worklist: bool = False
    delta_exchange: bool = False  # row shards: sparse delta rounds (PG_FLAG_DELTA_EXCHANGE)

    def to_c(self) -> abi.PgConfig:
        c = abi.PgConfig()
        c.round_limit = self.round_limit
        c.infinity_threshold = self.infinity_threshold
        c.improvement_abs = self.improvement_abs
        c.improvement_rel = self.improvement_rel
        c.integrality_eps = self.integrality_eps
        c.nnz_budget = self.nnz_budget
        c.vector_threshold = self.vector_threshold
        c.worker_count = self.worker_count
        c.scalar_mode = int(self.scalar_mode)
        c.device = self.device
        c.loop_mode = int(self.loop_mode)
        c.flags = ((abi.PG_FLAG_ROWCHECK if self.row_check else 0) |
                   (abi.PG_FLAG_WORKLIST if self.worklist else 0) |
                   (abi.PG_FLAG_DELTA_EXCHANGE if self.delta_exchange else 0))
        return c


@dataclass
class PropagationResult:
    bounds: VariableBounds
    status: PropagationStatus = PropagationStatus.Converged
    rounds_executed: int = 0
    total_bound_changes: int = 0
    per_round_changes: list = field(default_factory=list)
    constraints_processed: int = 0
    elapsed_ns: int = 0


def new_c_result(n: int, round_limit: int, out=None):
    """Allocate output arrays (or take the caller's `out` = (lower, upper),
    e.g. page-locked buffers reused across calls) and a PgResult pointing at
    them."""
    if out is None:
        lo = np.empty(n, dtype=np.float64)
        up = np.empty(n, dtype=np.float64)
    else:
        lo, up = out
        for a in (lo, up):
            if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.shape == (n,)
                    and a.flags.c_contiguous and a.flags.writeable):
                raise ValueError(f"out arrays must be writable contiguous float64 of shape ({n},)")
    prc = np.zeros(max(round_limit, 1), dtype=np.int64)
    r = abi.PgResult()
    r.lower = abi.ptr(lo, C.c_double)
    r.upper = abi.ptr(up, C.c_double)
    r.per_round_changes = abi.ptr(prc, C.c_int64)
    r.per_round_capacity = prc.shape[0]
    return r, lo, up, prc


def result_from_c(r: abi.PgResult, lo, up, prc) -> PropagationResult:
    return PropagationResult(
        bounds=VariableBounds(lo, up),
        status=PropagationStatus(r.status),
        rounds_executed=int(r.rounds_executed),
        total_bound_changes=int(r.total_bound_changes),
        per_round_changes=[int(x) for x in prc[: r.rounds_executed]],
        constraints_processed=int(r.constraints_processed),
        elapsed_ns=int(r.elapsed_ns),
    )
