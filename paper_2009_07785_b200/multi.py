"""Multi-GPU drivers: one process per GPU.

Work is spread only where the path shards naturally:

  * node sharding (config C4): K independent branch-and-bound node bound
    vectors over a shared matrix; node k goes to rank k * world // K ... in
    contiguous slices, the matrix is replicated, and there is no per-round
    communication (weak scaling).
  * row sharding (config C5): one instance split into `world` contiguous,
    nnz-balanced row ranges; every rank holds all columns.  Each round every
    rank propagates its rows and the shards' results are merged with ONE NCCL
    max all-reduce over the ordered-bits bound keys (lower keys and negated
    upper keys) plus the infeasibility flag, inside the device-resident loop
    (pg_session_attach_comm).  Max/min merges are exact and rows are never
    split, so the result is bit-identical to one GPU.

A single instance of configs C1-C3 stays on one GPU (north star): `--gpus N`
runs N replicas there.

torch.distributed (any backend) is used only to broadcast the 128-byte NCCL
unique id; the data path is the engine's own NCCL communicator.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi
from .engine import Session
from .model import EngineConfig, ProblemInstance, PropagationResult


def row_shards(row_ptr: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Contiguous row ranges with balanced entry counts (a row is never split)."""
    m = int(row_ptr.shape[0] - 1)
    nnz = int(row_ptr[-1])
    cuts = [0]
    for g in range(1, world):
        target = nnz * g / world
        r = int(np.searchsorted(row_ptr, target, side="left"))
        cuts.append(min(max(r, cuts[-1]), m))
    cuts.append(m)
    return [(cuts[g], cuts[g + 1]) for g in range(world)]


def node_shards(K: int, world: int) -> list[tuple[int, int]]:
    """Contiguous node slices, sizes differing by at most one."""
    base, extra = divmod(K, world)
    out, k = [], 0
    for g in range(world):
        size = base + (1 if g < extra else 0)
        out.append((k, k + size))
        k += size
    return out


def shard_instance(inst: ProblemInstance, r0: int, r1: int) -> ProblemInstance:
    """Rows [r0, r1) of an instance, all columns (bounds and integrality kept)."""
    rp = inst.matrix.row_ptr
    k0, k1 = int(rp[r0]), int(rp[r1])
    return ProblemInstance.from_arrays(
        (rp[r0:r1 + 1] - k0).astype(np.int32), inst.matrix.col_idx[k0:k1],
        inst.matrix.values[k0:k1], inst.lhs[r0:r1], inst.rhs[r0:r1], inst.bounds.lower,
        inst.bounds.upper, inst.integral, num_cols=inst.num_cols(), name=f"{inst.name}[{r0}:{r1}]")


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    abi.check(abi.load_library().pg_nccl_unique_id(buf), "pg_nccl_unique_id")
    return bytes(buf)


class RowShardedSession:
    """This rank's row shard of one instance, merged over NCCL every round."""

    def __init__(self, inst: ProblemInstance, cfg: EngineConfig, rank: int, world: int,
                 group=None, uid: bytes | None = None, force_comm: bool = False,
                 shard: ProblemInstance | None = None):
        """world == 1 is the plain single-GPU engine (nothing to exchange)
        unless force_comm attaches a one-rank communicator (tests).  `shard`:
        this rank's rows already cut (e.g. in pinned host memory)."""
        self.rank, self.world = rank, world
        self.r0, self.r1 = row_shards(inst.matrix.row_ptr, world)[rank]
        self.shard = shard if shard is not None else shard_instance(inst, self.r0, self.r1)
        self.session = Session(self.shard, cfg)
        self.comm = world > 1 or force_comm
        if not self.comm:
            return
        if uid is None:
            if world > 1:
                import torch.distributed as dist
                obj = [nccl_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(obj, src=0, group=group)
                uid = obj[0]
            else:
                uid = nccl_unique_id()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        abi.check(abi.load_library().pg_session_attach_comm(self.session._h, buf, rank, world),
                  "pg_session_attach_comm")

    def propagate(self, lower=None, upper=None, out=None) -> PropagationResult:
        return self.session.propagate(lower, upper, out)

    def run(self, download=False, out=None) -> PropagationResult:
        return self.session.run(download, out)

    def close(self):
        self.session.close()


def propagate_nodes_sharded(inst: ProblemInstance, cfg: EngineConfig, lower: np.ndarray,
                            upper: np.ndarray, rank: int, world: int):
    """This rank's slice of K node bound vectors ([K, n] arrays); returns
    (k0, k1, lower_out, upper_out, status, rounds) for its nodes."""
    k0, k1 = node_shards(lower.shape[0], world)[rank]
    with Session(inst, cfg) as s:
        lo, up, st, rd = s.propagate_batch(lower[k0:k1], upper[k0:k1])
    return k0, k1, lo, up, st, rd
