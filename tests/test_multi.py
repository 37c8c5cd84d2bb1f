"""CPU, world_size 2 over gloo: the host-side logic of the multi-GPU paths.

Row sharding (config C5): each rank runs the restated cpu_par round over its
nnz-balanced row shard, the shards are merged by MAX on lower / MIN on upper
bounds and MAX on the infeasibility flag -- exactly the single NCCL max
all-reduce of the GPU path over lower keys and NEGATED upper keys -- and every
rank commits the same merged bounds.  The trajectory must be bit-identical to
the unsharded cpu_par.  Node sharding (config C4): contiguous node slices,
results gathered, identical to one process.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from instances import generators as G
from paper_2009_07785_b200.model import EngineConfig, PropagationStatus
from paper_2009_07785_b200.multi import node_shards, row_shards, shard_instance

PAR = EngineConfig(row_check=False)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _key(x):
    """ordered-bits key of the GPU path (kernels.cuh key_enc)"""
    b = np.asarray(x, dtype=np.float64).view(np.int64)
    return np.where(b >= 0, b, b ^ np.int64(0x7FFFFFFFFFFFFFFF))


def _unkey(k):
    k = np.asarray(k, dtype=np.int64)
    return np.where(k >= 0, k, k ^ np.int64(0x7FFFFFFFFFFFFFFF)).view(np.float64)


def _row_sharded_worker(rank, world, port, insts, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    for inst in insts:
        r0, r1 = row_shards(inst.matrix.row_ptr, world)[rank]
        n = inst.num_cols()
        lo = np.where(np.abs(inst.bounds.lower) >= 1e20, np.sign(inst.bounds.lower) * np.inf,
                      inst.bounds.lower)
        up = np.where(np.abs(inst.bounds.upper) >= 1e20, np.sign(inst.bounds.upper) * np.inf,
                      inst.bounds.upper)
        per_round, status = [], None
        for rnd in range(1, PAR.round_limit + 1):
            lo_out, up_out = lo.copy(), up.copy()
            inf = O.round_rows(inst, PAR, r0, r1, lo, up, lo_out, up_out)
            # the GPU merge: one MAX all-reduce over [lb keys, -ub keys, flag]
            buf = torch.from_numpy(np.concatenate([_key(lo_out), -_key(up_out), [int(inf)]]))
            dist.all_reduce(buf, op=dist.ReduceOp.MAX)
            b = buf.numpy()
            lo_out, up_out, inf = _unkey(b[:n]), _unkey(-b[n:2 * n]), bool(b[2 * n])
            ch, cinf = O.commit(lo, up, lo_out, up_out)
            per_round.append(ch)
            if inf or cinf:
                status = PropagationStatus.Infeasible
            elif ch == 0:
                status = PropagationStatus.Converged
            elif rnd == PAR.round_limit:
                status = PropagationStatus.RoundLimit
            lo, up = lo_out, up_out
            if status is not None:
                break
        out.append((int(status), per_round, lo, up))
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def _spawn(fn, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_row_shards_balanced_and_contiguous():
    inst = G.gen_powerlaw(20000, 20000, 5, cap=2000)
    rp = inst.matrix.row_ptr
    for world in (1, 2, 3, 4, 8):
        sh = row_shards(rp, world)
        assert sh[0][0] == 0 and sh[-1][1] == inst.num_rows()
        assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
        sizes = [int(rp[r1] - rp[r0]) for r0, r1 in sh]
        longest = int(np.diff(rp).max())
        assert max(sizes) - min(sizes) <= 2 * longest + 1
        parts = [shard_instance(inst, r0, r1) for r0, r1 in sh]
        assert sum(p.matrix.nnz() for p in parts) == inst.matrix.nnz()


def test_node_shards():
    for K, world in ((8192, 8), (10, 3), (3, 4)):
        sh = node_shards(K, world)
        assert sh[0][0] == 0 and sh[-1][1] == K
        sizes = [b - a for a, b in sh]
        assert max(sizes) - min(sizes) <= 1


def test_row_sharded_merge_is_bit_identical_gloo():
    insts = [G.gen_setpart(4000, 20000, 20, f_fixed=0.2, seed=5001),
             G.gen_setpart(4000, 20000, 20, f_fixed=0.2, seed=5002, infeasible=True),
             G.gen_random(3000, 2500, 11, mean_row_nnz=9.0, integral_fraction=0.5),
             G.gen_longrows(2000, 4000, 3001, long_every=100, long_min=1500, long_max=2500)]
    res = _spawn(_row_sharded_worker, 2, insts)
    for i, inst in enumerate(insts):
        ref = O.propagate_parallel(inst, PAR)
        for rank in (0, 1):
            status, per_round, lo, up = res[rank][i]
            assert status == int(ref.status), (inst.name, rank)
            assert per_round == ref.per_round_changes, (inst.name, rank)
            assert np.array_equal(O.canon(lo), O.canon(ref.bounds.lower))
            assert np.array_equal(O.canon(up), O.canon(ref.bounds.upper))
    assert res[0][1][0] == int(PropagationStatus.Infeasible)  # the infeasible C5 variant


def _delta_worker(rank, world, port, insts, cap_div, q):
    """PG_FLAG_DELTA_EXCHANGE's protocol (engine.cu enqueue_round, kernels.cuh
    k_delta_compact / k_delta_apply): compact this rank's changed columns as
    (col, lb key, -ub key), all-gather [count, infeasible]; when every count
    is <= cap all-gather the items padded to the max count and max-merge
    them, else fall back to the dense max all-reduce."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    for inst in insts:
        r0, r1 = row_shards(inst.matrix.row_ptr, world)[rank]
        n = inst.num_cols()
        cap = max(1, n // cap_div)
        lo = np.where(np.abs(inst.bounds.lower) >= 1e20, np.sign(inst.bounds.lower) * np.inf,
                      inst.bounds.lower)
        up = np.where(np.abs(inst.bounds.upper) >= 1e20, np.sign(inst.bounds.upper) * np.inf,
                      inst.bounds.upper)
        per_round, status, sparse = [], None, 0
        for rnd in range(1, PAR.round_limit + 1):
            lo_out, up_out = lo.copy(), up.copy()
            inf = O.round_rows(inst, PAR, r0, r1, lo, up, lo_out, up_out)
            klo, knup = _key(lo_out), -_key(up_out)
            changed = np.nonzero((klo != _key(lo)) | (knup != -_key(up)))[0]
            cnt = torch.tensor([changed.shape[0], int(inf)], dtype=torch.int64)
            cnts = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(cnts, cnt)
            maxc = max(int(c[0]) for c in cnts)
            if maxc <= cap:
                sparse += 1
                items = np.zeros((maxc, 3), dtype=np.int64)
                items[:changed.shape[0]] = np.stack([changed, klo[changed], knup[changed]], 1)
                got = [torch.zeros((maxc, 3), dtype=torch.int64) for _ in range(world)]
                dist.all_gather(got, torch.from_numpy(items))
                mlo, mnup = _key(lo), -_key(up)  # the round's input keys on every rank
                for r in range(world):
                    it = got[r].numpy()[: int(cnts[r][0])]
                    np.maximum.at(mlo, it[:, 0], it[:, 1])
                    np.maximum.at(mnup, it[:, 0], it[:, 2])
                lo_out, up_out = _unkey(mlo), _unkey(-mnup)
                inf = any(int(c[1]) for c in cnts)
            else:
                buf = torch.from_numpy(np.concatenate([klo, knup, [int(inf)]]))
                dist.all_reduce(buf, op=dist.ReduceOp.MAX)
                b = buf.numpy()
                lo_out, up_out, inf = _unkey(b[:n]), _unkey(-b[n:2 * n]), bool(b[2 * n])
            ch, cinf = O.commit(lo, up, lo_out, up_out)
            per_round.append(ch)
            if inf or cinf:
                status = PropagationStatus.Infeasible
            elif ch == 0:
                status = PropagationStatus.Converged
            elif rnd == PAR.round_limit:
                status = PropagationStatus.RoundLimit
            lo, up = lo_out, up_out
            if status is not None:
                break
        out.append((int(status), per_round, lo, up, sparse))
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cap_div", [16, 400])
def test_row_sharded_delta_exchange_gloo(cap_div):
    """the sparse delta rounds give the unsharded trajectory bit for bit, with
    the product's cap (n/16) and with a small cap that forces dense fallbacks"""
    insts = [G.gen_setpart(4000, 20000, 20, f_fixed=0.2, seed=5001),
             G.gen_setpart(4000, 20000, 20, f_fixed=0.2, seed=5002, infeasible=True),
             G.gen_random(3000, 2500, 11, mean_row_nnz=9.0, integral_fraction=0.5)]
    res = _spawn(_delta_worker, 3, insts, cap_div)
    total_sparse = 0
    for i, inst in enumerate(insts):
        ref = O.propagate_parallel(inst, PAR)
        for rank in (0, 1, 2):
            status, per_round, lo, up, sparse = res[rank][i]
            assert status == int(ref.status), (inst.name, rank)
            assert per_round == ref.per_round_changes, (inst.name, rank)
            assert np.array_equal(O.canon(lo), O.canon(ref.bounds.lower))
            assert np.array_equal(O.canon(up), O.canon(ref.bounds.upper))
            assert sparse <= len(per_round)
        total_sparse += res[0][i][4]
        if cap_div == 16 and i == 0:  # C5-like: every round after the first is sparse
            assert res[0][i][4] >= 1
    assert total_sparse >= 1


def _node_worker(rank, world, port, inst, lo, up, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    k0, k1 = node_shards(lo.shape[0], world)[rank]
    mine = [O.propagate_parallel(inst, PAR, lo[k], up[k]) for k in range(k0, k1)]
    gathered = [None] * world
    dist.all_gather_object(gathered, [(int(r.status), r.rounds_executed, r.bounds.lower,
                                       r.bounds.upper) for r in mine])
    q.put((rank, [x for part in gathered for x in part]))
    dist.barrier()
    dist.destroy_process_group()


def test_node_sharded_batch_gloo():
    inst = G.gen_random(3000, 3000, 4, mean_row_nnz=8.0, integral_fraction=0.5)
    root = O.propagate_parallel(inst, PAR)
    lo, up = G.gen_nodes(inst, root.bounds.lower, root.bounds.upper, K=10, seed_base=4_000_000)
    res = _spawn(_node_worker, 2, inst, lo, up)
    for rank in (0, 1):
        assert len(res[rank]) == 10
        for k in range(10):
            ref = O.propagate_parallel(inst, PAR, lo[k], up[k])
            st, rd, l, u = res[rank][k]
            assert st == int(ref.status) and rd == ref.rounds_executed
            assert np.array_equal(O.canon(l), O.canon(ref.bounds.lower))
