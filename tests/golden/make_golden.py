"""Generate the golden vectors that pin the oracle (run in the CPU container).

Everything here is produced by the REFERENCE itself -- its sources compiled
unmodified into oracle/_ref/libpropgate_ref.so by oracle/build_ref.sh -- and
committed as small .npz fixtures, so tests/test_oracle.py can check the C
restatement (oracle/liboracle.so) and the generator restatement
(instances/libpgen.so) without /root/reference present.

  propcore.npz    compute_row_activities / residual_activities /
                  compute_bound_candidates / classify_constraint / tighten on
                  random rows (test_util.hpp:75-97 recipe, injected infinities)
  fixtures.npz    the 6 MPS fixtures (tests/fixtures, parsed by the reference's
                  parse_mps_file) with cpu_seq and cpu_par results
  cascade.npz     gen_cascade(m) results, m in {2,3,4,5,10,50,200}
  suite.npz       the acceptance suite's 500 instances (acceptance.cpp:56-75):
                  instance digests (generator check), cpu_par/cpu_seq statuses,
                  rounds, per-round changes, bound digests; full bounds for the
                  first 60 instances
  c1.npz          config C1 (gen_random 10k x 10k, mean 8, 50% int), seeds 1-5
  partition.npz   partition_row_blocks on random row-length patterns
  rounds.npz      propagate_round_parallel on random snapshots
  triplets.npz    csr_from_triplets (model.cpp:37-80): duplicates, cancelling
                  sums, summation-order-sensitive runs, empty rows, range errors

usage: python tests/golden/make_golden.py [triplets]   (needs oracle/_ref built;
       `triplets` regenerates triplets.npz only)
"""
from __future__ import annotations

import ctypes as C
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2009_07785_b200 import abi  # noqa: E402
from instances import generators as G  # noqa: E402
from paper_2009_07785_b200.model import EngineConfig, ProblemInstance  # noqa: E402

FIXTURE_DIR = "/root/reference/proj/tests/fixtures"
PAR = EngineConfig(row_check=False)


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        if a.dtype == np.float64:
            a = np.where(a == 0.0, 0.0, a)  # -0.0 == +0.0
        h.update(a.tobytes())
    return h.hexdigest()


def inst_digest(inst: ProblemInstance) -> str:
    return digest(inst.matrix.row_ptr, inst.matrix.col_idx, inst.matrix.values, inst.lhs, inst.rhs,
                  inst.bounds.lower, inst.bounds.upper, inst.integral)


def res_record(r):
    return (int(r.status), r.rounds_executed, list(r.per_round_changes), r.total_bound_changes,
            digest(r.bounds.lower, r.bounds.upper))


def propcore_vectors(rng, trials=3000):
    """Rows per test_util.hpp:75-97: len 1..10, coefs +-U[0.1,10], bounds
    U[-50,50] sorted, each side infinite with p = 0.2."""
    ref = O.ref_lib()
    cfg = PAR.to_c()
    rows = []
    for _ in range(trials):
        L = int(rng.integers(1, 11))
        coefs = rng.choice([-1.0, 1.0], L) * rng.uniform(0.1, 10.0, L)
        lo = rng.uniform(-50, 50, L)
        up = rng.uniform(-50, 50, L)
        lo, up = np.minimum(lo, up), np.maximum(lo, up)
        lo[rng.random(L) < 0.2] = -np.inf
        up[rng.random(L) < 0.2] = np.inf
        rows.append((coefs, lo, up))
    flat_len = np.array([len(c) for c, _, _ in rows], dtype=np.int32)
    coefs = np.concatenate([c for c, _, _ in rows])
    lower = np.concatenate([lo for _, lo, _ in rows])
    upper = np.concatenate([up for _, _, up in rows])
    act = np.zeros((trials, 4))
    res = np.zeros((len(coefs), 2))
    cand = np.zeros((len(coefs), 2, 2))   # [entry][integral?][lo,up]
    sides = np.zeros((trials, 2))
    klass = np.zeros(trials, dtype=np.int32)
    tight = np.zeros((len(coefs), 2))
    tkind = np.zeros(len(coefs), dtype=np.int32)
    off = 0
    for t, (cf, lo, up) in enumerate(rows):
        L = len(cf)
        cols = np.arange(L, dtype=np.int32)
        cfc = np.ascontiguousarray(cf)
        loc = np.ascontiguousarray(lo)
        upc = np.ascontiguousarray(up)
        out4 = np.zeros(4)
        ref.ref_row_activities(abi.ptr(cols, C.c_int32), abi.ptr(cfc, C.c_double), L,
                               abi.ptr(loc, C.c_double), abi.ptr(upc, C.c_double), L,
                               abi.ptr(out4, C.c_double))
        act[t] = out4
        mn = out4[0] if out4[2] == 0 else -np.inf
        mx = out4[1] if out4[3] == 0 else np.inf
        # sides around the activity range: lhs/rhs each finite with p 0.75
        lhs = mn + rng.uniform(-5, 20) if np.isfinite(mn) and rng.random() < 0.75 else -np.inf
        rhs = mx - rng.uniform(-5, 20) if np.isfinite(mx) and rng.random() < 0.75 else np.inf
        sides[t] = (lhs, rhs)
        klass[t] = ref.ref_classify(abi.ptr(out4, C.c_double), lhs, rhs, C.byref(cfg))
        for k in range(L):
            o2 = np.zeros(2)
            ref.ref_residual(abi.ptr(out4, C.c_double), cf[k], lo[k], up[k], abi.ptr(o2, C.c_double))
            res[off + k] = o2
            for integ in (0, 1):
                c2 = np.zeros(2)
                ref.ref_candidates(cf[k], lhs, rhs, o2[0], o2[1], integ, C.byref(cfg),
                                   abi.ptr(c2, C.c_double))
                cand[off + k, integ] = c2
            t2 = np.zeros(2)
            tkind[off + k] = ref.ref_tighten(lo[k], up[k], cand[off + k, 0, 0], cand[off + k, 0, 1],
                                             C.byref(cfg), abi.ptr(t2, C.c_double))
            tight[off + k] = t2
        off += L
    return dict(row_len=flat_len, coefs=coefs, lower=lower, upper=upper, act=act, res=res,
                cand=cand, sides=sides, klass=klass, tight=tight, tkind=tkind)


def save_instance(prefix, inst, out):
    out[prefix + "row_ptr"] = inst.matrix.row_ptr
    out[prefix + "col_idx"] = inst.matrix.col_idx
    out[prefix + "values"] = inst.matrix.values
    out[prefix + "lhs"] = inst.lhs
    out[prefix + "rhs"] = inst.rhs
    out[prefix + "lower"] = inst.bounds.lower
    out[prefix + "upper"] = inst.bounds.upper
    out[prefix + "integral"] = inst.integral


def save_result(prefix, r, out):
    out[prefix + "status"] = np.int32(r.status)
    out[prefix + "rounds"] = np.int32(r.rounds_executed)
    out[prefix + "per_round"] = np.array(r.per_round_changes, dtype=np.int64)
    out[prefix + "lo"] = r.bounds.lower
    out[prefix + "up"] = r.bounds.upper


def triplet_cases():
    """(name, m, n, rows, cols, vals) inputs of the csr_from_triplets vectors"""
    rng = np.random.default_rng(37)
    cases = []
    k = 600
    v = rng.integers(-3, 4, k).astype(np.float64)  # small integers: many sums cancel to 0
    cases.append(("dups", 50, 40, rng.integers(0, 50, k), rng.integers(0, 6, k), v))
    cases.append(("empty", 5, 3, np.zeros(0, int), np.zeros(0, int), np.zeros(0)))
    cases.append(("sparse_rows", 100, 10, np.array([7, 7, 93, 3, 93]), np.array([2, 1, 9, 0, 9]),
                  np.array([1.5, -2.0, 0.25, 4.0, -0.25])))
    cases.append(("signed_zero", 3, 3, np.array([0, 0, 1, 2, 2]), np.array([1, 1, 2, 0, 0]),
                  np.array([-0.0, 0.0, -0.0, 1e-300, -1e-300])))
    # input order decides the rounding of a run: (1e16 + 1) - 1e16 vs (1e16 - 1e16) + 1
    cases.append(("order", 2, 2, np.array([0, 1, 0, 1, 0, 1]), np.array([1, 1, 1, 1, 1, 1]),
                  np.array([1e16, 1e16, 1.0, -1e16, -1e16, 1.0])))
    k = 50000
    rows = rng.integers(0, 2000, k)
    cols = rng.integers(0, 3000, k)
    dup = rng.integers(0, k, k // 10)
    rows = np.concatenate([rows, rows[dup]])
    cols = np.concatenate([cols, cols[dup]])
    vals = rng.uniform(-10, 10, rows.shape[0])
    vals[k:] = np.where(rng.random(dup.shape[0]) < 0.3, -vals[dup], vals[k:])
    cases.append(("medium", 2000, 3000, rows, cols, vals))
    cases.append(("bad_row", 4, 4, np.array([0, 1, 2, 3, 4, 0]), np.array([0, 1, 2, 3, 0, 9]),
                  np.ones(6)))
    cases.append(("bad_col_first", 4, 4, np.array([0, 1, 2, 0, 9]), np.array([0, 1, 2, -1, 0]),
                  np.ones(5)))
    cases.append(("bad_both", 4, 4, np.array([0, -1]), np.array([0, 7]), np.ones(2)))
    return cases


def triplet_vectors():
    out = {}
    for name, m, n, r, c, v in triplet_cases():
        out[f"{name}/in"] = np.array([m, n], dtype=np.int64)
        out[f"{name}/rows"] = np.asarray(r, dtype=np.int32)
        out[f"{name}/cols"] = np.asarray(c, dtype=np.int32)
        out[f"{name}/vals"] = np.asarray(v, dtype=np.float64)
        try:
            rp, ci, vo = O.csr_from_triplets(r, c, v, m, n, impl="reference")
            out[f"{name}/row_ptr"] = rp
            out[f"{name}/col_idx"] = ci
            out[f"{name}/values"] = vo
        except IndexError as e:
            out[f"{name}/error"] = np.array(str(e))
    return out


def main():
    assert O.ref_available(), "build oracle/_ref first (oracle/build_ref.sh)"
    if sys.argv[1:] == ["triplets"]:
        np.savez_compressed(os.path.join(HERE, "triplets.npz"), **triplet_vectors())
        return
    rng = np.random.default_rng(20090778)
    np.savez_compressed(os.path.join(HERE, "propcore.npz"), **propcore_vectors(rng))

    out = {}
    names = []
    for base, _, files in sorted(os.walk(FIXTURE_DIR)):
        for f in sorted(files):
            if f.endswith(".mps"):
                path = os.path.join(base, f)
                name = os.path.splitext(f)[0]
                inst = O.ref_parse_mps(path)
                names.append(name)
                save_instance(name + "/", inst, out)
                for eng, fn in (("seq", O.ref_propagate_sequential), ("par", O.ref_propagate_parallel)):
                    save_result(f"{name}/{eng}/", fn(inst, PAR), out)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "fixtures.npz"), **out)

    out = {}
    for m in (2, 3, 4, 5, 10, 50, 200):
        inst = O.ref_gen_cascade(m)
        out[f"{m}/digest"] = np.array(inst_digest(inst))
        for eng, fn in (("seq", O.ref_propagate_sequential), ("par", O.ref_propagate_parallel)):
            save_result(f"{m}/{eng}/", fn(inst, PAR), out)
    np.savez_compressed(os.path.join(HERE, "cascade.npz"), **out)

    params = G.acceptance_suite_params(500)
    recs = {"params": np.array(params, dtype=np.int64)}
    inst_dig, par_dig, seq_dig = [], [], []
    par_meta, seq_meta = [], []
    par_prc, seq_prc = [], []
    full = {}
    for i, (r, c, seed, mx) in enumerate(params):
        inst = O.ref_gen_random(r, c, seed, max_nnz=mx)
        inst_dig.append(inst_digest(inst))
        par = O.ref_propagate_parallel(inst, PAR)
        seq = O.ref_propagate_sequential(inst, PAR)
        par_dig.append(digest(par.bounds.lower, par.bounds.upper))
        seq_dig.append(digest(seq.bounds.lower, seq.bounds.upper))
        par_meta.append((int(par.status), par.rounds_executed, par.total_bound_changes))
        seq_meta.append((int(seq.status), seq.rounds_executed, seq.total_bound_changes))
        par_prc.append(",".join(map(str, par.per_round_changes)))
        seq_prc.append(",".join(map(str, seq.per_round_changes)))
        if i < 60:
            full[f"{i}/par_lo"] = par.bounds.lower
            full[f"{i}/par_up"] = par.bounds.upper
            full[f"{i}/seq_lo"] = seq.bounds.lower
            full[f"{i}/seq_up"] = seq.bounds.upper
    recs.update(inst_digest=np.array(inst_dig), par_digest=np.array(par_dig),
                seq_digest=np.array(seq_dig), par_meta=np.array(par_meta),
                seq_meta=np.array(seq_meta), par_prc=np.array(par_prc),
                seq_prc=np.array(seq_prc), **full)
    np.savez_compressed(os.path.join(HERE, "suite.npz"), **recs)

    out = {}
    for seed in range(1, 6):
        inst = O.ref_gen_random(10_000, 10_000, seed, mean_row_nnz=8.0, integral_fraction=0.5)
        out[f"{seed}/digest"] = np.array(inst_digest(inst))
        for eng, fn in (("seq", O.ref_propagate_sequential), ("par", O.ref_propagate_parallel)):
            r = fn(inst, PAR)
            out[f"{seed}/{eng}/status"] = np.int32(r.status)
            out[f"{seed}/{eng}/rounds"] = np.int32(r.rounds_executed)
            out[f"{seed}/{eng}/per_round"] = np.array(r.per_round_changes, dtype=np.int64)
            out[f"{seed}/{eng}/digest"] = np.array(digest(r.bounds.lower, r.bounds.upper))
    np.savez_compressed(os.path.join(HERE, "c1.npz"), **out)

    # partition_row_blocks on random length patterns (test_par_engine.cpp:82-100)
    lib = O.ref_lib()
    out = {}
    cases = []
    for t in range(300):
        rows = int(rng.integers(1, 60))
        lens = np.where(rng.random(rows) < 0.05, 1024 + rng.integers(0, 2000, rows),
                        rng.integers(0, 120, rows)).astype(np.int32)
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        ncols = int(max(1, lens.max()))
        ci = np.concatenate([np.arange(L, dtype=np.int32) for L in lens]) if lens.sum() else np.zeros(0, np.int32)
        inst = ProblemInstance.from_arrays(rp, ci, np.ones(len(ci)), np.full(rows, -np.inf),
                                           np.full(rows, np.inf), np.zeros(ncols), np.ones(ncols))
        starts = np.zeros(rows + 1, np.int32)
        kinds = np.zeros(rows, np.int32)
        nb = C.c_int32()
        p = inst.to_c()
        cfg = PAR.to_c()
        lib.ref_partition(C.byref(p), C.byref(cfg), abi.ptr(starts, C.c_int32),
                          abi.ptr(kinds, C.c_int32), C.byref(nb))
        out[f"{t}/lens"] = lens
        out[f"{t}/starts"] = starts[: nb.value + 1]
        out[f"{t}/kinds"] = kinds[: nb.value]
        cases.append(t)
    out["count"] = np.int32(len(cases))
    np.savez_compressed(os.path.join(HERE, "partition.npz"), **out)

    # one round on random snapshots (propagate_round_parallel)
    out = {}
    for t in range(12):
        inst = O.ref_gen_random(int(rng.integers(50, 800)), int(rng.integers(50, 800)),
                                int(rng.integers(1, 1 << 30)), mean_row_nnz=7.0, integral_fraction=0.4)
        lo = inst.bounds.lower.copy()
        up = inst.bounds.upper.copy()
        # a perturbed snapshot: tighten some finite bounds a little
        sel = rng.random(lo.shape[0]) < 0.2
        lo = np.where(sel & np.isfinite(lo), lo + 0.5, lo)
        r = O.ref_propagate_round_parallel(inst, PAR, lo, up)
        save_instance(f"{t}/", inst, out)
        out[f"{t}/lb_in"] = lo
        out[f"{t}/ub_in"] = up
        out[f"{t}/lb_out"] = r["lower"]
        out[f"{t}/ub_out"] = r["upper"]
        out[f"{t}/outcome"] = np.array([r["changed"], r["infeasible"], r["changes"]], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "rounds.npz"), **out)
    np.savez_compressed(os.path.join(HERE, "triplets.npz"), **triplet_vectors())
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
