"""CPU: pin the oracle (C restatement, oracle/liboracle.so) and the generator
restatement (libpgen.so) against golden vectors produced by the reference
itself (tests/golden/make_golden.py, compiled reference in oracle/_ref).

Bit-exact everywhere: integer/index work, statuses, round counts, per-round
change counts, and every bound (-0.0 == +0.0).
"""
import ctypes as C
import hashlib
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2009_07785_b200 import abi
from instances import generators as G
from paper_2009_07785_b200.model import EngineConfig, ProblemInstance, PropagationStatus

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
PAR = EngineConfig(row_check=False)


def load(name):
    return np.load(os.path.join(GOLD, name), allow_pickle=False)


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        if a.dtype == np.float64:
            a = np.where(a == 0.0, 0.0, a)
        h.update(a.tobytes())
    return h.hexdigest()


def inst_digest(inst):
    return digest(inst.matrix.row_ptr, inst.matrix.col_idx, inst.matrix.values, inst.lhs, inst.rhs,
                  inst.bounds.lower, inst.bounds.upper, inst.integral)


def same(a, b):
    return np.array_equal(O.canon(np.asarray(a)), O.canon(np.asarray(b)))


def instance_from(z, prefix):
    return ProblemInstance.from_arrays(z[prefix + "row_ptr"], z[prefix + "col_idx"], z[prefix + "values"],
                                       z[prefix + "lhs"], z[prefix + "rhs"], z[prefix + "lower"],
                                       z[prefix + "upper"], z[prefix + "integral"],
                                       num_cols=z[prefix + "lower"].shape[0])


# ---- propcore (test_propcore.cpp hand KATs + golden random rows) ---------------------

def _act(cols, coefs, lo, up):
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    coefs = np.ascontiguousarray(coefs, dtype=np.float64)
    lo = np.ascontiguousarray(lo, dtype=np.float64)
    up = np.ascontiguousarray(up, dtype=np.float64)
    out = np.zeros(4)
    O.oracle_lib().orc_row_activities(abi.ptr(cols, C.c_int32), abi.ptr(coefs, C.c_double),
                                      len(cols), abi.ptr(lo, C.c_double), abi.ptr(up, C.c_double),
                                      abi.ptr(out, C.c_double))
    return out


def _cand(a, lhs, rhs, mn, mx, integral):
    out = np.zeros(2)
    cfg = PAR.to_c()
    O.oracle_lib().orc_candidates(a, lhs, rhs, mn, mx, integral, C.byref(cfg), abi.ptr(out, C.c_double))
    return out


def test_propcore_hand_kats():
    inf = np.inf
    # test_propcore.cpp:15-26 row {x: 1, y: -2}, l = (0, 1), u = (2, 3)
    assert list(_act([0, 1], [1.0, -2.0], [0.0, 1.0], [2.0, 3.0])) == [-6.0, 0.0, 0, 0]
    # :28-37 single infinite term isolated
    assert list(_act([0], [1.0], [-inf], [5.0])) == [0.0, 5.0, 1, 0]
    # :39-45 empty row
    assert list(_act([], [], [], [])) == [0.0, 0.0, 0, 0]
    # :137-143 2x <= 10 with residual 0 -> x <= 5
    assert list(_cand(2.0, -inf, 10.0, 0.0, -inf, 0)) == [-inf, 5.0]
    # :145-149 integral rounding 10/3 -> 3
    assert _cand(3.0, -inf, 10.0, 0.0, -inf, 1)[1] == 3.0
    # :151-156 infinite side non-binding, lhs side -> -3
    assert list(_cand(1.0, 2.0, inf, 0.0, 5.0, 0)) == [-3.0, inf]
    # :158-163 negative coefficient swaps sides
    assert list(_cand(-2.0, -inf, 6.0, 0.0, -inf, 0)) == [-3.0, inf]
    # :165-175 1e21 reaches the infinity threshold, 1e19 kept
    assert _cand(1e-20, -inf, 10.0, 0.0, -inf, 0)[1] == inf
    assert _cand(1e-18, -inf, 10.0, 0.0, -inf, 0)[1] == 1e19


def test_propcore_golden_rows():
    z = load("propcore.npz")
    nrows = len(z["row_len"])
    ne = len(z["coefs"])
    act = np.zeros((nrows, 4))
    klass = np.zeros(nrows, np.int32)
    res = np.zeros((ne, 2))
    cand = np.zeros((ne, 2, 2))
    tight = np.zeros((ne, 2))
    tkind = np.zeros(ne, np.int32)
    arrs = {k: np.ascontiguousarray(z[k]) for k in ("row_len", "coefs", "lower", "upper", "sides")}
    cfg = PAR.to_c()
    O.oracle_lib().orc_propcore_rows(
        nrows, abi.ptr(arrs["row_len"], C.c_int32), abi.ptr(arrs["coefs"], C.c_double),
        abi.ptr(arrs["lower"], C.c_double), abi.ptr(arrs["upper"], C.c_double),
        abi.ptr(arrs["sides"], C.c_double), C.byref(cfg), abi.ptr(act, C.c_double),
        abi.ptr(klass, C.c_int32), abi.ptr(res, C.c_double), abi.ptr(cand, C.c_double),
        abi.ptr(tight, C.c_double), abi.ptr(tkind, C.c_int32))
    assert same(act, z["act"])
    assert np.array_equal(klass, z["klass"])
    assert same(res, z["res"])
    assert same(cand, z["cand"])
    assert np.array_equal(tkind, z["tkind"])
    assert same(tight, z["tight"])
    # the KATs exercise every classification and tighten outcome
    assert set(np.unique(z["klass"])) == {0, 1, 2}
    assert set(np.unique(z["tkind"])) >= {0, 1, 2, 4}


# ---- engines ----------------------------------------------------------------------------

def test_mps_fixtures():
    z = load("fixtures.npz")
    assert len(z["names"]) == 6
    for name in z["names"]:
        inst = instance_from(z, f"{name}/")
        for eng, fn in (("seq", O.propagate_sequential), ("par", O.propagate_parallel)):
            r = fn(inst, PAR)
            p = f"{name}/{eng}/"
            assert int(r.status) == int(z[p + "status"]), (name, eng)
            assert r.rounds_executed == int(z[p + "rounds"]), (name, eng)
            assert r.per_round_changes == list(z[p + "per_round"]), (name, eng)
            assert same(r.bounds.lower, z[p + "lo"]) and same(r.bounds.upper, z[p + "up"]), (name, eng)
    assert int(z["toy_infeasible/seq/status"]) == int(PropagationStatus.Infeasible)


@pytest.mark.parametrize("m", [2, 3, 4, 5, 10, 50, 200])
def test_cascade(m):
    z = load("cascade.npz")
    inst = G.gen_cascade(m)
    assert inst_digest(inst) == str(z[f"{m}/digest"])  # generator restatement
    for eng, fn in (("seq", O.propagate_sequential), ("par", O.propagate_parallel)):
        r = fn(inst, PAR)
        p = f"{m}/{eng}/"
        assert int(r.status) == int(z[p + "status"]) and r.rounds_executed == int(z[p + "rounds"])
        assert r.per_round_changes == list(z[p + "per_round"])
        assert same(r.bounds.lower, z[p + "lo"]) and same(r.bounds.upper, z[p + "up"])


def test_acceptance_suite():
    """acceptance.cpp criterion 1 instances: generator restatement bit-exact;
    restated cpu_par and cpu_seq bit-exact with the reference."""
    z = load("suite.npz")
    params = z["params"]
    assert [tuple(p) for p in params] == G.acceptance_suite_params(500)
    for i, (r, c, seed, mx) in enumerate(params):
        inst = G.gen_random(int(r), int(c), int(seed), max_nnz=int(mx))
        assert inst_digest(inst) == str(z["inst_digest"][i]), i
        par = O.propagate_parallel(inst, PAR)
        seq = O.propagate_sequential(inst, PAR)
        assert (int(par.status), par.rounds_executed, par.total_bound_changes) == tuple(z["par_meta"][i])
        assert (int(seq.status), seq.rounds_executed, seq.total_bound_changes) == tuple(z["seq_meta"][i])
        assert ",".join(map(str, par.per_round_changes)) == str(z["par_prc"][i])
        assert ",".join(map(str, seq.per_round_changes)) == str(z["seq_prc"][i])
        assert digest(par.bounds.lower, par.bounds.upper) == str(z["par_digest"][i]), i
        assert digest(seq.bounds.lower, seq.bounds.upper) == str(z["seq_digest"][i]), i
        if i < 60:
            assert same(par.bounds.lower, z[f"{i}/par_lo"]) and same(seq.bounds.upper, z[f"{i}/seq_up"])


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_config1(seed):
    z = load("c1.npz")
    inst = G.config_instance("c1", seed)
    assert inst_digest(inst) == str(z[f"{seed}/digest"])
    for eng, fn in (("seq", O.propagate_sequential), ("par", O.propagate_parallel)):
        r = fn(inst, PAR)
        p = f"{seed}/{eng}/"
        assert int(r.status) == int(z[p + "status"]) and r.rounds_executed == int(z[p + "rounds"])
        assert r.per_round_changes == list(z[p + "per_round"])
        assert digest(r.bounds.lower, r.bounds.upper) == str(z[p + "digest"])


def test_partition_row_blocks():
    z = load("partition.npz")
    lib = O.oracle_lib()
    for t in range(int(z["count"])):
        lens = z[f"{t}/lens"]
        rows = len(lens)
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        ci = np.concatenate([np.arange(L, dtype=np.int32) for L in lens]) if lens.sum() else np.zeros(0, np.int32)
        ncols = int(max(1, lens.max()))
        inst = ProblemInstance.from_arrays(rp, ci, np.ones(len(ci)), np.full(rows, -np.inf),
                                           np.full(rows, np.inf), np.zeros(ncols), np.ones(ncols))
        starts = np.zeros(rows + 1, np.int32)
        kinds = np.zeros(rows, np.int32)
        nb = C.c_int32()
        p = inst.to_c()
        cfg = PAR.to_c()
        lib.orc_partition_row_blocks(C.byref(p), C.byref(cfg), abi.ptr(starts, C.c_int32),
                                     abi.ptr(kinds, C.c_int32), C.byref(nb))
        assert np.array_equal(starts[: nb.value + 1], z[f"{t}/starts"])
        assert np.array_equal(kinds[: nb.value], z[f"{t}/kinds"])


def test_round_parallel():
    z = load("rounds.npz")
    for t in range(12):
        inst = instance_from(z, f"{t}/")
        r = O.propagate_round_parallel(inst, PAR, z[f"{t}/lb_in"], z[f"{t}/ub_in"])
        assert [r["changed"], r["infeasible"], r["changes"]] == list(z[f"{t}/outcome"])
        assert same(r["lower"], z[f"{t}/lb_out"]) and same(r["upper"], z[f"{t}/ub_out"])


def test_config_validation():
    lib = O.oracle_lib()
    for bad in [EngineConfig(round_limit=0), EngineConfig(infinity_threshold=0.0),
                EngineConfig(improvement_rel=0.0), EngineConfig(integrality_eps=0.0),
                EngineConfig(vector_threshold=0), EngineConfig(nnz_budget=10, vector_threshold=64),
                EngineConfig(worker_count=-1)]:
        c = bad.to_c()
        assert lib.orc_validate(C.byref(c)) == abi.PG_EINVAL
    c = EngineConfig().to_c()
    assert lib.orc_validate(C.byref(c)) == 0


def test_rowcheck_mode_verdicts_match_seq():
    """The row-check mode (the GPU default) on the suite: infeasibility
    verdicts equal cpu_seq's."""
    for r, c, seed, mx in G.acceptance_suite_params(120):
        inst = G.gen_random(r, c, seed, max_nnz=mx)
        rc = O.propagate_parallel(inst, EngineConfig(row_check=True))
        seq = O.propagate_sequential(inst, PAR)
        assert (rc.status == PropagationStatus.Infeasible) == (seq.status == PropagationStatus.Infeasible)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_restatement_vs_compiled_reference_live():
    """When the compiled reference is present: live cross-check on fresh seeds
    (cpu_par bit-exact incl. a wide row > nnz_budget; cpu_seq bit-exact)."""
    rng = np.random.default_rng(7)
    for _ in range(20):
        inst = G.gen_random(int(rng.integers(20, 600)), int(rng.integers(20, 600)),
                            int(rng.integers(1, 1 << 40)), mean_row_nnz=float(rng.uniform(3, 60)),
                            integral_fraction=0.5)
        for mine, ref in ((O.propagate_parallel, O.ref_propagate_parallel),
                          (O.propagate_sequential, O.ref_propagate_sequential)):
            a, b = mine(inst, PAR), ref(inst, PAR)
            assert (a.status, a.rounds_executed, a.per_round_changes) == (b.status, b.rounds_executed, b.per_round_changes)
            assert same(a.bounds.lower, b.bounds.lower) and same(a.bounds.upper, b.bounds.upper)
    n = 5000
    vals = [0.5 if j % 7 else -2.0 for j in range(n)]
    inst = ProblemInstance.from_arrays([0, n], list(range(n)), vals, [-np.inf], [10.0], [0.0] * n, [1.0] * n)
    a, b = O.propagate_parallel(inst, PAR), O.ref_propagate_parallel(inst, PAR)
    assert same(a.bounds.upper, b.bounds.upper)


def test_f32_mode_matches_reference():
    """ScalarMode::Narrow32 (model.hpp:129) restated; vs the compiled reference."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    from paper_2009_07785_b200.model import ScalarMode
    cfg = EngineConfig(row_check=False, scalar_mode=ScalarMode.Narrow32)
    for r, c, seed, mx in G.acceptance_suite_params(60):
        inst = G.gen_random(r, c, seed, max_nnz=mx)
        a, b = O.propagate_parallel(inst, cfg), O.ref_propagate_parallel(inst, cfg)
        assert (a.status, a.rounds_executed, a.per_round_changes) == (b.status, b.rounds_executed, b.per_round_changes)
        assert same(a.bounds.lower, b.bounds.lower) and same(a.bounds.upper, b.bounds.upper)
        a, b = O.propagate_sequential(inst, cfg), O.ref_propagate_sequential(inst, cfg)
        assert same(a.bounds.lower, b.bounds.lower) and same(a.bounds.upper, b.bounds.upper)


def _triplet_cases():
    d = load("triplets.npz")
    names = sorted({k.split("/")[0] for k in d.files})
    return d, names


def test_csr_from_triplets_golden():
    """csr_from_triplets (model.cpp:37-80): the C restatement reproduces the
    reference's CSR (order, duplicate sums, dropped zeros) and its
    out_of_range messages on every golden case"""
    d, names = _triplet_cases()
    assert len(names) >= 9
    for name in names:
        m, n = (int(x) for x in d[f"{name}/in"])
        args = (d[f"{name}/rows"], d[f"{name}/cols"], d[f"{name}/vals"], m, n)
        if f"{name}/error" in d.files:
            with pytest.raises(IndexError, match=str(d[f"{name}/error"])):
                O.csr_from_triplets(*args)
            continue
        rp, ci, v = O.csr_from_triplets(*args)
        np.testing.assert_array_equal(rp, d[f"{name}/row_ptr"])
        np.testing.assert_array_equal(ci, d[f"{name}/col_idx"])
        assert v.tobytes() == d[f"{name}/values"].tobytes(), name


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_csr_from_triplets_vs_reference_live():
    rng = np.random.default_rng(5)
    for trial in range(5):
        m, n, k = 300, 200, 20000
        r = rng.integers(0, m, k)
        c = rng.integers(0, 8 if trial % 2 else n, k)
        v = rng.integers(-2, 3, k).astype(np.float64) if trial < 3 else rng.normal(size=k)
        a = O.csr_from_triplets(r, c, v, m, n)
        b = O.csr_from_triplets(r, c, v, m, n, impl="reference")
        for x, y in zip(a, b):
            assert x.tobytes() == y.tobytes()
