"""GPU parity: the CUDA engine (through the C-ABI) against the oracle.

Contracts:
  * vs cpu_par (propagate_parallel), row check off: status, rounds_executed,
    per_round_changes and every bound BIT-IDENTICAL (-0.0 == +0.0);
  * with the Step-2 row check on: bit-identical to the oracle's cpu_par +
    row-check mode, and verdicts identical to cpu_seq;
  * vs cpu_seq on both-converged instances: identical integer bounds,
    continuous bounds within |a-b| <= 1e-8 + 1e-5|b| (harness.cpp:17-20,
    PAPER.md:754); the 1e-9-relative pass rate is reported.
KATs mirror tests/test_par_engine.cpp and tests/test_seq_engine.cpp.
"""
import numpy as np
import pytest

from oracle import oracle as O
from instances import generators as G
from paper_2009_07785_b200.engine import (RoundSnapshot, Session, partition_row_blocks,
                                          propagate_gpu, propagate_round_gpu)
from paper_2009_07785_b200.model import (EngineConfig, LoopMode, ProblemInstance,
                                         PropagationStatus, VariableBounds, kInf)

pytestmark = pytest.mark.gpu

PAR = EngineConfig(row_check=False)
ROWCHECK = EngineConfig(row_check=True)


def assert_bit_exact(gpu, ref, what=""):
    assert gpu.status == ref.status, (what, gpu.status, ref.status)
    assert gpu.rounds_executed == ref.rounds_executed, (what, gpu.rounds_executed, ref.rounds_executed)
    assert gpu.per_round_changes == ref.per_round_changes, what
    assert gpu.total_bound_changes == ref.total_bound_changes, what
    assert np.array_equal(O.canon(gpu.bounds.lower), O.canon(ref.bounds.lower)), what
    assert np.array_equal(O.canon(gpu.bounds.upper), O.canon(ref.bounds.upper)), what


def make_instance(triplets, m, n, lhs, rhs, lower, upper, integral=None):
    rows = [[] for _ in range(m)]
    for r, c, v in triplets:
        rows[r].append((c, v))
    rp, ci, va = [0], [], []
    for r in rows:
        for c, v in sorted(r):
            ci.append(c)
            va.append(v)
        rp.append(len(ci))
    return ProblemInstance.from_arrays(rp, ci, va, lhs, rhs, lower, upper,
                                       integral if integral is not None else [0] * n, num_cols=n)


# ---- test_par_engine.cpp KATs ---------------------------------------------------

def test_round_cascade_first_round_one_change():  # test_par_engine.cpp:102-116
    inst = G.gen_cascade(3)
    snap = RoundSnapshot(inst.bounds)
    out = propagate_round_gpu(inst, snap, PAR)
    assert out.changed and not out.infeasible and out.changes == 1
    assert snap.bounds_out.upper[1] == 0.0
    assert snap.bounds_out.upper[2] == 1e6


def test_round_fixed_point_reports_no_change():  # :118-131
    inst = G.gen_cascade(4)
    fixed = propagate_gpu(inst, PAR)
    assert fixed.status == PropagationStatus.Converged
    out = propagate_round_gpu(inst, RoundSnapshot(fixed.bounds), PAR)
    assert not out.changed and out.changes == 0


def test_round_competing_uppers_merge_to_min():  # :133-152
    inst = make_instance([(0, 0, 1.0), (1, 0, 1.0)], 2, 1, [-kInf, -kInf], [5.0, 3.0], [0.0], [10.0])
    snap = RoundSnapshot(inst.bounds)
    out = propagate_round_gpu(inst, snap, PAR)
    assert out.changes == 1
    assert snap.bounds_out.upper[0] == 3.0


@pytest.mark.parametrize("m", [2, 10, 50, 200])
def test_cascade_one_round_per_link(m):  # :154-160, acceptance criteria 2/3
    r = propagate_gpu(G.gen_cascade(m), PAR)
    if m + 1 <= 100:
        assert r.status == PropagationStatus.Converged and r.rounds_executed == m + 1
    else:
        assert r.status == PropagationStatus.RoundLimit and r.rounds_executed == 100
    assert_bit_exact(r, O.propagate_parallel(G.gen_cascade(m), PAR), f"cascade{m}")


def test_fixed_point_converges_in_one_round():  # :162-173
    inst = G.gen_cascade(5)
    first = propagate_gpu(inst, PAR)
    second = propagate_gpu(inst.with_bounds(first.bounds.lower, first.bounds.upper), PAR)
    assert second.status == PropagationStatus.Converged and second.rounds_executed == 1


def test_round_limit_enforced():  # :175-181
    r = propagate_gpu(G.gen_cascade(50), EngineConfig(round_limit=5, row_check=False))
    assert r.status == PropagationStatus.RoundLimit and r.rounds_executed == 5


def test_merge_order_independent():  # :212-245
    rng = np.random.default_rng(71)
    uppers = 1.0 + rng.integers(0, 1000, 40).astype(float)
    for _ in range(5):
        rng.shuffle(uppers)
        inst = make_instance([(i, 0, 1.0) for i in range(40)], 40, 1, [-kInf] * 40, list(uppers),
                             [0.0], [1e6])
        assert propagate_gpu(inst, PAR).bounds.upper[0] == uppers.min()


def test_wide_row_matches():  # :272-292 (5000 entries: chunked long-row path)
    n = 5000
    vals = [0.5 if j % 7 else -2.0 for j in range(n)]
    inst = ProblemInstance.from_arrays([0, n], list(range(n)), vals, [-kInf], [10.0],
                                       [0.0] * n, [1.0] * n)
    gpu = propagate_gpu(inst, PAR)
    assert_bit_exact(gpu, O.propagate_parallel(inst, PAR), "wide")
    seq = O.propagate_sequential(inst, PAR)
    assert gpu.status == seq.status
    assert O.bounds_equal(seq.bounds.upper, gpu.bounds.upper).all()


def test_infeasible_toy():  # :294-304
    inst = make_instance([(0, 0, 1.0)], 1, 1, [5.0], [kInf], [0.0], [1.0])
    assert propagate_gpu(inst, PAR).status == PropagationStatus.Infeasible
    assert propagate_gpu(inst, ROWCHECK).status == PropagationStatus.Infeasible


# ---- test_seq_engine.cpp KATs ---------------------------------------------------

def test_crossed_input_zero_rounds():  # test_seq_engine.cpp:66-72
    inst = make_instance([(0, 0, 1.0)], 1, 1, [-kInf], [10.0], [2.0], [1.0])
    r = propagate_gpu(inst, ROWCHECK)
    assert r.status == PropagationStatus.Infeasible and r.rounds_executed == 0
    assert r.bounds.lower[0] == 2.0 and r.bounds.upper[0] == 1.0


def test_integer_fixing_example():  # :45-56
    inst = make_instance([(0, 0, 1.0), (0, 1, 1.0), (1, 0, 1.0)], 2, 2, [-kInf, 1.0], [1.0, kInf],
                         [0.0, 0.0], [1.0, 1.0], [1, 1])
    r = propagate_gpu(inst, ROWCHECK)
    assert r.status == PropagationStatus.Converged
    assert list(r.bounds.lower) == [1.0, 0.0] and list(r.bounds.upper) == [1.0, 0.0]


def test_verdict_counterexample_rowcheck():
    """x - y <= -1e-4 with x = y = 1e4 fixed: cpu_seq says
    Infeasible, cpu_par Converged; the row check restores cpu_seq's verdict."""
    inst = make_instance([(0, 0, 1.0), (0, 1, -1.0)], 1, 2, [-kInf], [-1e-4], [1e4, 1e4], [1e4, 1e4])
    assert O.propagate_sequential(inst, PAR).status == PropagationStatus.Infeasible
    assert propagate_gpu(inst, PAR).status == PropagationStatus.Converged
    assert propagate_gpu(inst, ROWCHECK).status == PropagationStatus.Infeasible


def test_config_validation_errors():
    inst = G.gen_cascade(3)
    for bad in [EngineConfig(round_limit=0), EngineConfig(infinity_threshold=0.0),
                EngineConfig(improvement_abs=0.0), EngineConfig(integrality_eps=-1.0),
                EngineConfig(vector_threshold=0), EngineConfig(nnz_budget=10, vector_threshold=64),
                EngineConfig(worker_count=-1)]:
        with pytest.raises(ValueError):
            propagate_gpu(inst, bad)


def test_empty_rows_and_columns():
    inst = ProblemInstance.from_arrays([0, 0, 2, 2], [0, 2], [1.0, 1.0], [-kInf, -kInf, -kInf],
                                       [1.0, 4.0, -1.0], [0.0, 0.0, 0.0, 0.0], [9.0] * 4)
    assert_bit_exact(propagate_gpu(inst, PAR), O.propagate_parallel(inst, PAR), "empty")
    assert_bit_exact(propagate_gpu(inst, ROWCHECK), O.propagate_parallel(inst, ROWCHECK), "empty rc")
    # empty row with rhs = -1 is infeasible for cpu_seq's row check
    assert propagate_gpu(inst, ROWCHECK).status == PropagationStatus.Infeasible


# ---- random suites ------------------------------------------------------------------

def _suite_compare(instances, stats):
    for inst in instances:
        gpu = propagate_gpu(inst, PAR)
        assert_bit_exact(gpu, O.propagate_parallel(inst, PAR), inst.name)
        gpu_rc = propagate_gpu(inst, ROWCHECK)
        assert_bit_exact(gpu_rc, O.propagate_parallel(inst, ROWCHECK), inst.name + " rowcheck")
        seq = O.propagate_sequential(inst, PAR)
        assert (gpu_rc.status == PropagationStatus.Infeasible) == (
            seq.status == PropagationStatus.Infeasible), inst.name
        if seq.status == PropagationStatus.Converged and gpu_rc.status == PropagationStatus.Converged:
            stats["both"] += 1
            integ = inst.integral.astype(bool)
            for a, b in [(seq.bounds.lower, gpu_rc.bounds.lower), (seq.bounds.upper, gpu_rc.bounds.upper)]:
                assert np.array_equal(a[integ], b[integ]), inst.name
                assert O.bounds_equal(a, b).all(), inst.name
            tight = all(O.bounds_equal(a, b, 1e-9, 1e-9).all() for a, b in
                        [(seq.bounds.lower, gpu_rc.bounds.lower), (seq.bounds.upper, gpu_rc.bounds.upper)])
            stats["tight"] += int(tight)


def test_acceptance_suite_parity():
    """The reference acceptance suite's 500 random instances (acceptance.cpp:56-75)."""
    stats = {"both": 0, "tight": 0}
    _suite_compare(G.acceptance_suite(500), stats)
    assert stats["both"] > 450
    print(f"\nboth converged {stats['both']}/500; within 1e-9 of cpu_seq: {stats['tight']}")


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_config1_parity(seed):
    stats = {"both": 0, "tight": 0}
    _suite_compare([G.config_instance("c1", seed)], stats)


def test_loop_modes_identical():
    inst = G.gen_random(3000, 2500, 99, mean_row_nnz=10.0, integral_fraction=0.5)
    a = propagate_gpu(inst, EngineConfig(row_check=False, loop_mode=LoopMode.Graph))
    b = propagate_gpu(inst, EngineConfig(row_check=False, loop_mode=LoopMode.Host))
    assert_bit_exact(a, b, "loop modes")


def test_round_api_matches_oracle_round():
    inst = G.gen_random(1500, 1200, 5, mean_row_nnz=9.0, integral_fraction=0.5)
    lo, up = inst.bounds.lower.copy(), inst.bounds.upper.copy()
    for _ in range(4):
        snap = RoundSnapshot(VariableBounds(lo, up))
        out = propagate_round_gpu(inst, snap, PAR)
        ref = O.propagate_round_parallel(inst, PAR, lo, up)
        assert out.changes == ref["changes"] and out.infeasible == ref["infeasible"]
        assert np.array_equal(O.canon(snap.bounds_out.lower), O.canon(ref["lower"]))
        assert np.array_equal(O.canon(snap.bounds_out.upper), O.canon(ref["upper"]))
        lo, up = snap.bounds_out.lower, snap.bounds_out.upper


def test_session_round_matches_oracle_round():
    """pg_session_round: the one-round API on a resident session (matrix set
    up once), chained like a branch-and-bound caller would."""
    inst = G.gen_powerlaw(20000, 20000, 5, cap=3000)
    lo, up = inst.bounds.lower.copy(), inst.bounds.upper.copy()
    for cfg in (EngineConfig(row_check=True), EngineConfig(row_check=False, worklist=True)):
        lo, up = inst.bounds.lower.copy(), inst.bounds.upper.copy()
        with Session(inst, cfg) as s:
            for _ in range(4):
                snap = RoundSnapshot(VariableBounds(lo, up))
                out = s.round(snap)
                ref = O.propagate_round_parallel(inst, PAR, lo, up)
                assert out.changes == ref["changes"] and out.infeasible == ref["infeasible"]
                assert np.array_equal(O.canon(snap.bounds_out.lower), O.canon(ref["lower"]))
                assert np.array_equal(O.canon(snap.bounds_out.upper), O.canon(ref["upper"]))
                lo, up = snap.bounds_out.lower, snap.bounds_out.upper
            # the session still solves normally afterwards (row check restored)
            assert_bit_exact(s.propagate(), O.propagate_parallel(inst, cfg), "after rounds")


@pytest.mark.parametrize("loop", [LoopMode.Graph, LoopMode.Host])
def test_small_budget_short_split_rows(loop):
    """nnz_budget < 32: split rows of nnz_budget < len <= 32 entries go on the
    short phase-2 queue; the persistent loop (Graph mode, small instance) and
    the per-phase kernels (Host mode) must both drain it."""
    inst = G.gen_random(3000, 2500, 21, mean_row_nnz=24.0, integral_fraction=0.5)
    for budget, vt in ((16, 8), (20, 4), (8, 8)):
        cfg = EngineConfig(row_check=False, nnz_budget=budget, vector_threshold=vt, loop_mode=loop)
        assert_bit_exact(propagate_gpu(inst, cfg), O.propagate_parallel(inst, cfg),
                         f"budget {budget}")


def test_bad_indices_rejected_without_poisoning_the_context():
    """Out-of-range col_idx / non-monotone row_ptr: PG_EINVAL, not a device
    fault (the reference has undefined behaviour here); later solves in the
    same process still work.  PG_EINVAL surfaces as ValueError, like the
    reference's std::invalid_argument."""
    inst = G.gen_random(500, 400, 3, mean_row_nnz=6.0)
    bad = G.gen_random(500, 400, 3, mean_row_nnz=6.0)
    bad.matrix.col_idx[7] = 400 + 12345
    with pytest.raises(ValueError) as e:
        propagate_gpu(bad, PAR)
    assert "col_idx" in str(e.value)
    bad2 = G.gen_random(500, 400, 3, mean_row_nnz=6.0)
    bad2.matrix.col_idx[3] = -5
    with pytest.raises(ValueError):
        propagate_gpu(bad2, EngineConfig(row_check=False, worklist=True))
    bad3 = G.gen_random(500, 400, 3, mean_row_nnz=6.0)
    rp = bad3.matrix.row_ptr
    rp[10], rp[11] = rp[11], rp[10] - 1
    with pytest.raises(ValueError) as e:
        propagate_gpu(bad3, PAR)
    assert "row_ptr" in str(e.value)
    assert_bit_exact(propagate_gpu(inst, PAR), O.propagate_parallel(inst, PAR), "after bad input")


def test_partition_matches_reference_partitioner():
    inst = G.gen_random(3000, 3000, 11, mean_row_nnz=40.0)
    starts, kinds = partition_row_blocks(inst, PAR)
    m = inst.num_rows()
    s2 = np.zeros(m + 1, np.int32)
    import ctypes as C
    from paper_2009_07785_b200 import abi
    k2 = np.zeros(m, np.int32)
    nb = C.c_int32()
    p = inst.to_c()
    c = PAR.to_c()
    O.oracle_lib().orc_partition_row_blocks(C.byref(p), C.byref(c), abi.ptr(s2, C.c_int32),
                                            abi.ptr(k2, C.c_int32), C.byref(nb))
    assert np.array_equal(starts, s2[: nb.value + 1]) and np.array_equal(kinds, k2[: nb.value])


def test_session_warm_start_and_batch():
    inst = G.gen_random(4000, 4000, 21, mean_row_nnz=8.0, integral_fraction=0.5)
    root = O.propagate_parallel(inst, PAR)
    lo, up = G.gen_nodes(inst, root.bounds.lower, root.bounds.upper, K=6, seed_base=77)
    with Session(inst, PAR) as s:
        r0 = s.propagate()
        assert_bit_exact(r0, root, "session root")
        blo, bup, bst, brd = s.propagate_batch(lo, up)
        for k in range(6):
            ref = O.propagate_parallel(inst, PAR, lo[k], up[k])
            assert bst[k] == int(ref.status) and brd[k] == ref.rounds_executed
            assert np.array_equal(O.canon(blo[k]), O.canon(ref.bounds.lower))
            assert np.array_equal(O.canon(bup[k]), O.canon(ref.bounds.upper))
            single = s.propagate(lo[k], up[k])
            assert_bit_exact(single, ref, f"node {k}")


@pytest.mark.parametrize("budget", [64, 256, 4096])
def test_nnz_budget_changes_long_row_order(budget):
    """Rows longer than nnz_budget are summed in nnz_budget chunks combined
    pairwise (par_engine.cpp:99-123); the GPU follows any budget."""
    inst = G.gen_random(800, 3000, 3, mean_row_nnz=300.0, integral_fraction=0.5)
    cfg = EngineConfig(row_check=False, nnz_budget=budget)
    assert_bit_exact(propagate_gpu(inst, cfg), O.propagate_parallel(inst, cfg), f"budget {budget}")


@pytest.mark.slow
def test_config2_full_size_bit_exact():
    """C2 (1M x 1M power-law, ~12M entries): the full solve is bit-identical
    to the restated cpu_par (status, rounds, per-round changes, bounds), with
    full sweeps and with worklist rounds (the bench's mode)."""
    inst = G.config_instance("c2")
    ref = O.propagate_parallel(inst, PAR)
    assert_bit_exact(propagate_gpu(inst, PAR), ref, "c2")
    assert_bit_exact(propagate_gpu(inst, EngineConfig(row_check=False, worklist=True)), ref,
                     "c2 worklist")


@pytest.mark.parametrize("worklist", [False, True])
@pytest.mark.parametrize("row_check", [False, True])
def test_worklist_modes_identical(worklist, row_check):
    """The device-side worklist is exact: same trajectory with it on and off."""
    for seed in (3, 8, 13):
        inst = G.gen_random(3000, 2500, seed, mean_row_nnz=9.0, integral_fraction=0.5)
        cfg = EngineConfig(row_check=row_check, worklist=worklist)
        assert_bit_exact(propagate_gpu(inst, cfg), O.propagate_parallel(inst, cfg), inst.name)
    inst = G.gen_powerlaw(20000, 20000, 77, cap=3000)
    cfg = EngineConfig(row_check=row_check, worklist=worklist, nnz_budget=256)
    assert_bit_exact(propagate_gpu(inst, cfg), O.propagate_parallel(inst, cfg), inst.name)


# ---- ScalarMode::Narrow32 (model.hpp:129) -------------------
def _f32(row_check=False, **kw):
    from paper_2009_07785_b200.model import ScalarMode
    return EngineConfig(row_check=row_check, scalar_mode=ScalarMode.Narrow32, **kw)


def test_f32_acceptance_suite_parity():
    """Float working copy, float activities/candidates, double acceptance:
    bit-identical to the oracle's run_parallel<float> (pinned to the reference
    in tests/test_oracle.py::test_f32_mode_matches_reference)."""
    cfg = _f32()
    for r, c, seed, mx in G.acceptance_suite_params(80):
        inst = G.gen_random(r, c, seed, max_nnz=mx)
        assert_bit_exact(propagate_gpu(inst, cfg), O.propagate_parallel(inst, cfg), (r, c, seed))


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("row_check", [False, True])
def test_f32_config1_parity(seed, row_check):
    inst = G.config_instance("c1", seed)
    cfg = _f32(row_check=row_check)
    assert_bit_exact(propagate_gpu(inst, cfg), O.propagate_parallel(inst, cfg), seed)


@pytest.mark.parametrize("budget", [64, 256])
def test_f32_chunked_long_rows(budget):
    """Rows longer than nnz_budget: float chunk partials combined pairwise."""
    inst = G.gen_random(300, 4000, 11, mean_row_nnz=400.0, integral_fraction=0.3)
    cfg = _f32(nnz_budget=budget, vector_threshold=64)
    assert_bit_exact(propagate_gpu(inst, cfg), O.propagate_parallel(inst, cfg), budget)


def test_f32_round_api_is_double():
    """propagate_round_parallel always works in double (par_engine.cpp:282)."""
    inst = G.gen_random(2000, 1500, 5, mean_row_nnz=8.0, integral_fraction=0.5)
    lo = np.array(inst.bounds.lower, dtype=float)
    up = np.array(inst.bounds.upper, dtype=float)
    sa = RoundSnapshot(VariableBounds(lo.copy(), up.copy()))
    sb = RoundSnapshot(VariableBounds(lo.copy(), up.copy()))
    oa = propagate_round_gpu(inst, sa, _f32())
    ob = propagate_round_gpu(inst, sb, PAR)
    assert oa.changes == ob.changes and oa.changes > 0
    assert np.array_equal(O.canon(sa.bounds_out.lower), O.canon(sb.bounds_out.lower))
    assert np.array_equal(O.canon(sa.bounds_out.upper), O.canon(sb.bounds_out.upper))


@pytest.mark.parametrize("mode", ["dense", "worklist", "f32", "host", "f32_worklist"])
def test_modes_on_edge_instances(mode):
    """Every engine mode on degenerate shapes: empty rows / columns, a single
    entry, all-infinite bounds, a crossed start (0 rounds), a chunked row."""
    from paper_2009_07785_b200.model import ScalarMode
    kw = dict(row_check=False)
    if "worklist" in mode:
        kw["worklist"] = True
    if "f32" in mode:
        kw["scalar_mode"] = ScalarMode.Narrow32
    if mode == "host":
        kw["loop_mode"] = LoopMode.Host
    cfg = EngineConfig(**kw)
    cases = [
        ProblemInstance.from_arrays([0, 0, 2, 2], [0, 2], [1.0, 1.0], [-kInf, -kInf, -kInf],
                                    [1.0, 4.0, -1.0], [0.0] * 4, [9.0] * 4),
        ProblemInstance.from_arrays([0, 1], [0], [2.0], [-kInf], [3.0], [-kInf], [kInf]),
        ProblemInstance.from_arrays([0, 2], [0, 1], [1.0, -1.0], [0.0], [0.0], [-kInf, 2.0],
                                    [kInf, 5.0]),
        ProblemInstance.from_arrays([0, 1], [0], [1.0], [-kInf], [1.0], [3.0], [2.0]),  # crossed
        G.gen_random(50, 3000, 17, mean_row_nnz=300.0, integral_fraction=0.5),
        G.gen_cascade(30),
    ]
    for k, inst in enumerate(cases):
        assert_bit_exact(propagate_gpu(inst, cfg), O.propagate_parallel(inst, cfg), (mode, k))


_GATHER_SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np
from oracle import oracle as O
from instances import generators as G
from paper_2009_07785_b200.engine import propagate_gpu
from paper_2009_07785_b200.model import EngineConfig
PAR = EngineConfig(row_check=False)
insts = [G.gen_powerlaw(100000, 100000, 20090778, cap=2000),
         G.gen_longrows(3000, 6000, 3001, long_every=100, long_min=1500, long_max=4000),
         G.gen_random(20000, 20000, 5, mean_row_nnz=8.0, integral_fraction=0.5),
         G.gen_setpart(20000, 100000, 20, seed=5001)]
for inst in insts:
    for wl in (False, True):
        g = propagate_gpu(inst, EngineConfig(row_check=False, worklist=wl))
        r = O.propagate_parallel(inst, PAR)
        assert int(g.status) == int(r.status) and g.rounds_executed == r.rounds_executed, inst.name
        assert list(g.per_round_changes) == list(r.per_round_changes), inst.name
        assert np.array_equal(O.canon(g.bounds.lower), O.canon(r.bounds.lower)), inst.name
        assert np.array_equal(O.canon(g.bounds.upper), O.canon(r.bounds.upper)), inst.name
print("ok")
"""


@pytest.mark.gpu
@pytest.mark.parametrize("gather", ["8", "16", "32"])
def test_gather_record_modes(gather):
    """every gather record (8 B float bounds with the exact 16 B record for
    bounds that are not floats, 16 B bounds + recomputed q, 32 B snapshot)
    forced on instances of every kind: bit-exact with the oracle"""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PG_SELL_GATHER=gather)
    p = subprocess.run([sys.executable, "-c", _GATHER_SCRIPT.format(root=root)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and "ok" in p.stdout, p.stdout + p.stderr
