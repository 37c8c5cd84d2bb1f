"""GPU parity at the benchmark configurations' FULL sizes,
against the reference itself.

The expected results are digests of the REFERENCE's `propagate_parallel`
(compiled from /root/reference into oracle/_ref, all host threads) committed
in tests/golden/digests.json by tests/golden/make_digests.py: status,
rounds_executed, per_round_changes, total changes and the sha256 of the
canonicalised bounds.  Bit-exact means all of them equal (acceptance.cpp:
104-117 asks for agreement on everything it benches; we ask for identity).
The instance's own sha256 is checked first, so a drifting generator is not
mistaken for an engine mismatch.

Also here: the reference's 6 MPS fixtures through the GPU, the bench's exact
mode (row check + worklist) on C2, and a run-to-run determinism check (the
GPU analogue of test_par_engine.cpp:183-210).
"""
import os

import numpy as np
import pytest

from instances import digest as D
from instances import generators as G
from paper_2009_07785_b200.engine import Session, node_overrides, propagate_gpu
from paper_2009_07785_b200.model import EngineConfig, ProblemInstance, PropagationStatus

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
DIG = D.load()


def want(cfg, seed):
    return DIG[cfg][str(seed)]


def check(res, w, what):
    diffs = D.compare(res, w["cpu_par"])
    assert not diffs, (what, diffs)


def instance(cfg, seed):
    inst = G.config_instance(cfg, seed)
    assert D.instance_sha(inst) == want(cfg, seed)["instance_sha256"], f"{cfg} generator drifted"
    return inst


@pytest.fixture(scope="module")
def c2():
    return instance("c2", 20090778)


@pytest.mark.parametrize("row_check,worklist", [(True, True), (False, False), (True, False)])
def test_c2_full_vs_reference(c2, row_check, worklist):
    """C2 in the bench's exact mode (row check on, worklist on) and the other
    modes: the reference cpu_par's result bit for bit (C2 is feasible, so
    the Step-2 row check never fires)."""
    cfg = EngineConfig(row_check=row_check, worklist=worklist)
    with Session(c2, cfg) as s:
        check(s.propagate(), want("c2", 20090778), f"c2 rc={row_check} wl={worklist}")


def test_c2_determinism_10_runs(c2):
    """10 solves of full-size C2 on one session, worklist on: identical
    per-round changes and bounds every time (red.max merges and ticketed
    slices must not make the result schedule-dependent)."""
    cfg = EngineConfig(worklist=True)
    with Session(c2, cfg) as s:
        first = D.result_digest(s.propagate())
        for _ in range(9):
            assert D.result_digest(s.propagate()) == first
    assert first == want("c2", 20090778)["cpu_par"]


def test_c2_second_seed_vs_reference():
    check(propagate_gpu(instance("c2", 20090779), EngineConfig(worklist=True)),
          want("c2", 20090779), "c2 seed 20090779")


@pytest.mark.slow
def test_c3_full_vs_reference():
    """C3 at full size: 1,000 rows of 100k-150k entries (126.5M entries,
    chunked rows: wide_row_activities order), both sweep modes."""
    inst = instance("c3", 3001)
    with Session(inst, EngineConfig(worklist=False)) as s:
        check(s.propagate(), want("c3", 3001), "c3 full sweeps")
    with Session(inst, EngineConfig(worklist=True)) as s:
        check(s.propagate(), want("c3", 3001), "c3 worklist")


@pytest.mark.slow
def test_c5_full_vs_reference():
    """C5 at full size (1M x 5M, 50M entries) and its infeasible variant."""
    inst = instance("c5", 5001)
    for wl in (True, False):
        with Session(inst, EngineConfig(worklist=wl)) as s:
            check(s.propagate(), want("c5", 5001), f"c5 wl={wl}")
    del inst
    bad = G.gen_setpart(seed=5001, infeasible=True)
    w = want("c5", 5001)["infeasible_variant"]
    assert D.instance_sha(bad) == w["instance_sha256"]
    r = propagate_gpu(bad, EngineConfig())
    assert r.status.name == w["cpu_seq_status"] == "Infeasible"
    r = propagate_gpu(bad, EngineConfig(row_check=False))
    assert r.status.name == w["cpu_par_status"]


@pytest.mark.slow
def test_c4_full_root_and_64_nodes():
    """C4 at full size: the 500k x 500k root fixpoint on the device, then
    branch-and-bound nodes 0..63 of the bench's node set, batched, each
    identical to the reference cpu_par solve of that node's bounds."""
    inst = instance("c4", 4)
    w = want("c4", 4)
    # row check off: the reference cpu_par; on (the bench's mode): the
    # restated cpu_par + row check (oracle, pinned to the reference)
    for rc, key in ((False, "nodes"), (True, "nodes_rowcheck")):
        with Session(inst, EngineConfig(worklist=True, row_check=rc)) as s:
            root = s.set_root()
            check(root, w, "c4 root")
            lo, up = G.gen_nodes(inst, root.bounds.lower, root.bounds.upper, K=len(w[key]))
            ptr, vs, ls, us = node_overrides(root.bounds.lower, root.bounds.upper, lo, up)
            st, rd, blo, bup, _ = s.propagate_nodes(ptr, vs, ls, us, want_bounds=True)
        for k, nd in enumerate(w[key]):
            got = D.node_digest(st[k], rd[k], blo[k], bup[k])
            assert got == nd, (key, k, got, nd)


def test_c1_seeds_vs_reference():
    for seed in (1, 2, 3, 4, 5):
        check(propagate_gpu(instance("c1", seed), EngineConfig(row_check=False)),
              want("c1", seed), f"c1 seed {seed}")


def test_mps_fixtures_on_gpu():
    """The reference's 6 MPS fixtures (tests/fixtures/*.mps, parsed by the
    reference's parse_mps_file into tests/golden/fixtures.npz): the GPU gives
    the reference cpu_par's result bit for bit, and cpu_seq's verdict with the
    row check on."""
    z = np.load(os.path.join(GOLD, "fixtures.npz"), allow_pickle=False)
    assert len(z["names"]) == 6
    for name in z["names"]:
        p = f"{name}/"
        inst = ProblemInstance.from_arrays(z[p + "row_ptr"], z[p + "col_idx"], z[p + "values"],
                                           z[p + "lhs"], z[p + "rhs"], z[p + "lower"],
                                           z[p + "upper"], z[p + "integral"],
                                           num_cols=z[p + "lower"].shape[0], name=str(name))
        r = propagate_gpu(inst, EngineConfig(row_check=False))
        q = f"{name}/par/"
        assert int(r.status) == int(z[q + "status"]), name
        assert r.rounds_executed == int(z[q + "rounds"]), name
        assert r.per_round_changes == list(z[q + "per_round"]), name
        assert D.bounds_sha(r.bounds.lower, r.bounds.upper) == D.bounds_sha(z[q + "lo"], z[q + "up"]), name
        rc = propagate_gpu(inst, EngineConfig(row_check=True))
        seq_inf = int(z[f"{name}/seq/status"]) == int(PropagationStatus.Infeasible)
        assert (rc.status == PropagationStatus.Infeasible) == seq_inf, name


@pytest.mark.parametrize("cfg_name,seed", [("c2", 20090778), ("c3", 3001)])
def test_narrow32_full_vs_reference(cfg_name, seed):
    """ScalarMode::Narrow32 at full size over the sliced-ELL copy: the
    reference's run_parallel<float> (float activities and candidates, double
    acceptance) bit for bit -- C3 in float is Infeasible in round 1, as the
    reference says."""
    from paper_2009_07785_b200.model import ScalarMode
    inst = instance(cfg_name, seed)
    r = propagate_gpu(inst, EngineConfig(row_check=False, scalar_mode=ScalarMode.Narrow32))
    diffs = D.compare(r, want(cfg_name, seed)["cpu_par_f32"])
    assert not diffs, diffs
