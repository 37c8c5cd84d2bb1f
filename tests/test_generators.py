"""CPU: the synthetic instance generators (SURVEY.md 8(d) recipes)."""
import os
import subprocess
import sys

import numpy as np

from instances import generators as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _digest(inst):
    import hashlib
    h = hashlib.sha256()
    for a in (inst.matrix.row_ptr, inst.matrix.col_idx, inst.matrix.values, inst.lhs, inst.rhs,
              inst.bounds.lower, inst.bounds.upper, inst.integral):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _canonical(inst):
    rp, ci = inst.matrix.row_ptr, inst.matrix.col_idx
    assert rp[0] == 0 and rp[-1] == len(ci) and np.all(np.diff(rp) >= 0)
    for i in range(min(inst.num_rows(), 2000)):
        assert np.all(np.diff(ci[rp[i]:rp[i + 1]]) > 0)  # strictly increasing columns
    assert np.all(inst.matrix.values != 0)
    assert np.all(inst.bounds.lower <= inst.bounds.upper)
    assert ci.min() >= 0 and ci.max() < inst.num_cols()


def test_powerlaw_shape():
    inst = G.gen_powerlaw(50000, 50000, 20090778)
    _canonical(inst)
    L = np.diff(inst.matrix.row_ptr)
    assert 10.5 < L.mean() < 13.5 and L.min() >= 4 and L.max() <= 10000
    assert 0.4 < inst.integral.mean() < 0.6
    assert 0.02 < np.isinf(inst.bounds.lower).mean() < 0.08


def test_longrows_shape():
    inst = G.gen_longrows(2000, 5000, 3001, long_every=100, long_min=2000, long_max=3000)
    _canonical(inst)
    L = np.diff(inst.matrix.row_ptr)
    assert np.all(L[::100] >= 2000) and np.all(L[::100] <= 3000)
    short = np.delete(L, np.arange(0, 2000, 100))
    assert 6.5 < short.mean() < 9.5


def test_setpart_planted_solution():
    inst = G.gen_setpart(5000, 25000, 50, f_fixed=0.2, seed=5001)
    _canonical(inst)
    assert np.all(np.diff(inst.matrix.row_ptr) == 50)
    assert np.all(inst.matrix.values == 1.0) and np.all(inst.lhs == 1.0) and np.all(inst.rhs == 1.0)
    assert np.all(inst.integral == 1) and np.all(inst.bounds.upper == 1.0)
    fixed = inst.bounds.lower == 1.0
    # every fixed column is an S1 column: no row holds two of them
    per_row = np.add.reduceat(fixed[inst.matrix.col_idx].astype(int), inst.matrix.row_ptr[:-1])
    assert per_row.max() <= 1
    bad = G.gen_setpart(5000, 25000, 50, f_fixed=0.2, seed=5001, infeasible=True)
    per_row = np.add.reduceat((bad.bounds.lower == 1.0)[bad.matrix.col_idx].astype(int),
                              bad.matrix.row_ptr[:-1])
    assert per_row.max() == 2


def test_nodes_branch_on_integer_columns():
    inst = G.gen_random(2000, 2000, 4, mean_row_nnz=8.0, integral_fraction=0.5)
    lo, up = G.gen_nodes(inst, inst.bounds.lower, inst.bounds.upper, K=50, seed_base=4_000_000)
    for k in range(50):
        d = np.flatnonzero((lo[k] != inst.bounds.lower) | (up[k] != inst.bounds.upper))
        assert 1 <= len(d) <= 8
        assert np.all(inst.integral[d] == 1)
        assert np.all(lo[k] <= up[k])


def test_thread_count_independent():
    code = ("import sys; sys.path.insert(0, %r); from instances import generators as G;"
            "import hashlib, numpy as np; i = G.gen_powerlaw(20000, 20000, 7);"
            "print(hashlib.sha256(np.ascontiguousarray(i.matrix.col_idx).tobytes() + "
            "i.matrix.values.tobytes() + i.rhs.tobytes()).hexdigest())" % ROOT)
    outs = set()
    for t in ("1", "3", "8"):
        env = dict(os.environ, OMP_NUM_THREADS=t)
        outs.add(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                                text=True, check=True).stdout.strip())
    assert len(outs) == 1


def test_acceptance_suite_params():
    p = G.acceptance_suite_params(500)
    assert len(p) == 500 and all(10 <= r <= 2000 and 10 <= c <= 2000 for r, c, _, _ in p)
    assert p[0][2] == 1000 and p[-1][2] == 1499
