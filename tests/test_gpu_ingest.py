"""GPU: on-device CSR build (csr_from_triplets, core/src/model.cpp:37-80) --
SURVEY.md 8(f) row 4.  Bit-exact against the reference's golden vectors and,
at larger sizes, against the C restatement (oracle/)."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2009_07785_b200.engine import csr_from_triplets_gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _same(mat, ref):
    rp, ci, v = ref
    np.testing.assert_array_equal(mat.row_ptr, rp)
    np.testing.assert_array_equal(mat.col_idx, ci)
    assert mat.values.tobytes() == v.tobytes()


@pytest.mark.gpu
def test_triplets_golden():
    d = np.load(os.path.join(GOLD, "triplets.npz"))
    for name in sorted({k.split("/")[0] for k in d.files}):
        m, n = (int(x) for x in d[f"{name}/in"])
        args = (d[f"{name}/rows"], d[f"{name}/cols"], d[f"{name}/vals"], m, n)
        if f"{name}/error" in d.files:
            with pytest.raises(IndexError, match=str(d[f"{name}/error"])):
                csr_from_triplets_gpu(*args)
            continue
        _same(csr_from_triplets_gpu(*args),
              (d[f"{name}/row_ptr"], d[f"{name}/col_idx"], d[f"{name}/values"]))


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,k,ncol", [(1_000_000, 1_000_000, 4_000_000, None),
                                        (100_000, 200_000, 2_000_000, 64),
                                        (1, 5_000_000, 1_000_000, None)])
def test_triplets_large_vs_oracle(m, n, k, ncol):
    rng = np.random.default_rng(m + k)
    r = rng.integers(0, m, k, dtype=np.int32)
    c = rng.integers(0, ncol or n, k, dtype=np.int32)
    v = rng.integers(-3, 4, k).astype(np.float64)
    v[::3] = rng.normal(size=v[::3].shape[0])
    _same(csr_from_triplets_gpu(r, c, v, m, n), O.csr_from_triplets(r, c, v, m, n))


@pytest.mark.gpu
def test_triplets_then_propagate():
    """ingest -> propagate: the device-built CSR drives the engine like the
    reference's own csr_from_triplets output"""
    from instances import generators as G
    from paper_2009_07785_b200.engine import propagate_gpu
    from paper_2009_07785_b200.model import EngineConfig, ProblemInstance
    inst = G.config_instance("c1")
    mat = inst.matrix
    rows = np.repeat(np.arange(mat.num_rows, dtype=np.int32), np.diff(mat.row_ptr))
    perm = np.random.default_rng(3).permutation(rows.shape[0])
    built = csr_from_triplets_gpu(rows[perm], mat.col_idx[perm], mat.values[perm],
                                  mat.num_rows, mat.num_cols)
    _same(built, (mat.row_ptr, mat.col_idx, mat.values))
    inst2 = ProblemInstance(built, inst.lhs, inst.rhs, inst.bounds, inst.integral)
    a = propagate_gpu(inst, EngineConfig())
    b = propagate_gpu(inst2, EngineConfig())
    assert a.status == b.status and a.rounds_executed == b.rounds_executed
    assert a.bounds.lower.tobytes() == b.bounds.lower.tobytes()
