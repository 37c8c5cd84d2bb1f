"""MPS ingest: the host-parallel reader behind
pg_mps_read (paper_2009_07785_b200/csrc/mps_reader.h) against the
reference's own parse_mps_file (compiled from its sources, oracle/_ref).

The CPU tests compare everything the parse decides -- dimensions, the
triplets (turned into CSR by the reference's csr_from_triplets), sides,
bounds, integrality, name, and the error messages of malformed files; the
GPU test builds the CSR on the device (pg_mps_to_csr) and propagates it."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2009_07785_b200.abi import MpsError
from paper_2009_07785_b200.engine import MpsFile

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")

FIX = "/root/reference/proj/tests/fixtures"


def same(a, b):
    return np.array_equal(O.canon(np.asarray(a, dtype=float)), O.canon(np.asarray(b, dtype=float)))


def check_against_reference(path, threads=0):
    ref = O.ref_parse_mps(path)
    f = MpsFile(path, threads=threads)
    assert (f.m, f.n) == (ref.num_rows(), ref.num_cols())
    rp, ci, va = O.csr_from_triplets(f.rows, f.cols, f.values, f.m, f.n, impl="reference")
    assert np.array_equal(rp, ref.matrix.row_ptr)
    assert np.array_equal(ci, ref.matrix.col_idx)
    assert same(va, ref.matrix.values)
    for a, b in ((f.lhs, ref.lhs), (f.rhs, ref.rhs), (f.lower, ref.bounds.lower),
                 (f.upper, ref.bounds.upper)):
        assert same(a, b)
    assert np.array_equal(f.integral, ref.integral)
    return f


@pytest.mark.skipif(not os.path.isdir(FIX), reason="reference fixtures not present")
def test_reference_fixtures():
    files = sorted(os.path.join(d, x) for d, _, fs in os.walk(FIX) for x in fs if x.endswith(".mps"))
    assert len(files) == 6
    for p in files:
        f = check_against_reference(p)
        assert f.name  # NAME section, else the file name


def write_mps(path, rows, cols, vals, m, n, kinds, rhs, ranges, bounds, intcols, name="t",
              split_entries=False, crlf=False):
    """A free-MPS writer for tests: row kinds 'L'/'G'/'E', an objective row,
    integer marker blocks, RANGES, BOUNDS lines (type, col, value|None)."""
    nl = "\r\n" if crlf else "\n"
    out = [f"NAME {name}", "* a comment line", "ROWS", " N obj"]
    out += [f" {kinds[i]} r{i}" for i in range(m)]
    out.append("COLUMNS")
    by_col = {}
    for r, c, v in zip(rows, cols, vals):
        by_col.setdefault(c, []).append((r, v))
    in_block = False
    for c in sorted(by_col):
        want = c in intcols
        if want != in_block:
            out.append(f"    MARKER 'MARKER' '{'INTORG' if want else 'INTEND'}'")
            in_block = want
        ents = by_col[c]
        if c % 3 == 0:
            ents = ents + [("obj", 1.5)]
        if split_entries:
            for r, v in ents:
                out.append(f"    x{c} {r if r == 'obj' else 'r' + str(r)} {v!r}")
        else:
            for k in range(0, len(ents), 2):
                pairs = " ".join(f"{r if r == 'obj' else 'r' + str(r)} +{v!r}" if v >= 0 else
                                 f"{r if r == 'obj' else 'r' + str(r)} {v!r}" for r, v in ents[k:k + 2])
                out.append(f"    x{c} {pairs}")
    if in_block:
        out.append("    MARKER 'MARKER' 'INTEND'")
    out.append("RHS")
    out += [f"    rhs r{i} {v!r}" for i, v in enumerate(rhs) if v is not None]
    out.append("RANGES")
    out += [f"    rng r{i} {v!r}" for i, v in ranges]
    out.append("BOUNDS")
    for t, c, v in bounds:
        out.append(f" {t} bnd x{c}" + ("" if v is None else f" {v!r}"))
    out.append("ENDATA")
    with open(path, "w", newline="") as fh:
        fh.write(nl.join(out) + nl)


def random_problem(seed, m=300, n=250, per_row=6):
    rng = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    for i in range(m):
        cs = rng.choice(n, size=per_row, replace=False)
        for c in cs:
            rows.append(i)
            cols.append(int(c))
            vals.append(float(np.round(rng.uniform(-10, 10), int(rng.integers(0, 6)))))
    kinds = [str(rng.choice(["L", "G", "E"])) for _ in range(m)]
    rhs = [None if rng.random() < 0.1 else float(np.round(rng.uniform(-50, 50), 3)) for _ in range(m)]
    ranges = [(i, float(np.round(rng.uniform(-5, 5), 2))) for i in range(m) if rng.random() < 0.1]
    types = ["LO", "UP", "FX", "FR", "MI", "PL", "BV", "UI", "LI", "lo"]
    bounds = []
    for c in range(n):
        if rng.random() < 0.6:
            t = str(rng.choice(types))
            v = None if t.upper() in ("FR", "MI", "PL", "BV") else float(np.round(rng.uniform(-20, 20), 2))
            if rng.random() < 0.05 and v is not None:
                v = 1e21 if v > 0 else -1e21  # normalised to an infinity
            bounds.append((t, c, v))
    intcols = set(int(c) for c in rng.choice(n, size=n // 3, replace=False))
    return rows, cols, vals, m, n, kinds, rhs, ranges, bounds, intcols


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_generated_files(tmp_path, seed):
    prob = random_problem(seed)
    for split, crlf in ((False, False), (True, False), (False, True)):
        p = str(tmp_path / f"g{seed}_{split}_{crlf}.mps")
        write_mps(p, *prob, split_entries=split, crlf=crlf)
        for threads in (1, 3, 8):
            check_against_reference(p, threads=threads)


def test_large_file_parallel_chunks(tmp_path):
    """Several MB of COLUMNS, so the section is cut into many chunks (column
    runs and marker blocks crossing chunk boundaries)."""
    prob = random_problem(7, m=20000, n=30000, per_row=8)
    p = str(tmp_path / "big.mps")
    write_mps(p, *prob, split_entries=True)
    assert os.path.getsize(p) > 4 << 20
    for threads in (1, 16):
        check_against_reference(p, threads=threads)


BAD = {
    "unknown_row": "NAME x\nROWS\n N obj\n L r0\nCOLUMNS\n x0 r1 1.0\nENDATA\n",
    "bad_value": "NAME x\nROWS\n N obj\n L r0\nCOLUMNS\n x0 r0 1.0q\nENDATA\n",
    "no_endata": "NAME x\nROWS\n N obj\n L r0\nCOLUMNS\n x0 r0 1.0\n",
    "bad_marker": "NAME x\nROWS\n L r0\nCOLUMNS\n M 'MARKER' 'FOO'\n x0 r0 1.0\nENDATA\n",
    "odd_columns": "NAME x\nROWS\n L r0\nCOLUMNS\n x0 r0\nENDATA\n",
    "bad_section": "NAME x\nROWZ\nENDATA\n",
    "dup_row": "NAME x\nROWS\n L r0\n G r0\nENDATA\n",
    "two_obj": "NAME x\nROWS\n N a\n N b\nENDATA\n",
    "row_type": "NAME x\nROWS\n Q r0\nENDATA\n",
    "data_first": " x0 r0 1\nNAME x\nENDATA\n",
    "bound_value": "NAME x\nROWS\n L r0\nCOLUMNS\n x0 r0 1\nBOUNDS\n UP b x0\nENDATA\n",
    "bound_type": "NAME x\nROWS\n L r0\nCOLUMNS\n x0 r0 1\nBOUNDS\n ZZ b x0 1\nENDATA\n",
    "rhs_row": "NAME x\nROWS\n L r0\nCOLUMNS\n x0 r0 1\nRHS\n rhs r9 1\nENDATA\n",
}


@pytest.mark.parametrize("case", sorted(BAD))
def test_error_messages_match_reference(tmp_path, case):
    p = str(tmp_path / f"{case}.mps")
    with open(p, "w") as fh:
        fh.write(BAD[case])
    with pytest.raises(ValueError) as ref:
        O.ref_parse_mps(p)
    with pytest.raises(MpsError) as got:
        MpsFile(p)
    assert str(got.value) == str(ref.value)


def test_missing_file():
    with pytest.raises(MpsError) as e:
        MpsFile("/nonexistent/x.mps")
    assert "cannot open" in str(e.value)


@pytest.mark.gpu
def test_device_csr_and_propagation(tmp_path):
    """pg_mps_to_csr on the device gives the reference's CSR byte for byte,
    and the parsed instance propagates bit-exactly."""
    from paper_2009_07785_b200.engine import propagate_gpu, read_mps
    from paper_2009_07785_b200.model import EngineConfig
    prob = random_problem(11, m=3000, n=2500, per_row=7)
    p = str(tmp_path / "dev.mps")
    write_mps(p, *prob)
    ref = O.ref_parse_mps(p)
    got = read_mps(p)
    assert np.array_equal(got.matrix.row_ptr, ref.matrix.row_ptr)
    assert np.array_equal(got.matrix.col_idx, ref.matrix.col_idx)
    assert same(got.matrix.values, ref.matrix.values)
    cfg = EngineConfig(row_check=False)
    a, b = propagate_gpu(got, cfg), O.ref_propagate_parallel(ref, cfg)
    assert a.status == b.status and a.rounds_executed == b.rounds_executed
    assert same(a.bounds.lower, b.bounds.lower) and same(a.bounds.upper, b.bounds.upper)
