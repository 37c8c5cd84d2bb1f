"""MPS ingest timing: the reference's parse_mps_file (oracle/_ref, one
thread, its own csr_from_triplets) against pg_mps_read (host threads) +
pg_mps_to_csr (device CSR), on an instance written as free MPS (C4 shape by
default: 500k x 500k, ~4M entries), both results compared array for array.
usage: python tools/mps_time.py [OUT.json] [config]"""
import json
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from instances import generators as G  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2009_07785_b200.engine import MpsFile  # noqa: E402


def write(inst, path):
    m, n = inst.num_rows(), inst.num_cols()
    A = inst.matrix
    rows = np.repeat(np.arange(m), np.diff(A.row_ptr))
    order = np.lexsort((rows, A.col_idx))  # column-major, as MPS lists entries
    integ = inst.integral.astype(bool)
    inf = float("inf")
    with open(path, "w") as f:
        f.write(f"NAME {inst.name}\nROWS\n N obj\n")
        kinds = []
        for i in range(m):
            l, h = inst.lhs[i], inst.rhs[i]
            k = "E" if l == h else ("G" if np.isfinite(l) and not np.isfinite(h) else "L")
            kinds.append(k)
            f.write(f" {k} r{i}\n")
        f.write("COLUMNS\n")
        block = False
        lines = []
        cols, rws, vls = A.col_idx[order], rows[order], A.values[order]
        for c, r, v in zip(cols.tolist(), rws.tolist(), vls.tolist()):
            if integ[c] != block:
                lines.append("    M 'MARKER' 'INTORG'" if integ[c] else "    M 'MARKER' 'INTEND'")
                block = bool(integ[c])
            lines.append(f"    x{c} r{r} {v!r}")
        if block:
            lines.append("    M 'MARKER' 'INTEND'")
        f.write("\n".join(lines) + "\n")
        f.write("RHS\n")
        for i in range(m):
            l, h = inst.lhs[i], inst.rhs[i]
            side = l if kinds[i] == "G" or kinds[i] == "E" else h
            if np.isfinite(side):
                f.write(f"    rhs r{i} {float(side)!r}\n")
        f.write("RANGES\n")
        for i in range(m):
            l, h = inst.lhs[i], inst.rhs[i]
            if kinds[i] == "L" and np.isfinite(l) and np.isfinite(h):
                f.write(f"    rng r{i} {float(h - l)!r}\n")
        f.write("BOUNDS\n")
        for j in range(n):
            lo, up = inst.bounds.lower[j], inst.bounds.upper[j]
            f.write(f" LO b x{j} {float(lo)!r}\n" if np.isfinite(lo) else f" MI b x{j}\n")
            f.write(f" UP b x{j} {float(up)!r}\n" if np.isfinite(up) else f" PL b x{j}\n")
        f.write("ENDATA\n")


def main(out, cfg):
    inst = G.config_instance(cfg)
    d = tempfile.mkdtemp()
    path = os.path.join(d, f"{cfg}.mps")
    t = time.perf_counter()
    write(inst, path)
    wsec = time.perf_counter() - t
    size = os.path.getsize(path)
    t = time.perf_counter()
    ref = O.ref_parse_mps(path)
    ref_s = time.perf_counter() - t
    # the CUDA context exists before the timed region (one tiny device CSR build)
    from paper_2009_07785_b200.engine import csr_from_triplets_gpu
    csr_from_triplets_gpu(np.zeros(1, np.int32), np.zeros(1, np.int32), np.ones(1), 1, 1)
    t = time.perf_counter()
    f = MpsFile(path)
    parse_s = time.perf_counter() - t
    t = time.perf_counter()
    got = f.instance()
    csr_s = time.perf_counter() - t
    same = (np.array_equal(got.matrix.row_ptr, ref.matrix.row_ptr) and
            np.array_equal(got.matrix.col_idx, ref.matrix.col_idx) and
            np.array_equal(O.canon(got.matrix.values), O.canon(ref.matrix.values)) and
            all(np.array_equal(O.canon(a), O.canon(b)) for a, b in
                ((got.lhs, ref.lhs), (got.rhs, ref.rhs), (got.bounds.lower, ref.bounds.lower),
                 (got.bounds.upper, ref.bounds.upper))) and
            np.array_equal(got.integral, ref.integral))
    res = {"config": cfg, "file_mb": round(size / 1e6, 1), "entries": int(ref.matrix.nnz()),
           "m": ref.num_rows(), "n": ref.num_cols(), "identical_to_reference": bool(same),
           "reference_parse_mps_file_s": round(ref_s, 3),
           "pg_mps_read_s": round(parse_s, 3), "threads": os.cpu_count(),
           "pg_mps_to_csr_s": round(csr_s, 3), "ours_total_s": round(parse_s + csr_s, 3),
           "speedup": round(ref_s / (parse_s + csr_s), 2), "write_s": round(wsec, 1)}
    print(json.dumps(res))
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    os.remove(path)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/mps_ingest.json",
         sys.argv[2] if len(sys.argv) > 2 else "c4")
