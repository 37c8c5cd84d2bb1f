"""Time the on-device CSR build (pg_csr_from_triplets, host arrays in/out)
against the reference's csr_from_triplets (oracle/_ref, 1 core) and the C
restatement on a C2-sized triplet set (12M triplets, 1M x 1M, ~3% duplicates,
shuffled).  usage: python tools/ingest_time.py [count]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2009_07785_b200.engine import csr_from_triplets_gpu  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 12_000_000
m = n = 1_000_000
rng = np.random.default_rng(11)
r = rng.integers(0, m, k, dtype=np.int32)
c = rng.integers(0, n, k, dtype=np.int32)
d = rng.integers(0, k, k // 32)
r[d[: len(d) // 2]] = r[d[len(d) // 2:]]
c[d[: len(d) // 2]] = c[d[len(d) // 2:]]
v = rng.uniform(-10, 10, k)
out = {"triplets": k, "m": m, "n": n}
gpu = []
for i in range(4):
    t = time.perf_counter()
    a = csr_from_triplets_gpu(r, c, v, m, n)
    gpu.append((time.perf_counter() - t) * 1e3)
out["gpu_ms_e2e"] = round(float(np.median(gpu[1:])), 2)
t = time.perf_counter()
b = O.csr_from_triplets(r, c, v, m, n)
out["port_ms"] = round((time.perf_counter() - t) * 1e3, 1)
assert a.row_ptr.tobytes() == b[0].tobytes() and a.col_idx.tobytes() == b[1].tobytes()
assert a.values.tobytes() == b[2].tobytes()
if O.ref_available():
    t = time.perf_counter()
    b = O.csr_from_triplets(r, c, v, m, n, impl="reference")
    out["reference_ms"] = round((time.perf_counter() - t) * 1e3, 1)
    assert a.values.tobytes() == b[2].tobytes()
out["nnz"] = int(a.col_idx.shape[0])
print(json.dumps(out))
