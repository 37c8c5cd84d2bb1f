"""Result digests for the benchmark configurations (test / bench checker).

A digest pins one propagation result without storing its bounds: status,
rounds_executed, per_round_changes, total changes and a sha256 over the
canonicalised (-0.0 -> +0.0) lower and upper bound vectors.  The committed
digests (tests/golden/digests.json) are produced by the reference compiled
from its own sources (oracle/_ref, `propagate_parallel`) by
tests/golden/make_digests.py; the GPU tests and bench.py compare the engine's
result to them, so the box needs neither /root/reference nor a CPU solve.
The instance itself is hashed too, so a generator that drifted is reported
as such and not as an engine mismatch.
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np

DIGESTS = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                       "golden", "digests.json")


def _canon(x) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.float64).copy()
    a[a == 0.0] = 0.0  # -0.0 == +0.0
    return a


def bounds_sha(lower, upper) -> str:
    h = hashlib.sha256()
    h.update(_canon(lower).tobytes())
    h.update(_canon(upper).tobytes())
    return h.hexdigest()


def instance_sha(inst) -> str:
    h = hashlib.sha256()
    for a in (inst.matrix.row_ptr, inst.matrix.col_idx, inst.matrix.values, inst.lhs, inst.rhs,
              inst.bounds.lower, inst.bounds.upper, inst.integral):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def result_digest(res) -> dict:
    return {"status": res.status.name, "rounds": int(res.rounds_executed),
            "per_round_changes": [int(c) for c in res.per_round_changes],
            "total_changes": int(res.total_bound_changes),
            "bounds_sha256": bounds_sha(res.bounds.lower, res.bounds.upper)}


def node_digest(status: int, rounds: int, lower, upper) -> dict:
    return {"status": int(status), "rounds": int(rounds), "bounds_sha256": bounds_sha(lower, upper)}


def load(path: str = DIGESTS) -> dict:
    with open(path) as f:
        return json.load(f)


def compare(res, want: dict) -> list[str]:
    """Differences between a result and a committed digest (empty = bit-exact)."""
    got = result_digest(res)
    return [f"{k}: got {got[k]!r}, reference {want[k]!r}" for k in
            ("status", "rounds", "per_round_changes", "total_changes", "bounds_sha256")
            if got[k] != want[k]]
