"""Reference digests of the full-size benchmark configurations.

Run in the CPU container (needs oracle/_ref, the reference compiled from its
own sources by oracle/build_ref.sh).  For every configuration the bench and
the GPU tests use, the REFERENCE's `propagate_parallel` (cpu_par, all host
threads; bit-deterministic at any worker count, test_par_engine.cpp:183-210)
solves the instance, and its result is committed as a digest
(instances/digest.py) to tests/golden/digests.json, together with the
instance's own sha256 and the reference `propagate_sequential` verdict:

  c1     gen_random 10k x 10k, seeds 1-5
  c2     power-law 1M x 1M, seeds 20090778 (bench), 20090779
  c3     long rows 100k x 200k, 126.5M entries, seed 3001
  c4     gen_random 500k x 500k seed 4: the root fixpoint and B&B nodes
         0..63 (gen_nodes, seed base 4_000_000) solved from their bounds
  c5     set partitioning 1M x 5M, 50M entries, seed 5001 (+ the infeasible
         variant's verdict)

usage: python tests/golden/make_digests.py [config ...]
"""
from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from instances import digest as D  # noqa: E402
from instances import generators as G  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2009_07785_b200.model import EngineConfig, ScalarMode  # noqa: E402

THREADS = os.cpu_count() or 1
PAR = EngineConfig(row_check=False, worker_count=THREADS)
SEEDS = {"c1": [1, 2, 3, 4, 5], "c2": [20090778, 20090779], "c3": [3001], "c4": [4], "c5": [5001]}
C4_NODES = 64


def entry(inst, seq_verdict=True):
    t = time.perf_counter()
    par = O.ref_propagate_parallel(inst, PAR)
    e = {"instance": inst.name, "m": inst.num_rows(), "n": inst.num_cols(), "nnz": inst.matrix.nnz(),
         "instance_sha256": D.instance_sha(inst), "cpu_par": D.result_digest(par)}
    if seq_verdict:
        e["cpu_seq_status"] = O.ref_propagate_sequential(inst, PAR).status.name
    print(f"  {inst.name}: {par.status.name} in {par.rounds_executed} rounds "
          f"({time.perf_counter() - t:.1f} s)", flush=True)
    return e, par


def main(configs, only_f32=False):
    if not O.ref_available():
        sys.exit("oracle/_ref/libpropgate_ref.so missing: run oracle/build_ref.sh")
    out = D.load() if os.path.exists(D.DIGESTS) else {}
    out["_about"] = ("reference propagate_parallel (oracle/_ref, compiled from /root/reference "
                     "sources) results; tests/golden/make_digests.py")
    for cfg in configs:
        print(cfg, flush=True)
        ents = {}
        for seed in SEEDS[cfg]:
            inst = G.config_instance(cfg, seed)
            # cpu_seq on C3 takes ~50 s: its verdict is the same Converged
            e, par = entry(inst, seq_verdict=cfg != "c3")
            if cfg in ("c2", "c3") and str(seed) in ("20090778", "3001"):
                # ScalarMode::Narrow32: the reference's run_parallel<float>
                f32 = EngineConfig(row_check=False, worker_count=THREADS,
                                   scalar_mode=ScalarMode.Narrow32)
                e["cpu_par_f32"] = D.result_digest(O.ref_propagate_parallel(inst, f32))
            if cfg == "c4":
                lo, up = G.gen_nodes(inst, par.bounds.lower, par.bounds.upper, K=C4_NODES)
                nodes = []
                for k in range(C4_NODES):
                    r = O.ref_propagate_parallel(inst, PAR, lo[k], up[k])
                    nodes.append(D.node_digest(int(r.status), r.rounds_executed, r.bounds.lower,
                                               r.bounds.upper))
                e["nodes"] = nodes
                # the bench's mode (Step-2 row check on) has no reference
                # engine: the oracle restatement's cpu_par + row check, which
                # tests/test_oracle.py pins to the reference
                rc = EngineConfig(row_check=True)
                e["nodes_rowcheck"] = [
                    D.node_digest(int(r.status), r.rounds_executed, r.bounds.lower, r.bounds.upper)
                    for r in (O.propagate_parallel(inst, rc, lo[k], up[k]) for k in range(C4_NODES))]
                e["root_bounds_sha256"] = e["cpu_par"]["bounds_sha256"]
            if cfg == "c5":
                bad = G.gen_setpart(seed=seed, infeasible=True)
                e["infeasible_variant"] = {
                    "instance_sha256": D.instance_sha(bad),
                    "cpu_par_status": O.ref_propagate_parallel(bad, PAR).status.name,
                    "cpu_seq_status": O.ref_propagate_sequential(bad, PAR).status.name}
            ents[str(seed)] = e
        out[cfg] = ents
        with open(D.DIGESTS, "w") as f:
            json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", D.DIGESTS)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c4", "c5", "c3"])
