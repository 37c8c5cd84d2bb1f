"""Parity artifact (GPU box): the engine against the reference's two
oracles, recorded as JSON.

  vs cpu_par  (propagate_parallel; the reference compiled from its sources):
              status, rounds, per-round changes and every bound identical
  vs cpu_seq  (propagate_sequential, the north-star oracle): identical
              infeasibility verdicts and integer-variable bounds; continuous
              bounds within the reference comparator |a-b| <= 1e-8 + 1e-5|b|
              (harness.cpp:17-20); and the 1e-9-relative pass rate -- per
              instance (every bound within 1e-9 relative, 1e-9 absolute near
              zero) and per bound

Instances: the reference acceptance suite's 500 random instances
(acceptance.cpp:56-75), C1 seeds 1-5, C2 (1M x 1M) seeds 20090778/9, C5.
usage: python tools/parity_report.py OUT.json
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from instances import generators as G  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2009_07785_b200.engine import propagate_gpu  # noqa: E402
from paper_2009_07785_b200.model import EngineConfig, PropagationStatus  # noqa: E402

THREADS = os.cpu_count() or 1


def close(a, b, t_abs, t_rel):
    return O.bounds_equal(a, b, t_abs, t_rel)


def one(inst):
    gpu = propagate_gpu(inst, EngineConfig(row_check=True))
    gpu_par = propagate_gpu(inst, EngineConfig(row_check=False))
    ref = O.ref_available()
    par = (O.ref_propagate_parallel if ref else O.propagate_parallel)(
        inst, EngineConfig(row_check=False, worker_count=THREADS))
    seq = (O.ref_propagate_sequential if ref else O.propagate_sequential)(inst, EngineConfig())
    par_ok = (gpu_par.status == par.status and gpu_par.rounds_executed == par.rounds_executed and
              gpu_par.per_round_changes == par.per_round_changes and
              np.array_equal(O.canon(gpu_par.bounds.lower), O.canon(par.bounds.lower)) and
              np.array_equal(O.canon(gpu_par.bounds.upper), O.canon(par.bounds.upper)))
    inf_g = gpu.status == PropagationStatus.Infeasible
    inf_s = seq.status == PropagationStatus.Infeasible
    r = {"name": inst.name, "nnz": int(inst.matrix.nnz()), "bit_exact_vs_cpu_par": bool(par_ok),
         "verdict_match_vs_cpu_seq": inf_g == inf_s, "gpu_status": gpu.status.name,
         "seq_status": seq.status.name, "gpu_rounds": gpu.rounds_executed,
         "seq_rounds": seq.rounds_executed}
    if gpu.status == seq.status == PropagationStatus.Converged:
        integ = inst.integral.astype(bool)
        lo_g, up_g, lo_s, up_s = gpu.bounds.lower, gpu.bounds.upper, seq.bounds.lower, seq.bounds.upper
        r["integer_bounds_identical"] = bool(np.array_equal(lo_g[integ], lo_s[integ]) and
                                             np.array_equal(up_g[integ], up_s[integ]))
        ok_tol = close(lo_s, lo_g, 1e-8, 1e-5) & close(up_s, up_g, 1e-8, 1e-5)
        ok_9 = close(lo_s, lo_g, 1e-9, 1e-9) & close(up_s, up_g, 1e-9, 1e-9)
        r["within_reference_comparator"] = bool(ok_tol.all())
        r["within_1e-9"] = bool(ok_9.all())
        r["bounds_within_1e-9"] = int(ok_9.sum())
        r["bounds"] = int(ok_9.size)
    return r


def main(out):
    t0 = time.time()
    groups = {"acceptance_suite_500": list(G.acceptance_suite(500)),
              "c1": [G.config_instance("c1", s) for s in range(1, 6)]}
    res = {}
    for gname, insts in groups.items():
        res[gname] = [one(i) for i in insts]
    res["c2"] = [one(G.config_instance("c2", s)) for s in (20090778, 20090779)]
    res["c5"] = [one(G.config_instance("c5", 5001))]
    summary = {}
    for g, rows in res.items():
        both = [r for r in rows if "within_1e-9" in r]
        summary[g] = {
            "instances": len(rows),
            "bit_exact_vs_cpu_par": sum(r["bit_exact_vs_cpu_par"] for r in rows),
            "verdict_match_vs_cpu_seq": sum(r["verdict_match_vs_cpu_seq"] for r in rows),
            "both_converged": len(both),
            "integer_bounds_identical": sum(r["integer_bounds_identical"] for r in both),
            "within_reference_comparator": sum(r["within_reference_comparator"] for r in both),
            "instances_within_1e-9": sum(r["within_1e-9"] for r in both),
            "bounds_within_1e-9": sum(r["bounds_within_1e-9"] for r in both),
            "bounds_compared": sum(r["bounds"] for r in both)}
    doc = {"about": __doc__.strip().split("\n\n")[0], "oracle": "reference compiled from its "
           "sources (oracle/_ref)" if O.ref_available() else "restated oracle",
           "seconds": round(time.time() - t0, 1), "summary": summary,
           "instances": {g: rows for g, rows in res.items() if g != "acceptance_suite_500"}}
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/parity_report.json")
