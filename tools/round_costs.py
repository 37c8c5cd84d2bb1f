"""Marginal device time per round of a graph solve: the same session solved
with round_limit = 1 .. R (solve time differences = the cost of each round
inside the CUDA graph, launch gaps included)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from instances import generators as G  # noqa: E402
from paper_2009_07785_b200.engine import Session  # noqa: E402
from paper_2009_07785_b200.model import EngineConfig  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
inst = G.config_instance(cfgname)
wl = cfgname in ("c2", "c4", "c5")
prev = 0.0
full = None
for lim in range(1, 60):
    with Session(inst, EngineConfig(worklist=wl, round_limit=lim)) as s:
        best = min(s.run().elapsed_ns for _ in range(7)) / 1e3
        r = s.run()
    print(f"limit {lim:2d}: rounds {r.rounds_executed:2d} {best:9.1f} us  (+{best - prev:7.1f})  {r.status}")
    prev = best
    if r.rounds_executed < lim:
        break
