"""One host-loop solve of a configuration (every kernel a separate launch),
for ncu captures of a given round's kernels, e.g.
  ncu -k regex:k_mark -s 3 -c 1 python tools/prof_solve.py c2   (round 4's marks)
With --rounds the per-round device state is printed (PG_DEBUG_ROUNDS)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from instances import generators as G  # noqa: E402
from paper_2009_07785_b200.engine import Session  # noqa: E402
from paper_2009_07785_b200.model import EngineConfig, LoopMode  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
if "--rounds" in sys.argv:
    os.environ["PG_DEBUG_ROUNDS"] = "1"
inst = G.config_instance(cfgname)
with Session(inst, EngineConfig(worklist=True, loop_mode=LoopMode.Host)) as s:
    r = s.run()
    print(r.status, r.rounds_executed, r.per_round_changes, r.elapsed_ns / 1e6, "ms")
