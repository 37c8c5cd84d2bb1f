"""One solve of a configuration (profiling driver): python tools/solve_once.py c2 [--host-loop]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from instances import generators as G  # noqa: E402
from paper_2009_07785_b200.engine import Session  # noqa: E402
from paper_2009_07785_b200.model import EngineConfig, LoopMode  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
host = "--host-loop" in sys.argv
inst = G.config_instance(cfgname)
cfg = EngineConfig(loop_mode=LoopMode.Host if host else LoopMode.Graph, worklist=cfgname in ("c2", "c5"))
with Session(inst, cfg) as s:
    r = s.run()
    print("status", int(r.status), "rounds", r.rounds_executed, "ms", r.elapsed_ns / 1e6)
