import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PG_TIMING"] = "1"
import torch  # noqa
from bench import pinned_copy  # noqa
from instances import generators as G  # noqa
from paper_2009_07785_b200.engine import propagate_gpu  # noqa
from paper_2009_07785_b200.model import EngineConfig  # noqa
inst = pinned_copy(G.config_instance(sys.argv[1] if len(sys.argv) > 1 else "c2"))
cfg = EngineConfig(worklist=len(sys.argv) > 2 and sys.argv[2] == "wl")
for i in range(3):
    t = time.perf_counter()
    r = propagate_gpu(inst, cfg)
    print(f"--- e2e {(time.perf_counter() - t) * 1e3:.2f} ms  solve {r.elapsed_ns / 1e6:.3f} ms", flush=True)
