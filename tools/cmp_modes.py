"""Time-to-fixpoint of a config under engine options (device time, L2 flushed)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from instances import generators as G  # noqa: E402
from paper_2009_07785_b200.engine import Session  # noqa: E402
from paper_2009_07785_b200.model import EngineConfig  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
inst = G.config_instance(cfgname)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, cfg in [("worklist on ", EngineConfig()), ("worklist off", EngineConfig(worklist=False))]:
    with Session(inst, cfg) as s:
        for _ in range(3):
            s.run()
        ts = []
        for _ in range(5):
            flush.zero_()
            torch.cuda.synchronize()
            r = s.run()
            ts.append(r.elapsed_ns / 1e6)
        print(f"{cfgname} {name}: {min(ts):.3f} ms  rounds {r.rounds_executed} {r.status.name}")
