"""Device-side timeline of one-shot pg_propagate calls (PG_TIMING=1 prints
the [pg gpu] marks of engine.cu's GpuTrace), from pinned host arrays as in
bench.py's e2e leg; wall time per call beside it."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PG_TIMING", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from instances import generators as G  # noqa: E402
from paper_2009_07785_b200.engine import propagate_gpu  # noqa: E402
from paper_2009_07785_b200.model import EngineConfig  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
inst = G.config_instance(cfgname)
pinned = bench.pinned_copy(inst)
out = bench.pinned_out(inst.num_cols()) if "--pageable" not in sys.argv else None
cfg = EngineConfig(worklist=cfgname in ("c2", "c5"))
walls = []
for i in range(int(os.environ.get("CALLS", "4"))):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = propagate_gpu(pinned, cfg, out=out)
    walls.append((time.perf_counter() - t) * 1e3)
    print(f"call {i}: {walls[-1]:.3f} ms status={r.status} rounds={r.rounds_executed}", file=sys.stderr)
print("median wall", np.median(walls[1:]), file=sys.stderr)
