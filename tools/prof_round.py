"""Profiling driver: one session of a config, a few isolated round-kernel
launches (for ncu -k regex:k_tiles) and one full solve."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from instances import generators as G  # noqa: E402
from paper_2009_07785_b200.engine import Session  # noqa: E402
from paper_2009_07785_b200.model import EngineConfig, LoopMode  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--solve", action="store_true")
ap.add_argument("--host-loop", action="store_true")
ap.add_argument("--debug-flags", type=lambda x: int(x, 0), default=0)
ap.add_argument("--worklist", action="store_true")
a = ap.parse_args()
inst = G.config_instance(a.config)
cfg = EngineConfig(loop_mode=LoopMode.Host if a.host_loop else LoopMode.Graph, worklist=a.worklist)
import ctypes as C  # noqa: E402
from paper_2009_07785_b200 import abi  # noqa: E402
if a.debug_flags:
    lib = abi.load_library()
    c = cfg.to_c()
    c.flags |= a.debug_flags
    p = inst.to_c()
    h = C.c_void_p()
    abi.check(lib.pg_session_create(C.byref(p), C.byref(c), C.byref(h)), "create")
    ns, b = C.c_double(), C.c_double()
    abi.check(lib.pg_session_time_round_kernel(h, a.reps, C.byref(ns), C.byref(b)), "time")
    print(f"k_round {ns.value/1e3:.1f} us (debug flags {a.debug_flags:#x})")
    if a.solve:
        from paper_2009_07785_b200.engine import new_c_result
        best = None
        for _ in range(3):
            r, lo, up, prc = new_c_result(inst.num_cols(), cfg.round_limit)
            r.lower = C.cast(None, C.POINTER(C.c_double))
            r.upper = C.cast(None, C.POINTER(C.c_double))
            abi.check(lib.pg_session_run(h, C.byref(r)), "run")
            best = r.elapsed_ns if best is None else min(best, r.elapsed_ns)
        print(f"solve status={r.status} rounds={r.rounds_executed} best={best/1e6:.3f} ms")
    sys.exit(0)
with Session(inst, cfg) as s:
    print(s.info())
    ns, b = s.time_round_kernel(a.reps)
    print(f"k_tiles {ns/1e3:.1f} us  {b/ns:.1f} GB/s")
    if a.solve:
        best = None
        for _ in range(5):
            r = s.run()
            best = r.elapsed_ns if best is None else min(best, r.elapsed_ns)
        print(f"solve status={int(r.status)} rounds={r.rounds_executed} best={best/1e6:.3f} ms")
