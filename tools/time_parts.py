"""Time k_round on C2's initial snapshot with timing-only switches."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_07785_b200 import abi
from instances import generators as G  # noqa: E402
from paper_2009_07785_b200.model import EngineConfig  # noqa: E402

inst = G.config_instance(sys.argv[1] if len(sys.argv) > 1 else "c2")
lib = abi.load_library()
for name, extra in [("full", 0), ("tiles only", 0x100), ("segments only", 0x200)]:
    c = EngineConfig().to_c()
    c.flags |= extra
    p = inst.to_c()
    h = C.c_void_p()
    abi.check(lib.pg_session_create(C.byref(p), C.byref(c), C.byref(h)), "create")
    ns, b = C.c_double(), C.c_double()
    abi.check(lib.pg_session_time_round_kernel(h, 10, C.byref(ns), C.byref(b)), "time")
    print(f"{name:14s} k_round {ns.value/1e3:8.1f} us")
    lib.pg_session_destroy(h)
