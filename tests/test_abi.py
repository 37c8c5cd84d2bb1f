"""CPU: the drop-in boundary.  The CUDA library loads without a GPU, exports
every entry point include/propgate_b200.h declares, validates configs like
EngineConfig::validate (core/src/model.cpp:21-35), and fails loudly (no CPU
fallback) when no device is present."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2009_07785_b200 import abi
from instances import generators as G
from paper_2009_07785_b200.model import EngineConfig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "propgate_b200.h")


def header_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pg_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_the_abi():
    names = header_functions()
    for must in ("pg_propagate", "pg_round", "pg_partition_row_blocks", "pg_session_create",
                 "pg_session_propagate", "pg_session_propagate_batch", "pg_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(abi.LIB_PATH)
    missing = [n for n in header_functions() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", abi.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (pg_[a-z_0-9]+)", out))
    assert set(header_functions()) <= exported


def test_library_is_sm100a_code():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", abi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_header():
    # sizes of the C structs as laid out by the C compiler
    src = os.path.join(ROOT, "build", "abi_sizes.c")
    exe = os.path.join(ROOT, "build", "abi_sizes")
    os.makedirs(os.path.dirname(src), exist_ok=True)
    with open(src, "w") as f:
        f.write('#include <stdio.h>\n#include <stddef.h>\n#include "propgate_b200.h"\n'
                'int main(void){printf("%zu %zu %zu %zu %zu\\n", sizeof(pg_problem), '
                'sizeof(pg_config), sizeof(pg_result), offsetof(pg_result, total_bound_changes), '
                'offsetof(pg_config, flags));return 0;}\n')
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", exe, src], check=True)
    got = list(map(int, subprocess.run([exe], capture_output=True, text=True).stdout.split()))
    assert got == [C.sizeof(abi.PgProblem), C.sizeof(abi.PgConfig), C.sizeof(abi.PgResult),
                   abi.PgResult.total_bound_changes.offset, abi.PgConfig.flags.offset]


def test_config_defaults_and_validation():
    lib = abi.load_library()
    c = abi.PgConfig()
    lib.pg_config_default(C.byref(c))
    ref = EngineConfig().to_c()
    for f, _ in abi.PgConfig._fields_:
        assert getattr(c, f) == getattr(ref, f), f
    assert lib.pg_config_validate(C.byref(c)) == abi.PG_OK
    for field, bad in [("round_limit", 0), ("infinity_threshold", 0.0), ("improvement_abs", 0.0),
                       ("improvement_rel", -1.0), ("integrality_eps", 0.0), ("vector_threshold", 0),
                       ("worker_count", -1), ("loop_mode", 7), ("scalar_mode", 3)]:
        d = abi.PgConfig()
        lib.pg_config_default(C.byref(d))
        setattr(d, field, bad)
        assert lib.pg_config_validate(C.byref(d)) == abi.PG_EINVAL, field
        assert lib.pg_last_error()
    d = abi.PgConfig()
    lib.pg_config_default(C.byref(d))
    d.nnz_budget, d.vector_threshold = 10, 64
    assert lib.pg_config_validate(C.byref(d)) == abi.PG_EINVAL
    assert b"nnz_budget must be >= vector_threshold" == lib.pg_last_error()


def test_partition_row_blocks_is_host_code():
    # partition_row_blocks (par_engine.cpp:14-41) needs no device: [2000, 3, 3] example
    lib = abi.load_library()
    from paper_2009_07785_b200.model import ProblemInstance
    import numpy as np
    lens = [2000, 3, 3]
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    ci = np.concatenate([np.arange(L, dtype=np.int32) for L in lens])
    inst = ProblemInstance.from_arrays(rp, ci, np.ones(len(ci)), [-np.inf] * 3, [np.inf] * 3,
                                       np.zeros(2000), np.ones(2000))
    starts = np.zeros(4, np.int32)
    kinds = np.zeros(3, np.int32)
    nb = C.c_int32()
    p = inst.to_c()
    cfg = EngineConfig().to_c()
    assert lib.pg_partition_row_blocks(C.byref(p), C.byref(cfg), abi.ptr(starts, C.c_int32),
                                       abi.ptr(kinds, C.c_int32), C.byref(nb)) == 0
    assert nb.value == 2 and list(starts[:3]) == [0, 1, 3] and list(kinds[:2]) == [2, 0]


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure mode")
def test_no_silent_cpu_fallback():
    from paper_2009_07785_b200.engine import propagate_gpu
    with pytest.raises(abi.EngineError, match="no CPU fallback|no CUDA device"):
        propagate_gpu(G.gen_cascade(3))
