"""ORACLE build helper (test infrastructure): the reference's bench harness
with a GPU engine, for SURVEY.md 8(f) row 1.

Copies the UNMODIFIED reference files core/include/propgate/harness.hpp and
core/src/harness.cpp from /root/reference into oracle/_ref/patched/ (git-
ignored; nothing of the reference is committed) and applies the patch
INTEGRATION.md describes:

  * EngineId gains Gpu (harness.hpp:65);
  * to_string(EngineId) names it "gpu" (harness.cpp:110-112);
  * run_engine dispatches Gpu to propgate::propagate_gpu from
    include/propgate_b200.hpp (harness.cpp:116-120).

Everything else of run_benchmark / bench_to_csv / bench_to_json (best-of-N
timing, exclusion of non-converged instances, geomean, percentiles, size
classes) runs as the reference wrote it.  Fails loudly if the anchors moved.

usage: python oracle/patch_harness.py REF_PROJ OUT_DIR
"""
import os
import sys


def patch(text, old, new, what):
    if text.count(old) != 1:
        sys.exit(f"patch_harness: anchor for {what} not found exactly once")
    return text.replace(old, new)


def main(ref, out):
    hpp_in = os.path.join(ref, "core/include/propgate/harness.hpp")
    cpp_in = os.path.join(ref, "core/src/harness.cpp")
    os.makedirs(os.path.join(out, "propgate"), exist_ok=True)
    h = open(hpp_in).read()
    h = patch(h, "enum class EngineId { Seq, Par };", "enum class EngineId { Seq, Par, Gpu };",
              "EngineId")
    open(os.path.join(out, "propgate", "harness.hpp"), "w").write(h)
    c = open(cpp_in).read()
    c = patch(c, '#include "propgate/harness.hpp"',
              '#include "propgate/harness.hpp"\n#include "propgate_b200.hpp"', "include")
    c = patch(c, 'return engine == EngineId::Seq ? "seq" : "par";',
              'return engine == EngineId::Seq ? "seq" : engine == EngineId::Par ? "par" : "gpu";',
              "to_string")
    c = patch(c, "return engine == EngineId::Seq ? propagate_sequential(instance, cfg)\n"
                 "                                 : propagate_parallel(instance, cfg);",
              "if (engine == EngineId::Gpu) return propagate_gpu(instance, cfg);\n"
              "  return engine == EngineId::Seq ? propagate_sequential(instance, cfg)\n"
              "                                 : propagate_parallel(instance, cfg);",
              "run_engine")
    open(os.path.join(out, "harness.cpp"), "w").write(c)
    print("patch_harness: ok ->", out)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
