"""GPU: the reference's own harness flow with the GPU engine substituted
through the C++ adapter include/propgate_b200.hpp (oracle/_ref/gpu_dropin,
built from tests/cpp/gpu_dropin.cpp against the unmodified reference)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "gpu_dropin")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(EXE), reason="oracle/_ref/gpu_dropin not built")
def test_reference_harness_with_gpu_engine():
    p = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "FAIL" not in p.stdout


HARNESS = os.path.join(ROOT, "oracle", "_ref", "harness_gpu")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(HARNESS), reason="oracle/_ref/harness_gpu not built")
def test_reference_bench_harness_with_gpu_engine(tmp_path):
    """the reference's run_benchmark / bench_to_csv /
    bench_to_json (harness.cpp, EngineId::Gpu patched into a build-time copy)
    over cascades, C1 seeds 1-5 and the 6 MPS fixtures (round-tripped through
    the reference's write_mps / parse_mps inside the driver), engines
    {seq, par, gpu}: every GPU result agrees (bit-identical with cpu_par,
    cpu_seq's verdicts and comparator), and the tables carry a gpu column
    with speedups computed by the reference code."""
    import csv
    import json

    import numpy as np

    z = np.load(os.path.join(ROOT, "tests", "golden", "fixtures.npz"), allow_pickle=False)
    mps = []
    for name in z["names"]:
        p = f"{name}/"
        path = str(tmp_path / f"{name}.pgi")
        with open(path, "wb") as f:
            m, n = z[p + "lhs"].shape[0], z[p + "lower"].shape[0]
            np.array([m, n, z[p + "col_idx"].shape[0]], dtype=np.int64).tofile(f)
            for key, dt in (("row_ptr", np.int32), ("col_idx", np.int32), ("values", np.float64),
                            ("lhs", np.float64), ("rhs", np.float64), ("lower", np.float64),
                            ("upper", np.float64), ("integral", np.uint8)):
                np.ascontiguousarray(z[p + key], dtype=dt).tofile(f)
        mps.append(path)
    out = str(tmp_path / "bench")
    r = subprocess.run([HARNESS, out, *mps], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
    table = json.load(open(out + ".json"))
    engines = {rec["engine"] for rec in table["records"]}
    assert engines == {"seq", "par", "gpu"}
    names = {rec["instance"] for rec in table["records"]}
    assert len(names) == 4 + 5 + 6
    gpu = [a for a in table["aggregates"] if a["engine"] == "gpu"]
    assert gpu and gpu[0]["included"] > 0 and gpu[0]["geo_mean_speedup"] > 0
    # cascade(200) hits the round limit in every engine: excluded from the
    # means, as harness.cpp:165-175 does
    assert "cascade200" in table["excluded"]
    with open(out + ".csv") as f:
        rows = [row for row in csv.reader(f) if row]
    assert any(row[1] == "gpu" for row in rows[1:])
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    for ext in (".csv", ".json"):
        with open(out + ext) as src, open(os.path.join(ROOT, "gpurun_out", "harness_gpu" + ext), "w") as dst:
            dst.write(src.read())
