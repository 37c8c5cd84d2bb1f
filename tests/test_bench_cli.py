"""bench.py's host-side contract on CPU: the multi-GPU launch form fails
loudly without the GPUs, the reference arm prints its JSON line, and the
parity check reads the committed reference digests."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(*args, timeout=300):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=timeout,
                          env={k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK")})


def test_gpus_n_without_the_gpus_fails_loudly():
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("this box has the GPUs")
    p = run("--gpus", "2", "--steps", "1")
    assert p.returncode == 2
    assert "needs 2 visible GPUs" in p.stderr


def test_world_size_mismatch_is_an_error():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"], cwd=ROOT,
                       capture_output=True, text=True, timeout=120,
                       env=dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0"))
    assert p.returncode == 2 and "WORLD_SIZE=2" in p.stderr


def test_reference_arm_line():
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    p = run("--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1")
    assert p.returncode == 0, p.stderr
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "ms" and line["higher_is_better"] is False
    assert line["config"]["workload"] == "c1" and line["status"] == "Converged"
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_parity_field_against_reference_digest():
    import bench
    from instances import generators as G
    from oracle import oracle as O
    from paper_2009_07785_b200.model import EngineConfig
    inst = G.config_instance("c1", 1)
    res = O.propagate_parallel(inst, EngineConfig(row_check=False))
    par, want = bench.parity("c1", 1, res)
    assert par == "bit-exact" and want["rounds"] == res.rounds_executed
    res.per_round_changes[0] += 1
    par, _ = bench.parity("c1", 1, res)
    assert par.startswith("MISMATCH") and "per_round_changes" in par
    assert bench.parity("c1", 12345, res)[0].startswith("unpinned")


def test_shard_launch_count():
    import bench
    info = {"slices": 10, "split_rows": 0, "shard_rounds": 4, "host_syncs": 3, "delta_graphs": 1,
            "held_rounds": 1}
    # 2 dense graphs x 4 rounds x (k_sell, k_commit, k_flag_to_slot) + 1 delta graph x 4 x
    # (k_sell, k_commit, k_delta_compact, k_delta_apply) + k_reset + 1 resume
    assert bench.shard_launches(info, False, True) == 2 * 4 * 3 + 4 * 4 + 1 + 1
    # split rows add k_split_finish and k_cand to every round
    info["split_rows"] = 5
    assert bench.shard_launches(info, False, True) == 2 * 4 * 5 + 4 * 6 + 1 + 1


def test_solve_launch_count():
    import bench
    info = {"slices": 10, "split_rows": 0, "persistent": 0}
    # k_sell + k_commit; the worklist adds its k_sell, k_commit_list, k_mark (+ k_mark_vars)
    assert bench.solve_launches(info, False) == (2, 1)
    assert bench.solve_launches(info, True) == (5, 2)
    info["split_rows"] = 3  # + k_split_finish + k_cand
    assert bench.solve_launches(info, True) == (7, 2)
