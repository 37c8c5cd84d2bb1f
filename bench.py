"""bench.py -- time-to-fixpoint of the B200 propagation engine.

Metric (BASELINE.json): time-to-fixpoint & GB/s per round vs the HBM
roofline; speedup vs the CPU reference.  One "step" = one full propagation
of one instance to its fixpoint (or infeasibility / round limit) from its
start bounds.

Default workload: config C2 -- synthetic 1M x 1M,
power-law row lengths (x_min 4.25, beta 1.5, cap 10k, ~12M entries), mixed
bounds incl. infinities, 50% integer, seed 20090778, on one B200.  The
instance (~200 MB in HBM) is larger than L2 and L2 is flushed between steps.

  value     device time-to-fixpoint per step (ms, CUDA events around the
            graph launch; inputs resident in HBM), max over ranks
  e2e       the same solve through the C-ABI entry point pg_propagate with
            pinned HOST buffers: H2D upload + on-device setup + solve + D2H
  roofline  the round kernels (k_sell + k_cand) timed alone with CUDA events:
            algorithmic bytes / mean launch time vs MEASURED_PEAKS hbm_gbs
  cpu_baseline  the reference's own cpu_seq (compiled from its sources into
            oracle/_ref; 1 core), best of a bounded number of solves

--gpus N > 1: a single instance stays on one GPU (north star), so N ranks run
N independent replicas (weak scaling); value = max over ranks.
--impl reference: the reference's cpu_par (oracle/_ref, all host threads) on
the same instance, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time-to-fixpoint & GB/s per round vs HBM roofline; geomean speedup vs CPU ref"


def b_round(m, n, nnz):
    """SURVEY.md 8(d) algorithmic bytes of one full propagation round."""
    return 12 * nnz + 4 * (m + 1) + 16 * m + 33 * n


def _ncu_traffic(config, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (tools/ncu_traffic.py -> profiles/roofline_traffic.json), or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "roofline_traffic.json")
    try:
        with open(path) as f:
            ks = json.load(f)[config]["kernels"]
        return next(int(v["dram_bytes"]) for k, v in ks.items() if kernel in k)
    except (OSError, KeyError, StopIteration, ValueError):
        return None


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.samples)}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_instance(config, seed):
    from instances import generators as G
    return G.config_instance(config, seed)


def pinned_copy(inst):
    """Instance arrays in page-locked host memory (the e2e H2D source)."""
    import torch

    from paper_2009_07785_b200.model import ProblemInstance

    def pin(a):
        t = torch.empty(a.shape, dtype={np.int32: torch.int32, np.float64: torch.float64,
                                        np.uint8: torch.uint8}[a.dtype.type], pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()

    return ProblemInstance.from_arrays(pin(inst.matrix.row_ptr), pin(inst.matrix.col_idx),
                                       pin(inst.matrix.values), pin(inst.lhs), pin(inst.rhs),
                                       pin(inst.bounds.lower), pin(inst.bounds.upper),
                                       pin(inst.integral), num_cols=inst.num_cols(),
                                       name=inst.name)


def run_reference(args, inst, rank, world):
    """The reference's own cpu_par (all host threads) on the same workload."""
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_2009_07785_b200.model import EngineConfig

    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libpropgate_ref.so not built (needs /root/reference at build time)"}))
        return
    threads = os.cpu_count() or 1
    cfg = EngineConfig(worker_count=threads)
    for _ in range(args.warmup):
        O.ref_propagate_parallel(inst, cfg)
    times, res = [], None
    t0 = time.perf_counter()
    for _ in range(args.steps):
        res = O.ref_propagate_parallel(inst, cfg)
        times.append(res.elapsed_ns / 1e6)
    wall = (time.perf_counter() - t0) * 1e3 / args.steps
    ms = float(np.mean(times))
    m, n, nnz = inst.num_rows(), inst.num_cols(), inst.matrix.nnz()
    line = {
        "impl": "reference", "metric": METRIC, "value": round(ms, 4), "unit": "ms",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": args.config, "instance": inst.name, "m": m,
                                        "n": n, "nnz": nnz, "engine": "propagate_parallel (cpu_par)"},
        "rounds": res.rounds_executed, "status": res.status.name,
        "rounds_per_s": round(res.rounds_executed / (ms / 1e3), 2),
        "gbs_per_round": round(b_round(m, n, nnz) * res.rounds_executed / (ms / 1e3) / 1e9, 3),
        "wall_ms_per_step": round(wall, 3),
        "cpu_baseline": {"value": round(ms, 4), "unit": "ms", "cores": threads,
                         "kind": "reference", "sample": f"{args.steps} full solves of {inst.name}"},
        "e2e": {"value": round(ms, 4), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(inst, budget_s=25.0):
    """cpu_seq of the reference (1 core), best of up to 3 solves within ~budget."""
    from oracle import oracle as O
    from paper_2009_07785_b200.model import EngineConfig

    ref = O.ref_available()
    fn = O.ref_propagate_sequential if ref else O.propagate_sequential
    cfg = EngineConfig()
    best, res, t0, runs = None, None, time.perf_counter(), 0
    while runs < 3 and (runs == 0 or time.perf_counter() - t0 < budget_s):
        res = fn(inst, cfg)
        runs += 1
        v = res.elapsed_ns / 1e6
        best = v if best is None else min(best, v)
    return {"value": round(best, 3), "unit": "ms", "cores": 1,
            "kind": "reference" if ref else "port",
            "sample": f"cpu_seq best of {runs} full solves of {inst.name} "
                      f"({res.status.name}, {res.rounds_executed} rounds)",
            "status": res.status.name, "rounds": res.rounds_executed}, res


def _gpu_setup(local, world):
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return torch, dist


def _max_over_ranks(torch, dist, world, local, v):
    if world > 1:
        t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        v = float(t.item())
    return v


def _common_line(args, world, ms, scaling, workload, extra_cfg):
    return {"metric": METRIC, "value": round(ms, 4), "unit": "ms", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": False, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": workload, **extra_cfg}}


def bench_single(args, inst, world, rank, local):
    """C1/C2/C3: one instance per GPU (N > 1: independent replicas)."""
    torch, dist = _gpu_setup(local, world)
    from paper_2009_07785_b200.engine import Session, propagate_gpu
    from paper_2009_07785_b200.model import EngineConfig

    from paper_2009_07785_b200.model import LoopMode
    cfg = EngineConfig(device=local, worklist=args.worklist,
                       loop_mode=LoopMode.Host if args.loop == "host" else LoopMode.Graph)
    m, n, nnz = inst.num_rows(), inst.num_cols(), inst.matrix.nnz()
    sess = Session(inst, cfg)
    info = sess.info()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{local}")
    for _ in range(args.warmup):
        r = sess.run()
    launches_per_round, per_solve = solve_launches(info, args.worklist)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    step_ms, rounds = [], []
    with ClockSampler(local) as clk:
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            r = sess.run()
            step_ms.append(r.elapsed_ns / 1e6)
            rounds.append(r.rounds_executed)
        barrier()
        wall_ms = (time.perf_counter() - t0) * 1e3
    ms = _max_over_ranks(torch, dist, world, local, float(np.sum(step_ms))) / args.steps
    R = rounds[-1]
    gpu_launches = sum(per_solve + rr * launches_per_round for rr in rounds)

    # dominant kernels alone (roofline), first-round snapshot
    k_ns, k_bytes = sess.time_round_kernel(reps=20)
    peak, peak_kind = hbm_peak()
    achieved = k_bytes / (k_ns * 1e-9) / 1e9

    # e2e through the C-ABI (pg_propagate) with pinned host buffers
    pinned = pinned_copy(inst)
    e2e = []
    for _ in range(args.e2e_steps + 1):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        re = propagate_gpu(pinned, cfg)
        e2e.append((time.perf_counter() - t1) * 1e3)
    e2e_ms = _max_over_ranks(torch, dist, world, local, float(np.median(e2e[1:])))
    assert re.status == r.status and re.rounds_executed == R

    line = _common_line(args, world, ms, "weak", args.config, {
        "instance": inst.name, "m": m, "n": n, "nnz": nnz,
        "parallelism": f"replicas x{world}" if world > 1 else "single-gpu",
        "worklist": args.worklist, "l2": "flushed between steps (256 MB write); instance > L2",
        "slices": info["slices"], "chains": info["chains"], "sell_elems": info["sell_elems"],
        "split_segments": info["segments"]})
    line.update({
        "rounds": R, "status": r.status.name,
        "rounds_per_s": round(R / (ms / 1e3), 1),
        "ms_per_round": round(ms / max(R, 1), 5),
        "gbs_per_round": round(b_round(m, n, nnz) * R / (ms / 1e3) / 1e9, 1),
        "round_roofline_frac": round(b_round(m, n, nnz) * R / (ms / 1e3) / 1e9 / peak, 4),
        "round_roofline_frac_8tbs": round(b_round(m, n, nnz) * R / (ms / 1e3) / 8e12, 4),
        "wall_ms_per_step": round(wall_ms / args.steps, 3),
        "roofline": {"kernel": "k_sell+k_cand (dense first round)", "bound": "hbm",
                     "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": _ncu_traffic(args.config, "k_sell"),
                     "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum of k_sell "
                                       "(dense first round), one ncu --set full capture "
                                       "(profiles/roofline_traffic.json)",
                     "bytes_per_launch": k_bytes, "launch_us": round(k_ns / 1e3, 3),
                     "share_of_round": round(k_ns / 1e6 / (ms / max(R, 1)), 3)},
        "e2e": {"value": round(e2e_ms, 3), "unit": "ms",
                "h2d_bytes_per_step": int(12 * nnz + 4 * (m + 1) + 16 * m + 17 * n),
                "d2h_bytes_per_step": int(16 * n + 8 * R)},
        "gpu_launches": int(gpu_launches),
        "clocks": clk.summary(),
    })
    if rank == 0 and not args.no_cpu_baseline:
        cb, _ = cpu_baseline(inst)
        line["cpu_baseline"] = cb
        line["speedup_vs_cpu_seq"] = round(cb["value"] / ms, 2)
        line["e2e_speedup_vs_cpu_seq"] = round(cb["value"] / e2e_ms, 2)
    sess.close()
    return line


def c4_nodes(inst, root_lo, root_up, k0, k1):
    from instances import generators as G
    from paper_2009_07785_b200.engine import node_overrides
    lo, up = G.gen_nodes(inst, root_lo, root_up, K=k1 - k0, seed_base=4_000_000 + k0)
    return lo, up, node_overrides(root_lo, root_up, lo, up)


def bench_nodes(args, inst, world, rank, local):
    """C4: K branch-and-bound child nodes of the root fixpoint, node-sharded
    (contiguous slices, matrix replicated, no per-round communication)."""
    torch, dist = _gpu_setup(local, world)
    from paper_2009_07785_b200.engine import Session
    from paper_2009_07785_b200.model import EngineConfig
    from paper_2009_07785_b200.multi import node_shards

    cfg = EngineConfig(device=local, worklist=True)
    k0, k1 = node_shards(args.nodes, world)[rank]
    sess = Session(inst, cfg)
    root = sess.set_root()
    _, _, (ptr, vs, ls, us) = c4_nodes(inst, root.bounds.lower, root.bounds.upper, k0, k1)
    for _ in range(args.warmup):
        sess.propagate_nodes(ptr[: min(65, len(ptr))], vs, ls, us)
    times = []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for _ in range(args.steps):
            st, rd, _, _, ns = sess.propagate_nodes(ptr, vs, ls, us)
            times.append(ns / 1e6)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = _max_over_ranks(torch, dist, world, local, float(np.mean(times)))
    K = args.nodes
    line = _common_line(args, world, ms, "strong", "c4", {
        "instance": inst.name, "m": inst.num_rows(), "n": inst.num_cols(),
        "nnz": inst.matrix.nnz(), "nodes": K, "parallelism": f"node-sharded x{world}",
        "root_rounds": root.rounds_executed, "warm_start": "root fixpoint + device worklist"})
    line.update({"nodes_per_s": round(K / (ms / 1e3), 1), "ms_per_node": round(ms / (k1 - k0), 4),
                 "rounds_mean": round(float(np.mean(rd)), 3),
                 "status_counts": {str(s): int((st == s).sum()) for s in np.unique(st)},
                 "clocks": clk.summary(), "gpu_launches": None,
                 "e2e": {"value": round(ms, 4), "unit": "ms",
                         "h2d_bytes_per_step": int(4 * len(ptr) + 20 * len(vs)),
                         "d2h_bytes_per_step": int(8 * (k1 - k0))}})
    if rank == 0 and not args.no_cpu_baseline:
        from oracle import oracle as O
        sample = 16
        lo, up, _ = c4_nodes(inst, root.bounds.lower, root.bounds.upper, 0, sample)
        fn = O.ref_propagate_sequential if O.ref_available() else O.propagate_sequential
        t = [fn(inst, EngineConfig(), lo[k], up[k]).elapsed_ns / 1e6 for k in range(sample)]
        per = float(np.mean(t))
        line["cpu_baseline"] = {"value": round(per * K, 1), "unit": "ms", "cores": 1,
                                "kind": "reference" if O.ref_available() else "port",
                                "sample": f"cpu_seq on nodes 0..{sample - 1}, mean {per:.2f} ms/node "
                                          f"x {K} nodes (extrapolated)"}
        line["speedup_vs_cpu_seq"] = round(per * K / ms, 2)
    sess.close()
    return line


def solve_launches(info, worklist):
    """Our kernels per round and per solve (engine.cu enqueue_round /
    enqueue_reset): k_sell (full sweep) + k_cand + k_commit, k_split_finish
    with split rows, and with the worklist the worklist k_sell +
    k_commit_list + k_mark; per solve k_reset (+ k_mark_vars).  The
    persistent loop is one kernel per solve (+ k_reset)."""
    per_round = ((2 if info["slices"] else 0) + 1 + (1 if info["split_rows"] else 0) +
                 (3 if worklist else 0))
    if info["persistent"]:
        per_round = 0
    per_solve = 1 + (1 if worklist else 0) + (1 if info["persistent"] else 0)
    return per_round, per_solve


def bench_rowshard(args, inst, world, rank, local):
    """C5: one 50M-entry set-partitioning instance, row-sharded over the
    GPUs; one NCCL max all-reduce merges the bound keys every round."""
    torch, dist = _gpu_setup(local, world)
    from paper_2009_07785_b200.model import EngineConfig, LoopMode
    from paper_2009_07785_b200.multi import RowShardedSession

    delta = bool(args.delta if args.delta is not None else world > 1)
    cfg = EngineConfig(device=local, worklist=args.worklist, delta_exchange=delta,
                       loop_mode=LoopMode.Host if args.loop == "host" else LoopMode.Graph)
    rs = RowShardedSession(inst, cfg, rank, world)
    for _ in range(args.warmup):
        r = rs.run()
    times = []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        gpu_launches = 0
        info = rs.session.info()
        per_round, per_solve = solve_launches(info, args.worklist)
        for _ in range(args.steps):
            r = rs.run()
            times.append(r.elapsed_ns / 1e6)
            # row shards: no k_commit_list; k_flag_to_slot, or the delta pair
            pr = (per_round - (1 if args.worklist else 0) + (2 if delta else 1)) if rs.comm \
                else per_round
            gpu_launches += per_solve + r.rounds_executed * pr
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = _max_over_ranks(torch, dist, world, local, float(np.mean(times)))
    m, n, nnz = inst.num_rows(), inst.num_cols(), inst.matrix.nnz()
    R = r.rounds_executed
    line = _common_line(args, world, ms, "strong", "c5", {
        "instance": inst.name, "m": m, "n": n, "nnz": nnz,
        "parallelism": (f"row-sharded x{world} (NCCL max all-reduce of bound keys"
                        + (", sparse delta all-gather when every rank changed <= n/16 columns)"
                           if delta else ")")) if world > 1
                       else "single-gpu (one row shard: no exchange)",
        "worklist": args.worklist, "delta_exchange": delta})
    line["delta_rounds"] = rs.session.info()["delta_rounds"]
    line.update({"rounds": R, "status": r.status.name, "rounds_per_s": round(R / (ms / 1e3), 1),
                 "gbs_per_round": round(b_round(m, n, nnz) * R / (ms / 1e3) / 1e9, 1),
                 "clocks": clk.summary(), "gpu_launches": gpu_launches,
                 "e2e": {"value": round(ms, 4), "unit": "ms", "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 8 * R}})
    if rank == 0 and not args.no_cpu_baseline:
        cb, _ = cpu_baseline(inst, budget_s=40.0)
        line["cpu_baseline"] = cb
        line["speedup_vs_cpu_seq"] = round(cb["value"] / ms, 2)
    rs.close()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--nodes", type=int, default=8192, help="C4: number of B&B nodes")
    ap.add_argument("--worklist", type=int, default=None,
                    help="device-side worklist (exact); default: on for c2 and c5 (few rows "
                         "change after the first rounds), off for c1/c3 (faster as full sweeps)")
    ap.add_argument("--delta", type=int, default=None,
                    help="c5: sparse delta exchange rounds (default: on when world > 1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--loop", default="graph", choices=["graph", "host"],
                    help="host: one launch per kernel per round (for ncu launch lists: ncu "
                         "cannot profile kernel nodes of graphs with conditional nodes)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.worklist is None:
        args.worklist = args.config in ("c2", "c5")
    args.worklist = bool(args.worklist)

    world, rank, local = dist_init()
    inst = make_instance(args.config, args.seed)
    if args.impl == "reference":
        run_reference(args, inst, rank, world)
        return
    if args.config == "c4":
        line = bench_nodes(args, inst, world, rank, local)
    elif args.config == "c5":
        line = bench_rowshard(args, inst, world, rank, local)
    else:
        line = bench_single(args, inst, world, rank, local)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
