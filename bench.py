"""bench.py -- time-to-fixpoint of the B200 propagation engine.

Metric (BASELINE.json): time-to-fixpoint & GB/s per round vs the HBM
roofline; speedup vs the CPU reference.  One "step" = one full propagation
of one instance to its fixpoint (or infeasibility / round limit) from its
start bounds.

Workloads (synthetic, seeded, generated in-process):

  N = 1 (default) C2: 1M x 1M, power-law row lengths (~12M entries), mixed
                  bounds incl. infinities, 50% integer, seed 20090778.
  N > 1 (default) C5: 1M x 5M set partitioning (50M entries), row-sharded
                  over the N GPUs, one merge per round over NCCL (dense
                  all-reduce of the bound keys, or sparse delta all-gathers
                  once few columns change); C4's node-sharded batch rides
                  along under "also".  `--config c2` runs N C2 replicas.
  --config c1|c3|c4|c5 one configuration; --config all: C1-C5 at N = 1 and
                  the geomean speedup vs cpu_seq over the >= 1M-entry ones.

Line fields:
  value      device time-to-fixpoint per step (ms, CUDA events around the
             device-resident loop on the engine's stream; inputs resident in
             HBM; L2 flushed by a 256 MB write before every step), max over
             ranks
  e2e        the same solve through the reference-facing C-ABI with HOST
             buffers (pinned), H2D and D2H inside the timed region
  parity     the timed configuration's result against the committed digest
             of the REFERENCE's own propagate_parallel (tests/golden/
             digests.json): "bit-exact" or the differences
  roofline   the dominant kernels of one dense round (k_sell + k_cand),
             timed alone with CUDA events on the engine stream: algorithmic
             bytes (SURVEY.md 8(d) B_round less the commit's share) / mean
             launch time vs MEASURED_PEAKS hbm_gbs
  cpu_baseline  the reference's cpu_seq (compiled from its own sources into
             oracle/_ref), 1 core, best of a bounded number of solves
--impl reference: the reference's cpu_par (oracle/_ref, all host threads) on
the same configuration as this arm at the same N; rank 0 only.
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
SEEDS = {"c1": 1, "c2": 20090778, "c3": 3001, "c4": 4, "c5": 5001}


def b_round(m, n, nnz):
    """SURVEY.md 8(d) algorithmic bytes of one full propagation round."""
    return 12 * nnz + 4 * (m + 1) + 16 * m + 33 * n


def _ncu_traffic(config, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (tools/ncu_traffic.py -> profiles/roofline_traffic.json), or None."""
    path = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)[config]
        ks = d["kernels"]
        return next(int(v["dram_bytes"]) for k, v in ks.items() if kernel in k), d.get("capture", "")
    except (OSError, KeyError, StopIteration, ValueError):
        return None, ""


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def host_cpu():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), "")
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


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


def pin(a):
    import torch
    t = torch.empty(a.shape, dtype={np.int32: torch.int32, np.float64: torch.float64,
                                    np.uint8: torch.uint8}[a.dtype.type], pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


def pinned_out(n):
    """Page-locked result buffers (the e2e D2H destination), reused across calls."""
    return pin(np.zeros(n)), pin(np.zeros(n))


def pinned_copy(inst):
    """Instance arrays in page-locked host memory (the e2e H2D source)."""
    from paper_2009_07785_b200.model import ProblemInstance
    return ProblemInstance.from_arrays(pin(inst.matrix.row_ptr), pin(inst.matrix.col_idx),
                                       pin(inst.matrix.values), pin(inst.lhs), pin(inst.rhs),
                                       pin(inst.bounds.lower), pin(inst.bounds.upper),
                                       pin(inst.integral), num_cols=inst.num_cols(),
                                       name=inst.name)


# ---- parity against the committed reference digests ---------------------------------

def parity(config, seed, res, key="cpu_par"):
    """The result against the reference propagate_parallel digest (the
    timed configuration's own instance; key cpu_par_f32: Narrow32);
    'unpinned' when no digest exists."""
    from instances import digest as D
    try:
        want = D.load()[config][str(seed)][key]
    except (OSError, KeyError):
        return "unpinned (no reference digest for this instance)", None
    diffs = D.compare(res, want)
    return ("bit-exact" if not diffs else "MISMATCH: " + "; ".join(diffs)), want


# ---- the reference arm ----------------------------------------------------------------

def run_reference(args, rank, world):
    """The reference's own cpu_par (all host threads) on this arm's
    configuration; rank 0 only."""
    if rank != 0:
        return None
    from oracle import oracle as O
    from paper_2009_07785_b200.model import EngineConfig

    if not O.ref_available():
        return {"impl": "reference", "unavailable":
                "oracle/_ref/libpropgate_ref.so not built (needs /root/reference at build time)"}
    config = args.config
    inst = make_instance(config, args.seed)
    threads = os.cpu_count() or 1
    cfg = EngineConfig(worker_count=threads)
    budget = args.ref_budget_s
    t0 = time.perf_counter()
    warm = 0
    for _ in range(min(args.warmup, 1)):
        O.ref_propagate_parallel(inst, cfg)
        warm += 1
    one = time.perf_counter() - t0
    # whole solves; as many of the K steps as fit the time budget (>= 1)
    steps = max(1, min(args.steps, int(budget / max(one, 1e-3))))
    times, res = [], None
    t0 = time.perf_counter()
    for _ in range(steps):
        res = O.ref_propagate_parallel(inst, cfg)
        times.append(res.elapsed_ns / 1e6)
    wall = (time.perf_counter() - t0) * 1e3 / steps
    ms = float(np.mean(times))
    m, n, nnz = inst.num_rows(), inst.num_cols(), inst.matrix.nnz()
    cpu = host_cpu()
    return {
        "impl": "reference", "metric": METRIC, "value": round(ms, 4), "unit": "ms",
        "n_gpus": world, "steps": steps, "warmup": warm, "ms_per_step": round(ms, 4),
        "higher_is_better": False, "scaling": "strong" if config == "c5" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": config, "instance": inst.name, "m": m, "n": n, "nnz": nnz,
                   "engine": "propagate_parallel (cpu_par), all host threads"},
        "rounds": res.rounds_executed, "status": res.status.name,
        "rounds_per_s": round(res.rounds_executed / (ms / 1e3), 2),
        "gbs_per_round": round(b_round(m, n, nnz) * res.rounds_executed / (ms / 1e3) / 1e9, 3),
        "wall_ms_per_step": round(wall, 3),
        "cpu_baseline": {"value": round(ms, 4), "unit": "ms", "cores": threads, "kind": "reference",
                         "sample": f"{steps} full solves of {inst.name} (steps capped by a "
                                   f"{budget:.0f} s budget)", **cpu},
        "e2e": {"value": round(ms, 4), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def cpu_baseline(inst, budget_s=25.0, lower=None, upper=None, cfg=None):
    """cpu_seq of the reference (1 core), best of up to 3 solves within ~budget
    (harness default best-of-3, harness.hpp:75)."""
    from oracle import oracle as O
    from paper_2009_07785_b200.model import EngineConfig

    ref = O.ref_available()
    fn = O.ref_propagate_sequential if ref else O.propagate_sequential
    cfg = cfg or EngineConfig()
    best, res, t0, runs = None, None, time.perf_counter(), 0
    while runs < 3 and (runs == 0 or time.perf_counter() - t0 < budget_s):
        res = fn(inst, cfg, lower, upper)
        runs += 1
        v = res.elapsed_ns / 1e6
        best = v if best is None else min(best, v)
    return {"value": round(best, 3), "unit": "ms", "cores": 1,
            "kind": "reference" if ref else "port",
            "sample": f"cpu_seq best of {runs} full solves of {inst.name} "
                      f"({res.status.name}, {res.rounds_executed} rounds)",
            "status": res.status.name, "rounds": res.rounds_executed, **host_cpu()}, res


# ---- GPU arm helpers ------------------------------------------------------------------

def _gpu_setup(local, world):
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return torch, dist


def _max_over_ranks(torch, dist, world, local, v):
    if world > 1:
        t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        v = float(t.item())
    return v


def _barrier(torch, dist, world):
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


def _common_line(args, world, ms, scaling, workload, extra_cfg):
    return {"metric": METRIC, "value": round(ms, 4), "unit": "ms", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": False, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, SURVEY.md 8(d))",
            "config": {"workload": workload, **extra_cfg}}


def solve_launches(info, worklist):
    """Our kernels per round and per solve (engine.cu enqueue_round /
    enqueue_reset): k_sell (full sweep) + k_commit, k_split_finish + k_cand
    with split rows, and with the worklist the worklist k_sell +
    k_commit_list + k_mark; per solve k_reset (+ k_mark_vars).  The
    persistent loop is one kernel per solve (+ k_reset)."""
    per_round = ((1 if info["slices"] else 0) + 1 + (2 if info["split_rows"] else 0) +
                 (3 if worklist else 0))
    if info["persistent"]:
        per_round = 0
    per_solve = 1 + (1 if worklist else 0) + (1 if info["persistent"] else 0)
    return per_round, per_solve


def shard_launches(info, worklist, delta):
    """Kernels of one row-sharded solve in unrolled graphs: every launched
    graph runs shard_rounds rounds (rounds past the decision return at once)
    of k_sell (+ worklist variant), [k_split_finish, k_cand], the exchange
    kernels (k_flag_to_slot; or k_delta_compact + k_delta_apply), k_commit,
    [k_mark]; plus k_reset (+ k_mark_vars) and one k_shard_resume per held
    round.  NCCL's own kernels are not counted."""
    base = ((2 if worklist else 1) if info["slices"] else 0) + (2 if info["split_rows"] else 0) + \
        1 + (1 if worklist else 0)
    R = max(info["shard_rounds"], 1)
    dg = info["delta_graphs"]
    return ((info["host_syncs"] - dg) * R * (base + 1) + dg * R * (base + 2) +
            1 + (1 if worklist else 0) + info["held_rounds"])


# ---- C1 / C2 / C3: one instance per GPU -------------------------------------------------

def bench_single(args, world, rank, local, config):
    torch, dist = _gpu_setup(local, world)
    from paper_2009_07785_b200.engine import Session, propagate_gpu
    from paper_2009_07785_b200.model import EngineConfig, LoopMode

    from paper_2009_07785_b200.model import ScalarMode
    seed = args.seed if args.seed is not None else SEEDS[config]
    inst = make_instance(config, seed)
    f32 = args.scalar == "f32"
    worklist = (args.worklist if args.worklist is not None else config in ("c2", "c5")) and not f32
    cfg = EngineConfig(device=local, worklist=worklist,
                       scalar_mode=ScalarMode.Narrow32 if f32 else ScalarMode.Wide64,
                       loop_mode=LoopMode.Host if args.loop == "host" else LoopMode.Graph)
    m, n, nnz = inst.num_rows(), inst.num_cols(), inst.matrix.nnz()
    sess = Session(inst, cfg)
    info = sess.info()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{local}")
    for _ in range(args.warmup):
        r = sess.run()
    launches_per_round, per_solve = solve_launches(info, worklist)

    step_ms, rounds = [], []
    with ClockSampler(local) as clk:
        _barrier(torch, dist, world)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            r = sess.run()
            step_ms.append(r.elapsed_ns / 1e6)
            rounds.append(r.rounds_executed)
        _barrier(torch, dist, world)
        wall_ms = (time.perf_counter() - t0) * 1e3
    ms = _max_over_ranks(torch, dist, world, local, float(np.sum(step_ms))) / args.steps
    R = rounds[-1]
    gpu_launches = sum(per_solve + rr * launches_per_round for rr in rounds)

    # the timed configuration's result (one more solve, bounds downloaded)
    # against the reference's own cpu_par digest
    par, _ = parity(config, seed, sess.run(download=True), "cpu_par_f32" if f32 else "cpu_par")

    # dominant kernels alone (roofline), first-round snapshot
    k_ns, k_bytes = sess.time_round_kernel(reps=20)
    peak, peak_kind = hbm_peak()
    achieved = k_bytes / (k_ns * 1e-9) / 1e9
    traffic, capture = _ncu_traffic(config, "k_sell")

    # e2e through the C-ABI (pg_propagate) with pinned host buffers
    pinned, out = pinned_copy(inst), pinned_out(inst.num_cols())
    e2e = []
    for _ in range(args.e2e_steps + 1):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        re = propagate_gpu(pinned, cfg, out=out)
        e2e.append((time.perf_counter() - t1) * 1e3)
    e2e_ms = _max_over_ranks(torch, dist, world, local, float(np.median(e2e[1:])))
    e2e_par, _ = parity(config, seed, re, "cpu_par_f32" if f32 else "cpu_par")

    line = _common_line(args, world, ms, "weak", config, {
        "instance": inst.name, "seed": seed, "m": m, "n": n, "nnz": nnz,
        "parallelism": f"replicas x{world}" if world > 1 else "single-gpu",
        "worklist": worklist, "row_check": True, "scalar": args.scalar,
        "l2": "flushed between steps (256 MB write); instance > L2" if config != "c1"
              else "flushed between steps (256 MB write)",
        "slices": info["slices"], "chains": info["chains"], "sell_elems": info["sell_elems"],
        "split_segments": info["segments"]})
    if f32:
        line["dtype"] = "f32 activities / candidates, f64 acceptance (ScalarMode::Narrow32)"
    line.update({
        "rounds": R, "status": r.status.name,
        "parity": par if par == e2e_par else f"timed: {par}; e2e: {e2e_par}",
        "parity_reference": "reference propagate_parallel digest (tests/golden/digests.json): "
                            "status, rounds, per_round_changes, sha256 of the bounds",
        "rounds_per_s": round(R / (ms / 1e3), 1),
        "ms_per_round": round(ms / max(R, 1), 5),
        "wall_ms_per_step": round(wall_ms / args.steps, 3),
        "roofline": {"kernel": "k_sell+k_cand (dense first round)", "bound": "hbm",
                     "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "frac_8tbs": round(achieved / 8000.0, 4),
                     "traffic": traffic,
                     "traffic_source": ("dram__bytes_read.sum + dram__bytes_write.sum of k_sell "
                                        "(dense first round) from a committed ncu --set full "
                                        f"capture ({capture or 'profiles/roofline_traffic.json'}), "
                                        "not this run") if traffic else None,
                     "bytes_per_launch": k_bytes,
                     "bytes_model": "12 nnz + 4(m+1) + 16m + 16n (B_round without the commit's 17n)",
                     "launch_us": round(k_ns / 1e3, 3),
                     "share_of_step": round(k_ns / 1e6 / ms, 3)},
        "e2e": {"value": round(e2e_ms, 3), "unit": "ms",
                "api": "pg_propagate (C-ABI) from pinned host arrays into pinned result buffers: "
                       "upload, device setup, solve, bounds download",
                "h2d_bytes_per_step": int(12 * nnz + 4 * (m + 1) + 16 * m + 17 * n),
                "d2h_bytes_per_step": int(16 * n + 8 * R)},
        "gpu_launches": int(gpu_launches),
        "clocks": clk.summary(),
    })
    if rank == 0 and not args.no_cpu_baseline:
        cb, _ = cpu_baseline(inst, budget_s=args.cpu_budget_s,
                             cfg=EngineConfig(scalar_mode=ScalarMode.Narrow32) if f32 else None)
        line["cpu_baseline"] = cb
        line["speedup_vs_cpu_seq"] = round(cb["value"] / ms, 2)
        line["e2e_speedup_vs_cpu_seq"] = round(cb["value"] / e2e_ms, 2)
    sess.close()
    return line


# ---- C4: batched branch-and-bound nodes, node-sharded ------------------------------------

def c4_nodes(inst, root_lo, root_up, k0, k1):
    from instances import generators as G
    from paper_2009_07785_b200.engine import node_overrides
    lo, up = G.gen_nodes(inst, root_lo, root_up, K=k1 - k0, seed_base=4_000_000 + k0)
    return lo, up, node_overrides(root_lo, root_up, lo, up)


def bench_nodes(args, world, rank, local, cpu=True):
    """C4: K branch-and-bound child nodes of the root fixpoint, node-sharded
    (contiguous slices, matrix replicated, no per-round communication)."""
    torch, dist = _gpu_setup(local, world)
    from instances import digest as D
    from paper_2009_07785_b200.engine import Session
    from paper_2009_07785_b200.model import EngineConfig
    from paper_2009_07785_b200.multi import node_shards

    seed = SEEDS["c4"]
    inst = make_instance("c4", seed)
    cfg = EngineConfig(device=local, worklist=True)
    K = args.nodes
    k0, k1 = node_shards(K, world)[rank]
    sess = Session(inst, cfg)
    root = sess.set_root()
    lo, up, (ptr, vs, ls, us) = c4_nodes(inst, root.bounds.lower, root.bounds.upper, k0, k1)
    for _ in range(args.warmup):
        sess.propagate_nodes(ptr[: min(65, len(ptr))], vs, ls, us)
    times, walls = [], []
    pvs, pls, pus, pptr = pin(vs), pin(ls), pin(us), pin(ptr)
    with ClockSampler(local) as clk:
        _barrier(torch, dist, world)
        for _ in range(args.steps):
            t1 = time.perf_counter()
            st, rd, _, _, ns = sess.propagate_nodes(pptr, pvs, pls, pus)
            walls.append((time.perf_counter() - t1) * 1e3)
            times.append(ns / 1e6)
        _barrier(torch, dist, world)
    ms = _max_over_ranks(torch, dist, world, local, float(np.mean(times)))
    e2e_ms = _max_over_ranks(torch, dist, world, local, float(np.median(walls)))

    # parity: this rank's nodes among 0..63 against the committed digests
    # (bench mode = row check on: the restated cpu_par + row check, pinned
    # to the reference by tests/test_oracle.py)
    par = "unpinned (no reference digest)"
    try:
        want = D.load()["c4"][str(seed)]
        root_ok = D.compare(root, want["cpu_par"])
        nodes = want["nodes_rowcheck"]
        lo_k = [k for k in range(k0, min(k1, len(nodes)))]
        bad = list(root_ok)
        if lo_k:
            sub = np.concatenate([[0], np.cumsum(np.diff(ptr)[: len(lo_k)])]).astype(np.int32)
            st2, rd2, blo, bup, _ = sess.propagate_nodes(sub, vs, ls, us, want_bounds=True)
            for i, k in enumerate(lo_k):
                if D.node_digest(st2[i], rd2[i], blo[i], bup[i]) != nodes[k]:
                    bad.append(f"node {k}")
        par = "bit-exact" if not bad else "MISMATCH: " + ", ".join(bad[:8])
        par += f" (root + nodes {lo_k[0]}..{lo_k[-1]})" if lo_k else " (root)"
    except (OSError, KeyError):
        pass
    line = _common_line(args, world, ms, "strong", "c4", {
        "instance": inst.name, "seed": seed, "m": inst.num_rows(), "n": inst.num_cols(),
        "nnz": inst.matrix.nnz(), "nodes": K, "parallelism": f"node-sharded x{world}",
        "root_rounds": root.rounds_executed,
        "warm_start": "root fixpoint + device worklist (round 1 visits only the rows of "
                      "branched columns)"})
    line.update({"nodes_per_s": round(K / (ms / 1e3), 1), "ms_per_node": round(ms / (k1 - k0), 5),
                 "rounds_mean": round(float(np.mean(rd)), 3),
                 "status_counts": {str(s): int((st == s).sum()) for s in np.unique(st)},
                 "parity": par,
                 "clocks": clk.summary(), "gpu_launches": int(args.steps),
                 "e2e": {"value": round(e2e_ms, 4), "unit": "ms",
                         "api": "pg_session_propagate_nodes from pinned host overrides; statuses "
                                "and rounds downloaded (node bounds stay on the device)",
                         "h2d_bytes_per_step": int(4 * len(ptr) + 20 * len(vs)),
                         "d2h_bytes_per_step": int(8 * (k1 - k0))}})
    if rank == 0 and cpu and not args.no_cpu_baseline:
        from oracle import oracle as O
        sample = 64
        lo_s, up_s, _ = c4_nodes(inst, root.bounds.lower, root.bounds.upper, 0, sample)
        fn = O.ref_propagate_sequential if O.ref_available() else O.propagate_sequential
        t = [fn(inst, EngineConfig(), lo_s[k], up_s[k]).elapsed_ns / 1e6 for k in range(sample)]
        per = float(np.mean(t))
        line["cpu_baseline"] = {"value": round(per * K, 1), "unit": "ms", "cores": 1,
                                "kind": "reference" if O.ref_available() else "port",
                                "sample": f"cpu_seq on nodes 0..{sample - 1}, mean {per:.2f} ms/node "
                                          f"x {K} nodes (extrapolated; cpu_seq re-sweeps every row "
                                          "of a node, seq_engine.cpp:29)", **host_cpu()}
        line["speedup_vs_cpu_seq"] = round(per * K / ms, 2)
        if O.ref_available():
            threads = os.cpu_count() or 1
            tp = [O.ref_propagate_parallel(inst, EngineConfig(worker_count=threads), lo_s[k],
                                           up_s[k]).elapsed_ns / 1e6 for k in range(16)]
            pp = float(np.mean(tp))
            line["cpu_par_per_node"] = {
                "value": round(pp, 3), "unit": "ms/node", "cores": threads, "kind": "reference",
                "sample": "propagate_parallel on nodes 0..15 from their bounds (the reference has "
                          "no warm start: every node is a full solve)",
                "extrapolated_ms": round(pp * K, 1), "speedup": round(pp * K / ms, 2)}
    sess.close()
    return line


# ---- C5: one instance row-sharded over the GPUs -------------------------------------------

def _allreduce_algbw(torch, dist, world, local, count):
    """NCCL all-reduce (max, int64) of the exchange's size through
    torch.distributed on the same GPUs: algbw = bytes / time."""
    if world < 2:
        return None
    t = torch.zeros(count, dtype=torch.int64, device=f"cuda:{local}")
    for _ in range(3):
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ms = _max_over_ranks(torch, dist, world, local, ms)
    return {"bytes": int(count * 8), "ms": round(ms, 4), "algbw_gbs": round(count * 8 / ms / 1e6, 1)}


def bench_rowshard(args, world, rank, local):
    """C5: one 50M-entry set-partitioning instance, row-sharded over the
    GPUs; the shards' bound keys merge every round over NCCL."""
    torch, dist = _gpu_setup(local, world)
    import ctypes as C

    from paper_2009_07785_b200 import abi
    from paper_2009_07785_b200.engine import Session, propagate_gpu
    from paper_2009_07785_b200.model import EngineConfig, LoopMode
    from paper_2009_07785_b200.multi import RowShardedSession

    seed = args.seed if args.seed is not None else SEEDS["c5"]
    inst = make_instance("c5", seed)
    worklist = args.worklist if args.worklist is not None else True
    delta = bool(args.delta if args.delta is not None else world > 1)
    cfg = EngineConfig(device=local, worklist=worklist, delta_exchange=delta,
                       loop_mode=LoopMode.Host if args.loop == "host" else LoopMode.Graph)
    m, n, nnz = inst.num_rows(), inst.num_cols(), inst.matrix.nnz()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{local}")
    rs = RowShardedSession(inst, cfg, rank, world)
    for _ in range(args.warmup):
        r = rs.run()
    times = []
    gpu_launches = 0
    with ClockSampler(local) as clk:
        _barrier(torch, dist, world)
        for _ in range(args.steps):
            flush.zero_()
            _barrier(torch, dist, world)
            r = rs.run()
            times.append(r.elapsed_ns / 1e6)
            info = rs.session.info()
            if rs.comm:
                gpu_launches += shard_launches(info, worklist, delta)
            else:
                pr, ps = solve_launches(info, worklist)
                gpu_launches += ps + r.rounds_executed * pr
        _barrier(torch, dist, world)
    ms = _max_over_ranks(torch, dist, world, local, float(np.mean(times)))
    info = rs.session.info()
    R = r.rounds_executed
    # parity: the row-sharded result against the reference cpu_par digest
    # (= the 1-GPU result: merges are exact and rows are never split); a
    # collective solve, so every rank runs it
    sharded = rs.run(download=True)
    par, _ = parity("c5", seed, sharded)

    # e2e: a one-shot call per rank from pinned host arrays -- this rank's
    # shard uploaded, device setup, communicator, solve, bounds downloaded
    if world > 1:
        from paper_2009_07785_b200.multi import shard_instance
        pshard = pinned_copy(shard_instance(inst, rs.r0, rs.r1))
        out = pinned_out(n)
        e2e = []
        for _ in range(args.e2e_steps):
            _barrier(torch, dist, world)
            t1 = time.perf_counter()
            one = RowShardedSession(inst, cfg, rank, world, shard=pshard)
            re = one.propagate(out=out)
            one.close()
            e2e.append((time.perf_counter() - t1) * 1e3)
        e2e_ms = _max_over_ranks(torch, dist, world, local, float(np.median(e2e)))
        e2e_api = ("per rank: pg_session_create of the rank's row shard from pinned host arrays "
                   "(upload + device setup), pg_session_attach_comm (NCCL communicator init), "
                   "solve, bounds download, destroy")
        h2d = int(12 * (inst.matrix.row_ptr[rs.r1] - inst.matrix.row_ptr[rs.r0]) +
                  20 * (rs.r1 - rs.r0) + 17 * n)
    else:
        pinned, out = pinned_copy(inst), pinned_out(n)
        e2e = []
        for _ in range(args.e2e_steps + 1):
            t1 = time.perf_counter()
            re = propagate_gpu(pinned, cfg, out=out)
            e2e.append((time.perf_counter() - t1) * 1e3)
        e2e_ms = float(np.median(e2e[1:]))
        e2e_api = ("pg_propagate (C-ABI) from pinned host arrays into pinned result buffers: upload, "
                   "device setup, solve, download")
        h2d = int(12 * nnz + 4 * (m + 1) + 16 * m + 17 * n)
    e2e_par, _ = parity("c5", seed, re)

    exchange = None
    single = None
    if world > 1:
        nccl_ver = None
        try:
            nccl_ver = ".".join(str(x) for x in torch.cuda.nccl.version())
        except Exception:
            pass
        exchange = {
            "nranks": world, "nccl": nccl_ver, "rounds": R,
            "dense_rounds": R - info["delta_rounds"], "delta_rounds": info["delta_rounds"],
            "held_rounds": info["held_rounds"], "host_syncs": info["host_syncs"],
            "rounds_per_graph": info["shard_rounds"],
            "dense_bytes_per_round": 16 * (n + 1),
            "delta_bytes_per_round": "24 B x capacity tier x ranks (fixed-size all-gather)",
            "allreduce_same_size": _allreduce_algbw(torch, dist, world, local, 2 * (n + 1)),
            "loop": "graphs of unrolled rounds, the host reads the round state once per graph"}
        # the same instance on ONE GPU in this run (rank 0 alone): the
        # strong-scaling reference point and the bit-identity check
        if rank == 0:
            s1 = Session(inst, EngineConfig(device=local, worklist=worklist))
            for _ in range(args.warmup):
                s1.run()
            t1 = []
            for _ in range(args.steps):
                flush.zero_()
                torch.cuda.synchronize()
                t1.append(s1.run().elapsed_ns / 1e6)
            r1 = s1.run(download=True)
            from instances import digest as D
            same = D.result_digest(r1) == D.result_digest(sharded)
            single = {"value": round(float(np.mean(t1)), 4), "unit": "ms",
                      "rounds": r1.rounds_executed, "bit_identical_to_sharded": same}
            s1.close()
        if world > 1:
            dist.barrier()
    line = _common_line(args, world, ms, "strong", "c5", {
        "instance": inst.name, "seed": seed, "m": m, "n": n, "nnz": nnz,
        "parallelism": (f"row-sharded x{world} (NCCL max all-reduce of the bound keys; sparse delta "
                        "all-gather rounds once few columns change)" if delta else
                        f"row-sharded x{world} (NCCL max all-reduce of the bound keys)")
                       if world > 1 else "single-gpu (one row shard: no exchange)",
        "worklist": worklist, "row_check": True, "delta_exchange": delta,
        "l2": "flushed between steps (256 MB write); instance > L2"})
    line.update({"rounds": R, "status": r.status.name,
                 "parity": par if par == e2e_par else f"timed: {par}; e2e: {e2e_par}",
                 "rounds_per_s": round(R / (ms / 1e3), 1),
                 "ms_per_round": round(ms / max(R, 1), 5),
                 "clocks": clk.summary(), "gpu_launches": int(gpu_launches),
                 "e2e": {"value": round(e2e_ms, 3), "unit": "ms", "api": e2e_api,
                         "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": int(16 * n + 8 * R)}})
    if exchange:
        line["exchange"] = exchange
    if single:
        line["single_gpu"] = single
    if rank == 0 and not args.no_cpu_baseline:
        cb, _ = cpu_baseline(inst, budget_s=args.cpu_budget_s)
        line["cpu_baseline"] = cb
        line["speedup_vs_cpu_seq"] = round(cb["value"] / ms, 2)
        line["e2e_speedup_vs_cpu_seq"] = round(cb["value"] / e2e_ms, 2)
    rs.close()
    return line


# ---- all configurations (N = 1): geomean ---------------------------------------------------

def bench_all(args, world, rank, local):
    lines = {}
    for cfg in ("c1", "c2", "c3", "c4", "c5"):
        a = argparse.Namespace(**vars(args))
        a.config = cfg
        a.seed = None
        a.worklist = None
        lines[cfg] = bench_one(a, world, rank, local)
        print(f"[bench all] {cfg}: {lines[cfg]['value']} ms, parity {lines[cfg].get('parity')}",
              file=sys.stderr, flush=True)
    big = [c for c in ("c2", "c3", "c4", "c5") if "speedup_vs_cpu_seq" in lines[c] and
           lines[c]["config"]["nnz"] >= 1_000_000]
    geo = float(np.exp(np.mean([np.log(lines[c]["speedup_vs_cpu_seq"]) for c in big]))) if big else None
    geo_e2e = [c for c in big if "e2e_speedup_vs_cpu_seq" in lines[c]]
    g2 = float(np.exp(np.mean([np.log(lines[c]["e2e_speedup_vs_cpu_seq"]) for c in geo_e2e]))) \
        if geo_e2e else None
    head = dict(lines["c2"])
    head["config"] = dict(head["config"], workload="all (headline line = c2; per-config below)")
    head["geomean_speedup_vs_cpu_seq"] = round(geo, 2) if geo else None
    head["geomean_over"] = big
    head["geomean_e2e_speedup_vs_cpu_seq"] = round(g2, 2) if g2 else None
    head["configs"] = {c: {k: v for k, v in ln.items() if k in (
        "value", "rounds", "status", "parity", "speedup_vs_cpu_seq", "e2e_speedup_vs_cpu_seq",
        "roofline", "e2e", "cpu_baseline", "config", "nodes_per_s", "cpu_par_per_node")}
        for c, ln in lines.items()}
    return head


def bench_one(args, world, rank, local):
    if args.config == "c4":
        return bench_nodes(args, world, rank, local)
    if args.config == "c5":
        return bench_rowshard(args, world, rank, local)
    return bench_single(args, world, rank, local, args.config)


def spawn_ranks(args):
    """--gpus N without a launcher: re-exec under torchrun, one rank per GPU."""
    try:
        import torch
        have = torch.cuda.device_count()
    except Exception:
        have = 0
    if have < args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs; this box has "
                         f"{have}. Nothing was run.\n")
        sys.exit(2)
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.run(cmd).returncode)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=None, choices=["c1", "c2", "c3", "c4", "c5", "all"],
                    help="default: c2 at N = 1, c5 (row-sharded) + c4 (node-sharded) at N > 1")
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--nodes", type=int, default=8192, help="C4: number of B&B nodes")
    ap.add_argument("--worklist", type=int, default=None,
                    help="device-side worklist (exact); default: on for c2, c4, c5, off for c1/c3")
    ap.add_argument("--delta", type=int, default=None,
                    help="c5: sparse delta exchange rounds (default: on when world > 1)")
    ap.add_argument("--scalar", default="f64", choices=["f64", "f32"],
                    help="f32: ScalarMode::Narrow32 (run_parallel<float>), c1-c3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-also", action="store_true", help="N > 1: skip the C4 line under 'also'")
    ap.add_argument("--cpu-budget-s", type=float, default=25.0)
    ap.add_argument("--ref-budget-s", type=float, default=150.0)
    ap.add_argument("--loop", default="graph", choices=["graph", "host"],
                    help="host: one launch per kernel per round (for ncu launch lists: ncu "
                         "cannot profile kernel nodes of graphs with conditional nodes)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.worklist is not None:
        args.worklist = bool(args.worklist)

    world, rank, local = dist_init()
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        sys.exit(2)
    if args.impl == "reference":
        if args.config is None:
            args.config = "c2" if args.gpus == 1 else "c5"
        if args.config == "all":
            args.config = "c2"
        line = run_reference(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if args.config is None:
        args.config = "c2" if world == 1 else "c5"
    if args.config == "all":
        if world > 1:
            sys.stderr.write("bench.py: --config all runs at N = 1\n")
            sys.exit(2)
        line = bench_all(args, world, rank, local)
    else:
        line = bench_one(args, world, rank, local)
        if world > 1 and args.config == "c5" and not args.no_also:
            also = bench_nodes(args, world, rank, local, cpu=False)
            if rank == 0:
                line["also"] = {"c4_node_sharded": {k: also.get(k) for k in (
                    "value", "unit", "nodes_per_s", "ms_per_node", "rounds_mean", "parity",
                    "status_counts", "e2e", "config")}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
