#!/usr/bin/env python
"""Benchmark of the B200 Goodput planner hot path (BASELINE.json metric).

One step = one per-window reconfiguration decision (solve_dp) on a config-1
window: 2 tenants, A100 7-slice lattice, S = 200 one-second slots, Poisson
arrivals (synthetic). Metric: candidate plans scored per
second, where one candidate plan = one reference DP transition
(solvers.hpp:424-469; 154,202,318 for the seed-100001 window).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1: one rank per GPU (bench.py re-launches itself under
torch.distributed.run when WORLD_SIZE is unset). Weak scaling for the headline:
every rank plans its own config-1 window (seed 100001 + rank) with no data-path
collective; after each step the per-window results (objective bits, plan
checksum) are all-gathered over NCCL. The config-4 Goodput-table leg shards its
4096 traces across the ranks (strong scaling), the config-5 leg gives each rank
its physical-GPU subproblems, and the lane-batch leg gives each rank its own
windows; every leg is timed as the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0
SAMPLE = os.path.join(ROOT, "tests", "golden", "c1", "c1_S60_100003.scn")  # bounded CPU sample
S200_WINDOW = os.path.join(ROOT, "tests", "golden", "c1", "c1_S200_100001.scn")  # the window our arm times
# reference DP transitions of that window (solvers.hpp:424-469), counted by the
# restatement and pinned to the device's counter by tests/test_gpu.py::test_c1_counters_match_oracle
C1_S200_TRANSITIONS = 154202318
METRIC = "candidate plans scored/sec (GB/s vs HBM roofline); per-window decision latency ms"
UNIT = "candidate plans/s"


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), "--query-gpu=" + q, "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                rows.append(parts)
        os.unlink(self.f.name)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i] == "Active"})
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def hbm_peak():
    try:
        d = json.load(open(PEAKS))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def c1_problem(seed, directory, pinned=False):
    from paper_2407_13126_b200 import scenario as SC
    from paper_2407_13126_b200 import workloads as W
    spec = W.c1_spec(seed)
    path = W.write_scenario(spec, directory, "c1_%d" % seed)
    sc = SC.load_scenario(path)
    p = SC.Problem(sc, 0)
    if pinned:  # forecast in pinned host memory for the end-to-end leg
        import torch
        t = torch.from_numpy(p.forecast.copy()).pin_memory()
        p._pinned = t
        import ctypes as C
        p.c.forecast = C.cast(t.data_ptr(), C.POINTER(C.c_int64))
    return p


def reference_cpu(steps, warmup, workers):
    """The unmodified reference solve_dp on the bounded sample (oracle/_ref)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import binding  # noqa: E402  (checker / CPU-baseline only)
    times = []
    for k in range(warmup + steps):
        secs, obj, enc = binding.ref_solve_inproc(SAMPLE, 0, workers)
        if k >= warmup:
            times.append(secs)
    return times


SAMPLE_TRANSITIONS = None


def sample_transitions():
    """Reference-defined transition count of the bounded sample (from the golden
    counters of the restatement, which the GPU tests pin to the device's)."""
    global SAMPLE_TRANSITIONS
    if SAMPLE_TRANSITIONS is None:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import binding
        from paper_2407_13126_b200 import scenario as SC
        p = SC.Problem(SC.load_scenario(SAMPLE), 0)
        _, _, st = binding.solve_window(p)
        SAMPLE_TRANSITIONS = st["transitions_ref"]
    return SAMPLE_TRANSITIONS


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    workers = os.cpu_count() or 1
    times = reference_cpu(args.steps, args.warmup, workers)
    tr = sample_transitions()
    value = tr * len(times) / sum(times)
    s200 = None
    if args.s200:  # one full config-1 window, the same one our arm times (seed 100001)
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import binding  # noqa: E402  (reference arm only)
        secs, obj, enc = binding.ref_solve_inproc(S200_WINDOW, 0, workers)
        s200 = {"window": os.path.relpath(S200_WINDOW, ROOT), "seconds": secs, "workers": workers,
                "transitions": C1_S200_TRANSITIONS, "value": C1_S200_TRANSITIONS / secs, "unit": UNIT,
                "objective_bits": bits(obj)}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "config-1-shaped window, S=60 (bounded sample of the S=200 window)",
                       "sample": os.path.relpath(SAMPLE, ROOT), "tenants": 2, "lattice": "a100 7-slice",
                       "parallelism": "host threads (SolveOptions::workers=%d)" % workers},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "reference",
                             "sample": "reference solve_dp on the S=60 config-1-shaped window, %d transitions" % tr},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if s200:
        line["decision_latency_ms_s200"] = 1e3 * s200["seconds"]
        line["s200"] = s200
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2407_13126_b200 import planner
    rank, world, local = env_rank()
    # one rank per GPU; --dist-backend gloo lets a functional N>1 check share
    # fewer GPUs (ranks wrap around the visible devices)
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    coll_dev = "cuda" if args.dist_backend == "nccl" else "cpu"
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    work = tempfile.mkdtemp(prefix="mgs_bench_")
    seed = 100001 + rank
    prob = c1_problem(seed, work)
    prob_e2e = c1_problem(seed, work, pinned=True)
    stream = torch.cuda.Stream()
    pl = planner.Planner(local)
    pl.lib.mgs_set_stream(pl.h, stream.cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    from paper_2407_13126_b200 import shard

    def combine(obj, opt):
        # per-window result of every shard (objective bits, plan checksum): one
        # NCCL all-gather over NVLink, the only collective of the step
        if world > 1:
            return shard.gather_rows([[shard.objective_key(obj), plan_checksum(opt)]], world, device=coll_dev)
        return [[shard.objective_key(obj), plan_checksum(opt)]]

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            opt, cfg, lab, obj, st = pl.solve_window(prob)
            combine(obj, opt)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clocks = Clocks(local)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        stats = []
        for k in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (outside the event pair)
            ev[k][0].record(stream)
            opt, cfg, lab, obj, st = pl.solve_window(prob)
            gathered = combine(obj, opt)
            ev[k][1].record(stream)
            stats.append(st)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clk = clocks.stop()
        step_ms = [a.elapsed_time(b) for a, b in ev]

        # end-to-end through the C ABI with host buffers (H2D forecast from
        # pinned memory, D2H plan + objective inside every step)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(args.steps):
            opt_e, cfg_e, lab_e, obj_e, st_e = pl.solve_window(prob_e2e)
            combine(obj_e, opt_e)
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        if world > 1:
            dist.barrier()

    tr_window = stats[-1]["transitions_ref"]
    dev_s = sum(step_ms) / 1e3
    trans_ms = sum(s["phase_ms"]["transitions"] for s in stats)
    trans_bytes = sum(s["transition_bytes"] for s in stats)
    launches = sum(s["kernel_launches"] for s in stats)
    my_dev_s, my_e2e_s = dev_s, e2e_s
    per_rank = [[rank, local, int(1e6 * dev_s), int(1e6 * e2e_s)]]
    if world > 1:
        per_rank = shard.gather_rows(per_rank, world, device=coll_dev)
        t = torch.tensor([dev_s, e2e_s], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s, e2e_s = t.tolist()
        n = torch.tensor([float(tr_window)], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(n, op=dist.ReduceOp.SUM)
        total_tr = n.item() * args.steps
    else:
        total_tr = float(tr_window) * args.steps
    # the legs below collect over all ranks (collectives inside), rank 0 prints
    legs = {}
    if args.batch > 0:
        legs["batch"] = batch_leg(pl, work, rank, world, args.batch, coll_dev)
    if args.table > 0:
        legs["goodput_table"] = table_leg(pl, work, stream, args.table, rank, world, coll_dev)
    if args.c5:
        legs["config5"] = c5_leg(pl, rank, world, coll_dev)
    if args.table > 0:
        legs["config4_dp"] = c4_dp_leg(pl, rank, world, coll_dev)
    if world == 1 and not args.no_cpu_baseline:
        legs["same_config"] = same_config_leg(pl)
    if rank != 0:
        pl.close()
        if world > 1:
            dist.destroy_process_group()
        return

    # parity check of the timed plan (seed 100001 golden from the reference)
    g = None
    gpath = os.path.join(ROOT, "tests", "golden", "c1", "c1_golden.json")
    if os.path.exists(gpath):
        g = json.load(open(gpath)).get("c1_S200_%d" % seed)
    peak, peak_kind = hbm_peak()
    # B_dp = sum_s(|F_s| R + |F_s+1| (R+8)) + 8 M S + |O| (13 M + 8), R = 24 + 4M
    st0 = stats[-1]
    M_, S_ = prob.M, prob.S
    R = 24 + 4 * M_
    b_dp = (st0["frontier_total"] + 1) * R + st0["frontier_total"] * (R + 8) + 8 * M_ * S_ + st0["options"] * (13 * M_ + 8)
    dp_ms = trans_ms / len(stats)  # device time of the DP graph per window (phase 3)
    achieved = b_dp / (dp_ms / 1e3) / 1e9 if dp_ms > 0 else 0.0
    traffic = measured_traffic()
    phases = {}
    for s in stats:
        for k, v in s["phase_ms"].items():
            phases[k] = phases.get(k, 0.0) + v / len(stats)
    line = {
        "metric": METRIC, "value": total_tr / dev_s, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dev_s / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config-1 window: 2 ResNet-18 tenants, A100 7-slice lattice (12 configs, 9864 options), "
                               "S=200 x 1 s slots, Poisson lambda 120/150, psi 0.5",
                   "seed": "100001+rank", "transitions_per_window": tr_window,
                   "transitions_gpu_evaluated_per_window": stats[-1]["transitions"],
                   "frontier_states_per_window": stats[-1]["frontier_total"], "parallelism": "dp%d" % world,
                   "collective": "per-step all-gather of (objective bits, plan checksum) over %s" % args.dist_backend,
                   "l2": "flushed between timed steps (256 MiB write)"},
        "per_rank": [{"rank": r[0], "device": r[1], "device_ms_per_step": r[2] / 1e3 / args.steps,
                      "e2e_ms_per_step": r[3] / 1e3 / args.steps} for r in per_rank],
        "gathered_window_results": [{"objective": shard.key_objective(g[0]), "plan_checksum": g[1]} for g in gathered],
        "decision_latency_ms": 1e3 * dev_s / args.steps,
        "phase_ms_per_window": phases,
        "e2e": {"value": total_tr / e2e_s, "unit": UNIT,
                "h2d_bytes_per_step": int(prob_e2e.forecast.nbytes + prob_e2e.slot_offset.nbytes +
                                          prob_e2e.slot_size.nbytes + prob_e2e.slot_start.nbytes),
                # options, configurations, labels and the objective: one packed read-back per solve
                "d2h_bytes_per_step": int(prob_e2e.S * (4 + 4 + 8) + 8),
                "decision_latency_ms": 1e3 * e2e_s / args.steps,
                "timing": "host wall clock around the C-ABI solve (pinned forecast in, plan out), max over ranks"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": "per-window DP graph (12 phase kernels x S steps in three graph branches, one graph launch)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if peak else None,
                     "traffic": traffic.get("bytes_per_window") if traffic else None,
                     "traffic_source": traffic.get("source") if traffic else None,
                     "peak_kind": peak_kind, "algorithmic_bytes_per_window": int(b_dp),
                     "dp_ms_per_window": dp_ms,
                     "library_transition_bytes_per_window": trans_bytes // max(1, len(stats))},
        "clocks": clk,
        "objective": obj,
    }
    if g:
        line["parity"] = {"golden": "c1_S200_%d" % seed, "objective_bits_equal": g["dp"]["obj"] == bits(obj)}
    line.update(legs)
    if world == 1 and not args.no_cpu_baseline:
        times = reference_cpu(1, 0, 1)
        tr = sample_transitions()
        line["cpu_baseline"] = {"value": tr / times[0], "unit": UNIT, "cores": 1, "kind": "reference",
                                "sample": "reference solve_dp, workers=1, S=60 config-1-shaped window "
                                          "(tests/golden/c1/c1_S60_100003.scn, %d transitions, %.2f s)" % (tr, times[0])}
    print(json.dumps(line), flush=True)
    pl.close()
    if world > 1:
        dist.destroy_process_group()


def measured_traffic():
    """DRAM bytes per C1 window from the committed ncu metrics pass (profiles/)."""
    path = os.path.join(ROOT, "profiles", "r2", "traffic_c1.json")
    try:
        return json.load(open(path))
    except (OSError, ValueError):
        return None


def plan_checksum(options) -> int:
    """FNV-1a over the chosen option indices (63-bit), for the per-step gather."""
    h = 1469598103934665603
    for o in options:
        h = ((h ^ (int(o) & 0xFFFFFFFF)) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h & 0x7FFFFFFFFFFFFFFF


def max_over_ranks(x, world, device):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def batch_leg(pl, work, rank, world, n, coll_dev):
    """Throughput with n independent C1 windows per rank (seeds 100001+rank*n ...)
    solved as batched lanes (mgs_solve_batch: windows share every DP kernel
    launch). Weak scaling: per-rank work fixed; time = max over ranks."""
    import torch
    from paper_2407_13126_b200 import shard
    probs = [c1_problem(100001 + rank * n + k, work) for k in range(n)]
    pl.solve_batch(probs)  # warm: capacity growth + graph capture for this lane count
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    t0 = time.perf_counter()
    opts, obj, status, stats, errs = pl.solve_batch(probs)
    dt = max_over_ranks(time.perf_counter() - t0, world, coll_dev)
    rows = [[100001 + rank * n + k, shard.objective_key(float(obj[k])), int(status[k])] for k in range(n)]
    rows = shard.gather_rows(rows, world, device=coll_dev)
    tr = sum(s["transitions_ref"] for s in stats) * world  # equal work per rank (same window shape)
    lanes = min(n, int(os.environ.get("MGS_BATCH_LANES", "32")))
    return {"workload": "%d config-1 windows per rank (%d total), %d lanes per launch" % (n, n * world, lanes),
            "value": tr / dt, "unit": UNIT, "ms_per_window": 1e3 * dt / n, "ok": sum(1 for r in rows if r[2] == 0),
            "windows": len(rows), "scaling": "weak",
            "timing": "host wall clock around mgs_solve_batch (host buffers in, plans out), max over ranks"}


def table_leg(pl, work, stream, n_traces, rank, world, coll_dev, reps=5):
    """Config 4: the Goodput table (ub_suffix) of a batch of 4-tenant, 600-slot
    MMPP traces sharing one window's tables (mgs_goodput_table_batch), the 4096
    traces sharded across the ranks (strong scaling). Device leg: traces
    resident in HBM, CUDA events on the planner's stream, max over ranks; e2e
    leg: host traces in, host ub_suffix out through the C ABI. Per-trace
    results are all-gathered (bound of slot 0 as IEEE bits)."""
    import numpy as np
    import torch
    from paper_2407_13126_b200 import scenario as SC
    from paper_2407_13126_b200 import shard
    from paper_2407_13126_b200 import workloads as W
    p = SC.Problem(SC.load_scenario(W.write_scenario(W.c2_spec(400000, steps=600, windows=1), work, "c4")), 0)
    lo, hi = shard.shard_range(n_traces, rank, world)
    mine = hi - lo
    traces = np.stack([W.mmpp_trace([40.0, 120.0, 12.0, 10.0], p.S, 400000 + k)
                       for k in range(lo, hi)]).astype(np.int32)  # seeds 400000..404095
    n_opt = len(pl.enumerate(p)["config"])
    with torch.cuda.stream(stream):
        d_arr = torch.from_numpy(traces).cuda()
        d_ub = torch.empty((mine, p.S + 1), dtype=torch.float64, device="cuda")
        d_best = torch.empty((mine, p.S), dtype=torch.float64, device="cuda")
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        npar = pl.goodput_table_batch_device(p, d_arr.data_ptr(), mine, d_best.data_ptr(), d_ub.data_ptr())
        torch.cuda.synchronize()
        evs = []
        for _ in range(reps):  # everything queued first: host latency never shows in the event pairs
            flush.zero_()  # traces are 39 MB < L2: flush between timed launches
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pl.goodput_table_batch_device(p, d_arr.data_ptr(), mine, d_best.data_ptr(), d_ub.data_ptr())
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        ms = [a.elapsed_time(b) for a, b in evs]
    t_ms = max_over_ranks(sum(ms) / len(ms), world, coll_dev)
    pinned = torch.from_numpy(traces).pin_memory().numpy()
    t0 = time.perf_counter()
    for _ in range(reps):
        ub_h, _ = pl.goodput_table_batch(p, pinned)
    e2e_ms = max_over_ranks((time.perf_counter() - t0) / reps * 1e3, world, coll_dev)
    rows = shard.gather_rows([[lo + i, shard.objective_key(float(ub_h[i, 0]))] for i in range(mine)], world, coll_dev)
    M, S = p.M, p.S
    algo = n_traces * M * S * 4 + world * npar * M * 8 + n_traces * S * 8 + n_traces * (S + 1) * 8
    peak, peak_kind = hbm_peak()
    scanned = n_traces * S * npar
    return {"workload": "config 4: %d MMPP traces x 4 tenants (ResNet-50/MobileNetV2/ViT-B/BERT-base) x 600 slots, "
                        "A100 lattice, %d options, %d Pareto placements; traces sharded over %d rank(s)"
                        % (n_traces, n_opt, npar, world),
            "value": scanned / (t_ms / 1e3),
            "unit": "Goodput-table cells scanned/s (trace x slot x Pareto placement)",
            "cells_scanned_per_batch": scanned,
            "cells_all_options_per_batch": n_traces * S * n_opt,
            "note": "the kernel scans only the Pareto-maximal placements; the other options can never win "
                    "(monotone rounding, csrc/table.cu) and are not counted",
            "ms_per_batch": t_ms, "traces_per_s": n_traces / (t_ms / 1e3), "scaling": "strong",
            "traces_gathered": len(rows),
            "e2e": {"ms_per_batch": e2e_ms, "h2d_bytes": int(traces.nbytes) * world,
                    "d2h_bytes": int(n_traces * (S + 1) * 8)},
            "roofline": {"bound": "hbm", "kernel": "k_table", "achieved": algo / (t_ms / 1e3) / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": algo / (t_ms / 1e3) / 1e9 / peak, "algorithmic_bytes": algo,
                         "peak_kind": peak_kind},
            "ub0": float(ub_h[0, 0]) if mine else None}


def c4_dp_leg(pl, rank, world, coll_dev, n=8):
    """Config 4's DP at the size the reference can pin: the
    M = 2 / S = 200 variant of the C4 generator (first two tenants of traces
    400000 + rank*n + k), n windows per rank solved as one lane batch."""
    import tempfile
    import torch
    from paper_2407_13126_b200 import scenario as SC
    from paper_2407_13126_b200 import shard
    from paper_2407_13126_b200 import workloads as W
    d = tempfile.mkdtemp(prefix="mgs_c4dp_")
    seeds = [400000 + rank * n + k for k in range(n)]
    probs = [SC.Problem(SC.load_scenario(W.write_scenario(W.c2_spec(sd, steps=200, windows=1, tenants=2), d,
                                                          "c4_%d" % sd)), 0) for sd in seeds]
    pl.solve_batch(probs)  # warm: capacity + graph for this lane count
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    t0 = time.perf_counter()
    opts, obj, status, stats, errs = pl.solve_batch(probs)
    dt = max_over_ranks(time.perf_counter() - t0, world, coll_dev)
    rows = shard.gather_rows([[sd, shard.objective_key(float(obj[k])), int(status[k])] for k, sd in enumerate(seeds)],
                             world, coll_dev)
    tr = sum(st["transitions_ref"] for st in stats) * world
    return {"workload": "config 4 DP variant: first two tenants of C4 traces, S=200, %d windows per rank as lanes" % n,
            "value": tr / dt, "unit": UNIT, "ms_per_window": 1e3 * dt / n, "windows": len(rows),
            "ok": sum(1 for r in rows if r[2] == 0), "scaling": "weak",
            "timing": "host wall clock around mgs_solve_batch, max over ranks"}


def c5_leg(pl, rank, world, coll_dev):
    """Config 5: 8 physical A100 MIG GPUs x 7 slices, 16 tenants, 1800 slots,
    decomposed into 8 independent two-tenant subproblems (tenants 2k, 2k+1 on
    MIG GPU k; workloads.c5_specs, seeds 500001..500008), each planned over its
    9 windows by the per-window loop (carried final ranges, oracle forecasts).
    Rank r plans the subproblems of shard_range(8, r, world) as batched lanes;
    per-window realized objectives are all-gathered; time = max over ranks."""
    import tempfile
    import torch
    from paper_2407_13126_b200 import driver
    from paper_2407_13126_b200 import scenario as SC
    from paper_2407_13126_b200 import shard
    from paper_2407_13126_b200 import workloads as W
    specs = W.c5_specs()
    lo, hi = shard.shard_range(len(specs), rank, world)
    d = tempfile.mkdtemp(prefix="mgs_c5_")
    scs = [SC.load_scenario(W.write_scenario(specs[k], d, "c5_gpu%d" % k)) for k in range(lo, hi)]
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    t0 = time.perf_counter()
    plans = driver.plan_scenarios(pl, scs) if scs else []
    torch.cuda.synchronize()
    dt = max_over_ranks(time.perf_counter() - t0, world, coll_dev)
    rows = [[lo + i, wp.window, shard.objective_key(wp.realized)] for i, ws in enumerate(plans) for wp in ws]
    rows = shard.gather_rows(rows, world, coll_dev) if world > 1 else rows
    windows = len(rows)
    return {"workload": "config 5: 8 MIG GPUs x 7 slices (A100 lattice), 16 tenants (2 per GPU), 1800 slots = "
                        "9 windows x 200; per-GPU two-tenant subproblems, %d per rank" % (hi - lo),
            "windows_planned": windows, "seconds": dt, "ms_per_window_decision": 1e3 * dt / max(1, windows) * world,
            "box_planning_latency_s": dt,
            "realized_total": sum(shard.key_objective(r[2]) for r in rows),
            "timing": "host wall clock around the per-window loop (forecast, batched solve, evaluate), max over ranks",
            "scaling": "strong (8 subproblems split over the ranks)"}


def same_config_leg(pl):
    """Like-for-like with the reference arm's bounded sample: the GPU on the same
    S=60 window (c1_S60_100003) the CPU baseline times."""
    import torch
    from paper_2407_13126_b200 import scenario as SC
    p = SC.Problem(SC.load_scenario(SAMPLE), 0)
    for _ in range(2):
        pl.solve_window(p)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 5
    for _ in range(reps):
        opt, cfg, lab, obj, st = pl.solve_window(p)
    dt = (time.perf_counter() - t0) / reps
    tr = st["transitions_ref"]
    return {"sample": os.path.relpath(SAMPLE, ROOT), "value": tr / dt, "unit": UNIT,
            "decision_latency_ms": 1e3 * dt, "transitions": tr,
            "timing": "host wall clock around the C-ABI solve (same call as the e2e leg)"}


def bits(x):
    import struct
    return "%016x" % struct.unpack("<Q", struct.pack("<d", float(x)))[0]


def relaunch(args):
    """--gpus N without a launcher: one rank per GPU under torch.distributed.run."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="collective backend for N>1 (gloo only for functional checks on fewer GPUs)")
    ap.add_argument("--batch", type=int, default=32, help="windows in the batched-lanes throughput leg (0: skip)")
    ap.add_argument("--table", type=int, default=4096, help="traces in the config-4 Goodput-table leg (0: skip)")
    ap.add_argument("--c5", type=int, default=1, help="run the config-5 leg (8 MIG GPUs x 16 tenants)")
    ap.add_argument("--s200", type=int, default=1, help="reference arm: also time one full S=200 window")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
