#!/usr/bin/env python
"""Benchmark of the tour-construction hot path (BASELINE.json metric).

A step is one synchronous ACO iteration over the whole colony (every ant builds a
tour against the frozen colony, then the completion step runs) on the C5
workload by default: 200,000-city mixed instance, m=1024 ants, k=16, alpha=1,
beta=2 (BASELINE.json configs[4], the config the >=40%-of-roofline target is
quoted on). Multi-GPU = independent replicas (the path shards by
ants but one GPU already holds every chain, so ranks run separate seeds).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]

Prints one JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "city-selection decisions/sec"
UNIT = "decisions/s"


def b_dec(k: int) -> int:
    """algorithmic bytes per candidate-hit decision = k*(4 idx + 8 coords + 4 tau) + 4."""
    return 16 * k + 4


def workload(name: str):
    from paper_1709_03187_b200.instances import CONFIGS

    spec = dict(CONFIGS[name])
    return spec


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def reduce_max_sum(values_max, values_sum, backend_device=None):
    """max over ranks of values_max, sum over ranks of values_sum (torch.distributed)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return list(values_max), list(values_sum)
    dev = backend_device or "cpu"
    tmax = torch.tensor(values_max, dtype=torch.float64, device=dev)
    tsum = torch.tensor(values_sum, dtype=torch.float64, device=dev)
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
    return tmax.tolist(), tsum.tolist()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 9 for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_reference_sample(spec, inst, seconds, threads):
    """O1 (the unmodified reference compiled in oracle/_ref) timed on the host cores."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    r = oracle.ref_sample_select(inst.xs, inst.ys, spec["m"], 1.0, 2.0, 0.95, 1.0, 12345, threads, seconds)
    rate = r["decisions"] * threads / r["busy_s"] if r["busy_s"] > 0 else 0.0
    return rate, r


def cpu_port_sample(spec, inst, threads, ants):
    """O2 (oracle/o2.c: the same north-star rule restated in C, pthreads over ants) on the
    host cores: the seeding iteration plus two partial iterations of a colony of `ants`
    ants on the same instance (the like-for-like CPU rate of the rule the GPU runs)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    o = oracle.O2(inst.xs, inst.ys, m=ants, k=spec["k"], seed=3, threads=threads)
    t0 = time.perf_counter()
    for _ in range(3):
        o.iterate()
    dt = time.perf_counter() - t0
    return o.counters()["decisions"] / dt, o.counters()["decisions"], dt


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def instance_sha256(inst) -> str:
    """sha256 of the instance as TSPLIB text (emit_tsplib, instance.hpp:251-261)."""
    import hashlib

    from paper_1709_03187_b200.instances import emit_tsplib

    return hashlib.sha256(emit_tsplib(inst).encode()).hexdigest()


# Dependent latencies of the operations on one decision's chain, measured on a B200
# (profiles/r01_ubench_latencies.txt: ub_latencies.cu; redux: ub_redux.cu), in SM cycles.
CHAIN_LATENCY = {"ldg_l1_hit": 66, "lds": 33, "shfl_up_fadd": 33, "shfl_idx": 36, "redux_min": 22}


def latency_roofline(spec, k, construct_ms, sm_mhz):
    """The synchronous iteration is one full construction long (n - 1 dependent decisions of
    one ant): the construction kernel's time per critical-chain
    decision against the sum of the measured latencies on that chain (row load from L1,
    bitmap probe, ceil(log2 k) shuffle-scan levels, the total's shuffle, the pick's
    reduction) - a floor of this design with zero issue overhead and no fallbacks."""
    if not sm_mhz:
        return None
    levels = max(1, (k - 1).bit_length())
    c = CHAIN_LATENCY
    floor = c["ldg_l1_hit"] + c["lds"] + levels * c["shfl_up_fadd"] + c["shfl_idx"] + c["redux_min"]
    achieved = construct_ms * 1e-3 * sm_mhz * 1e6 / (spec["n"] - 1)
    return {"bound": "latency", "unit": "cycles per decision of the critical (full-construction) ant",
            "achieved": achieved, "floor": floor, "frac": floor / achieved,
            "floor_terms": {**c, "scan_levels": levels},
            "note": "construction-kernel time x SM clock / (n - 1); floor = sum of the chain's measured "
                    "dependent latencies (profiles/r01_ubench_latencies.txt, ub_redux.cu)"}


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return {}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return 0
    spec = workload(args.config)
    from paper_1709_03187_b200.instances import make_config_instance

    inst = make_config_instance(args.config)
    threads = os.cpu_count() or 1
    per_step = max(2.0, min(8.0, 150.0 / max(1, args.steps + args.warmup)))
    rates, decisions, busy = [], 0, 0.0
    t_all = time.perf_counter()
    for s in range(args.warmup + args.steps):
        rate, r = cpu_reference_sample(spec, inst, per_step, threads)
        if s >= args.warmup:
            rates.append(rate)
            decisions += r["decisions"]
            busy += r["busy_s"]
    value = decisions * threads / busy if busy else 0.0
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: n={spec['n']} m={spec['m']} (reference rule: Independent Roulette "
                               f"over all unvisited cities, construction.hpp:246-281)", "threads": threads},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{decisions} paco::select_next calls on the {args.config} instance with a "
                                   f"{spec['m']}-ant ColonyPheromone; remaining-candidate counts drawn from the "
                                   f"workload's full/partial mix; {per_step:.0f}s per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t_all,
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1709_03187_b200 import Colony, Mode, RunConfig, make_config_instance, run as paco_run

    torch.cuda.set_device(local)
    spec = workload(args.config)
    inst = make_config_instance(args.config)
    k = spec["k"]
    cfg = RunConfig(ants=spec["m"], iterations=args.warmup + args.steps, alpha=1.0, beta=2.0, rho=0.5,
                    partial_prob=0.95, max_mod_frac=1.0, candidates=k, seed=1 + rank, device=local,
                    synchronous=True)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")

    col = Colony(inst, cfg, Mode.partial_aco)
    for _ in range(args.warmup):
        col.iterate(1)
    c0 = col.counters()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms, construct_ms = [], []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (torch stream, synchronised below)
            torch.cuda.synchronize()
            col.iterate(1)  # library-recorded CUDA events on the engine stream
            c_ms, u_ms, _ = col.timing()
            step_ms.append(c_ms + u_ms)
            construct_ms.append(c_ms)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    c1 = col.counters()
    decisions = c1["decisions"] - c0["decisions"]
    fallbacks = c1["fallbacks"] - c0["fallbacks"]
    total_ms = sum(step_ms)
    col.close()

    # asynchronous engine (f3, the reference's default): the config's full iteration budget
    # after seeding as one barrier-free call, same instance and seed
    acfg = RunConfig(**{**cfg.__dict__, "synchronous": False, "iterations": spec["iterations"]})
    acol = Colony(inst, acfg, Mode.partial_aco)
    acol.iterate(1)
    a0 = acol.counters()
    torch.cuda.synchronize()
    acol.iterate(spec["iterations"] - 1)
    a_ms = acol.timing()[0]
    a_dec = acol.counters()["decisions"] - a0["decisions"]
    acol.close()

    # end to end through the public C-ABI call (paco_run, the drop-in for paco::run):
    # host coordinates in, the config's whole iteration budget, g_best tour out
    ecfg = RunConfig(**{**cfg.__dict__, "iterations": spec["iterations"]})
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = paco_run(inst, ecfg, Mode.partial_aco)
    e2e_s = time.perf_counter() - t0
    e2e_dec = rep.counters["decisions"]

    dev = f"cuda:{local}" if world > 1 else None
    (tmax, e2emax), (dsum, e2esum, tours_sum) = reduce_max_sum(
        [total_ms, e2e_s], [decisions, e2e_dec, spec["m"] * args.steps], dev)
    if rank != 0:
        return 0
    value = dsum / (tmax / 1e3)
    c_ms_avg = sum(construct_ms) / len(construct_ms)
    bytes_per_launch = b_dec(k) * (decisions / args.steps)
    achieved = bytes_per_launch / (c_ms_avg / 1e3) / 1e9
    peaks = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json"))
    peak = float(peaks.get("hbm_gbs", 6650.0))
    # traffic: DRAM bytes per launch from the committed ncu --set full capture of THIS config
    # (profiles/ncu_summary.json, keyed by config); null when the config has no capture
    ncu = load_json(os.path.join(ROOT, "profiles", "ncu_summary.json")).get("k_construct", {}).get(args.config, {})
    traffic = ncu.get("dram_bytes_per_launch")
    l2_traffic = ncu.get("l2_bytes_per_launch")
    l2peak = load_json(os.path.join(ROOT, "profiles", "l2_peak.json"))
    l2_gbs = l2peak.get("l2_read_gbs")
    dec_per_iter = decisions / args.steps
    clk = clocks.summary()
    latency = latency_roofline(spec, k, c_ms_avg, clk.get("sm_mhz"))
    cpu = port = None
    host = {"cpu_model": cpu_model(), "threads": os.cpu_count() or 1}
    if world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        try:
            rate, r = cpu_reference_sample(spec, inst, args.cpu_seconds, threads)
            cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"{r['decisions']} paco::select_next calls (unmodified reference, IR rule) on the "
                             f"{args.config} instance, {args.cpu_seconds:.0f}s on {threads} threads",
                   "iteration_s_extrapolated": dec_per_iter / rate if rate else None}
        except Exception as e:  # the reference harness is test infrastructure; report, do not fail
            cpu = {"value": None, "unit": UNIT, "cores": threads, "kind": "reference", "sample": f"unavailable: {e}"}
        try:
            ants = min(spec["m"], 4 * threads)
            prate, pdec, pdt = cpu_port_sample(spec, inst, threads, ants)
            port = {"value": prate, "unit": UNIT, "cores": threads, "kind": "port",
                    "sample": f"O2 (the north-star rule restated in C, oracle/o2.c) on the {args.config} instance: "
                              f"seeding + 2 partial iterations of a {ants}-ant colony, {pdec} decisions in "
                              f"{pdt:.1f}s on {threads} threads",
                    "iteration_s_extrapolated": dec_per_iter / prate if prate else None,
                    "gpu_speedup_same_rule": value / prate if prate else None}
        except Exception as e:
            port = {"value": None, "unit": UNIT, "cores": threads, "kind": "port", "sample": f"unavailable: {e}"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tmax / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config}: {spec['n']}-city {spec['kind']} EUC_2D, m={spec['m']}, "
                               f"k={k}, alpha=1, beta=2, partial_prob=0.95, max_mod_frac=1.0",
                   "step": "one synchronous ACO iteration (weights, construction, completion step)",
                   "l2": "flushed (512 MiB write) before every timed step; per-step working set "
                         "(neighbour slices + tours) exceeds L2",
                   "parallelism": f"replicas x{world}",
                   "instance_sha256": instance_sha256(inst)},
        "tours_per_s": tours_sum / (tmax / 1e3),
        "fallback_frac": fallbacks / max(1, decisions),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "k_construct",
                     "bytes_per_decision": b_dec(k), "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks
                     else "fallback 6650 GB/s (B200_PROFILING.md)",
                     "traffic_source": (f"profiles/ncu_summary.json k_construct.{args.config} (ncu --set full, "
                                        "dram__bytes_read+write per launch)") if traffic is not None else
                                       f"no ncu capture committed for {args.config}",
                     "l2": {"achieved": achieved, "peak": l2_gbs, "unit": "GB/s",
                            "frac": achieved / l2_gbs if l2_gbs else None,
                            "traffic": l2_traffic,
                            "peak_source": "profiles/l2_peak.json (ub_l2_bw.cu, L2-resident read bandwidth "
                                           "measured on a B200)" if l2_gbs else None,
                            "note": "the per-decision tables (candidate rows, 25.6 MB at C5) are L1/L2-resident: "
                                    "same algorithmic bytes against the L2 bandwidth"},
                     "latency": latency},
        "cpu_baseline": cpu,
        "cpu_baseline_port": port,
        "host": {**host, "gpu_iteration_ms": tmax / args.steps,
                 "reference_iteration_s_extrapolated": (cpu or {}).get("iteration_s_extrapolated"),
                 "port_iteration_s_extrapolated": (port or {}).get("iteration_s_extrapolated"),
                 "note": "host-core time for one iteration of this config = decisions per GPU iteration / "
                         "host rate (the reference's own rule for `reference`, the same rule for `port`)"},
        "e2e": {"value": e2esum / e2emax, "unit": UNIT, "h2d_bytes_per_step": 16 * inst.n / ecfg.iterations,
                "d2h_bytes_per_step": (4 * inst.n + 8) / ecfg.iterations, "iterations": ecfg.iterations,
                "note": "paco_run: coordinates H2D, grid+k-NN build, the config's whole iteration budget incl. "
                        "seeding, g_best D2H",
                "wall_s": e2e_s, "device_ms": {"setup": rep.setup_ms, "construct": rep.construct_ms,
                                               "weights_and_updates": rep.update_ms}},
        "async": {"value": a_dec / (a_ms / 1e3), "unit": UNIT, "iterations": spec["iterations"] - 1,
                  "ms": a_ms, "note": "synchronous=False (engine.hpp:213-244): one barrier-free launch for the "
                                      "config's iteration budget after seeding; weights rebuilt concurrently"},
        # per synchronous partial-mode step: k_weights, k_ant_order (longest ants first),
        # k_construct, k_lengths (n >= 4096), k_update, k_publish (profiles/r02_launches_c5.csv)
        "gpu_launches": (6 if spec["n"] >= 4096 else 5) * args.steps,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        if args.impl == "reference":
            # the reference arm is a CPU measurement on rank 0 only; other ranks exit without work
            return run_reference_arm(args, rank, world)
        dist.init_process_group("nccl")
    try:
        if args.impl == "reference":
            return run_reference_arm(args, rank, world)
        return run_ours(args, rank, world, local)
    finally:
        if world > 1:
            import torch.distributed as dist

            if dist.is_initialized():
                dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
