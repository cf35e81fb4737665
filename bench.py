#!/usr/bin/env python
"""Benchmark of the iterative-Shor stage loop (BASELINE.json metric:
"amplitude updates/s per mulmod step; s per full iterative-Shor run; HBM GB/s").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one non-identity stage of the iterative circuit on the resident
state (the controlled modular-multiplication permutation fused with phase,
Hadamard, |psi|^2 reduction, host measurement and collapse). At N=1 the
workload is config 4 of BASELINE.json: N = 4294967213 = 57139 * 75167, a = 5,
t = 64 (paper-convention state 2^33 x 16 B = 137 GB; ours 2 x 68.7 GB), which
fits one B200. value = N / (device time per stage). The state (68.7 GB) is
540x the 126 MB L2, so no L2 flush is needed between steps.

--impl reference times the unmodified reference engine (oracle/_ref, compiled
from /root/reference/proj/src) on this box's host cores on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "amplitude updates/s per mulmod step"
UNIT = "amp-updates/s"

WORKLOADS = {
    # config 4 (BASELINE.json configs[3]): ~33-bit semiprime on 1 GPU
    "c4": dict(N=4294967213, a=5, p=57139, q=75167,
               desc="config 4: N=4294967213=57139*75167, a=5 (order 2147417454), t=64"),
    # config 3 (BASELINE.json configs[2]): ~24-bit semiprime
    "c3": dict(N=16777207, a=2, p=4093, q=4099,
               desc="config 3: N=16777207=4093*4099, a=2 (order 2794836), t=48"),
    # 31-qubit profiling size: 34 GB per buffer (the sharded exchange at ~8k bands)
    "n31": dict(N=2146005049, a=3, p=46301, q=46349,
                desc="31-qubit profiling size: N=2146005049=46301*46349, a=3, t=62"),
    # profiling size for the round-robin tiled variant (config 4's): 17 GB per buffer
    "n30": dict(N=1073217479, a=2, p=32749, q=32771,
                desc="30-qubit profiling size: N=1073217479=32749*32771, a=2 (order 536575980), t=60"),
    # an orbit of N / 6 (p - 1, q - 1 share 2 * 3 * ...): the compressed stages at low density
    "n30r6": dict(N=1087482493, a=2, p=32971, q=32983,
                  desc="30-qubit size with a small orbit: N=1087482493=32971*32983, a=2 (order 181236090 = N/6)"),
    # profiling size: 4.3 GB per buffer (34x L2), fast ncu replays
    "n29": dict(N=268435247, a=3, p=12589, q=21323,
                desc="29-qubit profiling size: N=268435247=12589*21323, a=3 (order 67100334), t=56"),
}
# the reference engine cannot hold config 4 (206 GB of buffers + up to 1.1 TB of u32
# gather tables, n=33 at its cap); its bounded sample is the config-3 problem.
REF_SAMPLE = "c3"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------ reference arm
def reference_sample(steps, warmup, threads):
    """Unmodified reference IterativeShorEngine::run on host cores (oracle/_ref).
    Each step = one full run (t stages) of the config-3 problem."""
    from oracle import Reference
    w = WORKLOADS[REF_SAMPLE]
    N, a = w["N"], w["a"]
    L, t = N.bit_length(), 2 * N.bit_length()
    ref = Reference()
    t0 = time.perf_counter()
    eng = ref.engine(N, a, L, t, shard_count=4, workers=threads, qubit_ceiling=33)
    construct_s = time.perf_counter() - t0
    for i in range(warmup):
        eng.time_runs(1, i, 1)
    secs = [eng.time_runs(1, warmup + i, 1) for i in range(steps)]
    run_s = min(secs)  # best of k
    return {"value": N * t / run_s, "s_per_run": run_s, "ms_per_stage": 1e3 * run_s / t,
            "s_per_run_all": secs, "construct_s": construct_s, "N": N, "t": t,
            "threads": threads, "runs": steps, "build": ref.build}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    steps = max(1, min(args.steps, 10))
    warm = 1 if args.warmup > 0 else 0
    try:
        r = reference_sample(steps, warm, threads)
    except Exception as exc:  # the reference is always present here; report loudly
        print(json.dumps({"impl": "reference", "unavailable": f"{type(exc).__name__}: {exc}"}))
        return 0
    sample = (f"best of {r['runs']} full IterativeShorEngine::run calls at N={r['N']} "
              f"(config-3 problem), t={r['t']}, workers={threads} on {cpu_model()}; reference "
              f"build {r['build']['variant']}: {r['build']['flags']}; config 4 is out of the "
              "reference's reach (n=33 needs 206 GB of buffers + up to 1.1 TB of u32 gather tables)")
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT,
        "n_gpus": ws, "steps": r["runs"], "warmup": warm,
        "ms_per_step": r["ms_per_stage"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic Shor state)",
        "config": {"workload": args.workload, "reference_sample": REF_SAMPLE,
                   "N": r["N"], "t": r["t"]},
        "s_per_run": r["s_per_run"], "construct_s": r["construct_s"],
        "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2308_05047_b200 as shs

    ws, rank, local = dist_env()
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    w = WORKLOADS[args.workload]
    N, a = w["N"], w["a"]
    prob = shs.FactoringProblem.make(N, a)
    t = prob.t
    err = shs.ErrorConfig()
    opts = shs.SimulatorOptions(device=local, qubit_ceiling=64)
    eng = shs.IterativeShorEngine(prob, err, opts)
    pows = eng.stage_multipliers()
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device=dev)
    seed, idx = 2308, rank

    # walk the real circuit: stage s with the observed prefix, measured by the
    # reference's sampling rule; timed steps cycle over stages 1..t-1 (never the
    # implicit-|1> first stage), all non-identity for this problem.
    state = {"s": 0, "prefix": 0}
    eng.state_init()

    def step():
        s = state["s"]
        p0, p1 = eng.stage_probs(s, state["prefix"])
        m = shs.sample_measurement(p1, seed, idx, s, err)
        b = m["sampled_bit"]
        eng.stage_collapse(b, p1 if b else p0)
        state["prefix"] = (state["prefix"] | (b << s)) & ((1 << t) - 1)
        state["s"] = s + 1 if s + 1 < t else 1
        return s, b

    for _ in range(max(args.warmup, 1)):
        step()
    timed_stages = []
    launches0 = eng.launch_count()
    clocks = ClockSampler(local)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    wall0 = time.perf_counter()
    timed_bits = []
    for _ in range(args.steps):
        s_, b_ = step()
        timed_stages.append(s_)
        timed_bits.append(b_)
    ev1.record(stream)
    ev1.synchronize()
    wall = time.perf_counter() - wall0
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clock_info = clocks.stop()
    launches = eng.launch_count() - launches0
    ms = ev0.elapsed_time(ev1)
    if ws > 1:
        tm = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        ms = float(tm.item())
    ms_per_step = ms / args.steps
    assert all(pows[s] != 1 for s in timed_stages)

    # per-kernel device times (CUDA events on the engine's stream) over extra stages
    eng.set_timing(True)
    for _ in range(max(3, min(args.steps, 6))):
        step()
    kt = eng.kernel_times()
    eng.set_timing(False)
    hbm_peak, peak_src = peaks()
    # algorithmic B/amplitude: a probs pass that is not the run's
    # last also writes h0 (speculative group-0 write, +16 B); the collapse (48 B)
    # then runs only when group 1 is kept
    spec_on = os.environ.get("SHS_SPEC", "1") != "0"

    def spec_at(s):
        return spec_on and s + 1 < t
    # orbit-compressed stages (the default from N >= 2^21): the
    # probs pass reads both sides of the r = ord(a) members and writes both
    # groups (64 B per member; 32 on a run's last stage), no collapse pass
    orb = eng.orbit_info()
    r_orb = orb["r"]
    orb_st = eng.orbit_stages()
    orbit_timed = r_orb > 0 and all(orb_st[s] for s in timed_stages)
    if orbit_timed:
        per_amp = {"probs": (64 if timed_stages[-1] + 1 < t else 32) * r_orb / N, "combine": 0,
                   "collapse": 0}
        step_bytes = [r_orb * (64 if s + 1 < t else 32) for s in timed_stages]
    else:
        per_amp = {"probs": 48 if spec_at(timed_stages[-1]) else 32, "combine": 0, "collapse": 48}
        step_bytes = [N * ((48 if spec_at(s) else 32) + (0 if spec_at(s) and b == 0 else 48))
                      for s, b in zip(timed_stages, timed_bits)]
    step_bpa = sum(step_bytes) / len(step_bytes) / N  # average algorithmic B/amp per timed stage
    kernels = {}
    for k, (tot, n) in kt.items():
        avg = tot / max(n, 1)
        b = per_amp[k] * N
        kernels[k] = {"avg_ms": avg, "launches": n, "algorithmic_bytes": b,
                      "achieved_gbs": (b / (avg * 1e-3) / 1e9) if avg > 0 and b else None}
    # device time of an average timed stage: probs + combine, plus the collapse
    # on the stages that run it (the speculative write skips it when group 0 is kept)
    ran = [not orbit_timed and not (spec_at(s) and b == 0) for s, b in zip(timed_stages, timed_bits)]
    stage_dev_ms = (kernels["probs"]["avg_ms"] + kernels["combine"]["avg_ms"] +
                    kernels["collapse"]["avg_ms"] * sum(ran) / len(ran))
    dom = max(("probs", "collapse"), key=lambda k: kernels[k]["avg_ms"])
    achieved = kernels[dom]["achieved_gbs"]
    tiled = eng.tile_plan(timed_stages[-1])["tiled"]
    kname = {"probs": ("k_tiled<1,0,1>" if orbit_timed else "k_tiled<1>") if tiled
             else "k_stage_probs<1,0>",
             "collapse": "k_tiled<0>" if tiled else "k_stage_collapse<1,0>"}[dom]
    traffic, traffic_src = None, None
    try:  # DRAM bytes per launch of this kernel from the committed ncu capture at this N
        with open(os.path.join(ROOT, "profiles", "r02", "ncu_summary.json")) as f:
            summ = json.load(f)
        ks = summ["kernels"][kname]
        if summ["N"] == N:
            traffic = ks["dram_bytes_per_launch"]
            traffic_src = (f"profiles/r02/ncu_summary.json {ks['name']}: dram__bytes_read.sum + "
                           f"dram__bytes_write.sum of one launch at this N "
                           f"({ks['dram_bytes_per_amp']} B/amp)")
    except (OSError, KeyError, ValueError):
        pass
    roofline = {"kernel": kname, "bound": "hbm", "achieved": achieved,
                "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                "peak_source": peak_src, "traffic": traffic, "traffic_source": traffic_src,
                "share_of_step": kernels[dom]["avg_ms"] / ms_per_step,
                "bytes_per_amp": per_amp[dom]}
    if orbit_timed:
        roofline["orbit"] = {"members": r_orb, "member_fraction": r_orb / N,
                             "bytes_per_member": 64,
                             "what": "k_tiled<true,false,true> (plan warps, producers, consumers, "
                                     "chains) + k_tile_fixup: both sides of every member read, both "
                                     "groups written, no collapse pass"}
        try:  # the measured ceiling of this access pattern (scripts/micro/fragment_bw.cu)
            with open(os.path.join(ROOT, "profiles", "r02", "fragment_bw.jsonl")) as f:
                pat = [json.loads(x) for x in f if x.strip()]
            ceil = next(x for x in pat if x["kernel"] == "streams" and x["stream_bytes"] == 512)
            roofline["orbit"]["pattern_ceiling"] = {
                "GBps": ceil["GBps"], "frac": achieved / ceil["GBps"],
                "source": "profiles/r02/fragment_bw.jsonl: 4736 row streams of 512 B reads and "
                          "2 x 512 B writes per step plus 2 random 256 B gathers, plain loads / "
                          "stores (DESIGN.md §3d)"}
        except (OSError, StopIteration, KeyError, ValueError):
            pass

    # the same stages with orbit compression off (the dense kernels), for scale
    dense_stages = None
    if orbit_timed and not args.no_dense_compare:
        eng.set_orbit(False)
        state["s"], state["prefix"] = 0, 0
        eng.state_init()
        for _ in range(max(args.warmup, 1)):
            step()
        nd = max(3, min(args.steps, 10))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        dbits, dst = [], []
        for _ in range(nd):
            s_, b_ = step()
            dst.append(s_)
            dbits.append(b_)
        e1.record(stream)
        e1.synchronize()
        dms = e0.elapsed_time(e1) / nd
        eng.set_timing(True)
        for _ in range(3):
            step()
        dkt = eng.kernel_times()
        eng.set_timing(False)
        pavg = dkt["probs"][0] / max(dkt["probs"][1], 1)
        dense_stages = {
            "ms_per_step": dms, "value": ws * N / (dms * 1e-3), "steps": nd,
            "probs_ms": pavg, "probs_frac_of_hbm": 48 * N / (pavg * 1e-3) / 1e9 / hbm_peak,
            "collapse_ms": dkt["collapse"][0] / max(dkt["collapse"][1], 1),
            "bits_1": sum(dbits),
            "what": "the same step loop from stage 1 with orbit compression off (dense tiled "
                    "kernels, speculative group-0 write); not the headline"}
        eng.set_orbit(True)

    # end to end: the public call a user makes (C ABI, host results), full run.
    # e2e.value: every stage swept, no sparse prefix (N amplitude updates per
    # stage, the reference's work, comparable with value); s_per_run: the default run()
    # with its sparse prefix (the first stages on the support of the state,
    # bit-identical results), the "s per full iterative-Shor run" metric.
    def timed_runs(sparse):
        eng.set_sparse(sparse)
        e2e_runs = max(1, args.e2e_runs)
        t0 = time.perf_counter()
        for i in range(e2e_runs):
            r = eng.run(seed, 1000 + i)
        sec = (time.perf_counter() - t0) / e2e_runs
        if ws > 1:
            tr = torch.tensor([sec], device=dev, dtype=torch.float64)
            dist.all_reduce(tr, op=dist.ReduceOp.MAX)
            sec = float(tr.item())
        return sec, r
    run_s_dense, res = timed_runs(False)
    run_s, res_sparse = timed_runs(True)
    sparse_stages = eng.sparse_stages()
    assert res_sparse.bits.j == res.bits.j and res_sparse.j_sampled == res.j_sampled

    value = ws * N / (ms_per_step * 1e-3)
    e2e_value = ws * N * t / run_s_dense
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: the deterministic iterative-Shor state from |1> (no dataset)",
        "config": {"workload": args.workload, "desc": w["desc"], "N": N, "a": a, "t": t,
                   "state_bytes_per_buffer": 16 * N, "device_bytes": eng.device_bytes(),
                   "l2": "state 540x larger than the 126 MB L2: no flush needed",
                   "parallelism": "1 GPU" if ws == 1 else f"{ws} independent replicas"},
        "s_per_run": run_s,
        "s_per_run_dense": run_s_dense,
        "sparse_prefix_stages": sparse_stages,
        "stage_hbm_gbs": step_bpa * N / (ms_per_step * 1e-3) / 1e9,
        "stage_frac_of_hbm": step_bpa * N / (ms_per_step * 1e-3) / 1e9 / hbm_peak,
        "stage_bytes_per_amp": step_bpa,
        "speculative_group0": {"on": spec_on, "timed_bits_1": sum(timed_bits),
                               "timed_steps": len(timed_bits),
                               "collapse_skipped": sum(1 for s, b in zip(timed_stages, timed_bits)
                                                       if spec_at(s) and b == 0)},
        "wall_ms_per_step": 1e3 * wall / args.steps,
        "device_ms_per_stage_kernels": stage_dev_ms,
        "roofline": roofline, "kernels": kernels, "dense_stages": dense_stages,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 16,
                "what": "IterativeShorEngine.run(seed, idx) through the C ABI with every stage "
                        "swept (set_sparse(False): no sparse prefix; the stages with whole-band "
                        "plans orbit-compressed, the rest dense): t stages, p0/p1 decided on "
                        "the device, bit string returned to the host; inputs are the problem "
                        "scalars (kernel arguments). The default run() (sparse prefix) is "
                        "s_per_run, same bit string",
                "s_per_run_default": run_s,
                "last_j": str(res.bits.j)},
        "gpu_launches": launches, "clocks": clock_info,
    }
    if rank == 0 and ws == 1 and not args.no_small:
        line["batched_small_n"] = small_n_throughput(shs)
        line["config3_error_models"] = config3_runs(shs)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            r = reference_sample(3, 1, os.cpu_count() or 1)
            line["cpu_baseline"] = {
                "value": r["value"], "unit": UNIT, "cores": r["threads"], "kind": "reference",
                "sample": f"best of 3 full IterativeShorEngine::run at N={r['N']}, t={r['t']} "
                          f"(config-3 problem; config 4 exceeds the reference's reach), "
                          f"workers={r['threads']}, construct {r['construct_s']:.1f}s untimed; "
                          f"{cpu_model()}; reference build {r['build']['variant']}: "
                          f"{r['build']['flags']}"}
        except Exception as exc:
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {type(exc).__name__}: {exc}"}
    if rank == 0:
        print(json.dumps(line))
    eng.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


def small_n_throughput(shs):
    """Configs 1-2 (BASELINE.json configs[0..1]): whole runs per second through
    the batched engine (shs_engine_run_batch), beside the unmodified reference's
    per-run time on one host core (its engine runs small problems single-threaded;
    the reference's campaign parallelism is one problem per worker thread)."""
    out = {}
    cases = {"config1_N15": [(15, 7)],
             "config2_N21_N35": [(21, a) for a in (2, 4, 5, 8, 10, 11, 13, 16, 17, 19, 20)] +
                                [(35, a) for a in range(2, 35) if math.gcd(a, 35) == 1]}
    shots = {"config1_N15": 100000, "config2_N21_N35": 1024}
    try:
        from oracle import Reference
        ref = Reference()
    except Exception:
        ref = None
    for name, problems in cases.items():
        engines = [shs.IterativeShorEngine(shs.FactoringProblem.make(N, a), shs.ErrorConfig(),
                                           shs.SimulatorOptions(qubit_ceiling=64))
                   for N, a in problems]
        import numpy as np
        bufs = [np.empty((shots[name], 2), dtype=np.uint64) for _ in engines]
        for e, b in zip(engines, bufs):
            e.run_batch_array(2, 0, shots[name], b)  # tables, buffers, warm
        t0 = time.perf_counter()  # the C-ABI call with host output buffers
        runs = 0
        for e, b in zip(engines, bufs):
            e.run_batch_array(2, 0, shots[name], b)
            runs += shots[name]
        dt = time.perf_counter() - t0
        entry = {"runs": runs, "seconds": dt, "runs_per_s": runs / dt,
                 "problems": len(problems), "shots_per_problem": shots[name]}
        if ref is not None:
            N, a = problems[0]
            t = 2 * N.bit_length()
            re = ref.engine(N, a, N.bit_length(), t, qubit_ceiling=33)
            k = 20000
            sec = re.time_runs(2, 0, k)
            entry["reference_cpu_runs_per_s_1core"] = k / sec
            entry["reference_sample"] = f"{k} IterativeShorEngine::run calls of N={N}, a={a}, 1 thread"
        if name == "config2_N21_N35":
            entry["statistics"] = config2_statistics(shs, engines, problems, ref)
        out[name] = entry
        for e in engines:
            e.close()
    out["campaign_L18_lockstep"] = lockstep_throughput(shs, ref)
    return out


def lockstep_throughput(shs, ref):
    """The largest problems of the reference's headline campaign (acceptance
    criteria 4-5: L = 9..18, M = 256 shots per problem): one L = 18 problem's
    256 shots through run_batch_array, served by the lockstep multi-shot path
    (DESIGN.md §6b), beside the reference engine's per-run time on one host core
    (its campaign runs one problem per worker thread)."""
    import numpy as np
    N, a, shots = 262139, 4242, 256
    e = shs.IterativeShorEngine(shs.FactoringProblem.make(N, a), shs.ErrorConfig(),
                                shs.SimulatorOptions(qubit_ceiling=64))
    buf = np.empty((shots, 2), dtype=np.uint64)
    e.run_batch_array(3, 0, shots, buf)  # warm
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        e.run_batch_array(3, 0, shots, buf)
    dt = (time.perf_counter() - t0) / reps
    t = e.problem.t
    e.close()
    entry = {"N": N, "a": a, "t": t, "shots": shots, "seconds": dt, "runs_per_s": shots / dt,
             "amp_updates_per_s": shots * N * t / dt}
    if ref is not None:
        re = ref.engine(N, a, N.bit_length(), t, qubit_ceiling=33)
        k = 8
        sec = re.time_runs(3, 0, k)
        entry["reference_cpu_runs_per_s_1core"] = k / sec
        entry["reference_sample"] = f"{k} IterativeShorEngine::run calls of N={N}, a={a}, 1 thread"
    return entry


def config2_statistics(shs, engines, problems, ref):
    """Config 2's success-probability statistics: run_problem (harness.cpp:109-148)
    for every coprime base of N = 21 and 35, M = 1024 shots each — runs on the
    batched engine, Shor post-processing on the device (§8 f4), tallies on the
    host — with the mean success / success+lucky fractions per N, beside the
    reference's run_problem for the same problems on one host core."""
    factors = {21: (3, 7), 35: (5, 7)}
    M = 1024
    probs = [shs.FactoringProblem.make(N, a, p=factors[N][0], q=factors[N][1], seed=1000 + i)
             for i, (N, a) in enumerate(problems)]
    for p, e in zip(probs, engines):
        shs.run_problem(p, M, engine=e)  # warm
    t0 = time.perf_counter()
    results = [shs.run_problem(p, M, engine=e) for p, e in zip(probs, engines)]
    dt = time.perf_counter() - t0
    out = {"M": M, "problems": len(probs), "seconds": dt,
           "shots_per_s": len(probs) * M / dt}
    for N in (21, 35):
        rs = [r for r in results if r.problem.N == N]
        out[f"N{N}"] = {"bases": len(rs),
                        "mean_success": statistics.mean(r.success_fraction() for r in rs),
                        "mean_success_lucky": statistics.mean(r.success_lucky_fraction()
                                                              for r in rs)}
    t0 = time.perf_counter()  # Ekerå's pipeline on the same shots (post_mode="ekera")
    ek = [shs.run_problem(p, M, engine=e, post_mode="ekera") for p, e in zip(probs, engines)]
    out["ekera"] = {"seconds": time.perf_counter() - t0}
    for N in (21, 35):
        rs = [r for r in ek if r.problem.N == N]
        out["ekera"][f"N{N}_mean_success"] = statistics.mean(r.success_fraction() for r in rs)
    import numpy as np
    j = np.zeros((1 << 20, 2), dtype=np.uint64)
    j[:, 0] = np.arange(1 << 20, dtype=np.uint64) * np.uint64(2654435761) % np.uint64(1 << 22)
    shs.shor_postprocess_array(j[:1024], 22, 4087, 1001)  # warm
    t0 = time.perf_counter()
    shs.shor_postprocess_array(j, 22, 4087, 1001)
    out["postprocess_bitstrings_per_s"] = len(j) / (time.perf_counter() - t0)
    if ref is not None:
        p = probs[-1]
        t0 = time.perf_counter()
        ref.run_problem(p.N, p.a, p.p, p.q, p.L, p.t, p.seed, M)
        out["reference_run_problem_shots_per_s_1core"] = M / (time.perf_counter() - t0)
    return out


def config3_runs(shs):
    """Config 3 (BASELINE.json configs[2]): N = 16777207, t = 48, full runs
    through the C ABI with each of the paper's error models at p_error = 0.01
    (acceptance criterion 8's settings, proj/tests/acceptance/acceptance_main.cpp:
    367-378): s per run with every stage dense (amplitude updates/s = N t / that)
    and with the default sparse prefix."""
    w = WORKLOADS["c3"]
    N, a = w["N"], w["a"]
    prob = shs.FactoringProblem.make(N, a)
    models = {"none": shs.ErrorConfig(),
              "classical_measure": shs.ErrorConfig(shs.ErrorKind.classical_measure, 0.01),
              "quantum_measure": shs.ErrorConfig(shs.ErrorKind.quantum_measure, 0.01,
                                                 shs.PauliProbs(0.005, 0.005, 0.0)),
              "amplitude_init": shs.ErrorConfig(shs.ErrorKind.amplitude_init,
                                                2.0 * math.sqrt(0.01 * 0.99)),
              "phase_init": shs.ErrorConfig(shs.ErrorKind.phase_init,
                                            math.acos(1.0 - 2.0 * 0.01) / math.pi),
              "bitflip": shs.ErrorConfig(shs.ErrorKind.bitflip, 0.01)}
    out = {"N": N, "a": a, "t": prob.t}
    for name, err in models.items():
        eng = shs.IterativeShorEngine(prob, err, shs.SimulatorOptions(qubit_ceiling=64))
        entry = {}
        for sparse in (False, True):  # every stage dense; the default run() (sparse prefix)
            eng.set_sparse(sparse)
            eng.run(7, 0)  # warm
            t0 = time.perf_counter()
            runs = 3
            for i in range(runs):
                eng.run(7, 1 + i)
            dt = (time.perf_counter() - t0) / runs
            if sparse:
                entry["s_per_run"] = dt
                entry["sparse_prefix_stages"] = eng.sparse_stages()
            else:
                entry["s_per_run_dense"] = dt
                entry["amp_updates_per_s_dense"] = N * prob.t / dt
        out[name] = entry
        eng.close()
    return out


def run_sharded(args):
    """N > 1 GPUs (one process per GPU under torchrun): one block shard of the
    config-4 state per rank (strong scaling: the same N as at 1 GPU). Peers
    attach through CUDA IPC (buffers, receive slots, stage digits, ordering
    events).

    A step here is one full iterative-Shor run, device-resident
    (ShardedShorEngine.run -> shs_shards_run): per stage the exchange v2
    all-to-all (pack -> NVLink -> unpack, in rounds), probs, the exact digit
    sum and the measurement on every device, collapse; no host round trip per
    stage. value = N * t * steps / device time (CUDA events on each rank's main
    stream, max over ranks) — every stage dense, so comparable with the 1-GPU
    line's e2e (s_per_run_dense)."""
    import torch
    import torch.distributed as dist

    import paper_2308_05047_b200 as shs

    ws, rank, local = dist_env()
    # SHS_BENCH_BACKEND=gloo lets the multi-rank path run with ranks sharing a GPU
    # (functional check: the kernels never wait on another rank's kernels)
    backend = os.environ.get("SHS_BENCH_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)
    cdev = dev if backend == "nccl" else None

    def max_over_ranks(x):
        tt = torch.tensor([float(x)], device=cdev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    w = WORKLOADS[args.workload]
    N, a = w["N"], w["a"]
    prob = shs.FactoringProblem.make(N, a)
    t = prob.t
    err = shs.ErrorConfig()
    opts = shs.SimulatorOptions(device=local, qubit_ceiling=64, combine="exact")
    shard = shs.Shard(prob, err, opts, rank, ws)
    group = shs.DistGroup(shard, attach_ipc=True, device=cdev)
    eng = shs.ShardedShorEngine(prob, err, opts, [shard], group)
    stream = torch.cuda.ExternalStream(shard.stream_handle(), device=dev)
    seed = 2308

    for i in range(max(args.warmup, 1)):  # the first run also prepares the exchange offsets
        eng.run(seed, 100 + i)
    launches0 = shard.launch_count()
    clocks = ClockSampler(local)
    dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    wall0 = time.perf_counter()
    ev0.record(stream)
    for i in range(args.steps):
        res = eng.run(seed, 1000 + i)
    ev1.record(stream)
    ev1.synchronize()
    wall = time.perf_counter() - wall0
    dist.barrier()
    clock_info = clocks.stop()
    ms_per_step = max_over_ranks(ev0.elapsed_time(ev1)) / args.steps
    wall_per_run = max_over_ranks(wall / args.steps)
    launches = shard.launch_count() - launches0

    shard.set_timing(True)  # one more run, every launch timed (serialised)
    eng.run(seed, 999)
    kt = shard.kernel_times()
    shard.set_timing(False)
    kms = {k: max_over_ranks(v[0] / max(v[1], 1)) for k, v in kt.items()}
    kn = {k: v[1] for k, v in kt.items()}
    nloc = shard.hi - shard.lo
    rounds = max(1, kn["pack"] // max(1, kn["probs"] - 1)) if kn["pack"] else 1
    pack_stage_ms = kms["pack"] * kn["pack"] / max(1, kn["probs"])  # per stage (all rounds)
    unpack_stage_ms = kms["unpack"] * kn["unpack"] / max(1, kn["probs"])
    # exchange v2 (exchange2.cuh): each element crosses once, sender -> receiver:
    # per GPU and direction 16 B x (N/G)(G-1)/G, the all-to-all minimum
    nvlink_bytes = 16 * nloc * (ws - 1) / ws
    nvlink_peak = 900.0  # GB/s per direction per GPU (NVLink 5, north_star)
    hbm_peak, peak_src = peaks()
    ex_gbs = nvlink_bytes / (pack_stage_ms * 1e-3) / 1e9 if pack_stage_ms else None
    local_ms = kms["probs"] + kms["collapse"]
    local_gbs = 80 * nloc / (local_ms * 1e-3) / 1e9 if local_ms else None

    line = {
        "metric": METRIC, "value": N * t / (ms_per_step * 1e-3), "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: the deterministic iterative-Shor state from |1> (no dataset)",
        "config": {"workload": args.workload, "desc": w["desc"], "N": N, "a": a, "t": t,
                   "step": "one full device-resident run (t stages, every stage dense)",
                   "shard_amplitudes": nloc, "parallelism": f"{ws} shards (block-sharded state)",
                   "backend": backend, "exchange_rounds": rounds,
                   "l2": "state far larger than L2: no flush needed"},
        "s_per_run": ms_per_step * 1e-3,
        "s_per_run_dense": ms_per_step * 1e-3,
        "sparse_prefix_stages": 0,
        "kernels_max_over_ranks_ms": kms,
        "per_stage_ms": {"pack": pack_stage_ms, "unpack": unpack_stage_ms,
                         "probs": kms["probs"], "collapse": kms["collapse"]},
        "roofline": {"kernel": "k_stage_probs + k_stage_collapse <kSrcBuffer> (shard-local)",
                     "bound": "hbm", "achieved": local_gbs, "peak": hbm_peak, "unit": "GB/s",
                     "frac": local_gbs / hbm_peak if local_gbs else None,
                     "peak_source": peak_src, "traffic": None, "bytes_per_amp": 80},
        "nvlink": {"kernel": "k_x2_pack (peer stores into the receivers' streams)",
                   "achieved": ex_gbs, "peak": nvlink_peak, "unit": "GB/s per direction",
                   "frac": ex_gbs / nvlink_peak if ex_gbs else None,
                   "bytes_per_gpu_per_direction_per_stage": nvlink_bytes,
                   "note": "one GPU per process; with ranks sharing a GPU (gloo) the streams go "
                           "through local HBM and this is not an NVLink number"},
        "e2e": {"value": N * t / wall_per_run, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 16 + 32 * t, "last_j": str(res.bits.j),
                "what": "ShardedShorEngine.run over the C ABI (shs_shards_run), wall clock per "
                        "run, bit string and stage trace returned to the host"},
        "gpu_launches": launches, "clocks": clock_info,
    }
    if rank == 0:
        print(json.dumps(line))
    shard.close()
    dist.destroy_process_group()
    return 0


def self_launch(args):
    """--gpus N > 1 without torchrun: relaunch this script as N ranks."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c4")
    ap.add_argument("--e2e-runs", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-small", action="store_true", help="skip the configs 1-2 batched line")
    ap.add_argument("--no-dense-compare", action="store_true",
                    help="skip timing the same stages with orbit compression off")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    ws = dist_env()[0]
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args)
    if ws != args.gpus:
        print(f"error: --gpus {args.gpus} but WORLD_SIZE={ws}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference_arm(args)
    if ws > 1:
        try:
            return run_sharded(args)
        except Exception as exc:  # one JSON line even when the multi-GPU path fails
            if dist_env()[1] == 0:
                print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": ws,
                                  "steps": args.steps, "warmup": args.warmup,
                                  "higher_is_better": True, "scaling": "strong",
                                  "config": {"workload": args.workload},
                                  "error": f"{type(exc).__name__}: {exc}"}))
            raise
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
