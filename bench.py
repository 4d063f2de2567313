#!/usr/bin/env python
"""Benchmark: one NS outer iteration (all SURVEY section 8(a) rows) per step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4]
                    [--mode auto|replicas|shard] [--impl reference]

Workload: C4 by default -- Bayesian logistic regression, d = 100, N = 10^4
synthetic rows, n_live = 20000, k = 10^4, p = d HRSS steps (BASELINE.json
configs[3], the largest configuration and the one quoted "sharded over 8
GPUs"; its energy is the batched X.theta contraction on the tensor cores).
--config picks another BASELINE configuration (C1, C2, C3a, C3b, C5).
Metric: constrained energy evaluations per second (D-0: every energy the
HRSS probes evaluate; with C4's Gaussian prior every probe is an evaluation),
plus NS iterations per second.

Timing window (independent of --steps): a run of a configuration takes
about REP_ITERS[config] iterations to its termination criterion; the K timed
iterations sit at fixed, evenly spaced offsets 4 + floor(i (T - 4) / K) of
that run (K > T: further runs with the next seeds), so the measured mix of
early and late iterations is the same whatever K is.  The iterations between
them run untimed.  Each timed iteration is bracketed by CUDA events on the
stream the library launches on, after a stream synchronisation and a 256 MiB
L2 flush outside the events.  A second run with the same seed replays the
same iterations in the library's event-timing mode (every kernel launched
eagerly between its own events) for the per-kernel roofline entry.

e2e: the public API end to end -- nss_init from host buffers (the problem's
data uploaded), nss_step with its info read back every iteration until the
termination criterion, nss_evidence -- wall clock, init evaluations included.

Multi-GPU: --gpus N starts N ranks itself (torchrun on
127.0.0.1) unless WORLD_SIZE is already set.  --mode shard runs ONE NS run
whose live set is sharded over the ranks (strong scaling); --mode replicas
an independent run per rank (weak scaling).  auto = replicas for C1/C2,
shard for C3a/C3b/C4/C5.  Times are the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import platform
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2601_23252_b200 import workloads as W  # noqa: E402

METRIC = "constrained energy evals/sec"
UNIT = "evals/s"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "traffic.json")
FP64_PATH = os.path.join(ROOT, "profiles", "r01_measured_fp64_tf32.json")  # scripts/fp64_peak.py (cuBLAS DGEMM)
N_SM = 148
FP32_LANES, FP64_LANES = 128, 64  # per SM per clock (FMA units)
# iterations a run takes to its termination criterion (R-19), measured on a
# B200 (profiles/r01_accuracy.md): the span the timed offsets are spread over
REP_ITERS = {"C1": 54, "C2": 250, "C3a": 2400, "C3b": 6400, "C4": 260, "C5": 46}
FIRST = 4  # iterations 1-3 of every run capture the iteration's graphs (host time): never timed
SHARDED = ("C3a", "C3b", "C4", "C5")


# ---------------------------------------------------------------------------
# algorithmic work models
# ---------------------------------------------------------------------------
def hrss_flops_model(prob):
    """fp32 flops of the warp/lane HRSS kernels: per HRSS step d(d+1) (L z)
    + 2d (normalise); per probe 2d (x + t v) plus the Gaussian prior 4d; per
    energy evaluation the energy's own flops."""
    d = prob.d
    per_step = d * (d + 1) + 2 * d
    per_probe = 2 * d + (4 * d if prob.prior_kind == W.PRIOR_GAUSS_DIAG else 0)
    k = prob.energy_kind
    if k == W.E_GAUSS:
        per_eval = 4 * d + 1
    elif k == W.E_MOG:
        per_eval = prob.n_comp * (4 * d + 3) + 2
    elif k == W.E_CORR_GAUSS:
        per_eval = 2 * d * d + 3 * d
    elif k == W.E_FUNNEL:
        per_eval = 2 * d + 10
    elif k == W.E_LOGREG:
        per_eval = prob.n_data * (2 * d + 6)
    else:
        per_eval = 0
    return per_step, per_probe, per_eval


def energy_pass_flops(prob):
    """Algorithmic flops of one batched energy evaluation (per probe row):
    logistic regression 2 N d (the X theta contraction); GP N^3/3 (Cholesky)
    + 2 N^2 (forward solve) + N^2 (D + 2) / 2 ... (kernel matrix) ."""
    if prob.energy_kind == W.E_LOGREG:
        return 2.0 * prob.n_data * prob.d
    if prob.energy_kind == W.E_GP_ARD:
        N, D = prob.n_data, prob.d_in
        return N ** 3 / 3.0 + 2.0 * N * N + 0.5 * N * N * (3 * D + 2)
    return 0.0


def read_json(path):
    try:
        return json.load(open(path))
    except Exception:
        return {}


# ---------------------------------------------------------------------------
# clocks under load (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------
def clocks_sampler_start(path):
    try:
        f = open(path, "w")
        p = subprocess.Popen(
            ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
             "--format=csv,noheader,nounits", "-lms", "100"], stdout=f, stderr=subprocess.DEVNULL)
        return p, f
    except Exception:
        return None, None


def clocks_sampler_stop(p, f, path, gpu_index):
    if p is None:
        return None
    p.terminate()
    try:
        p.wait(timeout=5)
    except Exception:
        p.kill()
    f.close()
    sm, mx, reasons = [], None, set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for line in open(path):
        parts = [t.strip() for t in line.split(",")]
        if len(parts) < 9 or parts[0] != str(gpu_index):
            continue
        try:
            sm.append(float(parts[1]))
            mx = float(parts[2])
        except ValueError:
            continue
        for nm, v in zip(names, parts[5:9]):
            if v.lower() == "active":
                reasons.add(nm)
    try:
        os.remove(path)
    except OSError:
        pass
    if not sm:
        return None
    return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# the oracle on the host: cpu_baseline and --impl reference
# ---------------------------------------------------------------------------
def host_cpu():
    model = platform.processor() or ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"host_cpu": model, "host_cores": os.cpu_count()}


def width_rule(d, c=1.0):
    """R-7 OPTIMAL width in whitened units: c 4 kappa sqrt(2 (d + 2) / (pi d))."""
    return c * 4.0 * 1.3035 * math.sqrt(2.0 * (d + 2) / (math.pi * d))


def _oracle_slice_sample(name, seconds, seed=1):
    """Bounded sample for the big configurations, whose whole iterations are
    out of reach of the oracle (C4 ~1e13 flops, C5 ~0.3 s per energy): the
    first iteration of a run, step by step -- HRSS steps of the oracle
    (nsso_slice_step: stepping-out, shrinkage, every energy of the real
    workload) from seeded prior draws, with the run's width rule (R-7: the
    live set is the prior, whose whitening is the identity for C4/C5's N(0, I)
    prior, so directions are uniform unit vectors and w = w*(d)) and E* = the
    median of 16 drawn energies (k/n = 1/2 at C4 and C5), until `seconds` of
    CPU time."""
    from oracle import nsso
    prob, cfg = W.workload(name)
    o = nsso.Oracle(prob, cfg, draw_live=False)
    rng = np.random.default_rng(seed)
    if prob.prior_kind == W.PRIOR_BOX:
        xs = prob.lo + (prob.hi - prob.lo) * rng.random((16, prob.d))
    else:
        xs = prob.mean + prob.sd * rng.standard_normal((16, prob.d))
    t0 = time.process_time()
    es = np.array([o.energy(x) for x in xs])
    e0_evals = len(es)
    e_star = float(np.sort(es)[8])
    live = np.nonzero(es < e_star)[0]
    w = width_rule(prob.d)
    steps = 0
    i0 = o.info()["energy_evals"]
    while time.process_time() - t0 < seconds:
        j = live[steps % live.size]
        v = rng.standard_normal(prob.d)
        v /= np.linalg.norm(v)
        o.slice_step(xs[j], es[j], v, w, e_star, 1, int(j), steps)
        steps += 1
    t = time.process_time() - t0
    evals = o.info()["energy_evals"] - i0 + e0_evals
    o.close()
    return evals, t, f"{name}: {steps} oracle HRSS steps (first iteration of a run: prior draws, width rule " \
                     f"w = {w:.3f}, E* = median of 16) + {e0_evals} energies, {t:.1f} s CPU, 1 thread, fp64"


def cpu_baseline(name, seconds=12.0):
    """The fp64 oracle, as it stands, on one host core (bounded sample)."""
    if name in ("C4", "C5"):
        evals, t, what = _oracle_slice_sample(name, seconds)
        return {"value": evals / t, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": what, **host_cpu()}
    from oracle import nsso
    prob, cfg = W.workload(name)
    evals, t_tot, iters, seed = 0, 0.0, 0, 1
    while t_tot < seconds and seed <= 8:
        cfg["seed"] = seed
        o = nsso.Oracle(prob, cfg)
        t0 = time.process_time()
        e0 = o.info()["energy_evals"]
        info = o.info()
        while (time.process_time() - t0) + t_tot < seconds and not info["terminated"]:
            info = o.step()
        t_tot += time.process_time() - t0
        evals += info["energy_evals"] - e0
        iters += info["iteration"]
        seed += 1
        o.close()
    return {"value": evals / t_tot, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{name}: {iters} oracle iterations from the start of {seed - 1} seeded runs "
                      f"({t_tot:.1f} s CPU, 1 thread, fp64)", "iterations_per_s": iters / t_tot, **host_cpu()}


def run_reference(args):
    """--impl reference: the fp64 oracle timed on the host (rank 0 only)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    from oracle import nsso
    prob, cfg = W.workload(args.config)
    evals, t_tot = 0, 0.0
    if args.config in ("C4", "C5"):
        per = max(2.0, 60.0 / max(args.steps + args.warmup, 1))
        for i in range(args.warmup):
            _oracle_slice_sample(args.config, per, seed=100 + i)
        for i in range(args.steps):
            e, t, what = _oracle_slice_sample(args.config, per, seed=i + 1)
            evals += e
            t_tot += t
        sample = f"{args.steps} bounded samples of {per:.0f} s: " + what.split(":", 1)[1]
    else:
        T = REP_ITERS.get(args.config, 50)
        seed = 1
        o = nsso.Oracle(prob, cfg)

        def fresh(o, seed):
            if o.info()["iteration"] >= T:
                o.close()
                cfg["seed"] = seed + 1
                return nsso.Oracle(prob, cfg), seed + 1
            return o, seed
        for _ in range(args.warmup):
            o, seed = fresh(o, seed)
            o.step()
        for _ in range(args.steps):
            o, seed = fresh(o, seed)
            e0 = o.info()["energy_evals"]
            t0 = time.perf_counter()
            info = o.step()
            t_tot += time.perf_counter() - t0
            evals += info["energy_evals"] - e0
        sample = f"{args.steps} oracle iterations of {args.config}"
    value = evals / t_tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, workloads.py)",
            "config": {"workload": f"{args.config} {prob.name}", "n_live": cfg["n_live"], "k": cfg["k"],
                       "steps_hrss": cfg["steps"], "d": prob.d},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                             **host_cpu()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def problem_bytes(prob):
    b = 0
    for a in (prob.lo, prob.hi, prob.mean, prob.sd, prob.w, prob.mu, prob.sigma, prob.prec, prob.data_x,
              prob.data_y):
        if a is not None:
            b += np.asarray(a).size * 8
    return b


def schedule(T, K):
    """(run, iteration) of the K timed iterations: evenly spaced offsets over
    iterations FIRST..T of a run, further runs when K > T - FIRST + 1."""
    span = max(T - FIRST + 1, 1)
    per_run = min(K, span)
    out = []
    for j in range(K):
        run, i = divmod(j, per_run)
        out.append((run, FIRST + (i * span) // per_run))
    return out


def relaunch_distributed(args):
    """--gpus N without a torchrun environment: start N ranks of this script."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ---------------------------------------------------------------------------
# the CUDA path
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--mode", default="auto", choices=["auto", "replicas", "shard"])
    ap.add_argument("--impl", default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(args)
    if args.impl == "reference":
        return run_reference(args)
    args.warmup = max(args.warmup, 3)  # timing rules: at least 3 warm-up steps (the line reports the count run)

    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    td = None
    if world > 1:
        import torch.distributed as td
        td.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2601_23252_b200 import dist as D
    from paper_2601_23252_b200 import nss

    mode = args.mode if args.mode != "auto" else ("shard" if args.config in SHARDED else "replicas")
    # shard at N = 1 only when asked: the NCCL world-1 sharded path (its overhead on one GPU)
    shard = mode == "shard" and (world > 1 or args.mode == "shard")
    prob, cfg = W.workload(args.config)
    T = REP_ITERS.get(args.config, 50)
    sched = schedule(T, args.steps)
    # a dedicated (non-default) stream: the library launches on it and the
    # timing events are recorded on it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    def new_run(seed):
        c = dict(cfg)
        c["max_dead"] = cfg["n_live"] + cfg["k"] * int(1.6 * T + 50)  # a whole run and its finalisation
        c["seed"] = seed if shard else seed + 1000 * rank
        if shard and world == 1:  # the world-1 NCCL sharded path
            return nss.Sampler(prob, c, stream=stream.cuda_stream, dist=(0, 1, D.nccl_unique_id()))
        if shard:
            return D.sharded_sampler(prob, c, stream=stream.cuda_stream)
        return nss.Sampler(prob, c, stream=stream.cuda_stream)

    # warm-up: W iterations of a throw-away run (module load, graph capture paths, clocks)
    s = new_run(99)
    engine = s.engine()
    for _ in range(args.warmup):
        s.step(sync=False)
    s.sync()
    s.close()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    per_step, per_probe, per_eval = hrss_flops_model(prob)

    def timed_pass(kernel_timing):
        """The scheduled iterations, each bracketed by CUDA events on the
        library's stream after a synchronisation and an L2 flush.
        kernel_timing False: the production path (each iteration one
        CUDA-graph replay; the batch engine's rounds in graph chunks) -- the
        metric.  True: the library's event-timing mode at the scheduled
        iterations only -- per-kernel durations for the roofline."""
        acc = {"ms": 0.0, "evals": 0, "probes": 0, "iters": 0, "launches": 0, "flops": 0.0, "ph": {},
               "short": 0}
        runs = sorted(set(r for r, _ in sched))
        for run in runs:
            its = [i for r, i in sched if r == run]
            sr = new_run(1 + run)
            cur = 0
            for it in its:
                if it - 1 > cur:
                    sr.steps(it - 1 - cur)  # untimed, asynchronous
                    cur = it - 1
                sr.sync()
                i0 = sr.info()
                if i0["terminated"]:
                    acc["short"] += 1
                l0 = sr.launch_count()
                if kernel_timing:
                    sr.set_kernel_timing(True)
                flush.zero_()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                sr.step(sync=False)
                b.record(stream)
                b.synchronize()
                acc["ms"] += a.elapsed_time(b)
                cur = it
                i1 = sr.info()
                if kernel_timing:
                    for nm, (ms, n) in sr.phase_times().items():
                        q = acc["ph"].setdefault(nm, [0.0, 0])
                        q[0] += ms
                        q[1] += n
                    sr.set_kernel_timing(False)
                acc["launches"] += sr.launch_count() - l0
                d_evals = i1["energy_evals"] - i0["energy_evals"]
                d_probes = i1["probes"] - i0["probes"]
                d_iters = i1["iteration"] - i0["iteration"]
                acc["evals"] += d_evals
                acc["probes"] += d_probes
                acc["iters"] += d_iters
                acc["flops"] += d_iters * cfg["k"] * cfg["steps"] * per_step + d_probes * per_probe + d_evals * per_eval
            sr.close()
        return acc

    # ---- timed region ----
    clk_path = os.path.join(ROOT, f".clocks_rank{rank}.csv")
    cp, cf = clocks_sampler_start(clk_path) if rank == 0 else (None, None)
    time.sleep(0.3 if cp else 0)
    if td is not None:
        td.barrier()
    torch.cuda.synchronize()
    A = timed_pass(False)  # the metric
    torch.cuda.synchronize()
    if td is not None:
        td.barrier()
    clocks = clocks_sampler_stop(cp, cf, clk_path, local) if rank == 0 else None
    B = timed_pass(True)   # per-kernel event timing (roofline, phase shares)
    tot_ms, evals, probes, iters, launches = A["ms"], A["evals"], A["probes"], A["iters"], A["launches"]
    ph_ms, alg_flops = B["ph"], B["flops"]

    t_max, tot_evals, tot_probes = tot_ms, float(evals), float(probes)
    if td is not None:
        tt = torch.tensor([tot_ms, float(evals), float(probes), float(launches)], dtype=torch.float64,
                          device="cuda")
        mx = tt.clone()
        td.all_reduce(mx, op=td.ReduceOp.MAX)
        td.all_reduce(tt, op=td.ReduceOp.SUM)
        t_max, tot_evals, tot_probes = mx[0].item(), tt[1].item(), tt[2].item()
        launches = int(tt[3].item())
    value = tot_evals / (t_max / 1e3)
    job_iters = iters if shard else iters * world

    # ---- end-to-end through the public API: init from host buffers, steps
    #      each reading back its step info until termination, evidence ----
    e2e = None
    if not args.no_e2e:
        torch.cuda.synchronize()
        if td is not None:
            td.barrier()
        t0 = time.perf_counter()
        se = new_run(10_000)
        info = se.info()
        n_steps = 0
        while not info["terminated"] and n_steps < 4 * T:
            info = se.step(sync=True)
            n_steps += 1
        lz, lz_err = se.evidence()
        t_e2e = time.perf_counter() - t0
        e2e_evals = float(info["energy_evals"] + info["init_evals"])
        se.close()
        if td is not None:
            tt = torch.tensor([t_e2e, e2e_evals], dtype=torch.float64, device="cuda")
            mx = tt.clone()
            td.all_reduce(mx, op=td.ReduceOp.MAX)
            td.all_reduce(tt, op=td.ReduceOp.SUM)
            t_e2e, e2e_evals = mx[0].item(), tt[1].item()
        from paper_2601_23252_b200.nss import nss_step_info
        import ctypes
        e2e = {"value": e2e_evals / t_e2e, "unit": UNIT,
               "h2d_bytes_per_step": problem_bytes(prob) / max(n_steps, 1),
               "d2h_bytes_per_step": float(ctypes.sizeof(nss_step_info)) + 8.0 * (cfg["n_volume_sims"] + 3) /
               max(n_steps, 1),
               "what": f"one whole run: nss_init from host buffers (problem data uploaded, {n_steps} x nss_step "
                       "with its step info read back, nss_evidence), wall clock; init evaluations included",
               "iterations": n_steps, "seconds": t_e2e, "log_z": lz, "log_z_err": lz_err}

    if rank == 0:
        peaks = read_json(PEAKS_PATH)
        traffic = read_json(TRAFFIC_PATH)
        mhz = peaks.get("sm_max_mhz", 1965.0)
        roof = roofline(prob, engine, ph_ms, alg_flops, peaks, traffic, mhz, B["ms"], B["evals"])
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if shard else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded, workloads.py)",
            "config": {"workload": f"{args.config} {prob.name}", "n_live": cfg["n_live"], "k": cfg["k"],
                       "steps_hrss": cfg["steps"], "d": prob.d, "engine": engine,
                       "parallelism": (f"shard x{world} (live set by gid segment; NCCL all-gather of candidates "
                                       "and moments; parent rows read from peers)" if shard
                                       else f"replicas x{world}"),
                       "l2": "flushed between timed iterations (256 MiB write)",
                       "window": f"{args.steps} iterations at fixed offsets over iterations {FIRST}..{T} of "
                                 f"{len(set(r for r, _ in sched))} run(s) (independent of --steps)"},
            "iterations_per_s": job_iters / (t_max / 1e3),
            "probes_per_s": tot_probes / (t_max / 1e3),
            "gpu_launches": launches,
            "phase_ms_per_step": {nm: v[0] / max(args.steps, 1) for nm, v in ph_ms.items()},
            "kernel_timing": "phase and kernel times from a second run with the same seed replaying the same "
                             "iterations in the library's event-timing mode (eager launches)",
            "roofline": roof,
        }
        if A["short"]:
            line["warning"] = f"{A['short']} timed iterations fell after the run's termination"
        if e2e:
            line["e2e"] = e2e
        if prob.energy_kind == W.E_GP_ARD:
            line["dtype"] = "f32 (GP energy f64)"
        if clocks:
            line["clocks"] = clocks
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args.config)
        print(json.dumps(line), flush=True)
    if td is not None:
        td.destroy_process_group()
    return 0


def roofline(prob, engine, ph_ms, alg_flops, peaks, traffic, mhz, step_ms, evals):
    """Roofline entry for the dominant kernel: the
    HRSS kernel (warp / lane engines: fp32 ALU bound), else the batched energy
    kernel (tensor-core logistic regression: bf16 tensor bound against the
    measured burst peak -- every launch is timed alone by its own events;
    GP: fp64 tensor against the measured DGEMM)."""
    hr_ms, hr_n = ph_ms.get("hrss", [0.0, 0])
    en_ms, en_n = ph_ms.get("energy", [0.0, 0])
    if engine != "batch":
        peak = N_SM * FP32_LANES * 2 * mhz * 1e6 / 1e12
        achieved = (alg_flops / max(hr_n, 1)) / ((hr_ms / max(hr_n, 1)) / 1e3) / 1e12 if hr_n else 0.0
        name = "k_hrss_lane (one probe per lane)" if engine == "lane" else "k_hrss (warp per chain)"
        return {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic.get(name.split()[0]),
                "kernel": name + " + fused energy", "kernel_ms_avg": hr_ms / max(hr_n, 1),
                "kernel_share_of_step": hr_ms / max(step_ms, 1e-9),
                "peak_source": f"148 SM x 128 FP32 lanes x 2 x {mhz:.0f} MHz (derived from B200_PROFILING.md)"}
    # batch engine: the energy passes, timed per launch; each evaluates the
    # probe rows of one round, and the rows over all launches are this rank's
    # energy evaluations
    flops_per_row = energy_pass_flops(prob)
    if prob.energy_kind == W.E_LOGREG:
        peak = peaks.get("bf16_tflops", 1590.0)
        bound, kname = "tensor", "k_lr_energy"
        src = "bf16_tflops (burst) of measured (MEASURED_PEAKS.json)" if "bf16_tflops" in peaks \
            else "1.59 PFLOP/s burst of fallback"
    else:
        fp64 = read_json(FP64_PATH).get("fp64_tflops")
        # DMMA (fp64 tensor) Cholesky updates and TRSM; the fused chain kernel
        # (default) runs the HRSS state machine and the GP energies in one launch
        bound, kname = "tensor", "k_gp_energy" if os.environ.get("NSS_GP_ROUNDS") else "k_gp_chains"
        if fp64:
            peak, src = fp64, "fp64 cuBLAS DGEMM of measured (profiles/r01_measured_fp64_tf32.json)"
        else:
            peak = N_SM * FP64_LANES * 2 * mhz * 1e6 / 1e12
            src = f"148 SM x 64 FP64 lanes x 2 x {mhz:.0f} MHz (derived)"
    achieved = evals * flops_per_row / (en_ms / 1e3) / 1e12 if en_ms > 0 else 0.0
    return {"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": traffic.get(kname), "kernel": kname, "kernel_ms_avg": en_ms / max(en_n, 1),
            "kernel_share_of_step": en_ms / max(step_ms, 1e-9), "flops_per_row": flops_per_row,
            "rows_per_launch": evals / max(en_n, 1), "peak_source": src}


if __name__ == "__main__":
    sys.exit(main())
