#!/usr/bin/env python
"""Benchmark: one NS outer iteration (all SURVEY section 8(a) rows) per step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2]
                    [--mode auto|replicas|shard] [--impl reference]

Workload (BASELINE.json configs[1]): C2, d=10 well-separated 4-component
Gaussian mixture, n_live=2000, k=200, p=10 HRSS steps, synthetic seeded data.
--config picks another BASELINE configuration (C1, C3a, C3b, C4, C5).
Metric: constrained energy evaluations per second (also NS iterations/s).

Timing: W warm-up iterations, then K timed iterations; each timed iteration is
bracketed by CUDA events on the stream the library launches on, and L2 is
flushed (a 256 MiB write) between timed iterations, outside the events.  The
metric pass runs the production path (one CUDA-graph replay per iteration); a
second pass of K iterations in the library's event-timing mode (every kernel
launched eagerly between its own events) gives the per-kernel durations of
the roofline entry and the phase times.  NS
runs terminate; when a run reaches its last representative iteration a new
seed is initialised outside the timed region, so every timed step is a real
iteration of a live run.

Multi-GPU (torchrun): --mode shard runs ONE NS run whose
HRSS chains are split over the ranks (NCCL all-gather of the new rows each
iteration; strong scaling: the job's work is fixed); --mode replicas runs an
independent run per rank (weak scaling).  auto = replicas for C1/C2 (an
iteration's HRSS there is a few tens of microseconds, below what splitting it
saves), shard for C3a/C3b/C4/C5.  Times are the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
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
RUN_LIMIT = {"C1": 40, "C2": 200, "C3a": 60, "C3b": 60, "C4": 20, "C5": 4}
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
def _oracle_slice_sample(name, seconds, seed=1):
    """Bounded sample for the big configurations, whose whole iterations are
    out of reach of the oracle (C4 ~1e13 flops, C5 ~0.3 s per energy): HRSS
    steps of the oracle (nsso_slice_step: stepping-out, shrinkage, every energy
    of the real workload) from seeded prior draws under a threshold E* set at
    the worst of 16 drawn energies, until `seconds` of CPU time."""
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
    e_star = es.max() + 1e-9 * abs(es.max())
    w = 2.0 * math.sqrt(2.0 / (math.pi * prob.d)) * 2.0
    steps = 0
    i0 = o.info()["energy_evals"]
    while time.process_time() - t0 < seconds:
        j = steps % 15
        x0 = xs[j] if es[j] < e_star else xs[(j + 1) % 16]
        e0 = es[j] if es[j] < e_star else es[(j + 1) % 16]
        v = rng.standard_normal(prob.d)
        v /= np.linalg.norm(v)
        o.slice_step(x0, e0, v, w, e_star, 1, j, steps)
        steps += 1
    t = time.process_time() - t0
    evals = o.info()["energy_evals"] - i0 + e0_evals
    o.close()
    return evals, t, f"{name}: {steps} oracle HRSS steps + {e0_evals} energies from seeded prior draws " \
                     f"(E* = worst of 16), {t:.1f} s CPU, 1 thread, fp64"


def cpu_baseline(name, seconds=12.0):
    """The fp64 oracle, as it stands, on one host core (bounded sample)."""
    if name in ("C4", "C5"):
        evals, t, what = _oracle_slice_sample(name, seconds)
        return {"value": evals / t, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": what}
    from oracle import nsso
    prob, cfg = W.workload(name)
    evals, t_tot, iters, seed = 0, 0.0, 0, 1
    while t_tot < seconds and seed <= 8:
        cfg["seed"] = seed
        o = nsso.Oracle(prob, cfg)
        t0 = time.process_time()
        info = o.info()
        for _ in range(RUN_LIMIT.get(name, 50)):
            info = o.step()
            if (time.process_time() - t0) + t_tot > seconds:
                break
        t_tot += time.process_time() - t0
        evals += info["energy_evals"]
        iters += info["iteration"]
        seed += 1
        o.close()
    return {"value": evals / t_tot, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{name}: {iters} oracle iterations over {seed - 1} seeded runs "
                      f"({t_tot:.1f} s CPU, 1 thread, fp64)", "iterations_per_s": iters / t_tot}


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
        lim = RUN_LIMIT.get(args.config, 50)
        seed = 1
        o = nsso.Oracle(prob, cfg)

        def fresh(o, seed):
            if o.info()["iteration"] >= lim:
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
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
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


# ---------------------------------------------------------------------------
# the CUDA path
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=600)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--mode", default="auto", choices=["auto", "replicas", "shard"])
    ap.add_argument("--impl", default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    assert args.warmup >= 3, "timing rules: at least 3 warm-up steps"

    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    td = None
    if world > 1:
        import torch.distributed as td
        td.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2601_23252_b200 import dist as D
    from paper_2601_23252_b200 import nss

    mode = args.mode if args.mode != "auto" else ("shard" if args.config in SHARDED else "replicas")
    shard = world > 1 and mode == "shard"
    prob, cfg = W.workload(args.config)
    lim = RUN_LIMIT.get(args.config, 50)
    # a dedicated (non-default) stream: the library launches on it and the
    # timing events are recorded on it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    state = {"seed": 1 if shard else 1 + 1000 * rank}

    def new_run(seed=None):
        c = dict(cfg)
        c["seed"] = state["seed"] if seed is None else seed
        if seed is None:
            state["seed"] += 1
        if shard:
            return D.sharded_sampler(prob, c, stream=stream.cuda_stream)
        return nss.Sampler(prob, c, stream=stream.cuda_stream)

    s = new_run()
    engine = s.engine()
    for _ in range(args.warmup):
        if s.info()["iteration"] >= lim:
            s.close()
            s = new_run()
        s.step(sync=False)
    torch.cuda.synchronize()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    per_step, per_probe, per_eval = hrss_flops_model(prob)

    # ---- timed region ----
    clk_path = os.path.join(ROOT, f".clocks_rank{rank}.csv")
    cp, cf = clocks_sampler_start(clk_path) if rank == 0 else (None, None)
    time.sleep(0.3 if cp else 0)
    if td is not None:
        td.barrier()
    torch.cuda.synchronize()
    def timed_pass(kernel_timing):
        """K iterations, each bracketed by CUDA events on the library's stream
        with the L2 flushed in between (outside the events).  kernel_timing
        False: the production path (each iteration one CUDA-graph replay) --
        the metric.  True: the library's event-timing mode (every kernel
        launched eagerly between its own events) -- per-kernel durations for
        the roofline only; its step time is not reported."""
        nonlocal s
        acc = {"ms": 0.0, "evals": 0, "probes": 0, "iters": 0, "launches": 0, "flops": 0.0, "ph": {}}
        done = 0
        while done < args.steps:
            if s.info()["iteration"] >= lim:
                s.close()
                s = new_run()
                for _ in range(2):
                    s.step(sync=False)
            s.set_kernel_timing(kernel_timing)
            i0 = s.info()
            l0 = s.launch_count()
            batch = min(args.steps - done, lim - i0["iteration"])
            evs = []
            for _ in range(batch):
                flush.zero_()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                s.step(sync=False)
                b.record(stream)
                evs.append((a, b))
            torch.cuda.synchronize()
            for a, b in evs:
                acc["ms"] += a.elapsed_time(b)
            i1 = s.info()
            if kernel_timing:
                for nm, (ms, n) in s.phase_times().items():
                    q = acc["ph"].setdefault(nm, [0.0, 0])
                    q[0] += ms
                    q[1] += n
            s.set_kernel_timing(False)
            acc["launches"] += s.launch_count() - l0
            d_evals = i1["energy_evals"] - i0["energy_evals"]
            d_probes = i1["probes"] - i0["probes"]
            d_iters = i1["iteration"] - i0["iteration"]
            acc["evals"] += d_evals
            acc["probes"] += d_probes
            acc["iters"] += d_iters
            acc["flops"] += d_iters * cfg["k"] * cfg["steps"] * per_step + d_probes * per_probe + d_evals * per_eval
            done += batch
        return acc

    A = timed_pass(False)  # the metric
    torch.cuda.synchronize()
    if td is not None:
        td.barrier()
    B = timed_pass(True)   # per-kernel event timing (roofline, phase shares)
    tot_ms, evals, probes, iters, launches = A["ms"], A["evals"], A["probes"], A["iters"], A["launches"]
    ph_ms, alg_flops = B["ph"], B["flops"]
    torch.cuda.synchronize()
    if td is not None:
        td.barrier()
    clocks = clocks_sampler_stop(cp, cf, clk_path, local) if rank == 0 else None

    t_max, tot_evals, tot_probes = tot_ms, float(evals), float(probes)
    if td is not None:
        tt = torch.tensor([tot_ms, float(evals), float(probes), float(launches)], dtype=torch.float64,
                          device="cuda")
        mx = tt.clone()
        td.all_reduce(mx, op=td.ReduceOp.MAX)
        td.all_reduce(tt, op=td.ReduceOp.SUM)
        t_max, tot_evals, tot_probes = mx[0].item(), tt[1].item(), tt[2].item()
    value = tot_evals / (t_max / 1e3)
    job_iters = iters if shard else iters * world

    # ---- context only (not the metric): the same iterations back to back,
    #      no flush and no per-step events, one event pair around the batch
    bb = None
    if not shard and world == 1:
        s2 = new_run(seed=20_000)
        for _ in range(3):
            s2.step(sync=False)
        s2.sync()
        nb = min(args.steps, lim - 3)
        ib0 = s2.info()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(nb):
            s2.step(sync=False)
        b.record(stream)
        torch.cuda.synchronize()
        ib1 = s2.info()
        ms_bb = a.elapsed_time(b)
        bb = {"us_per_iteration": 1e3 * ms_bb / max(ib1["iteration"] - ib0["iteration"], 1),
              "evals_per_s": (ib1["energy_evals"] - ib0["energy_evals"]) / (ms_bb / 1e3),
              "what": f"{nb} iterations back to back, L2 warm, no per-step events (context, not the metric)"}
        s2.close()

    # ---- end-to-end through the public API: init from host buffers, K steps
    #      each reading back its step info, evidence at the end ----
    s.close()
    torch.cuda.synchronize()
    if td is not None:
        td.barrier()
    e2e_steps = min(args.steps, lim)
    t0 = time.perf_counter()
    se = new_run(seed=10_000 + (0 if shard else rank))
    e_start = se.info()["energy_evals"]
    info = se.info()
    for _ in range(e2e_steps):
        info = se.step(sync=True)
    lz, lz_err = se.evidence()
    t_e2e = time.perf_counter() - t0
    e2e_evals = float(info["energy_evals"] - e_start)
    se.close()
    if td is not None:
        tt = torch.tensor([t_e2e, e2e_evals], dtype=torch.float64, device="cuda")
        mx = tt.clone()
        td.all_reduce(mx, op=td.ReduceOp.MAX)
        td.all_reduce(tt, op=td.ReduceOp.SUM)
        t_e2e, e2e_evals = mx[0].item(), tt[1].item()
    e2e_value = e2e_evals / t_e2e

    if rank == 0:
        peaks = read_json(PEAKS_PATH)
        traffic = read_json(TRAFFIC_PATH)
        mhz = peaks.get("sm_max_mhz", 1965.0)
        roof = roofline(prob, engine, ph_ms, alg_flops, peaks, traffic, mhz, tot_ms, B["evals"])
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if shard else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded, workloads.py)",
            "config": {"workload": f"{args.config} {prob.name}", "n_live": cfg["n_live"], "k": cfg["k"],
                       "steps_hrss": cfg["steps"], "d": prob.d, "engine": engine,
                       "parallelism": (f"shard x{world} (HRSS chain blocks, NCCL all-gather)" if shard
                                       else f"replicas x{world}"),
                       "l2": "flushed between timed iterations (256 MiB write)",
                       "runs": f"new seed every {lim} iterations (outside the timed region)"},
            "iterations_per_s": job_iters / (t_max / 1e3),
            "probes_per_s": tot_probes / (t_max / 1e3),
            "gpu_launches": launches,
            "back_to_back": bb,
            "phase_ms_per_step": {nm: v[0] / max(args.steps, 1) for nm, v in ph_ms.items()},
            "kernel_timing": "phase and kernel times from a second pass of K iterations in the library's "
                             "event-timing mode (eager launches); the metric pass replays the iteration's "
                             "CUDA graph with events only around each iteration",
            "roofline": roof,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": problem_bytes(prob) / e2e_steps,
                    "d2h_bytes_per_step": 96 + 8 * (cfg["n_volume_sims"] + 3) / e2e_steps,
                    "what": "nss_init from host buffers + K x nss_step(info) + nss_evidence, wall clock",
                    "log_z": lz, "log_z_err": lz_err},
        }
        if args.config == "C5" or prob.energy_kind == W.E_GP_ARD:
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
    kernel (tensor-core logistic regression: bf16 tensor bound; GP: fp64 ALU)."""
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
        peak = peaks.get("bf16_tflops_sustained", 1400.0)
        bound, kname = "tensor", "k_lr_energy"
        src = "bf16_tflops_sustained of measured (MEASURED_PEAKS.json)" if "bf16_tflops_sustained" in peaks \
            else "1.4 PFLOP/s sustained of fallback"
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
