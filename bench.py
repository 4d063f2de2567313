#!/usr/bin/env python
"""Benchmark: one NS outer iteration (all SURVEY section 8(a) rows) per step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl reference]

Workload (BASELINE.json configs[1]): C2, d=10 well-separated 4-component
Gaussian mixture, n_live=2000, k=200, p=10 HRSS steps, synthetic seeded data.
Metric: constrained energy evaluations per second (also NS iterations/s).

Timing: W warm-up iterations, then K timed iterations; each timed iteration is
bracketed by CUDA events on the stream the library launches on, and L2 is
flushed (a 256 MiB write) between timed iterations, outside the events.  NS
runs terminate; when a run reaches its last representative iteration a new
seed is initialised outside the timed region, so every timed step is a real
iteration of a live run.  Multi-GPU (torchrun): one independent run per rank
(weak scaling, no data-path collective yet), max of the per-rank times.
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
# FP32 pipe: 148 SMs x 128 FMA lanes x 2 flop at the max SM clock (B200_PROFILING.md)
N_SM, FP32_LANES = 148, 128
RUN_LIMIT = {"C1": 40, "C2": 200, "C3a": 60, "C3b": 60, "C4": 20, "C5": 10}


def flops_model(prob, cfg):
    """Algorithmic fp32 flops of the HRSS kernel:
    per HRSS step d(d+1) (L z) + 2d (normalise); per probe 2d (x + t v) plus the
    Gaussian prior 4d; per energy evaluation the energy's own flops."""
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


def read_peaks():
    try:
        return json.load(open(PEAKS_PATH))
    except Exception:
        return {}


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
    if not sm:
        return None
    return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(name, seconds=12.0):
    """The fp64 oracle, as it stands, on one host core: evals/s over whole runs
    of the same workload (bounded sample: up to `seconds` of CPU work)."""
    from oracle import nsso
    prob, cfg = W.workload(name)
    evals, t_tot, iters, seed = 0, 0.0, 0, 1
    while t_tot < seconds and seed <= 8:
        cfg["seed"] = seed
        o = nsso.Oracle(prob, cfg)
        t0 = time.process_time()
        lim = RUN_LIMIT.get(name, 50)
        for _ in range(lim):
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
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import nsso
    prob, cfg = W.workload(args.config)
    o = nsso.Oracle(prob, cfg)
    lim = RUN_LIMIT.get(args.config, 50)
    seed = 1
    for _ in range(args.warmup):
        if o.info()["iteration"] >= lim:
            seed += 1
            cfg["seed"] = seed
            o = nsso.Oracle(prob, cfg)
        o.step()
    evals, t_tot = 0, 0.0
    for _ in range(args.steps):
        if o.info()["iteration"] >= lim:
            seed += 1
            cfg["seed"] = seed
            o = nsso.Oracle(prob, cfg)
        e0 = o.info()["energy_evals"]
        t0 = time.perf_counter()
        info = o.step()
        t_tot += time.perf_counter() - t0
        evals += info["energy_evals"] - e0
    value = evals / t_tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, workloads.py)",
            "config": {"workload": f"{args.config} {prob.name}", "n_live": cfg["n_live"], "k": cfg["k"],
                       "steps_hrss": cfg["steps"], "d": prob.d},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{args.steps} oracle iterations of {args.config}"},
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=600)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2")
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
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2601_23252_b200 import nss

    prob, cfg = W.workload(args.config)
    lim = RUN_LIMIT.get(args.config, 50)
    # a dedicated (non-default) stream: the library launches on it and the
    # timing events are recorded on it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    seed_base = 1 + 1000 * rank
    state = {"seed": seed_base}

    def new_run():
        c = dict(cfg)
        c["seed"] = state["seed"]
        state["seed"] += 1
        return nss.Sampler(prob, c, stream=stream.cuda_stream)

    s = new_run()
    for _ in range(args.warmup):
        if s.info()["iteration"] >= lim:
            s.close()
            s = new_run()
        s.step(sync=False)
    torch.cuda.synchronize()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    per_step, per_probe, per_eval = flops_model(prob, cfg)

    # ---- timed region ----
    clk_path = os.path.join(ROOT, f".clocks_rank{rank}.csv")
    cp, cf = clocks_sampler_start(clk_path) if rank == 0 else (None, None)
    time.sleep(0.3 if cp else 0)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    tot_ms, evals, probes, iters, launches = 0.0, 0, 0, 0, 0
    hrss_ms, hrss_n, alg_flops = 0.0, 0, 0.0
    done = 0
    while done < args.steps:
        if s.info()["iteration"] >= lim:
            ms, n = s.kernel_time()
            hrss_ms += ms
            hrss_n += n
            s.close()
            s = new_run()
            for _ in range(2):
                s.step(sync=False)
        s.set_kernel_timing(True)
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
            tot_ms += a.elapsed_time(b)
        i1 = s.info()
        ms, n = s.kernel_time()
        hrss_ms += ms
        hrss_n += n
        s.set_kernel_timing(False)
        launches += s.launch_count() - l0
        d_evals = i1["energy_evals"] - i0["energy_evals"]
        d_probes = i1["probes"] - i0["probes"]
        d_iters = i1["iteration"] - i0["iteration"]
        evals += d_evals
        probes += d_probes
        iters += d_iters
        alg_flops += d_iters * cfg["k"] * cfg["steps"] * per_step + d_probes * per_probe + d_evals * per_eval
        done += batch
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clocks = clocks_sampler_stop(cp, cf, clk_path, local) if rank == 0 else None
    if cp:
        try:
            os.remove(clk_path)
        except OSError:
            pass

    t_max = tot_ms
    tot_evals = evals
    if dist is not None:
        tt = torch.tensor([tot_ms, float(evals), float(iters)], dtype=torch.float64, device="cuda")
        mx = tt.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(tt, op=dist.ReduceOp.SUM)
        t_max = mx[0].item()
        tot_evals = tt[1].item()
    value = tot_evals / (t_max / 1e3)

    # ---- end-to-end through the public API: init from host buffers, K steps
    #      each reading back its step info, evidence at the end ----
    torch.cuda.synchronize()
    e2e_steps = min(args.steps, lim)
    t0 = time.perf_counter()
    c = dict(cfg)
    c["seed"] = 10_000 + rank
    se = nss.Sampler(prob, c, stream=stream.cuda_stream)
    e_start = se.info()["energy_evals"]
    for _ in range(e2e_steps):
        info = se.step(sync=True)
    lz, lz_err = se.evidence()
    t_e2e = time.perf_counter() - t0
    e2e_evals = info["energy_evals"] - e_start
    se.close()
    e2e_value = e2e_evals / t_e2e * world
    s.close()

    if rank == 0:
        peaks = read_peaks()
        mhz = peaks.get("sm_max_mhz", 1965.0)
        peak = N_SM * FP32_LANES * 2 * mhz * 1e6 / 1e12
        achieved = (alg_flops / max(hrss_n, 1)) / ((hrss_ms / max(hrss_n, 1)) / 1e3) / 1e12 if hrss_n else 0.0
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, workloads.py)",
            "config": {"workload": f"{args.config} {prob.name}", "n_live": cfg["n_live"], "k": cfg["k"],
                       "steps_hrss": cfg["steps"], "d": prob.d, "parallelism": f"replicas x{world}",
                       "l2": "flushed between timed iterations (256 MiB write)",
                       "runs": f"new seed every {lim} iterations (outside the timed region)"},
            "iterations_per_s": iters * world / (t_max / 1e3),
            "probes_per_s": probes * world / (t_max / 1e3),
            "gpu_launches": launches,
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": None,
                         "kernel": "k_hrss (warp-per-chain HRSS + fused energy)",
                         "kernel_ms_avg": hrss_ms / max(hrss_n, 1),
                         "kernel_share_of_step": hrss_ms / max(tot_ms, 1e-9),
                         "peak_source": f"148 SM x 128 FP32 lanes x 2 x {mhz:.0f} MHz (derived, B200_PROFILING.md)"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": problem_bytes(prob) / e2e_steps,
                    "d2h_bytes_per_step": 96 + 8 * (cfg["n_volume_sims"] + 3) / e2e_steps,
                    "what": "nss_init from host buffers + K x nss_step(info) + nss_evidence, wall clock",
                    "log_z": lz, "log_z_err": lz_err},
        }
        if clocks:
            line["clocks"] = clocks
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args.config)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
