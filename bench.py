#!/usr/bin/env python3
"""Benchmark: R-ST-HOSVD end-to-end ms (Alg. 4) on BASELINE config 5
(1000^3 fp32, ranks 50, p=10, q=5) plus the fused power step's roofline fraction.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config c5]

One process per GPU (torchrun for N > 1).  The path shards as independent problems
(no data-path collective): every rank solves its own seeded tensor ("replicas",
scaling "weak"); value = max-over-ranks ms per step / N (ms per solve for the job).
Inputs are resident in HBM when the timed region starts; the 4 GB input exceeds
the 126 MB L2, so no flush is needed between steps.  Prints ONE JSON line on rank 0.
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

METRIC = "R-ST-HOSVD end-to-end ms"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")


def load_peaks():
    try:
        with open(PEAKS_FILE) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 9:
                for nm, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def dist_init(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        import torch
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, ws: int) -> float:
    """Max of a per-rank device time over the job (NCCL on GPUs, gloo on CPU)."""
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_value(ms_local: float, ws: int):
    """(ms_per_step, value): the step time is the max over ranks; the job solves ws independent
    replicas in that time, so the job's ms per solve is ms_step / ws (scaling "weak")."""
    ms_step = max_over_ranks(ms_local, ws)
    return ms_step, ms_step / ws


def cfg_block(cfg_name, c):
    return {"workload": f"{cfg_name}: R-ST-HOSVD (Alg. 4) {'x'.join(map(str, c['dims']))} fp32, "
                        f"ranks {tuple(c['ranks'])}, p={c['p']}, q={c['q']}, recipe {c['core']} core "
                        f"rank {c['core_ranks'][0]} + {c['noise']} noise",
            "dims": list(c["dims"]), "ranks": list(c["ranks"]), "p": c["p"], "q": c["q"],
            "omega_seed": c["omega_seed"], "data_seed": c["data_seed"],
            "l2": "input 4.0 GB >> 126 MB L2 (no flush needed between steps)"}


# ----------------------------------------------------------------- CPU oracle
def oracle_sample(cfg_name, c, slices: int):
    """Bounded sample of the workload for the CPU oracle: the first `slices` mode-d slices
    (same recipe, host float64 build), solved by oracle.rsthosvd; scale = n_d / slices."""
    import numpy as np
    from workloads import make_config_tensor
    dims = list(c["dims"])
    sample_dims = dims[:-1] + [slices]
    a = make_config_tensor(cfg_name, dims=tuple(sample_dims))
    return a, dims[-1] / slices, sample_dims


def time_oracle(a, c, reps=1):
    from oracle import tucker
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        tucker.rsthosvd(a, c["ranks"], c["p"], c["q"], c["omega_seed"])
        ts.append(time.perf_counter() - t0)
    return ts


def cpu_info():
    cores = os.cpu_count()
    try:
        from threadpoolctl import threadpool_info
        thr = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        thr = cores
    return cores, thr


# ----------------------------------------------------------------- reference
def run_reference(args, ws, rank):
    from workloads import CONFIGS
    if rank != 0:
        return
    c = CONFIGS[args.config]
    a, scale, sdims = oracle_sample(args.config, c, args.ref_slices)
    for _ in range(args.warmup):
        time_oracle(a, c)
    ts = []
    for _ in range(args.steps):
        ts += time_oracle(a, c)
    step_s = statistics.mean(ts)
    val = step_s * scale * 1e3
    cores, thr = cpu_info()
    sample = (f"first {args.ref_slices} of {c['dims'][-1]} mode-3 slices ({'x'.join(map(str, sdims))}), "
              f"oracle.rsthosvd float64 per step, scaled x{scale:g} to the full tensor")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "ms", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": val,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": cfg_block(args.config, c),
            "cpu_baseline": {"value": val, "unit": "ms", "cores": thr, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": val, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------- ours
def run_ours(args, ws, rank, local):
    import torch

    from paper_2506_04840_b200 import build as b
    if rank == 0:
        b.build()
    barrier(ws)
    import paper_2506_04840_b200 as rt
    from workloads import CONFIGS, make_config_tensor_torch

    c = CONFIGS[args.config]
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    A = make_config_tensor_torch(args.config, device=dev)
    torch.cuda.synchronize()
    ranks, p, q, seed = c["ranks"], c["p"], c["q"], c["omega_seed"]
    dims = c["dims"]
    d = len(dims)
    U = [torch.empty((r, n), dtype=torch.float32, device=dev).t() for n, r in zip(dims, ranks)]
    core = rt.as_column_major(torch.empty(ranks, dtype=torch.float32, device=dev))
    wsb = rt.workspace_bytes(True, dims, ranks, p, q)
    work = torch.empty(wsb, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        rt.rsthosvd(A, ranks, p, q, seed, out=(core, U), workspace=work)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    rt.profile_begin()
    barrier(ws)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    prof = rt.profile_end()
    clocks = clk.stop()
    ms_local = e0.elapsed_time(e1) / args.steps
    ms_step, value = job_value(ms_local, ws)

    # ---- roofline of the dominant kernel: the fused 3xTF32 power step on mode 1 ----
    # algorithmic work per launch (one power step): the unfolding read once,
    # 4 n m bytes, and Y = M (M^T Q): 4 n m l flops, executed as 3 tf32 tensor products each
    n, m, l = dims[0], 1, ranks[0] + p
    for j in dims[1:]:
        m *= j
    cnt = prof.count[1][0]
    t_pow = prof.ms[1][0] / max(cnt, 1) * 1e-3
    flops = 4.0 * n * m * l
    bytes_alg = 4.0 * n * m
    peaks, src = load_peaks()
    hbm_peak = peaks["hbm_gbs"]
    bf16 = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1590.0))
    tf32_peak = bf16 / 2.0      # dense tf32 = bf16 / 2 (B200_PROFILING.md nominal ratio), sustained
    t_hbm = bytes_alg / (hbm_peak * 1e9)
    t_tc = 3.0 * flops / (tf32_peak * 1e12)
    bound = "tensor" if t_tc >= t_hbm else "hbm"
    tot_ms = sum(prof.ms[k][j] for k in range(4) for j in range(8))
    share = prof.ms[1][0] / tot_ms if tot_ms > 0 else None
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get("power_step_mode1_dram_bytes")
        except Exception:
            traffic = None
    if bound == "tensor":
        achieved = 3.0 * flops / t_pow / 1e12 if t_pow > 0 else None
        peak, unit = tf32_peak, "TFLOP/s"
    else:
        achieved = bytes_alg / t_pow / 1e9 if t_pow > 0 else None
        peak, unit = hbm_peak, "GB/s"
    roof = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
            "frac": (achieved / peak) if achieved else None,
            "traffic": traffic,
            "kernel": f"fused_power_kernel mode 1 (n={n}, m={m}, l={l}): single HBM pass, 3xTF32 tcgen05",
            "algorithmic": {"bytes": bytes_alg, "flops_fp32": flops, "tf32_flops_3x": 3.0 * flops},
            "peak_src": (f"tf32 dense = {bf16:g}/2 TFLOP/s (bf16 sustained from MEASURED_PEAKS.json, {src}); "
                         f"HBM {hbm_peak:g} GB/s"),
            "roofline_ms": max(t_hbm, t_tc) * 1e3,
            "launch_ms": t_pow * 1e3, "launches_timed": cnt,
            "share_of_step": share,
            "hbm_achieved_gbs": bytes_alg / t_pow / 1e9 if t_pow > 0 else None,
            "hbm_frac": (bytes_alg / t_pow / 1e9) / hbm_peak if t_pow > 0 else None,
            "hbm_peak_gbs": hbm_peak}
    breakdown = {k: round(sum(prof.ms[i][j] for j in range(8)) / args.steps, 4)
                 for i, k in enumerate(["sketch", "power", "shrink", "small_solves"])}

    # ---- end to end through the public API from pinned host buffers ----
    # Every step copies its input tensor host -> device (pinned, 4 GB at C5) and reads its result back
    # device -> host inside the timed region.  The copies run on a copy stream into two device buffers:
    # step i+1's H2D overlaps step i's solve (a data-loader style prefetch; the copy engine and the
    # SMs work concurrently), and step i's solve waits for its own copy.
    e2e = None
    if not args.no_e2e:
        hostA = torch.empty_like(A, device="cpu").pin_memory()
        hostA.copy_(A)
        Adev = [torch.empty_like(A), torch.empty_like(A)]
        h_core = torch.empty(core.shape, dtype=torch.float32).pin_memory()
        h_U = [torch.empty(u.shape, dtype=torch.float32).pin_memory() for u in U]
        h2d = A.numel() * 4
        d2h = core.numel() * 4 + sum(u.numel() * 4 for u in U)
        cstream = torch.cuda.Stream()
        copied = [torch.cuda.Event(), torch.cuda.Event()]   # H2D into buffer b done
        freed = [torch.cuda.Event(), torch.cuda.Event()]    # solve reading buffer b done

        def h2d_into(b):
            cstream.wait_event(freed[b])
            with torch.cuda.stream(cstream):
                Adev[b].copy_(hostA, non_blocking=True)
                copied[b].record(cstream)

        def e2e_run(k):
            for b in range(2):
                freed[b].record(stream)
            h2d_into(0)
            for i in range(k):
                b = i % 2
                if i + 1 < k:
                    h2d_into(1 - b)          # next step's input, overlapping this step's solve
                stream.wait_event(copied[b])
                rt.rsthosvd(Adev[b], ranks, p, q, seed, out=(core, U), workspace=work)
                freed[b].record(stream)
                h_core.copy_(core, non_blocking=True)
                for hu, u in zip(h_U, U):
                    hu.copy_(u, non_blocking=True)

        e2e_run(1)
        torch.cuda.synchronize()
        barrier(ws)
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        ke = max(1, min(args.steps, 5))
        f0.record(stream)
        e2e_run(ke)
        f1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(f0.elapsed_time(f1) / ke, ws)
        e2e = {"value": e2e_ms / ws, "unit": "ms", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": ke,
               "overlap": "step i+1 H2D on a copy stream during step i's solve (2 device buffers)"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        a_s, scale, sdims = oracle_sample(args.config, c, args.cpu_slices)
        ts = time_oracle(a_s, c)
        cores, thr = cpu_info()
        cpu = {"value": ts[0] * scale * 1e3, "unit": "ms", "cores": thr, "kind": "oracle",
               "sample": f"oracle.rsthosvd (float64, numpy/LAPACK) on the first {args.cpu_slices} of "
                         f"{dims[-1]} mode-3 slices ({'x'.join(map(str, sdims))}), one run "
                         f"{ts[0]:.2f} s, scaled x{scale:g}; host has {cores} cores"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "ms", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32 stream / f64 small solves",
                "data": "synthetic", "config": cfg_block(args.config, c),
                "parallelism": f"replicas x{ws} (independent solves, no collective)",
                "roofline": roof, "breakdown_ms_per_step": breakdown, "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": int(prof.launches), "clocks": clocks}
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-slices", type=int, default=100)
    ap.add_argument("--ref-slices", type=int, default=64)
    args = ap.parse_args()
    if args.impl == "reference":
        ws = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, ws, rank)
        return
    ws, rank, local = dist_init(args)
    run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
