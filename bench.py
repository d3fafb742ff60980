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
def host_tensor(cfg_name):
    """The benchmarked tensor itself, on the host: make_config_tensor_torch (seeded, built on the
    GPU when there is one, else on the CPU), copied to a Fortran-ordered float32 numpy array."""
    import torch
    from workloads import make_config_tensor_torch
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    A = make_config_tensor_torch(cfg_name, device=dev)
    a = A.cpu().numpy()
    del A
    if dev == "cuda":
        torch.cuda.empty_cache()
    return a


def time_oracle(a, c):
    """One full oracle.rsthosvd solve (float64, numpy/LAPACK) of the whole tensor; seconds."""
    from oracle import tucker
    t0 = time.perf_counter()
    tucker.rsthosvd(a, c["ranks"], c["p"], c["q"], c["omega_seed"])
    return time.perf_counter() - t0


def cpu_info():
    cores = os.cpu_count()
    try:
        from threadpoolctl import threadpool_info
        thr = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        thr = cores
    return cores, thr


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------- reference
def run_reference(args, ws, rank):
    """The reference arm is the float64 CPU oracle (the paper ships no code), timed on
    the full benchmarked tensor, no extrapolation: min(W, 1) warm-up solve, then up to K timed
    solves, stopping early once --ref-budget seconds are spent (>= 1 timed solve); `steps` reports
    the solves actually timed, so value x steps is the time this arm really ran."""
    from workloads import CONFIGS
    if rank != 0:
        return
    c = CONFIGS[args.config]
    a = host_tensor(args.config)
    for _ in range(min(args.warmup, 1)):
        time_oracle(a, c)
    ts = []
    t_start = time.perf_counter()
    for _ in range(max(args.steps, 1)):
        ts.append(time_oracle(a, c))
        if time.perf_counter() - t_start > args.ref_budget:
            break
    val = statistics.mean(ts) * 1e3
    cores, thr = cpu_info()
    sample = (f"oracle.rsthosvd float64 (numpy/LAPACK) on the full {'x'.join(map(str, c['dims']))} tensor "
              f"(the benchmarked tensor, host copy), mean of {len(ts)} timed solve(s) after "
              f"{min(args.warmup, 1)} warm-up; {thr} BLAS threads on {cores} cores ({cpu_model()})")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "ms", "n_gpus": args.gpus,
            "steps": len(ts), "steps_requested": args.steps, "warmup": min(args.warmup, 1),
            "ms_per_step": val,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": cfg_block(args.config, c),
            "cpu_baseline": {"value": val, "unit": "ms", "cores": thr, "kind": "oracle",
                             "sample": sample, "runs_s": [round(t, 3) for t in ts]},
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
    # headline: profiling OFF (no per-launch events inside the programmatic-dependent-launch chain)
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
    clocks = clk.stop()
    ms_local = e0.elapsed_time(e1) / args.steps
    ms_step, value = job_value(ms_local, ws)

    # separate profiled pass (same K steps): per-kernel device times for the roofline and the
    # breakdown; CUDA events on the launching stream around every library launch
    clk2 = ClockSampler(local)
    clk2.start()
    rt.profile_begin()
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(args.steps):
        step()
    p1.record(stream)
    torch.cuda.synchronize()
    prof = rt.profile_end()
    clocks_prof = clk2.stop()
    ms_prof = p0.elapsed_time(p1) / args.steps
    launches_per_step = int(prof.launches) / max(args.steps, 1)

    # ---- roofline of the dominant kernel: the fused power step on mode 1 ----
    # algorithmic work per launch (one power step): the unfolding read once,
    # 4 n m bytes, and Y = M (M^T Q): 4 n m l flops, executed as 3 tensor products each: fp16
    # two-plane operands on the pair engine (kind::f16 runs at the bf16 rate), or
    # 3xTF32 when RTK_PAIR_F16=0
    n, m, l = dims[0], 1, ranks[0] + p
    for j in dims[1:]:
        m *= j
    cnt = prof.count[1][0]
    t_pow = prof.ms[1][0] / max(cnt, 1) * 1e-3
    flops = 4.0 * n * m * l
    bytes_alg = 4.0 * n * m
    peaks, src = load_peaks()
    hbm_peak = peaks["hbm_gbs"]
    bf16_burst = peaks.get("bf16_tflops", 1590.0)
    bf16_sus = peaks.get("bf16_tflops_sustained", bf16_burst)
    # dense fp16 = bf16, dense tf32 = bf16 / 2 (B200_PROFILING.md nominal ratios).  The kernel is
    # timed alone-ish at full clocks inside a sub-second region, so the BURST figure is the
    # denominator; the sustained one is reported beside it
    f16 = os.environ.get("RTK_PAIR_F16", "1") != "0"
    tf32_peak = bf16_burst / (1.0 if f16 else 2.0)
    tf32_sus = bf16_sus / (1.0 if f16 else 2.0)
    prec = "3xFP16" if f16 else "3xTF32"
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
            "kernel": (f"pair_power_kernel mode 1 (n={n}, m={m}, l={l}): single HBM pass on a CTA pair, "
                       f"{prec} tcgen05"),
            "algorithmic": {"bytes": bytes_alg, "flops_fp32": flops, "tensor_flops_3x": 3.0 * flops},
            "peak_src": ((f"fp16 dense = bf16 burst {bf16_burst:g}" if f16 else f"tf32 dense = bf16 burst {bf16_burst:g}/2")
                         + f" TFLOP/s (MEASURED_PEAKS.json, {src}); HBM {hbm_peak:g} GB/s (MEASURED_PEAKS.json)"),
            "tensor_frac": (3.0 * flops / t_pow / 1e12) / tf32_peak if t_pow > 0 else None,
            "tensor_frac_vs_sustained": (3.0 * flops / t_pow / 1e12) / tf32_sus if t_pow > 0 else None,
            "sustained_tensor_peak": tf32_sus,
            "roofline_ms": max(t_hbm, t_tc) * 1e3,
            "launch_ms": t_pow * 1e3, "launches_timed": cnt,
            "timed_in": "separate profiled pass (CUDA events around each launch on its stream)",
            "share_of_step": share,
            "hbm_achieved_gbs": bytes_alg / t_pow / 1e9 if t_pow > 0 else None,
            "hbm_frac": (bytes_alg / t_pow / 1e9) / hbm_peak if t_pow > 0 else None,
            "hbm_frac_8tbs": (bytes_alg / t_pow / 1e9) / 8000.0 if t_pow > 0 else None,
            "hbm_peak_gbs": hbm_peak, "clocks_profiled_pass": clocks_prof,
            "ms_per_step_profiled": ms_prof}
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
        # the oracle on the full benchmarked tensor (its host copy), one solve, no extrapolation
        a_host = A.cpu().numpy()
        t_or = time_oracle(a_host, c)
        del a_host
        cores, thr = cpu_info()
        cpu = {"value": t_or * 1e3, "unit": "ms", "cores": thr, "kind": "oracle",
               "sample": f"oracle.rsthosvd (float64, numpy/LAPACK) on the full {'x'.join(map(str, dims))} "
                         f"benchmarked tensor (host copy of the same bytes), one solve; {thr} BLAS threads, "
                         f"{cores} cores ({cpu_model()})"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "ms", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32 stream (3xFP16 / 3xTF32 split products) / f64 small solves",
                "data": "synthetic", "config": cfg_block(args.config, c),
                "parallelism": f"replicas x{ws} (independent solves, no collective)",
                "roofline": roof, "breakdown_ms_per_step": breakdown, "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": int(round(launches_per_step * args.steps)),
                "gpu_launches_per_step": launches_per_step, "clocks": clocks}
        print(json.dumps(line), flush=True)


def run_shard(args, ws, rank, local):
    """--shard: ONE C5 solve per step with A split along its last mode over the ws ranks
    (rtk_rsthosvd_shard): each GPU holds and streams 1/ws of the tensor, an NCCL
    all-reduce sums the n_k x l panel Y after every streaming pass, the small solves and mode d run
    redundantly.  Strong scaling: value = max-over-ranks ms per (whole-problem) solve."""
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
    dims = list(c["dims"])
    begin, count = rt.shard_bounds(dims[-1], ws, rank)
    A = make_config_tensor_torch(args.config, device=dev)
    S = rt.as_column_major(A[..., begin:begin + count])
    del A
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    ranks, p, q, seed = c["ranks"], c["p"], c["q"], c["omega_seed"]
    if ws > 1:
        import torch.distributed as dist

        def allreduce(t):
            dist.all_reduce(t)
    else:
        def allreduce(t):
            return None
    U = [torch.empty((r, n), dtype=torch.float32, device=dev).t() for n, r in zip(dims, ranks)]
    core = rt.as_column_major(torch.empty(ranks, dtype=torch.float32, device=dev))

    def step():
        rt.rsthosvd_shard(S, dims, begin, ranks, p, q, seed, allreduce=allreduce, root=rank == 0, out=(core, U))

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    stream = torch.cuda.current_stream(dev)
    barrier(ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    clocks = clk.stop()
    ms_step = max_over_ranks(e0.elapsed_time(e1) / args.steps, ws)
    if rank == 0:
        line = {"metric": METRIC, "value": ms_step, "unit": "ms", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32 stream (3xFP16 / 3xTF32 split products) / f64 small solves",
                "data": "synthetic", "config": cfg_block(args.config, c),
                "parallelism": f"last-mode shard x{ws}: n_{len(dims)} = {dims[-1]} split into slabs of "
                               f"{dims[-1] // ws}-{-(-dims[-1] // ws)} per GPU, one n_k x l fp64 all-reduce per "
                               "streaming pass (NCCL), mode d redundant",
                "roofline": None, "cpu_baseline": None, "e2e": None, "clocks": clocks}
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
    ap.add_argument("--shard", action="store_true",
                    help="one solve per step with A split along its last mode over the GPUs (strong scaling)")
    ap.add_argument("--ref-budget", type=float, default=150.0,
                    help="reference arm: stop timing further oracle solves after this many seconds")
    args = ap.parse_args()
    if args.impl == "reference":
        ws = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, ws, rank)
        return
    ws, rank, local = dist_init(args)
    if args.shard:
        run_shard(args, ws, rank, local)
    else:
        run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
