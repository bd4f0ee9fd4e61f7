#!/usr/bin/env python
"""Benchmark: batched OMP signals/s on B200 (BASELINE.json metric), one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--mode bf16] [--impl ours|reference]

A "step" is one ompBatch over the whole per-rank batch: S iterations of correlation screen,
exact selection, factor append and residual on device-resident inputs.
Multi-GPU (torchrun): the global batch of the config is sharded contiguously across ranks
(BASELINE.json configs[3]: "B=100,000 batch-sharded across 1/2/4/8 B200"); A is generated on
rank 0 and broadcast once over NCCL; there is no per-iteration collective.  Step time is the
max over ranks of CUDA-event time (barrier + synchronize on both sides).

`--impl reference` times the FP64 CPU oracle (the only reference this paper-tier run has) on a
bounded sample of the same workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "OMP signals/sec"
# the paper's own GPU numbers for the exact workload shapes it published (BASELINE.md §1a, App. B
# Table 2 rows 9-10: best of its naive / v0 GPU times, B = 100, other hardware): vs_baseline
PAPER_SIGNALS_PER_S = {"t2m1024": 100 / 0.546, "t2m2048": 100 / 4.392}
UNIT = "signals/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="c4")
    p.add_argument("--batch", type=int, default=None, help="override the config's global batch")
    p.add_argument("--mode", default="bf16", choices=["bf16", "3xtf32", "simt"])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--e2e-steps", type=int, default=2)
    p.add_argument("--oracle-sample", type=int, default=None, help="signals in the CPU oracle sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--dist-backend", default="nccl", help="nccl (default); gloo only for single-GPU testing")
    p.add_argument("--algo", default="auto", choices=["auto", "residual", "projection"],
                   help="iteration formulation (ompSetAlgorithm); auto = the library's cost model")
    p.add_argument("--small-limit", type=int, default=-1,
                   help="small-batch persistent-kernel limit (-1 library default, 0 never)")
    p.add_argument("--no-kernel-profile", action="store_true",
                   help="time the steps through the CUDA-graph path without per-kernel events; the kernel "
                        "split then comes from one extra profiled step (small-batch latency runs)")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        return self.summary()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower() == "active"})
        busy = [v for v in sm if v > 0.5 * (max(mx) if mx else 0)] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


def tensor_peak(peaks, mode):
    """Dense tensor peak for the screen's dtype.  The BURST figure: the screen runs in ~2 ms bursts
    between L2-bound update launches that draw far less power, so the sustained (4 s of back-to-back
    GEMMs) figure understates what it can reach inside the step (measured above it, r01e/r01h)."""
    base = (peaks or {}).get("bf16_tflops", 1650.0)
    src = "MEASURED_PEAKS bf16_tflops (burst)" if peaks else "fallback 1.65 PF"
    if mode == "bf16":
        return base, src
    if mode == "3xtf32":
        return base / 2.0 / 3.0, src + " x nominal tf32/bf16 ratio 1/2, /3 for the three products"
    return 74.4, "FP32 SIMT 148 SM x 128 lanes x 2 x 1.965 GHz"


def l2_peak():
    """Measured L2 gather bandwidth of this GPU model (scripts/l2_probe.cu, committed result)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "l2_probe_b200.json")))
        return float(d["l2_gather_sustained_gbs"]), "profiles/l2_probe_b200.json l2_gather_sustained_gbs"
    except Exception:
        return 20500.0, "fallback 20.5 TB/s (scripts/l2_probe.cu on B200)"


def ncu_traffic(kernel_key: str, config_name: str):
    """dram bytes per launch of the dominant kernel from the committed ncu --set full summary."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        return d["configs"][config_name][kernel_key]["dram_bytes_per_launch"]
    except Exception:
        return None


# ------------------------------------------------------------------------------ roofline model
def kernel_work(cfg, B, mode, path="residual", n_iter=None):
    """Algorithmic work per launch (SURVEY §8(d) per signal-iteration; DESIGN.md §6 states each figure),
    summed over the signals each launch actually processes: with n_iter (iterations each signal ran,
    from the step's own result) the launch at iteration k covers the live[k] = #{b : n_iter_b > k}
    signals at support size k (eps stops, live-set compaction); the per-launch figure is the mean
    over the S launches.  Without n_iter: all B signals for all S iterations."""
    import numpy as np
    M, N, S = cfg["M"], cfg["N"], cfg["S"]
    Mp = -(-M // 64) * 64
    ks = np.arange(S, dtype=np.float64)
    if n_iter is None:
        live = np.full(S, float(B))
    else:
        ni = np.asarray(n_iter).reshape(-1)
        live = np.array([(ni > k).sum() for k in range(S)], dtype=np.float64)
    per_launch = lambda f: float((live * f).sum() / S)   # noqa: E731  (f: per signal at iteration k)
    if path == "projection":
        Np = -(-N // 256) * 256
        # update: argmax over the p row, append, p = P0 - sum_j x_j G[s_j, :] (k+1 Gram rows from L2)
        hbm = per_launch(4.0 * Np * 3 + 4.0 * ks * (ks + 1) / 2 + 4.0 * (ks + 2) * 3)   # p read + P0 read + p write, F
        l2 = per_launch(4.0 * Np * (ks + 1))
        p0_simt = os.environ.get("OMP_B200_P0", "") == "simt"
        return {
            # P0 = A^T Y once per batch: 2 M N flops per signal (3xTF32 split-K on the tensor cores, or
            # the FP32 FFMA GEMM with OMP_B200_P0=simt)
            "correlation": ("alu" if p0_simt else "tensor3", 2.0 * M * N * B, "TFLOP/s", None),
            "update": ("l2", hbm + l2, "GB/s", {"hbm_bytes": hbm, "l2_gather_bytes": l2}),
            "init": ("hbm", B * 4.0 * (2 * M + Mp), "GB/s", None),
        }
    groups = 2 * math.ceil(N / 256)                # 128-atom screen groups (Np / 128)
    planes = {"bf16": 2.0, "3xtf32": 8.0, "simt": 0.0}[mode]
    # update = exact selection + factor append + residual, split into streamed (HBM) and gathered (L2)
    hbm = per_launch(4.0 * Mp                      # fp32 residual row read by the selection
                     + 8.0 * 4 * groups            # screen partials: TOPK = 4 float2 per group
                     + 4.0 * ks * (ks + 1) / 2     # packed F_k staged once
                     + 4.0 * (ks + 2) * 3          # new F column, x, u
                     + 4.0 * M                     # y
                     + (4.0 + planes) * Mp)        # residual written: fp32 + screen planes
    l2 = per_launch(4.0 * Mp * (ks + 1 + 1))       # (k+1) gathered atom rows + ~1 candidate row
    k = (S - 1) / 2.0
    return {
        # screen GEMM: 2 M N flops per live signal-iteration (the contraction C = A^T R)
        "correlation": ("tensor", per_launch(2.0 * M * N + 0 * ks), "TFLOP/s", None),
        # standalone argmax over the FP32 C (SIMT mode): 4N bytes per signal
        "select": ("hbm", per_launch(4.0 * N + 0 * ks), "GB/s", None),
        "update": ("l2", hbm + l2, "GB/s", {"hbm_bytes": hbm, "l2_gather_bytes": l2}),
        "init": ("hbm", B * (4.0 * M + (4.0 + planes) * Mp), "GB/s", None),
        # small-batch persistent kernel, all S iterations: per iteration the atom table once (phase A,
        # exact correlation over all N atoms) + the per-signal append/residual bytes (L2-resident)
        "small": ("l2", S * (4.0 * N * Mp + B * (4.0 * Mp * (k + 3) + 4.0 * k * (k + 1) / 2 + 4.0 * M)), "GB/s",
                  {"hbm_bytes": B * 4.0 * (M + S + S * (S + 1) / 2), "l2_gather_bytes": S * (4.0 * N * Mp + B * 4.0 * Mp * (k + 3))}),
    }


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, world, rank)
    import torch
    import torch.distributed as dist
    from synth import config, make_dictionary, make_signals
    from paper_2407_06434_b200 import OMP

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (there is no CPU fallback)")
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if world > 1:
        # NCCL's init log on stderr shows the ranks and the transports it picked (NVLink / NVLS)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
    cfg = config(args.config)
    B_total = args.batch or cfg["B"]
    per = -(-B_total // world)
    lo, hi = rank * per, min(B_total, (rank + 1) * per)
    B = max(0, hi - lo)
    M, N, S, eps = cfg["M"], cfg["N"], cfg["S"], cfg["eps"]
    eps32 = None if eps is None else float(np.float32(eps))
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    comm = dev if args.dist_backend == "nccl" else torch.device("cpu")

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=comm)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # inputs: A and the whole batch on rank 0 (device-resident); with N > 1 the library's distributed
    # driver broadcasts A once and, every step, scatters Y's slices from rank 0 and gathers the results
    # back to it (the timed span runs from the scatter to the gather)
    A_np = make_dictionary(M, N, cfg["seed"])
    Y_np = None
    if rank == 0:
        Y_np = make_signals(A_np, range(B_total), cfg["seed"], cfg["sparsity"], cfg["sigma"], device=dev)
    Y = torch.from_numpy(Y_np).to(dev) if rank == 0 else None

    # ompCreate (validation, norms, screen planes, Gram G = A^T A) timed on its own;
    # with N > 1 this includes the broadcast of A over NCCL (max over ranks)
    barrier()
    torch.cuda.synchronize()
    t_setup = time.perf_counter()
    if world > 1:
        from paper_2407_06434_b200.distributed import DistributedOMP
        dist_omp = DistributedOMP(torch.from_numpy(A_np).to(dev) if rank == 0 else None, mode=args.mode,
                                  device=dev)
        h = dist_omp.handle
        A = dist_omp.A.to(dev)
        solve = lambda: dist_omp.batch(Y, S, eps32)          # noqa: E731  (None on ranks != 0)
    else:
        dist_omp = None
        A = torch.from_numpy(A_np).to(dev)
        h = OMP(A, mode=args.mode)
        solve = lambda: h.batch(Y, S, eps32)                 # noqa: E731
    torch.cuda.synchronize()
    setup_ms = max_over_ranks((time.perf_counter() - t_setup) * 1e3)
    if args.small_limit != -1:
        h.set_small_batch_limit(args.small_limit)
    if args.algo != "auto":
        h.set_algorithm(args.algo)

    # warm-up (untimed)
    for _ in range(args.warmup):
        res = solve()
    torch.cuda.synchronize()
    barrier()

    # timed region: the graph path the library runs by default; with kernel profiling (default) the
    # captured graph carries an event-record node at every kernel boundary, so each kernel's time is
    # measured live inside the timed steps, on the library's launch stream
    h.profile(not args.no_kernel_profile)
    h.profile_read(reset=True)
    props = torch.cuda.get_device_properties(dev)
    clocks = ClockSampler(f"{props.pci_domain_id:08X}:{props.pci_bus_id:02X}:{props.pci_device_id:02X}.0")
    clocks.start()
    step_ms = []
    launches = 0
    # inputs smaller than 2x L2 (126 MB): flush L2 between timed steps by writing 256 MB
    y_bytes = B * M * 4
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev) if y_bytes < (252 << 20) else None
    for _ in range(args.steps):
        if flush is not None:
            flush.zero_()
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = solve()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        step_ms.append(max_over_ranks(e0.elapsed_time(e1)))
        launches += h.launch_count()
        h.profile_read(reset=False)      # per-kernel event pairs of this step
    clk = clocks.stop()
    kern = h.profile_read(reset=True)
    if args.no_kernel_profile:           # kernel split from one extra, profiled step
        h.profile(True)
        solve()
        torch.cuda.synchronize()
        kern = h.profile_read(reset=True)
    h.profile(False)
    ms = statistics.mean(step_ms)
    value = B_total / (ms / 1e3)
    if world > 1:
        # every rank's own launches; the line reports the sum over ranks
        t = torch.tensor([launches], dtype=torch.float64, device=comm)
        dist.all_reduce(t)
        launches = int(t.item())

    # end to end through the public API: pinned host Y in, host results out, every step.  N = 1:
    # ompBatchHost (copies inside the library call); N > 1: the distributed driver on rank 0's pinned
    # host batch (H2D to rank 0, scatter, solve, gather, D2H of the gathered results)
    e2e = None
    if not args.no_e2e and B > 0:
        outs = (torch.empty((B_total, S), dtype=torch.float32).pin_memory(),
                torch.empty((B_total, S), dtype=torch.int32).pin_memory(),
                torch.empty((B_total,), dtype=torch.float32).pin_memory(),
                torch.empty((B_total,), dtype=torch.int32).pin_memory(),
                torch.empty((B_total,), dtype=torch.int32).pin_memory()) if rank == 0 else None
        Yh = torch.from_numpy(Y_np).pin_memory() if rank == 0 else None

        def e2e_step():
            if world == 1:
                h.batch_host(Yh.numpy(), S, eps32, out=tuple(o.numpy() for o in outs))
                return
            r = dist_omp.batch(Yh.to(dev, non_blocking=True) if rank == 0 else None, S, eps32)
            if rank == 0:
                for o, f in zip(outs, ("X", "support", "resid_norm", "n_iter", "status")):
                    o.copy_(getattr(r, f), non_blocking=True)

        e2e_step()                       # warm the staging buffers
        torch.cuda.synchronize()
        e2e_ms = []
        for _ in range(args.e2e_steps):
            barrier()
            torch.cuda.synchronize()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            e2e_step()
            t1.record(stream)
            torch.cuda.synchronize()
            barrier()
            e2e_ms.append(max_over_ranks(t0.elapsed_time(t1)))
        e2e = {"value": B_total / (statistics.mean(e2e_ms) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(B_total * M * 4),
               "d2h_bytes_per_step": int(B_total * (8 * S + 12))}

    # roofline of the dominant kernel (events measured live over the timed steps, this rank)
    path = h.last_path()
    n_iter_here = None
    if B > 0:
        if world == 1:
            n_iter_here = res.n_iter.cpu().numpy()
        else:
            # this rank's slice of the gathered result is on rank 0 only: count its iterations from its
            # own per-launch live counts instead (every rank runs the same S launches)
            n_iter_here = rank_n_iter(dist_omp, res, rank, world, B_total, comm)
    work = kernel_work(cfg, B, args.mode, path, n_iter_here)
    dom = max((k for k in kern if k in work), key=lambda k: kern[k][0])
    bound, per_launch, unit, split = work[dom]
    peak_mode = args.mode
    if bound == "tensor3":                 # the projection path's P0: 3xTF32 whatever the screen mode
        bound, peak_mode = "tensor", "3xtf32"
    t_launch = kern[dom][0] / max(1, kern[dom][1]) / 1e3
    peaks = measured_peaks()
    if bound == "tensor":
        achieved = per_launch / t_launch / 1e12
        peak, peak_src = tensor_peak(peaks, peak_mode)
    elif bound == "alu":
        # FP32 FFMA peak: 148 SMs x 128 lanes x 2 flops x 1.965 GHz (guide unit counts and max clock)
        achieved = per_launch / t_launch / 1e12
        peak, peak_src = 74.4, "FP32 FFMA: 148 SM x 128 lanes x 2 x 1.965 GHz (DESIGN.md §6)"
    elif bound == "l2":
        # the update kernel's bytes all pass through L2 (the atom-row gather hits it; the streamed rows
        # come from HBM through it): its roof is the L2 read bandwidth measured on a B200 by
        # scripts/l2_probe.cu with the kernel's own access pattern (profiles/l2_probe_b200.json)
        achieved = per_launch / t_launch / 1e9
        peak, peak_src = l2_peak()
        roofline_extra = {"hbm_bytes": split["hbm_bytes"], "l2_gather_bytes": split["l2_gather_bytes"],
                          "hbm_floor_ms": split["hbm_bytes"] / ((peaks or {}).get("hbm_gbs", 6650.0) * 1e6),
                          "l2_floor_ms": per_launch / (peak * 1e6)}
    else:
        achieved = per_launch / t_launch / 1e9
        peak = (peaks or {}).get("hbm_gbs", 6650.0)
        peak_src = "MEASURED_PEAKS hbm_gbs" if peaks else "fallback 6.65 TB/s"
    roofline = {"bound": bound, "kernel": dom, "achieved": achieved, "peak": peak, "unit": unit,
                "frac": achieved / peak, "traffic": ncu_traffic(dom, args.config), "peak_source": peak_src,
                "work_per_launch": per_launch, "launch_ms": t_launch * 1e3}
    if bound == "l2":
        roofline.update(roofline_extra)
    # the measured peaks were taken at ~1.96 GHz; a long bench step runs power-capped (clocks.sm_mhz):
    # the same fraction against the peak scaled to the clock the step actually ran at (context)
    if bound in ("l2", "alu") and clk.get("sm_mhz") and clk.get("sm_max_mhz"):
        roofline["frac_at_bench_clock"] = roofline["frac"] * clk["sm_max_mhz"] / clk["sm_mhz"]
    other = {k: kern[k] for k in kern if k in work and k != dom and kern[k][1] > 0}
    roofline["others"] = {}
    for k, (tot_ms, n_l) in other.items():
        b2, w2, u2, _ = work[k]
        pm2 = args.mode
        if b2 == "tensor3":
            b2, pm2 = "tensor", "3xtf32"
        t2 = tot_ms / n_l / 1e3
        if b2 in ("tensor", "alu"):
            tp, tsrc = (74.4, "FP32 FFMA") if b2 == "alu" else tensor_peak(peaks, pm2)
            roofline["others"][k] = {"bound": b2, "achieved_tflops": w2 / t2 / 1e12, "launch_ms": t2 * 1e3,
                                     "frac": w2 / t2 / 1e12 / tp, "peak": tp, "peak_source": tsrc}
            if b2 == "tensor" and peaks and peaks.get("bf16_tflops_sustained"):
                sus = tp * peaks["bf16_tflops_sustained"] / peaks.get("bf16_tflops", tp)
                roofline["others"][k]["frac_vs_sustained"] = w2 / t2 / 1e12 / sus
        else:
            bp = l2_peak()[0] if b2 == "l2" else (peaks or {}).get("hbm_gbs", 6650.0)
            roofline["others"][k] = {"bound": b2, "achieved_gbs": w2 / t2 / 1e9, "launch_ms": t2 * 1e3,
                                     "frac": w2 / t2 / 1e9 / bp}
    kernels = {k: {"ms_total": v[0], "launches": v[1], "share": v[0] / max(1e-9, sum(x[0] for x in kern.values()))}
               for k, v in kern.items()}

    # CPU baseline: the oracle on a bounded sample (rank 0, N = 1) + parity of that sample
    cpu = None
    parity_rep = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, parity_rep = cpu_baseline(args, cfg, A_np, Y_np, res, lo)
    elif rank == 0 and world > 1 and not args.no_cpu_baseline:
        # parity of the gathered multi-GPU result on the shard boundaries (no oracle timing at N > 1)
        parity_rep = shard_parity(cfg, A_np, Y_np, res, world)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": (value / PAPER_SIGNALS_PER_S[args.config]) if args.config in PAPER_SIGNALS_PER_S else None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.config}: M={M} N={N} S={S} B={B_total}"
                                   + (f" sigma={cfg['sigma']} eps={eps:.4g}" if eps else " noiseless"),
                       "M": M, "N": N, "S": S, "global_batch": B_total, "per_gpu_batch": per,
                       "mode": args.mode, "screen_dtype": {"bf16": "bf16", "3xtf32": "tf32x3", "simt": "none"}[args.mode],
                       "l2": ("L2 flushed between timed steps (256 MB write; Y %.1f MB/rank)" if flush is not None
                              else "inputs larger than L2 (Y %.0f MB/rank)") % (y_bytes / 1e6),
                       "path": path,
                       "parallelism": f"batch-shard x{world}",
                       "collectives": ("none" if world == 1 else
                                       f"{args.dist_backend.upper()}: A broadcast once (setup); per step scatter Y from rank 0, "
                                       "gather the packed results to rank 0 (inside the timed span)")},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
            "kernels": kernels,
            "setup_ms": setup_ms,
        }
        if parity_rep is not None:
            line["parity"] = parity_rep
        print(json.dumps(line), flush=True)
    if dist_omp is not None:
        dist_omp.close()
    else:
        h.close()
    if world > 1:
        dist.destroy_process_group()


def rank_n_iter(dist_omp, res, rank, world, B_total, comm):
    """Iterations each signal of this rank's slice ran: rank 0 has the gathered result and scatters
    the slices' n_iter back (outside the timed region)."""
    import torch
    import torch.distributed as dist
    from paper_2407_06434_b200.distributed import shard_bounds
    per = -(-B_total // world)
    mine = torch.zeros(per, dtype=torch.int32, device=comm)
    chunks = None
    if rank == 0:
        ni = res.n_iter.to(comm)
        chunks = []
        for r in range(world):
            a, b, _ = shard_bounds(B_total, world, r)
            c = torch.zeros(per, dtype=torch.int32, device=comm)
            c[: b - a] = ni[a:b]
            chunks.append(c)
    dist.scatter(mine, chunks, src=0)
    lo, hi, _ = shard_bounds(B_total, world, rank)
    return mine[: hi - lo].cpu().numpy()


def shard_parity(cfg, A_np, Y_np, res, world):
    """Oracle parity of the gathered result at the ends of every rank's slice (8 signals each)."""
    from oracle import host_cores, omp_batch as oracle_batch
    from paper_2407_06434_b200.distributed import shard_bounds
    from parity import compare_batch
    B = len(Y_np)
    rows = sorted({b for r in range(world) for (lo, hi, _) in [shard_bounds(B, world, r)]
                   for b in list(range(lo, min(hi, lo + 4))) + list(range(max(lo, hi - 4), hi))})
    eps32 = None if cfg["eps"] is None else float(np.float32(cfg["eps"]))
    ora = oracle_batch(A_np, Y_np[rows], cfg["S"], eps32, workers=host_cores())
    rep = compare_batch(res.support.cpu().numpy(), res.X.cpu().numpy(), res.resid_norm.cpu().numpy(),
                        res.n_iter.cpu().numpy(), res.status.cpu().numpy(), ora, A_np.shape[1], rows=rows)
    return rep.as_dict()


def oracle_sample_size(args, cfg, cores):
    if args.oracle_sample:
        return args.oracle_sample
    per_signal_s = {"tiny": 3e-4, "c2": 0.012, "c3": 0.25, "c4": 3.4, "c5": 0.06}.get(cfg["name"], 1.0)
    target = 20.0   # ~20 s of wall time on `cores` workers
    return int(max(cores, min(4096, round(target * cores / per_signal_s))))


def cpu_baseline(args, cfg, A_np, Y_np, res, lo):
    from oracle import host_cores, omp_batch as oracle_batch
    from parity import compare_batch
    cores = host_cores()
    n = min(len(Y_np), oracle_sample_size(args, cfg, cores))
    rows = np.unique(np.linspace(0, len(Y_np) - 1, n).astype(int))
    eps32 = None if cfg["eps"] is None else float(np.float32(cfg["eps"]))
    t0 = time.perf_counter()
    ora = oracle_batch(A_np, Y_np[rows], cfg["S"], eps32, workers=cores)
    wall = time.perf_counter() - t0
    cpu = {"value": len(rows) / wall, "unit": UNIT, "cores": min(cores, len(rows)), "kind": "oracle",
           "sample": f"{len(rows)} signals of {cfg['name']} spread over the batch (rows {rows[0]}..{rows[-1]}), "
                     f"FP64 numpy QR per step, one process per core, BLAS threads = 1; {wall:.1f} s wall"}
    rep = compare_batch(res.support.cpu().numpy(), res.X.cpu().numpy(), res.resid_norm.cpu().numpy(),
                        res.n_iter.cpu().numpy(), res.status.cpu().numpy(), ora, A_np.shape[1], rows=list(rows))
    return cpu, rep.as_dict()


def run_reference(args, world, rank):
    """The reference arm: the FP64 CPU oracle as it stands, timed on the host cores (rank 0 only)."""
    if rank != 0:
        return
    from oracle import host_cores, omp_batch as oracle_batch
    from synth import config, make_dictionary, make_signals
    cfg = config(args.config)
    B_total = args.batch or cfg["B"]
    cores = host_cores()
    n = oracle_sample_size(args, cfg, cores) if args.oracle_sample is None else args.oracle_sample
    n = max(1, min(B_total, n // 2))   # each step is a bounded sample; keep the whole run ~minutes
    A_np = make_dictionary(cfg["M"], cfg["N"], cfg["seed"])
    eps32 = None if cfg["eps"] is None else float(np.float32(cfg["eps"]))
    times = []
    steps = max(1, args.steps)
    for s in range(args.warmup + steps):
        rows = (np.arange(n) * max(1, B_total // n) + s) % B_total
        Y = make_signals(A_np, rows, cfg["seed"], cfg["sparsity"], cfg["sigma"])
        t0 = time.perf_counter()
        oracle_batch(A_np, Y, cfg["S"], eps32, workers=cores)
        if s >= args.warmup:
            times.append(time.perf_counter() - t0)
    ms = statistics.mean(times) * 1e3
    value = n / (ms / 1e3)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg['name']}: M={cfg['M']} N={cfg['N']} S={cfg['S']} B={B_total}",
                   "global_batch": B_total, "step_sample": n},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": min(cores, n), "kind": "oracle",
                         "sample": f"{n} signals per step of {cfg['name']}, FP64 numpy QR per OMP step, "
                                   f"one process per core"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


if __name__ == "__main__":
    main()
