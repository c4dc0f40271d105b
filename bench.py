#!/usr/bin/env python3
"""bench.py -- per-cell FE local assembly throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A "step" is one pass of the hot path (femgpu_assemble: element matrices of
every cell of one config mesh) over inputs already resident in HBM.  At N>1
(torchrun, one rank per GPU, NCCL) every rank assembles its own shard -- a
full config-size jittered mesh with its own seed (weak scaling, no data-path
collective; a barrier and a max-reduce of the step time only).

Prints ONE JSON line (rank 0).  See DESIGN.md §Measurement for every key.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_CONFIG = "c2"  # BASELINE.json configs[1]: the metric's headline config


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=0,
                    help="timed steps (0 = auto: enough for >= 2 s of timed region)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-graph", action="store_true",
                    help="time direct launches (per-launch events) instead of a CUDA-graph replay")
    ap.add_argument("--partition", default="weak", choices=["weak", "strong"],
                    help="weak: a full config mesh per GPU; strong: one mesh split contiguously")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=3.0,
                    help="wall seconds per CPU-baseline sample (all host threads)")
    return ap.parse_args()


# ----------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)
# ----------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for n, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------
def dist_setup(args):
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.impl == "ours":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return rank, world, local


def load_peaks():
    peaks = {"hbm_gbs": None, "fp64_tflops": None, "hbm_source": None, "fp64_source": None}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        peaks["hbm_gbs"] = mp.get("hbm_gbs")
        peaks["hbm_source"] = "measured (MEASURED_PEAKS.json copy)"
    except OSError:
        peaks["hbm_gbs"] = 6650.0
        peaks["hbm_source"] = "fallback (B200_PROFILING.md)"
    # FP64 has no MEASURED_PEAKS entry: our mma.sync f64 (DMMA) microbenchmark on
    # this pool's B200 (tools/fp64_peak.cu -> profiles/fp64_peak_r01.txt).
    peaks["fp64_tflops"] = 37.0
    peaks["fp64_source"] = "measured DMMA peak, profiles/fp64_peak_r01.txt"
    peaks["dfma_tflops"] = 33.9
    peaks["dfma_source"] = "measured DFMA peak, profiles/fp64_peak_r01.txt"
    return peaks


def f_alg(cfg_name):
    """Reference-derived algorithmic flops/cell: min over femopt plans of
    flop_count(optimize(IR)) (tests/golden/<cfg>.json, written by the reference)."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "falg.json")) as f:
            meta = json.load(f)
        return min(p["flops_per_cell"] for p in meta[cfg_name].values())
    except (OSError, KeyError, ValueError):
        return None


def profile_traffic(cfg_name):
    """dram bytes per launch from the committed ncu --set full capture, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        return d.get(cfg_name, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def uses_dmma(cfg_name, kernel_name):
    """Whether the committed ncu capture of this kernel executed DMMA instructions
    (None if unknown): a DFMA-only kernel's FP64 ceiling is the DFMA peak."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f).get(cfg_name, {})
    except (OSError, ValueError):
        return None
    if ncu_flops(cfg_name, kernel_name) is None:
        return None
    b = d.get("fp64_flops_ncu_breakdown", {})
    return b.get("sm__ops_path_tensor_src_fp64", 0) > 0


def ncu_flops(cfg_name, kernel_name):
    """F_exec as SURVEY.md §8d defines it: FP64 flops executed per cell, counted by
    ncu (tools/ncu_flops.py; DFMA = 2, DADD/DMUL = 1, DMMA = 2mnk), if the committed
    capture is of the kernel this form runs."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f).get(cfg_name, {})
    except (OSError, ValueError):
        return None
    k = d.get("fp64_flops_ncu_kernel") or ""
    base = kernel_name.split("<")[0]
    ok = base in k or (base == "pair_kernel" and "pair_" in k)
    return d.get("fp64_flops_per_cell_ncu") if ok else None


# ----------------------------------------------------------------------------
def cpu_reference_rate(cfg, seconds: float, nthreads: int, coords, coeffs):
    """The reference's CPU path (femopt-optimized emitted C, oracle/_ref) on a
    bounded sample: fastest femopt plan, all threads.  Returns (cells/s, info)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import refkernel as rk

    best = None
    for plan in rk.plans_for(cfg):
        if not rk.available(cfg, plan):
            continue
        K = rk.RefKernel(cfg, plan)
        # calibrate sample size to ~`seconds` of wall time
        n = K.chunk * max(1, nthreads)
        st = K.prepare(coords[:n], coeffs[:n])
        t0 = time.perf_counter()
        K.run_prepared(st, nthreads)
        dt = time.perf_counter() - t0
        n = int(min(coords.shape[0], max(n, n * seconds / max(dt, 1e-6))))
        n = max(K.chunk, n // K.chunk * K.chunk)
        st = K.prepare(coords[:n], coeffs[:n])
        times = []
        for _ in range(3):
            t0 = time.perf_counter()
            K.run_prepared(st, nthreads)
            times.append(time.perf_counter() - t0)
        rate = n / min(times)
        if best is None or rate > best[0]:
            best = (rate, {"plan": plan, "cells": n, "flops_per_cell": K.flops_per_cell})
    if best is None:
        return None, {"error": "reference sources missing (oracle/_ref/src)"}
    return best


def run_reference_arm(args, rank, world):
    """--impl reference: the reference's own CPU implementation of the path."""
    from paper_1604_05872_b200 import fe

    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refkernel as rk

    cfg = fe.CONFIGS[args.config]
    nthreads = os.cpu_count() or 1
    coords, coeffs = fe.cell_inputs(cfg)
    rate, info = cpu_reference_rate(cfg, args.cpu_seconds, nthreads, coords, coeffs)
    if rate is None:
        print(json.dumps({"impl": "reference", "unavailable": info["error"]}))
        return
    K = rk.RefKernel(cfg, info["plan"])
    n = info["cells"]
    st = K.prepare(coords[:n], coeffs[:n])
    for _ in range(args.warmup):
        K.run_prepared(st, nthreads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        K.run_prepared(st, nthreads)
    dt = (time.perf_counter() - t0) / args.steps
    value = n / dt
    line = {
        "impl": "reference", "metric": "element matrices/s", "value": value, "unit": "elem/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded jittered cube mesh, seeded dofs)",
        "config": {"workload": f"{args.config}: {cfg.description}", "cells_per_step": n,
                   "sample": f"first {n} cells of the {cfg.ncells}-cell mesh"},
        "gflops": value * info["flops_per_cell"] / 1e9,
        "cpu_baseline": {"value": value, "unit": "elem/s", "cores": nthreads, "kind": "reference",
                         "sample": f"{n} cells, femopt plan '{info['plan']}' emitted C, "
                                   f"cc -O3 -march=native, {rk.cpu_model()}"},
        "e2e": {"value": value, "unit": "elem/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
def run_ours(args, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1604_05872_b200 import fe, femgpu

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_1604_05872_b200 import shard

    cfg = fe.CONFIGS[args.config]
    coords, coeffs, _ = shard.shard_inputs(cfg, rank, world, args.partition)
    E = coords.shape[0]
    form = femgpu.Form.from_config(cfg)
    x = torch.from_numpy(coords).to(dev)
    c = torch.from_numpy(coeffs).to(dev)
    out = torch.empty((E, cfg.n, cfg.n), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        form.assemble(x, c, out, stream=stream)

    clk = ClockSampler(local).__enter__()  # sample clocks across warm-up and timed region
    w0 = time.perf_counter()
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize(dev)
    est_ms = (time.perf_counter() - w0) * 1e3 / max(3, args.warmup)
    if args.steps <= 0:  # auto: a timed region of >= 2 s (clock samples under load)
        args.steps = int(max(20, min(5000, 2000.0 / max(est_ms, 1e-3))))
    t_wait = time.perf_counter()
    while not clk.lines and time.perf_counter() - t_wait < 3.0:
        step()
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    per_launch = []
    clk.lines.clear()
    graph = None
    if not args.no_graph:
        # the K launches replayed from a CUDA graph: back to back on the device,
        # no host-side launch gaps (a 60 us kernel would otherwise be timed
        # with the Python/ctypes launch overhead between launches)
        try:
            g_stream = torch.cuda.Stream(dev)
            g_stream.wait_stream(stream)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=g_stream):
                for _ in range(args.steps):
                    form.assemble(x, c, out, stream=g_stream)
            stream.wait_stream(g_stream)
            graph.replay()  # warm replay
            torch.cuda.synchronize(dev)
        except Exception as exc:  # noqa: BLE001 -- fall back to direct launches
            print(f"# graph capture unavailable ({exc}); timing direct launches", file=sys.stderr)
            graph = None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    evs = []
    if graph is not None:
        ev0.record(stream)
        graph.replay()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    else:
        ev0.record(stream)
        for _ in range(args.steps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step()
            b.record(stream)
            evs.append((a, b))
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    clk.__exit__(None, None, None)
    total_ms = ev0.elapsed_time(ev1)
    # mean launch duration of the dominant (only) kernel: back-to-back graph
    # replay -> total / K; direct launches -> per-launch events
    per_launch = [a.elapsed_time(b) for a, b in evs] if evs else [total_ms / args.steps]
    total_ms = shard.max_over_ranks(total_ms, dev)  # max over ranks (NCCL), device-timed
    ms_per_step = total_ms / args.steps
    cells_all = int(shard.max_over_ranks(float(E), dev)) * world if args.partition == "weak" \
        else cfg.ncells
    value = cells_all / (ms_per_step / 1e3)

    # ---- end to end through the host C ABI (pinned buffers, copies timed) ----
    e2e = None
    if args.e2e_steps > 0:
        hx = torch.from_numpy(coords).pin_memory()
        hc = torch.from_numpy(coeffs).pin_memory()
        hA = torch.empty((E, cfg.n, cfg.n), dtype=torch.float64).pin_memory()
        form.assemble_host_ptr(E, hx.data_ptr(), hc.data_ptr(), hA.data_ptr())  # warm-up
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            form.assemble_host_ptr(E, hx.data_ptr(), hc.data_ptr(), hA.data_ptr())
        dt = shard.max_over_ranks((time.perf_counter() - t0) / args.e2e_steps, dev)
        # spot check the host path against the device result (first cells)
        ok = bool(torch.equal(hA[:64], out[:64].cpu()))
        e2e = {"value": cells_all / dt, "unit": "elem/s",
               "h2d_bytes_per_step": int(hx.numel() * 8 + hc.numel() * 8),
               "d2h_bytes_per_step": int(hA.numel() * 8), "matches_device": ok,
               "api": "femgpu_assemble_host (chunked 3-stream H2D/kernel/D2H pipeline)"}
        del hx, hc, hA

    if rank != 0:
        return
    peaks = load_peaks()
    F_model = form.info["flops_per_cell"]
    F_ncu = ncu_flops(args.config, form.info["kernel_name"])
    F_exec = F_ncu if F_ncu else F_model
    Fa = f_alg(args.config)
    F_roof = min(F_exec, Fa) if Fa else F_exec
    bpc = cfg.bytes_per_cell()
    avg_launch_s = (sum(per_launch) / len(per_launch)) / 1e3
    # the bound is whichever floor is longer: algorithmic bytes at the measured HBM
    # bandwidth or algorithmic flops at the measured FP64 (DMMA) peak
    # FP64 ceiling of the pipe the kernel runs on: DMMA (tensor) or, for a
    # DFMA-only kernel, the DFMA peak (they share one datapath, tools/fp64_mix.cu)
    if uses_dmma(args.config, form.info["kernel_name"]) is False:
        peaks["fp64_tflops"], peaks["fp64_source"] = peaks["dfma_tflops"], peaks["dfma_source"]
    hbm_bound = bpc / peaks["hbm_gbs"] >= F_roof / (peaks["fp64_tflops"] * 1e3)
    if hbm_bound:
        achieved = E * bpc / avg_launch_s / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "peak_source": peaks["hbm_source"]}
    else:
        achieved = E * F_roof / avg_launch_s / 1e12
        roof = {"bound": "tensor", "pipe": "fp64 " + ("DFMA" if "DFMA" in peaks["fp64_source"] else "DMMA"),
                "achieved": achieved,
                "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
                "frac": achieved / peaks["fp64_tflops"], "peak_source": peaks["fp64_source"]}
    tr = profile_traffic(args.config)
    roof["traffic"] = tr
    roof["algorithmic_per_launch"] = (E * bpc) if hbm_bound else E * F_roof
    # roofline time (slower of FP64 and HBM) -> fraction of the whole-step roofline
    t_roof = E * max(F_roof / (peaks["fp64_tflops"] * 1e12), bpc / (peaks["hbm_gbs"] * 1e9))
    line = {
        "metric": "element matrices/s", "value": value, "unit": "elem/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": args.partition, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded jittered cube mesh, seeded dofs; BASELINE config shapes)",
        "config": {"workload": f"{args.config}: {cfg.description}", "cells_per_gpu": E,
                   "n": cfg.n, "nq": cfg.nq, "parallelism": f"cells sharded x{world} ({args.partition})",
                   "l2": "inputs+outputs per step > 126 MB L2 (no flush needed)",
                   "kernel": form.info["kernel_name"], "schedule": form.info["schedule"],
                   "timing": ("CUDA events around one CUDA-graph replay of the K launches"
                              if graph is not None else "CUDA events around K direct launches")},
        "gflops": value * F_roof / 1e9,
        "flops_per_cell": {"F_exec_ncu": F_ncu, "F_exec_model": F_model, "F_alg_reference": Fa,
                           "F_roof": F_roof,
                           "rule": "F_roof = min(F_alg, F_exec); F_exec = ncu-counted FP64 flops "
                                   "(profiles/ncu_flops_r01) when present, else the kernel's model"},
        "bytes_per_cell": bpc,
        "roofline": roof,
        "roofline_step_frac": t_roof / (ms_per_step / 1e3),
        "gpu_launches": args.steps * form.info["kernels_per_launch"],
        "clocks": clk.summary(),
    }
    if e2e:
        line["e2e"] = e2e
    if not args.no_cpu_baseline:
        nthreads = os.cpu_count() or 1
        try:
            rate, info = cpu_reference_rate(cfg, args.cpu_seconds, nthreads, coords, coeffs)
        except Exception as exc:  # noqa: BLE001 -- baseline is reported, never fatal
            rate, info = None, {"error": repr(exc)}
        if rate is not None:
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import refkernel as rk
            line["cpu_baseline"] = {
                "value": rate, "unit": "elem/s", "cores": nthreads, "kind": "reference",
                "sample": f"{info['cells']} cells of {args.config}, femopt plan '{info['plan']}' "
                          f"emitted C (cc -O3 -march=native), {rk.cpu_model()}"}
        else:
            line["cpu_baseline"] = {"value": None, "unit": "elem/s", "cores": nthreads,
                                    "kind": "reference", "sample": info.get("error")}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_setup(args)
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
    else:
        run_ours(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
