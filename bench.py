#!/usr/bin/env python3
"""bench.py -- per-cell FE local assembly throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--configs c1,...,c5]
                    [--headline c5] [--partition strong|weak] [--impl ours|reference]

A "step" is one pass of the hot path -- ``femgpu_assemble``: the element
matrices of every cell of one BASELINE config mesh -- over inputs already
resident in HBM.  Every config is timed in one invocation (graph-replayed
steps, roofline, e2e, parity, clocks, and at N=1 the reference's CPU path as
``cpu_baseline``) under the ``configs`` key; the top-level keys repeat the
headline config's (default c5, the largest: 5.8 GB and ~0.9 MFLOP per cell).

Multi-GPU (north_star): cells are split contiguously across the
N GPUs of one box (``--partition strong``, default); ``weak`` gives every rank
its own full mesh.  ``--gpus N`` launches N ranks itself (torch.distributed.run,
one process per GPU, NCCL) when not already under torchrun, and fails loudly
if fewer than N GPUs are visible.  The path needs no exchange: NCCL carries a
barrier and the max over ranks of each timed region only.

Prints ONE JSON line (rank 0).  DESIGN.md §6 documents every key.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_ORDER = ("c1", "c2", "c3", "c4", "c5")
HEADLINE = "c5"  # the largest config (BASELINE.json metric names none)
METRIC = "element matrices/s"
DATA = "synthetic (seeded jittered cube mesh, seeded dofs; BASELINE config shapes)"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--configs", default=",".join(CONFIG_ORDER),
                    help="comma-separated configs to time (all five by default)")
    ap.add_argument("--config", default=None, help="time only this config (alias)")
    ap.add_argument("--headline", default=HEADLINE)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--partition", default="strong", choices=["strong", "weak"],
                    help="strong: one mesh split contiguously (north_star); weak: a mesh per GPU")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-graph", action="store_true",
                    help="time direct launches (per-launch events) instead of a CUDA-graph replay")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=1.0,
                    help="wall seconds per CPU-baseline sample (all host threads)")
    ap.add_argument("--ref-step-seconds", type=float, default=0.3,
                    help="reference arm: wall seconds of CPU work per step and config")
    a = ap.parse_args(argv)
    a.configs = [a.config] if a.config else [c.strip() for c in a.configs.split(",") if c.strip()]
    if a.headline not in a.configs:
        a.headline = a.configs[-1]
    a.warmup = max(3, a.warmup)
    return a


def config_dict(cfg, world: int, partition: str) -> dict:
    """The workload, identical in both arms (the driver compares them)."""
    cells = cfg.ncells * (world if partition == "weak" else 1)
    return {"workload": f"{cfg.name}: {cfg.description}", "cells": cells, "n": cfg.n,
            "nq": cfg.nq, "bytes_per_cell": cfg.bytes_per_cell(),
            "parallelism": (f"cells split contiguously over {world} GPU(s), no exchange"
                            if partition == "strong" else
                            f"one full mesh per GPU x{world} (weak), no exchange"),
            "l2": "inputs+outputs per step > 126 MB L2 (no flush needed)"}


# ----------------------------------------------------------------------------
# launching: --gpus N spawns N ranks (torch.distributed.run) unless under torchrun
# ----------------------------------------------------------------------------
def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(args) -> int:
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} CUDA devices, {have} visible "
              "(refusing to report a smaller run as N GPUs)", file=sys.stderr, flush=True)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    print("# " + " ".join(cmd), file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def dist_setup(args):
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # NCCL init log (rank count, transports) on stderr; stdout carries the JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        print(f"# rank {rank}/{world} on cuda:{local} "
              f"({torch.cuda.get_device_name(local)}), NCCL {torch.cuda.nccl.version()}",
              file=sys.stderr, flush=True)
    return rank, world, local


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
                 "--format=csv,noheader,nounits", "-lms", "50"],
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
# roofline inputs, measured on this box where possible
# ----------------------------------------------------------------------------
def load_peaks(dev_index: int) -> dict:
    import ctypes

    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks["hbm_gbs"] = float(json.load(f)["hbm_gbs"])
        peaks["hbm_source"] = "measured copy bandwidth (MEASURED_PEAKS.json hbm_gbs, burst)"
    except (OSError, KeyError, ValueError):
        peaks["hbm_gbs"] = 6650.0
        peaks["hbm_source"] = "of fallback (B200_PROFILING.md: 6.65 TB/s)"
    # FP64 has no MEASURED_PEAKS entry: measure DFMA and DMMA (mma.sync .f64) on
    # this GPU now (tools/fp64_peak.cu built as tools/libpeaks.so)
    so = os.path.join(ROOT, "tools", "libpeaks.so")
    try:
        L = ctypes.CDLL(so)
        L.peaks_fp64.argtypes = [ctypes.POINTER(ctypes.c_double)] * 2
        a, b = ctypes.c_double(), ctypes.c_double()
        if L.peaks_fp64(ctypes.byref(a), ctypes.byref(b)) != 0:
            raise OSError("peaks_fp64 failed")
        peaks.update(dfma_tflops=a.value, dmma_tflops=b.value,
                     fp64_source=f"measured in this run on cuda:{dev_index} (tools/libpeaks.so: "
                                 "DFMA 512 thr x 4 CTA/SM, DMMA m16n8k8 256 thr x 2 CTA/SM, best of 5)")
    except OSError as exc:
        peaks.update(dfma_tflops=33.9, dmma_tflops=37.0,
                     fp64_source=f"committed measurement profiles/fp64_peak_r01.txt ({exc})")
    return peaks


def f_alg(cfg_name):
    """Reference-derived algorithmic flops/cell: min over femopt plans of
    flop_count(optimize(IR)) (tests/golden/falg.json, written by the reference)."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "falg.json")) as f:
            meta = json.load(f)
        return min(p["flops_per_cell"] for p in meta[cfg_name].values())
    except (OSError, KeyError, ValueError):
        return None


KERNEL_SOURCES = {"helm_quad": "helm_quad.cu", "helm_": "helmholtz.cu", "pair_": "pair.cu",
                  "burgers_quad": "burgers_quad.cu", "burgers": "burgers.cu", "elas_": "elasticity.cu",
                  "svk_mma": "svk_mma.cu"}


def kernel_source_sha(kernel_name: str):
    """sha of the kernel's .cu source with // comments and blank lines dropped (a
    capture stays valid across comment edits, not across code edits)."""
    for prefix, fn in KERNEL_SOURCES.items():
        if kernel_name.startswith(prefix):
            path = os.path.join(ROOT, "paper_1604_05872_b200", "csrc", fn)
            try:
                with open(path, encoding="utf-8") as f:
                    lines = [ln.split("//", 1)[0].rstrip() for ln in f]
            except OSError:
                return None
            code = "\n".join(ln for ln in lines if ln)
            return hashlib.sha1(code.encode()).hexdigest()[:12]
    return None


def ncu_capture(cfg_name: str, kernel_name: str):
    """The committed ncu --set full capture of this config's kernel (profiles/
    ncu_summary.json) if it is of the kernel this form runs AND of its current
    source (sha of the .cu file recorded at capture time); else None (stale)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f).get(cfg_name, {})
    except (OSError, ValueError):
        return None
    base = kernel_name.split("<")[0]
    if base not in (d.get("kernel") or ""):
        return None
    sha = kernel_source_sha(kernel_name)
    if not sha or d.get("src_sha") != sha:
        return None
    return d


# ----------------------------------------------------------------------------
# host side of e2e: NUMA-local pinned buffers, PCIe ceiling
# ----------------------------------------------------------------------------
def gpu_local_cpus(dev_index: int):
    """CPUs of the GPU's NUMA node (sysfs local_cpulist), or None."""
    import torch

    try:
        p = torch.cuda.get_device_properties(dev_index)
        bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bus}/local_cpulist") as f:
            spec = f.read().strip()
        cpus = set()
        for part in spec.split(","):
            if "-" in part:
                lo, hi = part.split("-")
                cpus.update(range(int(lo), int(hi) + 1))
            elif part:
                cpus.add(int(part))
        cpus &= os.sched_getaffinity(0)
        return cpus or None
    except (OSError, ValueError, AttributeError):
        return None


def pcie_bandwidth(dev, nbytes=1 << 29):
    """Pinned H2D and D2H GB/s, each alone and both at once (the e2e pipeline
    runs them concurrently on the two copy engines)."""
    import torch

    n = nbytes // 8
    h1 = torch.empty(n, dtype=torch.float64).pin_memory()
    h2 = torch.empty(n, dtype=torch.float64).pin_memory()
    d1 = torch.empty(n, dtype=torch.float64, device=dev)
    d2 = torch.empty(n, dtype=torch.float64, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    res = {}

    def timed(fns, reps=3):
        for fn, s in fns:
            with torch.cuda.stream(s):
                fn()
        torch.cuda.synchronize(dev)
        best = 1e30
        for _ in range(reps):
            t0 = time.perf_counter()
            for fn, s in fns:
                with torch.cuda.stream(s):
                    fn()
            torch.cuda.synchronize(dev)
            best = min(best, time.perf_counter() - t0)
        return best

    h2d = (lambda: d1.copy_(h1, non_blocking=True), s1)
    d2h = (lambda: h2.copy_(d2, non_blocking=True), s2)
    res["h2d_gbs"] = nbytes / timed([h2d]) / 1e9
    res["d2h_gbs"] = nbytes / timed([d2h]) / 1e9
    t = timed([h2d, d2h])
    res["duplex_gbs_each"] = nbytes / t / 1e9
    del h1, h2, d1, d2
    return res


# ----------------------------------------------------------------------------
# the reference's CPU path (oracle/_ref): cpu_baseline and the reference arm
# ----------------------------------------------------------------------------
def cpu_reference_rate(cfg, seconds: float, nthreads: int, coords, coeffs, steps=3):
    """femopt-optimized emitted C (oracle/_ref) on a bounded sample: every femopt
    plan, all threads, best of ``steps``; returns (cells/s, info) of the fastest."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refkernel as rk

    best = None
    for plan in rk.plans_for(cfg):
        if not rk.available(cfg, plan):
            continue
        K = rk.RefKernel(cfg, plan)
        n = min(coords.shape[0], K.chunk * max(1, nthreads))
        n = max(K.chunk, n // K.chunk * K.chunk)
        st = K.prepare(coords[:n], coeffs[:n])
        t0 = time.perf_counter()
        K.run_prepared(st, nthreads)
        dt = time.perf_counter() - t0
        n = int(min(coords.shape[0], max(n, n * seconds / max(dt, 1e-6))))
        n = max(K.chunk, n // K.chunk * K.chunk)
        st = K.prepare(coords[:n], coeffs[:n])
        times = []
        for _ in range(steps):
            t0 = time.perf_counter()
            K.run_prepared(st, nthreads)
            times.append(time.perf_counter() - t0)
        rate = n / min(times)
        if best is None or rate > best[0]:
            best = (rate, {"plan": plan, "cells": n, "flops_per_cell": K.flops_per_cell,
                           "times": times, "kernel": K, "state": st})
    if best is None:
        return None, {"error": "reference sources missing (oracle/_ref/src)"}
    return best


def run_reference_arm(args, rank, world):
    """--impl reference: the reference's own CPU implementation of the path
    (femopt's optimized emitted C, all host threads), every config, rank 0 only."""
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refkernel as rk

    from paper_1604_05872_b200 import fe

    nthreads = os.cpu_count() or 1
    per_cfg = {}
    for name in args.configs:
        cfg = fe.CONFIGS[name]
        coords, coeffs = fe.cell_inputs(cfg)
        rate, info = cpu_reference_rate(cfg, args.ref_step_seconds, nthreads, coords, coeffs,
                                        steps=1)
        if rate is None:
            print(json.dumps({"impl": "reference", "unavailable": info["error"]}), flush=True)
            return
        K, st, n = info["kernel"], info["state"], info["cells"]
        for _ in range(args.warmup):
            K.run_prepared(st, nthreads)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            K.run_prepared(st, nthreads)
        dt = (time.perf_counter() - t0) / args.steps
        value = n / dt
        sample = (f"first {n} of {cfg.ncells} cells of {name} per step, femopt plan "
                  f"'{info['plan']}' emitted C (cc -O3 -march=native -ffp-contract=off), "
                  f"{nthreads} threads, {rk.cpu_model()}")
        per_cfg[name] = {
            "metric": METRIC, "value": value, "unit": "elem/s", "ms_per_step": dt * 1e3,
            "config": config_dict(cfg, world, args.partition),
            "gflops": value * info["flops_per_cell"] / 1e9,
            "cpu_baseline": {"value": value, "unit": "elem/s", "cores": nthreads,
                             "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": "elem/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }
        print(f"# reference {name}: {value:.4g} elem/s ({info['plan']}, {n} cells/step)",
              file=sys.stderr, flush=True)
    h = per_cfg[args.headline]
    line = {"impl": "reference", "metric": METRIC, "value": h["value"], "unit": "elem/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": h["ms_per_step"], "higher_is_better": True,
            "scaling": "weak" if args.partition == "weak" else "strong", "vs_baseline": None,
            "dtype": "f64", "data": DATA, "config": h["config"], "gflops": h["gflops"],
            "cpu_baseline": h["cpu_baseline"], "e2e": h["e2e"], "headline": args.headline,
            "configs": per_cfg}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------
def time_config(args, name, rank, world, local, peaks, pcie):
    import numpy as np  # noqa: F401
    import torch
    import torch.distributed as dist

    from paper_1604_05872_b200 import fe, femgpu, shard

    dev = torch.device("cuda", local)
    cfg = fe.CONFIGS[name]
    coords, coeffs, first = shard.shard_inputs(cfg, rank, world, args.partition)
    E = coords.shape[0]
    form = femgpu.Form.from_config(cfg)
    x = torch.from_numpy(coords).to(dev)
    c = torch.from_numpy(coeffs).to(dev)
    out = torch.empty((E, cfg.n, cfg.n), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    steps = args.steps

    def step(s=stream):
        form.assemble(x, c, out, stream=s)

    clk = ClockSampler(local).__enter__()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    t_wait = time.perf_counter()  # at least one clock sample under load
    while not clk.lines and time.perf_counter() - t_wait < 3.0:
        step()
        torch.cuda.synchronize(dev)
    graph = None
    if not args.no_graph:
        # the K launches replayed from one CUDA graph: back to back on the device,
        # no host launch gaps (c1's 60 us kernel would otherwise be timed with them)
        g_stream = torch.cuda.Stream(dev)
        g_stream.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=g_stream):
            for _ in range(steps):
                form.assemble(x, c, out, stream=g_stream)
        stream.wait_stream(g_stream)
        graph.replay()  # warm replay
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    evs = []
    n_clk0 = len(clk.lines)
    if graph is not None:
        ev0.record(stream)
        graph.replay()
        ev1.record(stream)
    else:
        ev0.record(stream)
        for _ in range(steps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step()
            b.record(stream)
            evs.append((a, b))
        ev1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clk.__exit__(None, None, None)
    if len(clk.lines) > n_clk0 + 2:  # keep only samples taken in the timed region if enough
        clk.lines = clk.lines[n_clk0:]
    local_ms = ev0.elapsed_time(ev1)
    per_launch = [a.elapsed_time(b) for a, b in evs] if evs else [local_ms / steps]
    total_ms = shard.max_over_ranks(local_ms, dev)  # max over ranks, device-timed
    ms_per_step = total_ms / steps
    cells_all = int(round(shard.sum_over_ranks(float(E), dev)))
    value = cells_all / (ms_per_step / 1e3)
    res = {"metric": METRIC, "value": value, "unit": "elem/s", "ms_per_step": ms_per_step,
           "config": config_dict(cfg, world, args.partition),
           "kernel": form.info["kernel_name"], "schedule": form.info["schedule"],
           "timing": ("CUDA events around one CUDA-graph replay of the K launches"
                      if graph is not None else "CUDA events around K direct launches"),
           "gpu_launches": steps * form.info["kernels_per_launch"], "clocks": clk.summary()}
    del graph

    # ---- parity: every cell of the timed output vs the reference's CPU path ----
    if not args.no_parity:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        try:
            import parity

            lw = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
            nthr = max(1, (os.cpu_count() or 1) // lw)
            p = parity.check(cfg, coords, coeffs, lambda a, b: out[a:b].cpu().numpy(),
                             nthreads=nthr)
            err = shard.max_over_ranks(p["max_frob_rel"], dev)
            chk = int(round(shard.sum_over_ranks(float(p["cells_checked"]), dev)))
            res["parity"] = {"max_frob_rel": err, "cells_checked": chk, "cells": cells_all,
                             "tol": 1e-12, "ok": bool(err <= 1e-12 and chk == cells_all),
                             "against": p["against"],
                             "buffer": "the output of the last timed step"}
        except Exception as exc:  # noqa: BLE001 -- reported, never silently dropped
            res["parity"] = {"error": repr(exc)}

    # ---- roofline of the dominant (only) kernel ----
    F_model = form.info["flops_per_cell"]
    cap = ncu_capture(name, form.info["kernel_name"])
    F_ncu = cap.get("fp64_flops_per_cell_ncu") if cap else None
    F_exec = F_ncu if F_ncu else F_model
    Fa = f_alg(name)
    F_roof = min(F_exec, Fa) if Fa else F_exec
    bpc = cfg.bytes_per_cell()
    avg_launch_s = (sum(per_launch) / len(per_launch)) / 1e3
    uses_dmma = bool(cap and cap.get("dmma_pipe_pct", 0) > 0) if cap else \
        form.info["kernel_name"].startswith(("helm_tensor", "burgers", "elas_tensor", "svk_mma"))
    fp64_peak = peaks["dmma_tflops"] if uses_dmma else peaks["dfma_tflops"]
    pipe = "fp64 DMMA" if uses_dmma else "fp64 DFMA"
    t_fp = F_roof / (fp64_peak * 1e12)
    t_hbm = bpc / (peaks["hbm_gbs"] * 1e9)
    if t_hbm >= t_fp:
        achieved = E * bpc / avg_launch_s / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "peak_source": peaks["hbm_source"],
                "algorithmic_per_launch": E * bpc, "per_unit": f"{bpc} B/cell"}
    else:
        achieved = E * F_roof / avg_launch_s / 1e12
        roof = {"bound": "tensor", "pipe": pipe, "achieved": achieved, "peak": fp64_peak,
                "unit": "TFLOP/s", "frac": achieved / fp64_peak,
                "peak_source": peaks["fp64_source"], "algorithmic_per_launch": E * F_roof,
                "per_unit": f"{F_roof:.0f} flop/cell"}
        roof["frac_of_chip_fp64"] = achieved / max(peaks["dmma_tflops"], peaks["dfma_tflops"])
    roof["traffic"] = cap.get("dram_bytes_per_launch") * E / cfg.ncells if cap else None
    roof["traffic_source"] = (f"ncu --set full, {cap.get('capture')}" if cap else
                              "no current ncu capture of this kernel's source")
    res["roofline"] = roof
    res["roofline_step_frac"] = E * max(t_fp, t_hbm) / (ms_per_step / 1e3)
    res["flops_per_cell"] = {"F_exec_ncu": F_ncu, "F_exec_model": F_model,
                             "F_alg_reference": Fa, "F_roof": F_roof,
                             "rule": "F_roof = min(F_alg, F_exec); F_exec = ncu-counted FP64 "
                                     "flops of a capture of the current kernel source, else the "
                                     "kernel's useful-flop model"}
    res["bytes_per_cell"] = bpc
    res["gflops"] = value * F_roof / 1e9

    # ---- end to end through the host C ABI (pinned host buffers, copies timed) ----
    del x, c
    if args.e2e_steps > 0:
        cpus = gpu_local_cpus(local)
        old = os.sched_getaffinity(0)
        if cpus:  # first touch of the pinned pages on the GPU's NUMA node
            os.sched_setaffinity(0, cpus)
        try:
            hx = torch.from_numpy(coords).pin_memory()
            hc = torch.from_numpy(coeffs).pin_memory()
            hA = torch.empty((E, cfg.n, cfg.n), dtype=torch.float64, pin_memory=True)
            hA.view(-1)[:: 512].zero_()
            form.assemble_host_ptr(E, hx.data_ptr(), hc.data_ptr(), hA.data_ptr())  # warm-up
            if world > 1:
                dist.barrier()
            times = []
            for _ in range(args.e2e_steps):
                t0 = time.perf_counter()
                form.assemble_host_ptr(E, hx.data_ptr(), hc.data_ptr(), hA.data_ptr())
                times.append(time.perf_counter() - t0)
        finally:
            os.sched_setaffinity(0, old)
        dt = shard.max_over_ranks(sum(times) / len(times), dev)
        h2d = int(hx.numel() * 8 + hc.numel() * 8)
        d2h = int(hA.numel() * 8)
        same = all(bool(torch.equal(hA[a:a + 65536], out[a:a + 65536].cpu()))
                   for a in range(0, E, 65536))
        e2e = {"value": cells_all / dt, "unit": "elem/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "matches_device": same,
               "step_ms": [round(t * 1e3, 2) for t in times],
               "api": "femgpu_assemble_host (chunked 3-stream H2D/kernel/D2H pipeline)",
               "numa_local_cpus": len(cpus) if cpus else None}
        if pcie:
            # ceiling: the copies overlap (two copy engines, full-duplex PCIe) and the
            # kernel hides behind them: while both directions stream each runs at the
            # duplex rate, the rest of the larger one at its rate alone; the kernel
            # time is the other floor
            both = min(h2d, d2h)
            t_copy = both / (pcie["duplex_gbs_each"] * 1e9) + \
                (h2d - both) / (pcie["h2d_gbs"] * 1e9) + (d2h - both) / (pcie["d2h_gbs"] * 1e9)
            floor = max(t_copy, avg_launch_s)
            e2e["pcie"] = pcie
            e2e["ceiling"] = cells_all / floor
            e2e["pcie_frac"] = floor / dt
        res["e2e"] = e2e
        del hx, hc, hA

    # ---- the reference's CPU path on this box (N=1 only) ----
    if not args.no_cpu_baseline and world == 1:
        nthreads = os.cpu_count() or 1
        try:
            rate, info = cpu_reference_rate(cfg, args.cpu_seconds, nthreads, coords, coeffs)
        except Exception as exc:  # noqa: BLE001 -- baseline is reported, never fatal
            rate, info = None, {"error": repr(exc)}
        if rate is not None:
            import refkernel as rk
            res["cpu_baseline"] = {
                "value": rate, "unit": "elem/s", "cores": nthreads, "kind": "reference",
                "sample": f"{info['cells']} cells of {name}, femopt plan '{info['plan']}' "
                          f"emitted C (cc -O3 -march=native -ffp-contract=off), best of 3, "
                          f"{rk.cpu_model()}"}
        else:
            res["cpu_baseline"] = {"value": None, "unit": "elem/s", "cores": nthreads,
                                   "kind": "reference", "sample": info.get("error")}
    del out, form
    torch.cuda.empty_cache()
    print(f"# {name}: {value:.4g} elem/s, {ms_per_step:.4f} ms/step, roofline "
          f"{roof['frac']:.3f} ({roof['bound']}), parity "
          f"{res.get('parity', {}).get('max_frob_rel')}", file=sys.stderr, flush=True)
    return res


def run_ours(args, rank, world, local):
    import torch

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    peaks = load_peaks(local)
    pcie = None
    if args.e2e_steps > 0:
        cpus = gpu_local_cpus(local)
        old = os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
        try:
            pcie = pcie_bandwidth(dev)
        finally:
            os.sched_setaffinity(0, old)
    per_cfg = {}
    for name in args.configs:
        per_cfg[name] = time_config(args, name, rank, world, local, peaks, pcie)
    if rank != 0:
        return
    h = per_cfg[args.headline]
    line = {"metric": METRIC, "value": h["value"], "unit": "elem/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": h["ms_per_step"],
            "higher_is_better": True,
            "scaling": "weak" if args.partition == "weak" else "strong", "vs_baseline": None,
            "dtype": "f64", "data": DATA, "config": h["config"]}
    for k in ("gflops", "roofline", "roofline_step_frac", "flops_per_cell", "bytes_per_cell",
              "gpu_launches", "clocks", "e2e", "cpu_baseline", "parity", "kernel", "schedule",
              "timing"):
        if k in h:
            line[k] = h[k]
    line["headline"] = args.headline
    line["peaks"] = peaks
    line["configs"] = per_cfg
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "ours" and "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
        run_reference_arm(args, rank, world)  # rank 0 only; the others exit 0
        return
    rank, world, local = dist_setup(args)
    run_ours(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
