#!/usr/bin/env python
"""Benchmark of the Escoin direct sparse convolution on B200.

One step = one pass of the hot path over one batch: every sparse CONV layer
of the workload (default: pruned ResNet-50 v1, its 16 sparse 3x3 layers,
BASELINE configs[3]) over the global batch of 128, through
escoin_sconv_forward (stretched CSR x dense NCHW, bias + ReLU fused).  Inputs
resident in HBM; L2 flushed before every step (a 256 MB write, outside the
per-step events).  The step is captured once as a CUDA graph and replayed.

Multi-GPU (torchrun, one rank per GPU): STRONG scaling by default — the
global batch is split contiguously (rank r owns images shard_range(128, r, G)),
weights are stretched on rank 0 and broadcast once over NCCL, the
specialised kernels are compiled once per node (rank 0 fills the cubin cache
ESCOIN_JIT_CACHE, the other ranks load it), no per-layer collectives; time =
MAX over ranks.  `--weak` gives every rank its own 128 images instead.

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle
instead (the reference arm for this tier).
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
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# cubins of the specialised kernels, shared by the ranks of this node (never shipped: .gpurunignore)
os.environ.setdefault("ESCOIN_JIT_CACHE", os.path.join(ROOT, "build", "jit_cache"))
os.makedirs(os.environ["ESCOIN_JIT_CACHE"], exist_ok=True)

from paper_1802_10280_b200 import inputs, shard, workloads  # noqa: E402

REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}
WL_NAMES = {"alexnet": "pruned AlexNet conv2-conv5 (4 sparse CONV layers)",
            "googlenet": "pruned GoogLeNet 19 sparse 3x3/5x5 CONV layers",
            "googlenet_1x1": "pruned GoogLeNet 37 1x1 CONV layers",
            "resnet50": "pruned ResNet-50 v1 16 sparse 3x3 CONV layers",
            "resnet50_v15": "pruned ResNet-50 v1.5 16 sparse 3x3 CONV layers (3 with stride 2)",
            "alexnet_conv1": "pruned AlexNet conv1 (11x11, stride 4; 80% sparse, NEXT-3)",
            "alexnet_convs": "AlexNet all 5 CONV layers: conv1 dense (unpruned), conv2-5 pruned (NEXT-2 stack)",
            "resnet50_convs": "ResNet-50 v1 all 53 CONV layers: 16 pruned 3x3, 37 dense (NEXT-2 stack)",
            "tiny": "tiny conv layer N=1 C=16 14x14 M=32 3x3"}
# escoin_csr_jit tunings compiled per layer (Q,P,CC,NS,warps,CTAs/SM; 0 = the library's model pick);
# escoin_csr_autotune_ex keeps the fastest under the bench's flushed-L2 conditions
# (Q is balanced over the groups: 48 -> 43 rows on 256 channels; "32,2,8,3,12,2,-1" = FFMA2 slot pairs, the
# res2 winner in r02u; "-1" = no instruction-prefetch pass)
# The two split-channel entries (ks = -2: auto count, compiled only where the grid is below one wave —
# GoogLeNet's 7x7 5x5 / 1x1 layers, r02y) are skipped on every other layer.
_KS = ",0,0,0,0,0,0,0,0,0,0,0,-2"
DEFAULT_JIT_TUNINGS = ("0;32,1,0,0,24,1;32,1,0,0,16,2;32,2,8,3,12,2,-1;32,1,0,0,32,1;48,1,0,0,16,2;"
                       "32,1,8,2,8,1" + _KS + ";32,1,2,2,16,1" + _KS)
# ResNet-50 (the headline): only the three tunings that won a stage in r02u/r02z — FFMA2 q32 w12 b2 (res2),
# q48->43 w16 b2 (res3, res4), q32 w24 b1 (res5) — which halves the fresh compile (the res5 kernels take
# ~5 min of one host core each)
RESNET_JIT_TUNINGS = "32,2,8,3,12,2,-1;48,1,0,0,16,2;32,1,0,0,24,1"
WL_JIT_TUNINGS = {"resnet50": RESNET_JIT_TUNINGS, "resnet50_v15": RESNET_JIT_TUNINGS}


def jit_tunings_for(workload):
    """The escoin_csr_jit tunings bench.py compiles for this workload (--jit-tunings overrides)."""
    return WL_JIT_TUNINGS.get(workload, DEFAULT_JIT_TUNINGS)
METRIC = "sparse-conv images/s (whole stack of sparse layers, global batch 128)"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="escoin", choices=["escoin", "reference"])
    p.add_argument("--workload", default="resnet50", choices=list(WL_NAMES))
    p.add_argument("--batch", type=int, default=None, help="GLOBAL batch (default: the workload's, 128)")
    p.add_argument("--weak", action="store_true", help="weak scaling: every rank runs its own --batch images")
    p.add_argument("--tune-variants", action="store_true",
                   help="autotune also over the compiled interpreter variants (default: specialised kernels only, "
                        "the variants only where no specialised kernel exists)")
    p.add_argument("--no-graph", action="store_true", help="time eager launches instead of the captured graph")
    p.add_argument("--engine", default="auto", choices=["auto", "sparse", "dense"],
                   help="per-layer engine: auto = escoin_select_engine (sparsity >= threshold -> sparse), or forced")
    p.add_argument("--sparsity", type=int, default=800, help="per-mille (ASSUMED 800, reading R#14)")
    p.add_argument("--skew", action="store_true",
                   help="skewed per-row sparsity (Beta(1,b) row densities, same mean; load-balance variant)")
    p.add_argument("--kernel", type=int, default=-1, help="sconv variant id (-1 = auto)")
    p.add_argument("--no-autotune", action="store_true", help="skip escoin_csr_autotune at setup")
    p.add_argument("--no-jit", action="store_true", help="skip the pattern-specialised kernels (escoin_csr_jit)")
    p.add_argument("--jit-tunings", default=None,
                   help="';'-separated escoin_csr_jit tunings compiled per layer (0 = the library's model pick); "
                        "autotune keeps the fastest")
    p.add_argument("--no-baselines", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--out", default=None, help="also write the JSON line to this file")
    p.add_argument("--dist-backend", default="nccl", help="torch.distributed backend for N > 1 (tests use gloo)")
    p.add_argument("--same-device", action="store_true",
                   help="all ranks on cuda:0 (multi-rank test of the driver on a 1-GPU box; not a measurement)")
    a = p.parse_args()
    if a.jit_tunings is None:
        a.jit_tunings = jit_tunings_for(a.workload)
    return a


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.rows = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        for r in self.rows:
            f = [x.strip() for x in r.split(",")]
            if len(f) < 4:
                continue
            try:
                s, m = float(f[0]), float(f[1])
                bits = int(f[3], 16)
            except ValueError:
                continue
            mx = m
            if bits & 0x1:  # idle sample: not under load
                continue
            sm.append(s)
            for b, n in REASON_BITS.items():
                if bits & b:
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ setup
class LayerRun:
    pass


def batch_range(args, wl, rank, world):
    """Global image range [n0, n0 + B) of this rank: strong scaling splits the global batch
    (shard.shard_range), weak scaling gives every rank its own full batch."""
    GB = args.batch or wl.batch
    if args.weak:
        return rank * GB, GB, GB * world
    a, b = shard.shard_range(GB, rank, world)
    return a, b - a, GB


def setup(args, wl, device, rank, world, torch, escoin, flush):
    n0, B, GB = batch_range(args, wl, rank, world)
    runs = []
    for L in wl.layers:
        r = LayerRun()
        r.L = L
        sp = args.sparsity if L.sparse else 0  # whole-stack workloads: layers the paper leaves dense
        if rank == 0:
            w = (inputs.layer_weights_skewed if getattr(args, "skew", False) and L.sparse else inputs.layer_weights)(
                wl.net, L, sp)
            bias = inputs.bias(wl.net, L.name, L.M)
            src = escoin.Csr.stretch(w, L.H, L.W, L.stride, L.pad)
            rp, ci, v = src.host_arrays()
            r.w_dense = w
        else:
            rp = ci = v = bias = None
            r.w_dense = None
        if world > 1:  # A3: weights replicated once from rank 0 (NCCL broadcast over NVLink)
            t = shard.broadcast_csr(rp, ci, v, bias, device)
            r.d_csr = t[:3]
            r.bias = t[3]
            r.csr = escoin.Csr.wrap_device(t[0].data_ptr(), t[1].data_ptr(), t[2].data_ptr(), t[1].numel(), L.M, L.C,
                                           L.H, L.W, L.K, L.stride, L.pad, device.index,
                                           torch.cuda.current_stream().cuda_stream)
            if args.kernel != -1:
                r.csr.set_kernel(args.kernel)
        else:
            r.csr = src
            r.csr.set_kernel(args.kernel)
            r.csr.to_device(device.index, torch.cuda.current_stream().cuda_stream)
            r.bias = torch.from_numpy(bias).to(device)
        r.nnz = int(r.csr.info()["nnz"])
        # NEXT-1 engine selection: the dense tcgen05 engine below the measured sparsity crossover
        eng = getattr(args, "engine", "auto")
        if eng == "dense" or (eng == "auto" and escoin.select_engine(L.M, L.C, L.K, r.nnz) == escoin.ENGINE_DENSE_TC):
            r.csr.set_kernel(escoin.KERNEL_DENSE_TC)
            r.engine = "dense_tc"
        else:
            r.engine = "sparse"
        x = inputs.activations(wl.net, L.name, n0, B, L.C, L.H, L.W)
        r.h_x = torch.from_numpy(x).pin_memory()
        r.x = r.h_x.to(device)
        r.out = torch.empty((B, L.M, L.E, L.F), dtype=torch.float32, device=device)
        r.tune = None
        r.h_out = torch.empty((B, L.M, L.E, L.F), dtype=torch.float32).pin_memory()
        r.flops = 2.0 * B * r.nnz * L.E * L.F
        r.alg_bytes = 4.0 * (B * L.C * L.H * L.W + B * L.M * L.E * L.F + 2 * r.nnz + L.M + 1 + L.M)
        runs.append(r)
    torch.cuda.synchronize()
    setup_t = {}
    if args.kernel == -1 and not args.no_jit:
        # pattern-specialised kernels (escoin_csr_jit): compiled at setup, untimed.  Every (layer,
        # tuning) is submitted at once; the library bounds concurrent compiler threads to the host's
        # cores and splits large layers into units compiled in parallel.  Rank 0 compiles into the
        # node's cubin cache (ESCOIN_JIT_CACHE) first; the other ranks then load the same cubins.
        tunings = [[int(v) for v in t.split(",")] if t.strip() not in ("", "0") else []
                   for t in args.jit_tunings.split(";")]

        def jit(task):
            r, tun = task
            if r.engine != "sparse":
                return None
            try:
                r.csr.jit(B, *tun)
            except escoin.EscoinError as e:
                if e.status != escoin.ERR_UNSUPPORTED:
                    raise
                return None
            st = r.csr.jit_stats()
            return st["compile_s"], st["cache_hits"], st["units"]
        tasks = [(r, t) for r in runs for t in tunings]
        tasks.sort(key=lambda rt: -rt[0].nnz)  # largest compiles first

        def compile_all():
            t0 = time.time()
            with ThreadPoolExecutor(max(1, min(len(tasks), 64))) as ex:
                for (r, _), res in zip(tasks, ex.map(jit, tasks)):
                    if res is not None:
                        r.jit_s = round(getattr(r, "jit_s", 0.0) + res[0], 2)
                        r.jit_hits = getattr(r, "jit_hits", 0) + res[1]
            return round(time.time() - t0, 1)
        if world > 1 and rank != 0:
            torch.distributed.barrier()  # rank 0 compiles first
        setup_t["jit_compile_wall_s"] = compile_all()
        if world > 1 and rank == 0:
            torch.distributed.barrier()
    t0 = time.time()
    for r in runs:
        if args.kernel == -1 and not args.no_autotune and r.engine == "sparse":
            # kernel customization (paper §3.4): measured once at setup, untimed, each candidate
            # timed alone after an L2 flush like the timed steps (escoin_csr_autotune_ex)
            flags = escoin.TUNE_JIT
            if args.tune_variants or getattr(r, "jit_s", None) is None:
                flags |= escoin.TUNE_VARIANTS
            kid, kms = r.csr.autotune_ex(B, r.x, r.out, r.bias, True, 5, torch.cuda.current_stream().cuda_stream,
                                         flush=flush, flags=flags)
            r.tune = {"kernel_id": kid, "ms": round(kms, 4)}
        r.kernel = r.csr.label()
        r.units = r.csr.jit_info()["units"] if r.csr.kernel() == escoin.KERNEL_JIT else 1
    setup_t["autotune_s"] = round(time.time() - t0, 1)
    torch.cuda.synchronize()
    return runs, n0, B, GB, setup_t


def fwd(escoin, r, stream):
    L = r.L
    escoin.sconv_forward(r.x.shape[0], L.C, L.H, L.W, L.M, L.K, L.stride, L.pad, r.csr, r.x, r.out, r.bias, True,
                         stream)


def time_device(torch, runs, steps, warmup, flush, step_fn):
    """Eager launches, per-step CUDA events around each layer; L2 flushed before every step."""
    s = torch.cuda.current_stream()
    for _ in range(warmup):
        flush.zero_()
        step_fn()
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(runs) + 1)] for _ in range(steps)]
    for k in range(steps):
        flush.zero_()
        if k == 0:  # ncu --nvtx --nvtx-include "layers/" captures exactly one launch per layer
            torch.cuda.nvtx.range_push("layers")
        ev[k][0].record(s)
        for i, r in enumerate(runs):
            step_fn(i)
            ev[k][i + 1].record(s)
        if k == 0:
            torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    per_layer = np.array([[ev[k][i].elapsed_time(ev[k][i + 1]) for i in range(len(runs))] for k in range(steps)])
    return per_layer  # ms [steps][layers]


def capture_step(torch, step_fn):
    """The whole step (every layer's launch, incl. multi-unit fork/join) as one CUDA graph."""
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):  # one eager pass on the capture stream first (module/bind warm-up)
        step_fn()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step_fn()
    torch.cuda.synchronize()
    return g


def time_graph(torch, g, steps, warmup, flush):
    """K replays of the step graph, each between its own events; L2 flushed before every step (outside)."""
    s = torch.cuda.current_stream()
    for _ in range(warmup):
        flush.zero_()
        g.replay()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include "timed/" profiles only these launches
    for a, b in ev:
        flush.zero_()
        a.record(s)
        g.replay()
        b.record(s)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    return np.array([a.elapsed_time(b) for a, b in ev])  # ms per step


def cpu_oracle_timed(wl, args, seconds, max_images):
    """Time only the oracle calls (inputs pre-generated) on a bounded image sample."""
    import oracle
    items = []
    for L in wl.layers:
        w = (inputs.layer_weights_skewed if getattr(args, "skew", False) else inputs.layer_weights)(
            wl.net, L, args.sparsity)
        items.append((L, oracle.csr_stretch(w, L.H, L.W, L.stride, L.pad), inputs.bias(wl.net, L.name, L.M)))
    el = 0.0
    n = 0
    while n < max_images and el < seconds:
        for L, (rp, ci, v), b in items:
            x = inputs.activations(wl.net, L.name, n, 1, L.C, L.H, L.W)
            ts = time.perf_counter()
            oracle.sconv(x, rp, ci, v, L.M, L.K, L.stride, L.pad, bias=b, relu=True)
            el += time.perf_counter() - ts
        n += 1
    return n, el, oracle.num_threads()


def cpu_model():
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def sm_peak_tflops(torch, device, sm_max_mhz):
    props = torch.cuda.get_device_properties(device)
    # FP32 FFMA: 128 lanes/SM x 2 flop x clock (B200_PROFILING / blackwell guide unit counts)
    return props.multi_processor_count * 128 * 2 * sm_max_mhz * 1e6 / 1e12, props.multi_processor_count


def load_traffic(workload):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(path)).get(workload, {})
    except Exception:
        return {}


def load_ffma_peak():
    """The FFMA microbenchmark's measured FP32 peak (profiles/ffma_peak.json), for context."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ffma_peak.json")))
        return {"tflops": d.get("best_tflops"), "source": "profiles/ffma_peak.json"}
    except Exception:
        return None


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank, world, _ = shard.world()
    if rank != 0:
        return 0
    wl = workloads.workload(args.workload)
    import oracle
    items = []
    for L in wl.layers:
        w = inputs.layer_weights(wl.net, L, args.sparsity)
        items.append((L, oracle.csr_stretch(w, L.H, L.W, L.stride, L.pad), inputs.bias(wl.net, L.name, L.M)))
    per_step_images = 8  # a bounded sample of the batch per step (keeps all host cores busy)
    xs = {L.name: inputs.activations(wl.net, L.name, 0, per_step_images, L.C, L.H, L.W) for L, _, _ in items}

    def step():
        for L, (rp, ci, v), b in items:
            oracle.sconv(xs[L.name], rp, ci, v, L.M, L.K, L.stride, L.pad, bias=b, relu=True)

    for _ in range(args.warmup):
        step()
    t = []
    for _ in range(args.steps):
        ts = time.perf_counter()
        step()
        t.append(time.perf_counter() - ts)
    ms = 1e3 * float(np.mean(t))
    value = per_step_images / (ms / 1e3)
    sample = "%d image(s) through all %d layers per step" % (per_step_images, len(items))
    line = {"metric": METRIC, "value": value, "unit": "images/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": WL_NAMES[args.workload], "global_batch": wl.batch,
                       "sparsity": args.sparsity / 1000.0, "sample": sample},
            "cpu_baseline": {"value": value, "unit": "images/s", "cores": oracle.num_threads(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    if args.out:
        open(args.out, "w").write(json.dumps(line) + "\n")
    return 0


# ------------------------------------------------------------------ main
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    from paper_1802_10280_b200 import escoin

    rank, world, local = shard.world()
    device = torch.device("cuda", 0 if args.same_device else local)
    torch.cuda.set_device(device)
    if world > 1:
        import datetime

        import torch.distributed as dist
        # setup compiles the specialised kernels while the other ranks wait at a barrier
        to = datetime.timedelta(minutes=60)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=device, timeout=to)
        else:
            dist.init_process_group(args.dist_backend, timeout=to)
    wl = workloads.workload(args.workload)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)
    runs, n0, B, GB, setup_t = setup(args, wl, device, rank, world, torch, escoin, flush)
    stream = torch.cuda.current_stream().cuda_stream
    images = GB if not args.weak else B * world  # images all ranks process per step

    def step_fn(i=None):
        s_ = torch.cuda.current_stream().cuda_stream  # the capture stream inside torch.cuda.graph
        if i is None:
            for r in runs:
                fwd(escoin, r, s_)
        else:
            fwd(escoin, runs[i], s_)

    graph = None if args.no_graph else capture_step(torch, step_fn)
    # one kernel launch per layer (linked units are one kernel); split-channel layers (_k) add the reduce
    launches_per_step = sum(2 if "_k" in r.kernel else 1 for r in runs)

    # ---------------- device-timed region (K steps, barrier + sync both sides)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        wall0 = time.perf_counter()
        if graph is not None:
            step_times = time_graph(torch, graph, args.steps, args.warmup, flush)
        else:
            step_times = time_device(torch, runs, args.steps, args.warmup, flush, step_fn).sum(1)
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    if world > 1:
        torch.distributed.barrier()
    step_ms_local = float(np.mean(step_times))
    step_ms = shard.max_over_ranks(step_ms_local, device)
    value = images / (step_ms / 1e3)
    # per-layer breakdown (the roofline's dominant kernel): the same launches eagerly, one event
    # pair per layer on the launching stream, same flush, same number of steps
    per_layer = time_device(torch, runs, args.steps, max(2, args.warmup // 2), flush, step_fn)
    layer_ms = per_layer.mean(0)
    layer_ms_min, layer_ms_med = per_layer.min(0), np.median(per_layer, 0)

    # ---------------- e2e through the C-ABI with host buffers
    # Every step copies each layer's input from pinned host memory, runs the
    # layer and copies its output back (escoin_sconv_forward_hostio).  Layers
    # run on their own streams so one layer's H2D overlaps another's compute
    # and D2H (PCIe is full duplex), and consecutive steps alternate between
    # two buffer sets per layer (double buffering), so step i+1's H2D does not
    # wait for step i's D2H of the same layer.
    e2e_streams = [[torch.cuda.Stream(device), torch.cuda.Stream(device)] for _ in runs]
    for r in runs:
        r.e2e_buf = [(r.x, r.out, r.h_out),
                     (torch.empty_like(r.x), torch.empty_like(r.out), torch.empty_like(r.h_out).pin_memory())]
    e2e_i = [0]

    def e2e_step():
        k = e2e_i[0] & 1
        e2e_i[0] += 1
        for r, sts in zip(runs, e2e_streams):
            L = r.L
            dx, dout, hout = r.e2e_buf[k]
            escoin.sconv_forward_hostio(B, L.C, L.H, L.W, L.M, L.K, L.stride, L.pad, r.csr, r.h_x, hout, dx,
                                        dout, r.bias, True, sts[k].cuda_stream)

    e2e_steps = max(4, min(args.steps, 20))
    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for sts in e2e_streams:
        for st in sts:
            st.wait_event(e0)
    for _ in range(e2e_steps):
        e2e_step()
    for sts in e2e_streams:
        for st in sts:
            torch.cuda.current_stream().wait_stream(st)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = shard.max_over_ranks(e0.elapsed_time(e1) / e2e_steps, device)
    h2d = sum(r.h_x.numel() * 4 for r in runs)
    d2h = sum(r.h_out.numel() * 4 for r in runs)

    # ---------------- roofline of the dominant kernel
    peaks = measured_peaks()
    clocks = clk.summary()
    sm_max = clocks.get("sm_max_mhz") or peaks.get("sm_max_mhz") or 1965.0
    peak_tf, nsm = sm_peak_tflops(torch, device, sm_max)
    dom = int(np.argmax(layer_ms))
    rd = runs[dom]
    achieved = rd.flops / (layer_ms[dom] / 1e3) / 1e12
    bound, peak_used, peak_basis = "alu", peak_tf, "FP32 FFMA %d SMs x 128 lanes x 2 x %.0f MHz (derived, DESIGN.md)" % (
        nsm, sm_max)
    if rd.engine == "dense_tc":  # 3xTF32 on tcgen05: three TF32 MMAs per FP32-accurate product
        tf32 = (peaks.get("bf16_tflops") or 2250.0) * 0.5
        bound, peak_used = "tensor", tf32 / 3.0
        peak_basis = "TF32 dense = 0.5 x measured BF16 %.0f TFLOP/s (nominal ratio), / 3 for 3xTF32" % (2 * tf32)
    traffic = load_traffic(args.workload).get(rd.L.name)
    layers_out = []
    for r, ms, mn, md in zip(runs, layer_ms, layer_ms_min, layer_ms_med):
        layers_out.append({"layer": r.L.name, "ms": round(float(ms), 5), "ms_min": round(float(mn), 5),
                           "ms_median": round(float(md), 5), "kernel": r.kernel, "nnz": r.nnz,
                           "jit_compile_s": getattr(r, "jit_s", None), "units": r.units, "engine": r.engine,
                           "autotune_ms": (r.tune or {}).get("ms"),
                           "gflop": round(r.flops / 1e9, 4),
                           "tflops": round(r.flops / (ms / 1e3) / 1e12, 3),
                           "frac_fp32": round(r.flops / (ms / 1e3) / 1e12 / peak_tf, 4),
                           "alg_gbs": round(r.alg_bytes / (ms / 1e3) / 1e9, 1)})

    line = {"metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded; He-normal weights magnitude-pruned, "
                                                      "U[0,1) activations)",
            "config": {"workload": WL_NAMES[args.workload], "global_batch": images, "batch_per_gpu": B,
                       "rank0_images": [n0, n0 + B],
                       "sparsity": args.sparsity / 1000.0, "sparsity_note": "ASSUMED 80% (paper prints none)",
                       "row_sparsity": "skewed Beta(1,b) per row" if args.skew else "uniform (magnitude pruning)",
                       "parallelism": "dp%d (batch-sharded, weights replicated)" % world,
                       "timing": "CUDA graph of the whole step" if graph is not None else "eager launches",
                       "l2": "flushed (256 MB write) before every step, outside the per-step events"},
            "roofline": {"bound": bound, "achieved": round(achieved, 3), "peak": round(peak_used, 2),
                         "unit": "TFLOP/s", "frac": round(achieved / peak_used, 4), "traffic": traffic,
                         "kernel": "sconv %s (%s)" % (rd.kernel, rd.L.name),
                         "peak_basis": peak_basis,
                         "hbm_view": {"alg_gbs": round(rd.alg_bytes / (layer_ms[dom] / 1e3) / 1e9, 1),
                                      "peak_gbs": peaks.get("hbm_gbs")},
                         "measured_ffma_peak": load_ffma_peak(),
                         "stack": {"gflop": round(sum(r.flops for r in runs) / 1e9, 3),
                                   "tflops_graph": round(sum(r.flops for r in runs) / (step_ms_local / 1e3) / 1e12, 3),
                                   "frac_graph": round(sum(r.flops for r in runs) / (step_ms_local / 1e3) / 1e12
                                                       / peak_tf, 4)}},
            "layers": layers_out,
            "e2e": {"value": images / (e2e_ms / 1e3), "unit": "images/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "setup": setup_t,
            "wall_s_timed_region": round(wall, 3)}

    if rank == 0 and world == 1 and not args.no_baselines:
        line["baselines"] = run_baselines(torch, escoin, runs, flush, stream, args, value)
    if rank == 0 and world == 1 and not args.no_cpu:
        n, el, cores = cpu_oracle_timed(wl, args, args.cpu_seconds, B)
        line["cpu_baseline"] = {"value": n / el, "unit": "images/s", "cores": cores, "kind": "oracle",
                                "sample": "%d image(s) x %d layers, fp64 oracle (OpenMP over (n,m))" % (n, len(runs)),
                                "cpu_model": cpu_model()}
        import oracle
        oracle.set_threads(1)  # per-core rate: one image through the stack on one thread
        n1, el1, _ = cpu_oracle_timed(wl, args, max(2.0, args.cpu_seconds / 4), 1)
        oracle.set_threads(cores)
        line["cpu_baseline"]["one_thread"] = {"value": n1 / el1, "unit": "images/s", "sample": "%d image(s)" % n1}
    if rank == 0:
        s = json.dumps(line)
        print(s, flush=True)
        if args.out:
            open(args.out, "w").write(s + "\n")
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def run_baselines(torch, escoin, runs, flush, stream, args, sconv_value):
    """im2col+cuBLAS, im2col+cuSPARSE, cuDNN and the paper's own mapping, same inputs/outputs."""
    import baselines as bl
    out = {}
    reps, warm = 5, 2
    s = torch.cuda.current_stream()

    def time_fn(fn):
        for _ in range(warm):
            flush.zero_()
            fn()
        torch.cuda.synchronize()
        tot = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            fn()
            b.record(s)
            torch.cuda.synchronize()
            tot.append(a.elapsed_time(b))
        return float(np.median(tot))

    B = runs[0].x.shape[0]
    names = {"cublas": "im2col+cublas_sgemm", "cublas_gemm": "im2col+cublas_sgemm_one_gemm_per_batch",
             "cusparse": "im2col+cusparse_spmm", "cudnn": "cudnn_fp32_dense",
             "cudnn_tf32": "cudnn_tf32_dense_tensorcore", "cudnn_bf16": "cudnn_bf16_dense_tensorcore"}
    for mode in ["cublas", "cublas_gemm", "cusparse", "cudnn", "cudnn_tf32", "cudnn_bf16"]:
        per = {}
        try:
            for r in runs:
                if mode.startswith("cudnn"):
                    op = bl.CudnnConv(r.L, r.w_dense, r.bias.cpu().numpy(), r.x.device,
                                      {"cudnn": "fp32", "cudnn_tf32": "tf32", "cudnn_bf16": "bf16"}[mode])
                else:
                    op = bl.LoweredConv(r.L, r.w_dense, r.bias.cpu().numpy(), r.x.device, mode)
                y = torch.empty_like(r.out)
                per[r.L.name] = time_fn(lambda: op(r.x, y))
                del op, y
            tot = sum(per.values())
            out[names[mode]] = {
                "images_per_s": B / (tot / 1e3), "ms_per_layer": {k: round(v, 4) for k, v in per.items()},
                "escoin_speedup": round(sconv_value / (B / (tot / 1e3)), 3)}
        except Exception as e:  # report, do not hide
            out[mode] = {"error": repr(e)[:300]}
        torch.cuda.empty_cache()
    # our own dense tcgen05 implicit GEMM (the north_star comparison point), TF32 and 3xTF32
    for nsplit, key in [(1, "dense_tcgen05_tf32"), (3, "dense_tcgen05_3xtf32")]:
        per = {}
        for r in runs:
            L = r.L
            wd = torch.from_numpy(np.ascontiguousarray(r.w_dense)).to(r.x.device)
            y = torch.empty_like(r.out)
            per[L.name] = time_fn(lambda: escoin.bench_dense_tc_forward(wd, r.x, r.bias, L.stride, L.pad, True,
                                                                        nsplit, out=y, stream=s))
            del wd, y
        tot = sum(per.values())
        out[key] = {"images_per_s": B / (tot / 1e3), "ms_per_layer": {k: round(v, 4) for k, v in per.items()},
                    "escoin_speedup": round(sconv_value / (B / (tot / 1e3)), 3)}
    # the paper's Pascal-era mapping (variant 0) on B200, as an ablation
    per = {}
    for r in runs:
        L = r.L
        c = escoin.Csr.stretch(r.w_dense, L.H, L.W, L.stride, L.pad)
        c.set_kernel(0)
        c.to_device(r.x.device.index, stream)
        per[L.name] = time_fn(lambda: escoin.sconv_forward(B, L.C, L.H, L.W, L.M, L.K, L.stride, L.pad, c, r.x,
                                                           r.out, r.bias, True, stream))
        c.free()
    tot = sum(per.values())
    out["escoin_paper_mapping"] = {"images_per_s": B / (tot / 1e3),
                                   "ms_per_layer": {k: round(v, 4) for k, v in per.items()},
                                   "escoin_speedup": round(sconv_value / (B / (tot / 1e3)), 3)}
    return out


if __name__ == "__main__":
    sys.exit(main())
