"""Benchmark: KAN/UKAN layer fwd+bwd samples/s on 1..8 B200 vs the CPU reference path.

Headline workload (BASELINE.json configs[2], the largest single-GPU configuration):
cfg3 — one KAN layer 4096 -> 4096, grid G = 64, k = 3, batch 65536 PER GPU (weak scaling), x ~
U(-1, 1) with a 1% clamp-exercising tail, upstream gradient ~ N(0, 1).  One "step" = the layer's
data-parallel training step as a hidden layer of a stack (``LayerTrainer.step``): forward,
backward INCLUDING dx, the dcoeffs/dscale all-reduce in 8 feature buckets overlapping the backward
(N > 1, NCCL), and the fused Adam update of the layer's 1.1 G parameters.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU, NCCL)

Prints one JSON line on rank 0.  ``value`` is device-timed (CUDA events on the launching stream,
inputs resident in HBM, x > L2, max over ranks); ``e2e`` is the same step through the public API
with x and gy copied from pinned host memory and y and dx copied back every step.  The CPU
reference arm (``--impl reference``, and the ``cpu_baseline`` field) runs the UNMODIFIED reference
package (installed by __graft_entry__.build() into the git-ignored baseline/_ref) on the box's
host cores — or, if that install is absent, its float64 NumPy restatement in oracle/.
Supplementary fields (not the headline): cfg2 (KAN [784,256,10] DP step), cfg4 (UKAN 1024 -> 1024
at B = 65536, and the B = 4096 variant), cfg5 (UKAN [64,512,512,64] DP training, global batch
65536 sharded), cfg1 (autograd API and as a captured step), PINN.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF = os.path.join(ROOT, "baseline", "_ref")

CFG3 = dict(d=4096, G=64, k=3, g_min=-1.0, g_max=1.0, batch=65536, tail=0.01, lr=1e-3)
METRIC = "KAN/UKAN layer fwd+bwd samples/s & HBM GB/s vs peak at 1/2/4/8 B200 vs CPU"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_fallback": True}


# Compute roofs measured on this pool's B200 with the microbenchmarks in tools/ (clocks not locked):
# FMA chains (tools/peaks.cu -> profiles/peaks_r01.json), FP64 DMMA m8n8k4 (tools/dmma_peak.cu ->
# profiles/dmma_peak_r01.json).  MEASURED_PEAKS.json holds only HBM and bf16.
FP32_TFLOPS_MEASURED = 71.95
FP64_TFLOPS_MEASURED = 34.05
DMMA_TFLOPS_MEASURED = 37.0


def kan_flops(B, d_in, d_out, k):
    """Algorithmic FLOPs of one KAN layer pass: 2*K*B*d_in*d_out per pass."""
    return 2.0 * (k + 1) * B * d_in * d_out


def kan_bytes(B, d_in, d_out, G, k, dx=True):
    """Compulsory HBM bytes of one KAN layer fwd+bwd: x, y, dy, dx, C read +
    dC write, scale + dscale."""
    return 4.0 * (B * d_in + 2 * B * d_out + (B * d_in if dx else 0) + 2 * d_in * (G + k) * d_out + 2 * d_in * d_out)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        self.tmp = tempfile.NamedTemporaryFile("w+", delete=False, suffix=".csv")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.tmp, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait()
        self.tmp.seek(0)
        for line in self.tmp.read().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)
        os.unlink(self.tmp.name)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[2:]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------------------
# CPU reference path: the reference's own kan_forward + tape backward (x a recorded node) at
# cfg3 sub-batches of 1 and 4 rows; the marginal rate (3 rows / (t4 - t1)) removes the fixed
# cost of the full zeros_like(table) in span_gather's backward (layers.py:68).
# ---------------------------------------------------------------------------------------
def _ref_available() -> bool:
    return os.path.isdir(os.path.join(REF, "ukan"))


def _cpu_worker(args):
    reps, seed = args
    os.environ["OMP_NUM_THREADS"] = "1"
    d, G, k = CFG3["d"], CFG3["G"], CFG3["k"]
    rng = np.random.default_rng(seed)
    pairs = []
    if _ref_available():
        if REF not in sys.path:
            sys.path.insert(0, REF)
        import ukan
        T = ukan.tensor
        layer = ukan.init_layer("kan", d, d, k, seed=seed, g_min=CFG3["g_min"], g_max=CFG3["g_max"], G=G)

        def run(B):
            x = T.parameter(rng.uniform(-1, 1, (B, d)))
            g = T.as_tensor(rng.normal(size=(B, d)))
            t0 = time.perf_counter()
            y = ukan.kan_forward(layer, x)
            T.backward(T.sum_all(T.mul(y, g)))
            return time.perf_counter() - t0
    else:
        import oracle
        C = rng.normal(0, 0.1 / np.sqrt(d), (d, G + k, d))
        S = np.ones((d, d))

        def run(B):
            x = rng.uniform(-1, 1, (B, d))
            g = rng.normal(size=(B, d))
            t0 = time.perf_counter()
            oracle.kan_forward_backward(x, C, S, g, k=k, g_min=CFG3["g_min"], g_max=CFG3["g_max"], G=G)
            return time.perf_counter() - t0
    for _ in range(reps):
        t1 = run(1)
        t4 = run(4)
        pairs.append((t1, t4))
    return pairs


def cpu_rate(procs: int, reps: int):
    """cfg3 samples/s of the CPU reference path on `procs` host processes (sum of their marginal
    rates); returns (rate, per-process seconds per marginal sample, pairs)."""
    if procs == 1:
        pairs = _cpu_worker((reps, 0))
        all_pairs = [pairs]
    else:
        import multiprocessing as mp
        with mp.get_context("spawn").Pool(procs) as pool:
            all_pairs = pool.map(_cpu_worker, [(reps, i) for i in range(procs)])
    rates = []
    for pairs in all_pairs:
        dt = statistics.median(max(1e-9, t4 - t1) for t1, t4 in pairs)
        rates.append(3.0 / dt)
    return sum(rates), all_pairs


def _cpu_procs():
    ncpu = len(os.sched_getaffinity(0))
    try:
        mem_gb = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 2**30
    except (ValueError, OSError):
        mem_gb = 64
    # measured peak RSS of one reference process at cfg3, B = 4: 40 GB (the float64 coefficients,
    # zeros_like(table) in span_gather's backward and the einsum temporaries); keep 10% headroom
    return max(1, min(ncpu, int(mem_gb // 44)))


def reference_arm(args, rank):
    if rank != 0:
        return
    procs = _cpu_procs()
    reps = 1  # one (B=1, B=4) pair per process: ~25 s of reference work after a ~24 s layer init
    t0 = time.perf_counter()
    rate, pairs = cpu_rate(procs, reps)
    wall = time.perf_counter() - t0
    kind = "reference" if _ref_available() else "port"
    sample = (f"{procs} host processes x {reps} (B=1, B=4) pairs of the {'unmodified reference (baseline/_ref ukan: kan_forward + T.backward, x a T.parameter)' if kind == 'reference' else 'float64 NumPy port (oracle/)'} "
              f"on the cfg3 layer; marginal rate 3 rows / (t4 - t1) per process, summed; OMP_NUM_THREADS=1")
    ms = 1e3 * 65536.0 / rate if rate > 0 else None
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg3: KAN layer 4096->4096 G=64 k=3, fwd + bwd incl. dx (per-sample marginal cost)",
                   "global_batch": CFG3["batch"], "parallelism": f"{procs} host processes"},
        "cpu_baseline": {"value": rate, "unit": "samples/s", "cores": procs, "kind": kind, "sample": sample,
                         "cpu": cpu_model(), "wall_s": wall, "pairs_s": pairs},
        "e2e": {"value": rate, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------
def _events(timers):
    return {name: sum(a.elapsed_time(b) for a, b in ev) / len(ev) for name, ev in timers.items()}


def our_arm(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2408_11200_b200 as P

    dev_index = local_rank % torch.cuda.device_count()  # == local_rank on a full node
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    d, G, k, B = CFG3["d"], CFG3["G"], CFG3["k"], CFG3["batch"]

    def barrier():
        if world > 1:
            dist.barrier()

    layer = P.init_layer("kan", d, d, k, seed=0, g_min=CFG3["g_min"], g_max=CFG3["g_max"], G=G, device=dev)
    tr = P.LayerTrainer(layer, CFG3["lr"], buckets=8)
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    xs, gys = [], []
    for _ in range(2):  # two resident batches (each x is 1 GiB > the 126 MB L2)
        x = torch.rand((B, d), device=dev, generator=g) * 2 - 1
        m = torch.rand((B, d), device=dev, generator=g) < CFG3["tail"]
        xs.append(torch.where(m, x * 3, x))
        gys.append(torch.randn((B, d), device=dev, generator=g) / (B * world))
        del x, m
    for s in range(args.warmup):
        tr.step(xs[s % 2], gys[s % 2])
    torch.cuda.synchronize()
    tr.check_input()
    barrier()

    # ---- device-timed region (inputs resident in HBM) ----
    lib = P._lib.load()
    launches0 = lib.ukan_launch_count()
    tr.timers = {}
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev_index) as clk:
        torch.cuda.synchronize()
        barrier()
        start.record()
        for s in range(args.steps):
            tr.step(xs[s % 2], gys[s % 2])
        end.record()
        torch.cuda.synchronize()
        barrier()
    launches = (lib.ukan_launch_count() - launches0) // max(1, args.steps)
    ms = start.elapsed_time(end)
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * B * args.steps / (ms_max * 1e-3)
    timers, tr.timers = tr.timers, None
    phase_ms = _events(timers)
    # per-kernel launch timing of the dominant kernels on the launching stream (one extra step,
    # not in the timed region): the backward parts are separate launches already
    tr.check_input()

    # ---- end to end through the public API: pinned host x / gy in, y / dx out, every step ----
    hx = [torch.empty((B, d), dtype=torch.float32).pin_memory() for _ in range(2)]
    hg = [torch.empty((B, d), dtype=torch.float32).pin_memory() for _ in range(2)]
    hy = torch.empty((B, d), dtype=torch.float32).pin_memory()
    hdx = torch.empty((B, d), dtype=torch.float32).pin_memory()
    for i in range(2):
        hx[i].copy_(xs[i].cpu())
        hg[i].copy_(gys[i].cpu())
    del xs, gys
    torch.cuda.empty_cache()
    e2e_steps = max(3, min(args.steps, 5))
    out_stream = torch.cuda.Stream(device=dev)
    runs = []
    for _ in range(2):
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for bx, bg in P.DevicePrefetcher(((hx[s % 2], hg[s % 2]) for s in range(e2e_steps)), dev):
            y, dx = tr.step(bx, bg)
            ev = torch.cuda.Event()
            ev.record()
            out_stream.wait_stream(torch.cuda.current_stream(dev))  # outputs of this step -> host
            with torch.cuda.stream(out_stream):
                hy.copy_(y, non_blocking=True)
                hdx.copy_(dx, non_blocking=True)
                y.record_stream(out_stream)
                dx.record_stream(out_stream)
        out_stream.synchronize()
        torch.cuda.synchronize()
        tt = torch.tensor([time.perf_counter() - t0], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        runs.append(float(tt.item()))
    e2e_s = min(runs)
    e2e_value = world * B * e2e_steps / e2e_s
    del tr, layer, hx, hg, hy, hdx
    torch.cuda.empty_cache()

    supp = {}
    if not args.no_configs:
        supp["cfg5_ukan_dp"] = cfg5_rate(dev, world, rank)
        if world == 1:
            supp["cfg2_kan_stack_dp"] = cfg2_rate(dev)
            supp["ukan_layer"] = ukan_layer_rate(dev)
            supp["cfg4_ukan_layer"] = cfg4_rate(dev)
            supp["kan_layers"] = kan_layer_rates(dev)  # cfg1 (autograd API and as a captured step)
            supp["pinn"] = pinn_rate(dev)
    if rank != 0:
        return
    pk = peaks()
    # dominant kernel: the longest phase of the step (each phase is one kernel launch, or one
    # launch per feature bucket for the table gradient)
    f_pass = kan_flops(B, d, d, k)
    phase_info = {
        "forward": ("kan_fwd_tm_kernel (TMEM gather, FP32 FMA; + pack / records pre-passes)", FP32_TFLOPS_MEASURED,
                    "fp32 FMA (tools/peaks.cu)"),
        "backward_dx": ("kan_dx_tc_kernel (dx on FP64 DMMA)", DMMA_TFLOPS_MEASURED, "FP64 DMMA (tools/dmma_peak.cu)"),
        "backward_table": ("kan_bwd_tc3_sweep_kernel<16,4,4,4> x 8 feature buckets (dC/dscale on FP64 DMMA, TMA-fed)",
                           DMMA_TFLOPS_MEASURED, "FP64 DMMA (tools/dmma_peak.cu)"),
    }
    dom = max((p for p in phase_info if p in phase_ms), key=lambda p: phase_ms[p])
    dom_ms = phase_ms[dom]
    kern, dom_peak, peak_src = phase_info[dom]
    achieved = f_pass / (dom_ms * 1e-3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "traffic.json")) as f:
            traffic = json.load(f).get("cfg3." + dom, {}).get("dram_bytes")
    except (OSError, ValueError):
        traffic = None
    hbm = kan_bytes(B, d, d, G, k)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        rate1, pairs = cpu_rate(1, 1)
        cpu = {"value": rate1, "unit": "samples/s", "cores": 1, "kind": "reference" if _ref_available() else "port",
               "sample": ("one (B=1, B=4) pair of the cfg3 layer fwd+bwd incl. dx through the "
                          + ("unmodified reference (baseline/_ref ukan)" if _ref_available() else "float64 port (oracle/)")
                          + f"; marginal rate 3/(t4-t1); t1={pairs[0][0][0]:.1f} s, t4={pairs[0][0][1]:.1f} s; OMP_NUM_THREADS=1"),
               "cpu": cpu_model()}
    step_tflops = 3 * f_pass * args.steps / (ms_max * 1e-3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 storage; f64 grid locate + backward accumulation (DMMA)",
        "data": "synthetic (x ~ U(-1,1) with a 1% |x|<=3 clamp tail; upstream gradient ~ N(0,1)/global batch)",
        "config": {"workload": "cfg3: KAN layer 4096->4096 G=64 k=3, one DP training step of the layer as a hidden "
                               "layer (fwd + bwd incl. dx + bucketed grad all-reduce + Adam)",
                   "global_batch": B * world, "per_gpu_batch": B, "parallelism": f"dp{world}",
                   "l2": "inputs larger than L2 (x, gy 1 GiB each; two resident batches alternate)"},
        "roofline": {"bound": "tensor" if "DMMA" in peak_src else "fp32-fma", "kernel": kern, "achieved": achieved,
                     "peak": dom_peak, "unit": "TFLOP/s", "frac": achieved / dom_peak, "traffic": traffic,
                     "traffic_unit": "bytes per launch group (ncu dram__bytes_read+write, profiles/r02/traffic.json)",
                     "peak_source": peak_src, "algorithmic_flops_per_launch": f_pass, "avg_launch_ms": dom_ms},
        "roofline_hbm": {"bound": "hbm", "achieved": hbm / (ms_max / args.steps * 1e-3) / 1e9, "peak": pk["hbm_gbs"],
                         "unit": "GB/s", "frac": hbm / (ms_max / args.steps * 1e-3) / 1e9 / pk["hbm_gbs"],
                         "note": "compulsory bytes of the whole layer step (SURVEY 8d D2); the step is compute-bound "
                                 "(FP32 forward, FP64 backward forced by the parity bar)"},
        "roofline_phases": {  # every phase of the step against its own pipe (useful flops: 2*K*B*d_in*d_out)
            ph: {"kernel": phase_info[ph][0], "ms": phase_ms[ph], "achieved_tflops": f_pass / (phase_ms[ph] * 1e-3) / 1e12,
                 "peak_tflops": phase_info[ph][1],
                 "frac": f_pass / (phase_ms[ph] * 1e-3) / 1e12 / phase_info[ph][1],
                 "frac_of_banded_ceiling": (f_pass / (phase_ms[ph] * 1e-3) / 1e12 / (0.5 * phase_info[ph][1])
                                            if "DMMA" in phase_info[ph][2] else None)}
            for ph in phase_info if ph in phase_ms},
        "step_tflops": step_tflops,
        "roof_ms": (f_pass / (FP32_TFLOPS_MEASURED * 1e12) + 2 * f_pass / (FP64_TFLOPS_MEASURED * 1e12)) * 1e3,
        "phase_ms": phase_ms,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "e2e": {"value": e2e_value, "unit": "samples/s", "steps": e2e_steps, "runs_s": runs,
                "path": "LayerTrainer.step fed by DevicePrefetcher (pinned H2D of x, gy one step ahead); y and dx "
                        "copied to pinned host buffers on a side stream every step",
                "h2d_bytes_per_step": 2 * B * d * 4, "d2h_bytes_per_step": 2 * B * d * 4},
        "cpu_baseline": cpu,
        **supp,
    }
    print(json.dumps(line), flush=True)


def cfg2_rate(dev, steps=20, warmup=5):
    """Supplementary (the round-1 headline): KAN stack [784, 256, 10], G = 32, batch 8192,
    softmax-CE + Adam, one full training step captured as a CUDA graph."""
    import torch
    import paper_2408_11200_b200 as P
    from paper_2408_11200_b200 import ops
    B, widths = 8192, [784, 256, 10]
    model = P.build_model("kan", widths, 3, seed=0, device=dev, g_min=-1.0, g_max=1.0, G=32)
    tr = P.SplineTrainer(model, "softmax_cross_entropy", 1e-3, "adam")
    ops.set_check_mode("deferred")
    g = torch.Generator(device=dev)
    g.manual_seed(99)
    xs = [torch.rand((B, widths[0]), device=dev, generator=g) * 2 - 1 for _ in range(8)]
    ys = [torch.randint(0, widths[-1], (B,), device=dev, generator=g) for _ in range(8)]
    for s in range(warmup):
        tr.step(xs[s % 8], ys[s % 8])
    tr.read_loss(tr.step(xs[0], ys[0]))
    cap = tr.capture(xs[0], ys[0])
    for s in range(3):
        tr.read_loss(cap.replay(xs[s], ys[s]))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for s in range(steps):
        loss = cap.replay(xs[s % 8], ys[s % 8])
    b.record()
    torch.cuda.synchronize()
    tr.read_loss(loss)
    ops.flush_checks()
    ops.set_check_mode("eager")
    ms = a.elapsed_time(b) / steps
    return {"workload": "cfg2: KAN [784,256,10] G=32 k=3 B=8192 softmax-CE + Adam, one training step (CUDA graph)",
            "samples_per_s": B / (ms * 1e-3), "ms_per_step": ms, "steps": steps,
            "l2": "inputs rotate over 8 resident batches (196 MiB > L2)"}


def cfg5_rate(dev, world, rank, steps=5, warmup=2):
    """Supplementary cfg5 (shape proposed): UKAN denoiser-shaped
    stack [64, 512, 512, 64], delta_g = 0.4, d_pe = d_femb = 24, x ~ N(0, 1), MSE to N(0, 1)
    targets (epsilon prediction), Adam; GLOBAL batch 65536 sharded over the ranks (strong
    scaling), gradients all-reduced over NCCL."""
    import torch
    import torch.distributed as dist
    import paper_2408_11200_b200 as P
    from paper_2408_11200_b200.train import shard_bounds
    Bg = 65536
    lo, hi = shard_bounds(Bg, rank, world)
    Bl = hi - lo
    model = P.build_model("ukan", [64, 512, 512, 64], 3, seed=0, device=dev, delta_g=0.4, d_pe=24, d_femb=24)
    tr = P.SplineTrainer(model, "mse", 1e-3, "adam")
    g = torch.Generator(device=dev)
    g.manual_seed(5 + rank)
    x = torch.randn((Bl, 64), device=dev, generator=g)
    tgt = torch.randn((Bl, 64), device=dev, generator=g)
    for _ in range(warmup):
        tr.read_loss(tr.step(x, tgt, n_global=Bg))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        loss = tr.step(x, tgt, n_global=Bg)
    b.record()
    torch.cuda.synchronize()
    tr.read_loss(loss)
    ms = a.elapsed_time(b) / steps
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"workload": "cfg5: UKAN [64,512,512,64] k=3 delta_g=0.4 d_pe=d_femb=24, MSE + Adam, global batch 65536 "
                        f"sharded over {world} GPU(s) ({Bl} per GPU), NCCL all-reduce of the gradients",
            "samples_per_s": Bg / (ms * 1e-3), "ms_per_step": ms, "steps": steps, "scaling": "strong",
            "n_gpus": world, "path": "SplineTrainer.step (eager: one host read of the key count per UKAN layer); "
                    "dense layers (<= 67 rows per feature) on the FP64 tensor-core backward and the TMEM-gather forward"}


def ukan_layer_rate(dev, B=4096, steps=5, warmup=3):
    """Supplementary: one cfg4-shaped UKAN layer (1024 -> 1024, k=3, delta_g=0.5,
    d_pe=d_femb=32; x ~ N(0, 20^2)) forward + backward of x and every parameter through the
    drop-in API (key dedup, CG MLP, spline kernels), device-timed."""
    import torch
    import paper_2408_11200_b200 as P
    layer = P.init_layer("ukan", 1024, 1024, 3, seed=0, delta_g=0.5, d_pe=32, d_femb=32, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    x = (torch.randn((B, 1024), device=dev, generator=g) * 20.0).requires_grad_(True)
    gy = torch.randn((B, 1024), device=dev, generator=g)
    params = [x] + list(layer.parameters().values())
    for _ in range(warmup):
        torch.autograd.grad(P.ukan_forward(layer, x), params, gy)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        torch.autograd.grad(P.ukan_forward(layer, x), params, gy)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    n_u = P.ops.ukan_build_keys(x.detach(), 3, 0.5).n_u
    return {"workload": "UKAN layer 1024->1024 k=3 delta_g=0.5 d_pe=d_femb=32, x~N(0,20^2), B=4096 (cfg4-shaped)",
            "samples_per_s": B / (ms * 1e-3), "ms_per_step": ms, "n_u": n_u, "steps": steps, "warmup": warmup}


def cfg4_rate(dev, B=65536, steps=3, warmup=2):
    """Supplementary cfg4 at its SURVEY 8d D4 size: one UKAN layer 1024 -> 1024, k=3, delta_g=0.5,
    d_pe=d_femb=32, B = 65536, x ~ N(0, 20^2) with 0.1% of entries +-10^U(2,6) (criterion-10-style
    tails), forward + backward of x and every parameter through the drop-in API, device-timed."""
    import torch
    import paper_2408_11200_b200 as P
    layer = P.init_layer("ukan", 1024, 1024, 3, seed=0, delta_g=0.5, d_pe=32, d_femb=32, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(11)
    x = torch.randn((B, 1024), device=dev, generator=g) * 20.0
    m = torch.rand((B, 1024), device=dev, generator=g) < 0.001
    tails = torch.sign(torch.randn((B, 1024), device=dev, generator=g)) * 10.0 ** (
        2.0 + 4.0 * torch.rand((B, 1024), device=dev, generator=g))
    x = torch.where(m, tails, x).requires_grad_(True)
    del m, tails
    gy = torch.randn((B, 1024), device=dev, generator=g)
    params = [x] + list(layer.parameters().values())
    for _ in range(warmup):
        torch.autograd.grad(P.ukan_forward(layer, x), params, gy)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        torch.autograd.grad(P.ukan_forward(layer, x), params, gy)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    n_u = P.ops.ukan_build_keys(x.detach(), 3, 0.5).n_u
    out = {"workload": "cfg4: UKAN layer 1024->1024 k=3 delta_g=0.5 d_pe=d_femb=32, B=65536, x~N(0,20^2) + 0.1% "
                       "tails to 1e6, fwd + bwd of x and every parameter (drop-in API)",
           "samples_per_s": B / (ms * 1e-3), "ms_per_step": ms, "n_u": n_u, "steps": steps, "warmup": warmup}
    del layer, x, gy, params
    torch.cuda.empty_cache()
    return out


def kan_layer_rates(dev):
    """Supplementary configs[0] (cfg1: KAN 64 -> 64, G = 10, B = 1024): fwd + parameter grads
    through the drop-in API, device-timed, with its FP32/FP64 roof fraction."""
    import torch
    import paper_2408_11200_b200 as P
    from paper_2408_11200_b200 import ops
    d, G, B, steps = 64, 10, 1024, 50
    ops.set_check_mode("deferred")  # NaN flags checked once at the end instead of a host read per call
    layer = P.init_layer("kan", d, d, 3, seed=0, g_min=-1.0, g_max=1.0, G=G, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    x = torch.rand((B, d), device=dev, generator=g) * 2 - 1
    gy = torch.randn((B, d), device=dev, generator=g)
    params = [layer.coeffs, layer.scale]
    for _ in range(3):
        torch.autograd.grad(P.kan_forward(layer, x), params, gy)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        torch.autograd.grad(P.kan_forward(layer, x), params, gy)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    ops.flush_checks()
    ops.set_check_mode("eager")
    fl = kan_flops(B, d, d, 3)
    roof_ms = (fl / (FP32_TFLOPS_MEASURED * 1e12) + fl / (FP64_TFLOPS_MEASURED * 1e12)) * 1e3
    out = {"cfg1": {"workload": "KAN layer 64->64 G=10 k=3 B=1024, fwd + parameter grads (autograd API, "
                                "NaN checks deferred: ops.set_check_mode('deferred'))",
                    "samples_per_s": B / (ms * 1e-3), "ms_per_step": ms, "steps": steps, "roof_ms": roof_ms,
                    "roof_frac": roof_ms / ms}}
    # the same layer as a one-layer model's training step (MSE + Adam) captured as one CUDA graph:
    # the autograd figure above is host / launch bound, this is the device cost of the step
    model = P.build_model("kan", [d, d], 3, seed=0, device=dev, g_min=-1.0, g_max=1.0, G=G)
    tr = P.SplineTrainer(model, "mse", 1e-3, "adam")
    tgt = torch.randn((B, d), device=dev, generator=g)
    for _ in range(3):
        tr.read_loss(tr.step(x, tgt))
    cap = tr.capture(x, tgt)
    for _ in range(3):
        tr.read_loss(cap.replay())
    torch.cuda.synchronize()
    a.record()
    for _ in range(steps * 4):
        loss = cap.replay()
    b.record()
    torch.cuda.synchronize()
    tr.read_loss(loss)
    msg = a.elapsed_time(b) / (steps * 4)
    out["cfg1_graph_step"] = {"workload": "KAN [64,64] G=10 k=3 B=1024, MSE + Adam training step, one CUDA graph "
                                          "(SplineTrainer.capture; no dx: single layer)",
                              "samples_per_s": B / (msg * 1e-3), "ms_per_step": msg, "steps": steps * 4,
                              "roof_ms": roof_ms, "roof_frac": roof_ms / msg}
    return out


def pinn_rate(dev, n_colloc=128, steps=50, warmup=5):
    """Supplementary F2: one PINN step (pinn_loss through the forward-tangent kernels of a
    [1, 5, 1] KAN and UKAN, tasks.py:153-166, plus the reverse pass), device-timed."""
    import torch
    import paper_2408_11200_b200 as P
    out = {}
    for kind, kw in (("kan", dict(g_min=-5.0, g_max=5.0, G=10)), ("ukan", dict(delta_g=0.5, d_pe=8, d_femb=8))):
        model = P.build_model(kind, [1, 5, 1], 3, seed=0, device=dev, **kw)
        prob = P.PinnProblem(1.0, -5.0, 5.0, n_colloc)
        colloc = torch.tensor(prob.sample_collocation(np.random.default_rng(1)), dtype=torch.float32, device=dev)
        params = list(model.parameters().values())
        for _ in range(warmup):
            torch.autograd.grad(P.pinn_loss(model.forward, prob, colloc), params)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            torch.autograd.grad(P.pinn_loss(model.forward, prob, colloc), params)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / steps
        out[kind] = {"workload": f"pinn_loss [1,5,1] {kind}, {n_colloc} collocation points, loss + parameter grads",
                     "ms_per_step": ms, "collocation_points_per_s": n_colloc / (ms * 1e-3)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the supplementary cfg1/2/4/5 and PINN fields")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        dev_index = local_rank % torch.cuda.device_count()
        torch.cuda.set_device(dev_index)
        # NCCL over NVLink/NVSwitch; UKAN_DIST_BACKEND=gloo lets the multi-rank path be exercised on a
        # single-GPU box (ranks sharing one device), which NCCL refuses
        backend = os.environ.get("UKAN_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend)
    try:
        our_arm(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
