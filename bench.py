"""Benchmark: KAN/UKAN layer fwd+bwd samples/s on 1..8 B200 vs the CPU reference path.

Workload (BASELINE.json configs[1]): KAN stack [784, 256, 10], grid G=32, k=3, batch 8192 per
GPU (weak scaling), MNIST-shaped synthetic classification (x ~ U(-1,1), labels ~ U{0..9}),
softmax cross-entropy, Adam — one full data-parallel training step per "step".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU, NCCL)

Prints one JSON line on rank 0.  `value` is device-timed (CUDA events, inputs resident in HBM,
max over ranks); `e2e` is the same metric through the public API with pinned host inputs copied
H2D and the loss read D2H every step.  The CPU reference arm (`--impl reference`, and the
`cpu_baseline` field) runs the float64 NumPy port of the reference in oracle/ — the reference
itself is pure Python/NumPy and cannot travel to the GPU box.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(widths=[784, 256, 10], G=32, k=3, g_min=-1.0, g_max=1.0, batch=8192, lr=1e-3, wd=0.0)
ROTATE = 8  # resident batches cycled through: 8 x 25.7 MB of x > 126 MB L2


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_fallback": True}


# CUDA-core roofs measured with tools/peaks.cu on this pool's B200 (profiles/peaks_r01.json):
# FMA-chain microbenchmarks, 148 SMs, clocks not locked.
FP32_TFLOPS_MEASURED = 71.95
FP64_TFLOPS_MEASURED = 34.05


def kan_flops(B, d_in, d_out, k):
    """Algorithmic FLOPs of one KAN layer pass: 2*K*B*d_in*d_out per pass."""
    return 2.0 * (k + 1) * B * d_in * d_out


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


# ---------------------------------------------------------------------------------------
# CPU reference arm (oracle port of the float64 NumPy reference)
# ---------------------------------------------------------------------------------------
def _cpu_worker(args):
    sub, seed = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import oracle
    rng = np.random.default_rng(seed)
    widths, k, G = CFG["widths"], CFG["k"], CFG["G"]
    params, cfgs = [], []
    for i in range(len(widths) - 1):
        d_in, d_out = widths[i], widths[i + 1]
        params.append({"coeffs": rng.normal(0, 0.1 / np.sqrt(d_in), (d_in, G + k, d_out)).astype(np.float32).astype(np.float64),
                       "scale": np.ones((d_in, d_out))})
        cfgs.append(dict(k=k, g_min=CFG["g_min"], g_max=CFG["g_max"], G=G))
    x = rng.uniform(-1, 1, (sub, widths[0])).astype(np.float32).astype(np.float64)
    y = rng.integers(0, widths[-1], sub)
    t0 = time.perf_counter()
    oracle.model_step("kan", params, cfgs, x, y, "softmax_cross_entropy", CFG["lr"])
    return time.perf_counter() - t0


def cpu_rate(sub: int, procs: int, reps: int):
    """samples/s of the reference algorithm (oracle port) on `procs` host processes, each
    running a full fwd+bwd+Adam step on a `sub`-row slice; median over reps."""
    import multiprocessing as mp
    times = []
    if procs == 1:
        _cpu_worker((sub, 0))  # warm-up
        for r in range(reps):
            times.append(_cpu_worker((sub, r + 1)))
        step = statistics.median(times)
        return sub / step, step
    with mp.get_context("spawn").Pool(procs) as pool:
        pool.map(_cpu_worker, [(sub, i) for i in range(procs)])  # warm-up
        for r in range(reps):
            t0 = time.perf_counter()
            pool.map(_cpu_worker, [(sub, 1000 * r + i) for i in range(procs)])
            times.append(time.perf_counter() - t0)
    step = statistics.median(times)
    return procs * sub / step, step


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_arm(args, rank):
    if rank != 0:
        return
    ncpu = len(os.sched_getaffinity(0))
    try:
        mem_gb = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 2**30
    except (ValueError, OSError):
        mem_gb = 64
    procs = max(1, min(ncpu, 32, int(mem_gb // 4)))
    sub = 16
    rate, step = cpu_rate(sub, procs, max(1, args.steps))
    line = {
        "impl": "reference", "metric": "KAN/UKAN layer fwd+bwd samples/s (KAN [784,256,10] training step)",
        "value": rate, "unit": "samples/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg2: KAN [784,256,10] G=32 k=3 softmax-CE Adam", "global_batch": CFG["batch"],
                   "parallelism": f"{procs} host processes"},
        "cpu_baseline": {"value": rate, "unit": "samples/s", "cores": procs, "kind": "port",
                         "sample": f"{procs} processes x {sub}-row sub-batch, full fwd+bwd+Adam step of the "
                                   f"float64 NumPy port (oracle/), median of {max(1, args.steps)} reps",
                         "cpu": cpu_model()},
        "e2e": {"value": rate, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------
def our_arm(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2408_11200_b200 as P
    from paper_2408_11200_b200 import ops

    dev_index = local_rank % torch.cuda.device_count()  # == local_rank on a full node
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    B = CFG["batch"]
    model = P.build_model("kan", CFG["widths"], CFG["k"], seed=0, device=dev, g_min=CFG["g_min"],
                          g_max=CFG["g_max"], G=CFG["G"])
    tr = P.SplineTrainer(model, "softmax_cross_entropy", CFG["lr"], "adam", weight_decay=CFG["wd"])
    ops.set_check_mode("deferred")
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    xs = [torch.rand((B, CFG["widths"][0]), device=dev, generator=g) * 2 - 1 for _ in range(ROTATE)]
    ys = [torch.randint(0, CFG["widths"][-1], (B,), device=dev, generator=g) for _ in range(ROTATE)]

    def barrier():
        if world > 1:
            dist.barrier()

    for s in range(args.warmup):
        tr.step(xs[s % ROTATE], ys[s % ROTATE])
    tr.read_loss(tr.step(xs[0], ys[0]))
    torch.cuda.synchronize()
    barrier()

    # ---- device-timed region (inputs resident in HBM) ----
    tr.timers = {}
    lib = P._lib.load()
    launches0 = lib.ukan_launch_count()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev_index) as clk:
        torch.cuda.synchronize()
        barrier()
        start.record()
        for s in range(args.steps):
            loss = tr.step(xs[s % ROTATE], ys[s % ROTATE])
        end.record()
        torch.cuda.synchronize()
        barrier()
    launches = (lib.ukan_launch_count() - launches0) // max(1, args.steps)
    ms = start.elapsed_time(end)
    tr.read_loss(loss)
    ops.flush_checks()
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * B * args.steps / (ms_max * 1e-3)
    timers, tr.timers = tr.timers, None
    kern_ms = {name: sum(a.elapsed_time(b) for a, b in ev) / len(ev) for name, ev in timers.items()}

    # ---- end-to-end through the public API: pinned host inputs, H2D, step, loss D2H ----
    hx = [torch.empty((B, CFG["widths"][0]), dtype=torch.float32).pin_memory() for _ in range(2)]
    hy = [torch.empty((B,), dtype=torch.int64).pin_memory() for _ in range(2)]
    for i in range(2):
        hx[i].copy_(xs[i].cpu())
        hy[i].copy_(ys[i].cpu())
    # the step captured as one CUDA graph (single process; N > 1 keeps the eager NCCL path)
    cap = tr.capture(xs[0], ys[0]) if world == 1 else None
    if cap is not None:
        for s in range(2):  # graph warm-up replays
            tr.read_loss(cap.replay(xs[s], ys[s]))
    # every step: its batch is copied from pinned host memory (DevicePrefetcher, one step ahead on
    # a side stream) and its loss is read back to the host.  Wall-clock timed: 3 runs of
    # max(steps, 60) steps, the median run reported (max over ranks per run).
    e2e_steps = max(args.steps, 60)
    runs = []
    for _ in range(3):
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for bx, by in P.DevicePrefetcher(((hx[s % 2], hy[s % 2]) for s in range(e2e_steps)), dev):
            tr.read_loss(cap.replay(bx, by) if cap is not None else tr.step(bx, by))
        torch.cuda.synchronize()
        t = torch.tensor([time.perf_counter() - t0], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        runs.append(float(t.item()))
    e2e_s = sorted(runs)[1]
    e2e_value = world * B * e2e_steps / e2e_s

    ukan = ukan_layer_rate(dev) if (world == 1 and not args.no_ukan) else None
    cfg_rates = kan_layer_rates(dev) if (world == 1 and not args.no_configs) else None
    pinn = pinn_rate(dev) if (world == 1 and not args.no_configs) else None
    if rank != 0:
        return
    pk = peaks()
    d0, d1, d2 = CFG["widths"]
    k = CFG["k"]
    # dominant kernel: the layer-0 (784->256) launches; pick whichever is longer
    f_fwd = kan_flops(B, d0, d1, k)
    f_bwd = kan_flops(B, d0, d1, k)  # table gradient only (layer 0 needs no dx)
    fwd_ms = kern_ms.get("layer0.kan_forward")
    bwd_ms = kern_ms.get("layer0.kan_backward")
    if bwd_ms and fwd_ms and bwd_ms >= fwd_ms:
        dom, dom_ms, dom_fl, dom_peak, bound = ("layer0 backward: kan_bwd_tc2_sweep (FP64 DMMA); its x-only record "
                                                "prep runs earlier on a side stream (ukan_kan_backward_prep)", bwd_ms,
                                                f_bwd, FP64_TFLOPS_MEASURED, "fp64-fma")
    else:
        dom, dom_ms, dom_fl, dom_peak, bound = ("layer0 forward: kan_pack + kan_fwd_records + kan_fwd_tm (TMEM gather)",
                                                fwd_ms, f_fwd, FP32_TFLOPS_MEASURED, "fp32-fma")
    achieved = dom_fl / (dom_ms * 1e-3) / 1e12
    # compulsory HBM bytes of the dominant launch
    R = CFG["G"] + k
    if "backward" in dom:
        hbm_bytes = 4.0 * (B * d0 + B * d1 + 2 * d0 * R * d1 + 3 * d0 * d1)
    else:
        hbm_bytes = 4.0 * (B * d0 + B * d1 + d0 * R * d1 + d0 * d1)
    step_fl = kan_flops(B, d0, d1, k) * 2 + kan_flops(B, d1, d2, k) * 3
    # DRAM bytes per launch of the dominant kernel group from the committed ncu --set full capture
    traffic = None
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")) as f:
            tj = json.load(f)
            grp = tj.get("layer0.kan_backward_sweep") if "backward" in dom else tj.get("layer0.kan_forward")
        traffic = grp["dram_bytes"] if grp else None
    except (OSError, ValueError, KeyError):
        traffic = None
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        sub = 16
        rate, step = cpu_rate(sub, 1, 3)
        cpu = {"value": rate, "unit": "samples/s", "cores": 1, "kind": "port",
               "sample": f"{sub}-row slice of the cfg2 batch, full fwd+bwd+Adam step of the float64 NumPy port "
                         f"(oracle/), median of 3 reps ({step:.1f} s/rep), OMP_NUM_THREADS=1",
               "cpu": cpu_model()}
    line = {
        "metric": "KAN/UKAN layer fwd+bwd samples/s (KAN [784,256,10] training step)",
        "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 storage; f64 grid locate + backward accumulation", "data": "synthetic",
        "config": {"workload": "cfg2: KAN [784,256,10] G=32 k=3 MNIST-shaped softmax-CE + Adam, one DP step",
                   "global_batch": B * world, "per_gpu_batch": B, "parallelism": f"dp{world}",
                   "l2": f"inputs rotate over {ROTATE} HBM-resident batches ({ROTATE * B * d0 * 4 / 2**20:.0f} MiB > 126 MB L2)"},
        "roofline": {"bound": bound, "kernel": dom, "achieved": achieved, "peak": dom_peak, "unit": "TFLOP/s",
                     "frac": achieved / dom_peak, "traffic": traffic,
                     "traffic_unit": "bytes per launch (ncu dram__bytes_read+write, profiles/traffic.json)",
                     "algorithmic_bytes_per_launch": hbm_bytes,
                     "peak_source": "tools/peaks.cu FMA microbenchmark on this pool's B200 (profiles/peaks_r01.json)",
                     "algorithmic_flops_per_launch": dom_fl, "avg_launch_ms": dom_ms},
        "roofline_hbm": {"bound": "hbm", "achieved": hbm_bytes / (dom_ms * 1e-3) / 1e9, "peak": pk["hbm_gbs"],
                         "unit": "GB/s", "frac": hbm_bytes / (dom_ms * 1e-3) / 1e9 / pk["hbm_gbs"],
                         "note": "compulsory bytes of the dominant launch; the kernel is compute-bound"},
        "step_tflops": step_fl * args.steps / (ms_max * 1e-3) / 1e12,
        "kernel_ms": kern_ms,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "e2e": {"value": e2e_value, "unit": "samples/s", "steps": e2e_steps, "runs_s": runs,
                "path": "SplineTrainer.capture -> CapturedStep.replay (one CUDA graph per step) fed by "
                        "DevicePrefetcher" if world == 1 else "SplineTrainer.step fed by DevicePrefetcher",
                "h2d_bytes_per_step": B * d0 * 4 + B * 8, "d2h_bytes_per_step": 8 + 4},
        "cpu_baseline": cpu,
        "ukan_layer": ukan,
        "kan_layers": cfg_rates,
        "pinn": pinn,
    }
    print(json.dumps(line), flush=True)


def ukan_layer_rate(dev, B=4096, steps=5, warmup=3):
    """Supplementary UKAN measurement (not the headline): one cfg4-shaped UKAN layer (1024 -> 1024,
    k=3, delta_g=0.5, d_pe=d_femb=32; x ~ N(0, 20^2)) forward + backward of x and every parameter
    through the drop-in API (key dedup, CG MLP on the tensor cores, spline kernels), device-timed."""
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


def kan_layer_rates(dev):
    """Supplementary single-layer KAN measurements at BASELINE configs[0] and configs[2] (SURVEY
    8d D4): forward + backward of every parameter (x is input data: no dx) through the drop-in
    API, device-timed (CUDA events), with the FP32/FP64 roof fraction of the layer's algorithmic
    flops (forward 2KBio on FP32, table gradient 2KBio on FP64)."""
    import torch
    import paper_2408_11200_b200 as P
    out = {}
    for name, (d, G, B, steps, outl) in {"cfg1": (64, 10, 1024, 50, 0.0), "cfg3": (4096, 64, 65536, 2, 0.01)}.items():
        layer = P.init_layer("kan", d, d, 3, seed=0, g_min=-1.0, g_max=1.0, G=G, device=dev)
        g = torch.Generator(device=dev)
        g.manual_seed(3)
        x = torch.rand((B, d), device=dev, generator=g) * 2 - 1
        if outl:
            m = torch.rand((B, d), device=dev, generator=g) < outl
            x = torch.where(m, x * 3, x)
        gy = torch.randn((B, d), device=dev, generator=g)
        params = [layer.coeffs, layer.scale]
        for _ in range(2):
            torch.autograd.grad(P.kan_forward(layer, x), params, gy)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            torch.autograd.grad(P.kan_forward(layer, x), params, gy)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / steps
        fl = 2.0 * 4 * B * d * d
        roof_ms = (fl / (FP32_TFLOPS_MEASURED * 1e12) + fl / (FP64_TFLOPS_MEASURED * 1e12)) * 1e3
        out[name] = {"workload": f"KAN layer {d}->{d} G={G} k=3 B={B}" + (", 1% clamp tail" if outl else "")
                     + ", fwd + parameter grads", "samples_per_s": B / (ms * 1e-3), "ms_per_step": ms,
                     "steps": steps, "roof_ms": roof_ms, "roof_frac": roof_ms / ms}
        del layer, x, gy
        torch.cuda.empty_cache()
    return out


def pinn_rate(dev, n_colloc=128, steps=50, warmup=5):
    """Supplementary F2 measurement: one PINN step (pinn_loss through the forward-tangent kernels of
    a [1, 5, 1] KAN and a [1, 5, 1] UKAN, tasks.py:153-166, plus the reverse pass through the
    tangent graph), device-timed; tiny and launch-bound by nature."""
    import numpy as np
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
    ap.add_argument("--no-ukan", action="store_true", help="skip the supplementary UKAN layer measurement")
    ap.add_argument("--no-configs", action="store_true", help="skip the supplementary cfg1 / cfg3 layer measurements")
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
