"""Per-step wall-clock distribution of the e2e loop (graph replay + prefetch) — profiling tool."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2408_11200_b200 as P
from paper_2408_11200_b200 import ops

dev = torch.device("cuda", 0)
B = 8192
model = P.build_model("kan", [784, 256, 10], 3, seed=0, device=dev, g_min=-1.0, g_max=1.0, G=32)
tr = P.SplineTrainer(model, "softmax_cross_entropy", 1e-3, "adam", weight_decay=1e-5)
ops.set_check_mode("deferred")
xs = [torch.rand((B, 784), device=dev) * 2 - 1 for _ in range(2)]
ys = [torch.randint(0, 10, (B,), device=dev) for _ in range(2)]
for s in range(3):
    tr.read_loss(tr.step(xs[s % 2], ys[s % 2]))
hx = [x.cpu().pin_memory() for x in xs]
hy = [y.cpu().pin_memory() for y in ys]
cap = tr.capture(xs[0], ys[0])
for s in range(3):
    tr.read_loss(cap.replay(xs[s % 2], ys[s % 2]))
N = 200
for mode in ("graph+prefetch", "graph+sync-copy", "eager+prefetch", "graph-resident"):
    ts = []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if mode == "graph+prefetch":
        for bx, by in P.DevicePrefetcher(((hx[s % 2], hy[s % 2]) for s in range(N)), dev):
            a = time.perf_counter(); tr.read_loss(cap.replay(bx, by)); ts.append(time.perf_counter() - a)
    elif mode == "graph+sync-copy":
        for s in range(N):
            a = time.perf_counter()
            tr.read_loss(cap.replay(hx[s % 2].to(dev, non_blocking=True), hy[s % 2].to(dev, non_blocking=True)))
            ts.append(time.perf_counter() - a)
    elif mode == "eager+prefetch":
        for bx, by in P.DevicePrefetcher(((hx[s % 2], hy[s % 2]) for s in range(N)), dev):
            a = time.perf_counter(); tr.read_loss(tr.step(bx, by)); ts.append(time.perf_counter() - a)
    else:
        for s in range(N):
            a = time.perf_counter(); tr.read_loss(cap.replay()); ts.append(time.perf_counter() - a)
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
    ts.sort()
    print(f"{mode:18s} {B * N / tot / 1e6:6.3f} M/s  step ms p10 {ts[N//10]*1e3:.3f} p50 {ts[N//2]*1e3:.3f} p90 {ts[9*N//10]*1e3:.3f} max {ts[-1]*1e3:.3f}")
