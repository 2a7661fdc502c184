"""Data-parallel training step for spline stacks (reference: train.step, train.py:142-150).

``SplineTrainer.step`` = forward through every layer (fused kernels), loss (fp64,
normalised by the GLOBAL batch), backward through every layer writing parameter gradients
straight into one flat fp32 gradient buffer, one bucketed NCCL all-reduce(sum) of that buffer
(per layer, issued as soon as the layer's backward is enqueued so it overlaps the backward of
the layers below), and one fused Adam (coupled L2) / SGD kernel over the flat parameter
buffer.  The loss is all-reduced too and guards the optimizer: a non-finite global loss skips
the update on the device and raises ``DivergedError`` when the host reads it — the
reference's check-before-update semantics (train.py:143-144) without a mid-step sync.

Everything runs through the C ABI; no autograd tape is recorded on this path (the autograd
``ops`` are the drop-in layer API; both call the same kernels).
"""
from __future__ import annotations

import ctypes
import math

import torch
import torch.distributed as dist

from . import _lib
from ._lib import check, ptr, stream_ptr
from .errors import ConfigError, DimensionError, DivergedError
from .layers import KanLayer, Model, UkanLayer
from . import ops


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous batch shard [lo, hi) of rank (remainder rows go to the first ranks)."""
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


class GradSync:
    """All-reduce(sum) helper over a torch.distributed group (NCCL on GPUs, gloo in CPU tests).
    World size 1 (or no initialised group) is a no-op."""

    def __init__(self, group=None):
        self.group = group
        self.enabled = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
        self.world = dist.get_world_size(group) if self.enabled else 1
        self.rank = dist.get_rank(group) if self.enabled else 0
        self._handles = []

    def allreduce_async(self, t: torch.Tensor) -> None:
        if self.enabled:
            self._handles.append(dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group, async_op=True))

    def wait(self) -> None:
        for h in self._handles:
            h.wait()
        self._handles = []


class FlatParams:
    """All parameters of a model as views into one contiguous fp32 buffer, with a matching
    flat gradient buffer.  Layer attributes are rebound to the views, so the layers (and the
    drop-in autograd API) read the flat storage directly."""

    def __init__(self, model: Model):
        named = list(model.parameters().items())
        dev = named[0][1].device
        self.names = [n for n, _ in named]
        self.numel = [p.numel() for _, p in named]
        total = sum(self.numel)
        self.data = torch.empty(total, device=dev, dtype=torch.float32)
        self.grad = torch.zeros(total, device=dev, dtype=torch.float32)
        self.views, self.gviews, self.offsets = {}, {}, {}
        off = 0
        for (name, p), n in zip(named, self.numel):
            self.data[off:off + n].copy_(p.detach().reshape(-1))
            self.views[name] = self.data[off:off + n].view(p.shape)
            self.gviews[name] = self.grad[off:off + n].view(p.shape)
            self.offsets[name] = (off, off + n)
            off += n
        for i, layer in enumerate(model.layers):
            for pname in layer.parameters():
                setattr(layer, pname, self.views[f"layer{i}.{pname}"])

    def layer_slice(self, i: int, model: Model) -> tuple[int, int]:
        names = [f"layer{i}.{p}" for p in model.layers[i].parameters()]
        return min(self.offsets[n][0] for n in names), max(self.offsets[n][1] for n in names)


class SplineTrainer:
    """One-process-per-GPU data-parallel trainer for KAN / UKAN stacks."""

    def __init__(self, model: Model, loss_kind: str, lr: float, optimizer: str = "adam",
                 weight_decay: float = 0.0, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                 group=None):
        if model.kind not in ("kan", "ukan"):
            raise ConfigError(f"SplineTrainer handles kan/ukan stacks, got {model.kind!r}")
        if loss_kind not in ("mse", "softmax_cross_entropy"):
            raise ConfigError(f"unknown loss kind {loss_kind!r}")
        self.lib = _lib.load()
        self.model = model
        self.loss_kind = loss_kind
        self.lr, self.optimizer, self.wd = lr, optimizer, weight_decay
        self.beta1, self.beta2, self.eps = beta1, beta2, eps
        self.flat = FlatParams(model)
        self.sync = GradSync(group)
        self.t = 0
        dev = self.flat.data.device
        self.m = torch.zeros_like(self.flat.data) if optimizer == "adam" else None
        self.v = torch.zeros_like(self.flat.data) if optimizer == "adam" else None
        self._loss_buf = None
        self.device = dev
        self.kernel_launches = 0
        self.timers = None  # optional {name: [(start_event, end_event), ...]} (bench.py)
        self._dev_state = None  # (step counter, lr, bias corrections) on the device once captured

    def _mark(self, name):
        """Record a CUDA event pair around one launch when timing is enabled."""
        trainer = self

        class _M:
            def __enter__(self_):
                if trainer.timers is not None:
                    self_.a = torch.cuda.Event(enable_timing=True)
                    self_.a.record()

            def __exit__(self_, *exc):
                if trainer.timers is not None:
                    b = torch.cuda.Event(enable_timing=True)
                    b.record()
                    trainer.timers.setdefault(name, []).append((self_.a, b))
        return _M()

    # -- per-layer forward / backward on raw buffers ------------------------------------
    def _fwd(self, layer, h):
        st = stream_ptr()
        B = h.shape[0]
        y = torch.empty((B, layer.d_out), device=self.device, dtype=torch.float32)
        if isinstance(layer, KanLayer):
          with self._mark(f"layer{self._li}.kan_forward"):
            nbytes = 0 if layer.base_weight is not None else self.lib.ukan_kan_forward_workspace_size(
                B, layer.d_in, layer.d_out, layer.G, layer.k)
            ws = torch.empty(nbytes, device=self.device, dtype=torch.uint8) if nbytes > 0 else None
            check(self.lib.ukan_kan_forward_ws(ptr(h), ptr(layer.coeffs), ptr(layer.scale), ptr(layer.base_weight),
                                               ptr(y), B, layer.d_in, layer.d_out, layer.G, layer.k,
                                               float(layer.g_min), float(layer.g_max), ptr(self._err), ptr(ws),
                                               nbytes, st), "kan_forward")
            self.kernel_launches += 1
            return y, None
        keys = ops.ukan_build_keys(h, layer.k, float(layer.delta_g))
        self.kernel_launches += 5
        table, cg_cache = ops.cg_forward_raw(keys.key_f, keys.key_g, layer.feature_embedding, layer.cg_w1,
                                             layer.cg_b1, layer.cg_w2, layer.cg_b2, layer.d_pe)
        ops.ukan_forward_into(h, keys.base_row, keys.seg_start, table, layer.scale, y, layer.k, float(layer.delta_g),
                              keys.max_rows)
        self.kernel_launches += 4
        return y, (keys, cg_cache, table)

    def _prep_first_layer(self, layer, x):
        """The first layer's backward records depend on x only: build them on a side stream while
        the layers above run forward and backward (ukan_kan_backward_prep)."""
        B = x.shape[0]
        nbytes = self.lib.ukan_kan_backward_workspace_size(B, layer.d_in, layer.d_out, layer.G, layer.k)
        if nbytes <= 0:
            return
        ws = torch.empty(nbytes, device=self.device, dtype=torch.uint8)
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(device=self.device)
        side = self._side
        side.wait_stream(torch.cuda.current_stream(self.device))
        prepared = ctypes.c_int32(0)
        with torch.cuda.stream(side):
            check(self.lib.ukan_kan_backward_prep(ptr(x), ptr(layer.base_weight), B, layer.d_in, layer.d_out, layer.G,
                                                  layer.k, float(layer.g_min), float(layer.g_max), ptr(ws), nbytes,
                                                  ctypes.byref(prepared), stream_ptr()), "kan_backward_prep")
        ev = torch.cuda.Event()
        ev.record(side)
        self._pre0 = (ws, nbytes, prepared.value == 1, ev)
        self.kernel_launches += prepared.value

    def _bwd(self, i, layer, h, gy, cache, need_dx):
        st = stream_ptr()
        B = h.shape[0]
        pre_ = f"layer{i}."
        gv = self.flat.gviews
        dx = torch.empty_like(h) if need_dx else None
        if isinstance(layer, KanLayer):
            flags = 0
            if i == 0 and getattr(self, "_pre0", None) is not None:
                ws, nbytes, prepared, ev = self._pre0
                torch.cuda.current_stream(self.device).wait_event(ev)
                flags = 1 if prepared else 0
                self._pre0 = None
            else:
                nbytes = self.lib.ukan_kan_backward_workspace_size(B, layer.d_in, layer.d_out, layer.G, layer.k)
                ws = torch.empty(nbytes, device=self.device, dtype=torch.uint8) if nbytes else None
            bw = layer.base_weight
            with self._mark(f"layer{i}.kan_backward"):
              check(self.lib.ukan_kan_backward_ws2(ptr(h), ptr(layer.coeffs), ptr(layer.scale), ptr(bw), ptr(gy),
                                                 ptr(dx), ptr(gv[pre_ + "coeffs"]), ptr(gv[pre_ + "scale"]),
                                                 ptr(gv.get(pre_ + "base_weight")) if bw is not None else None,
                                                 B, layer.d_in, layer.d_out, layer.G, layer.k, float(layer.g_min),
                                                 float(layer.g_max), ptr(ws), nbytes, flags, st), "kan_backward")
            self.kernel_launches += 2 if need_dx else 1
            return dx
        keys, cg_cache, table = cache
        n_u = keys.n_u
        dtable = torch.empty_like(table)
        ops.ukan_backward_into(h, keys.base_row, keys.seg_start, table, layer.scale, gy, dx, dtable,
                               gv[pre_ + "scale"], layer.k, float(layer.delta_g), keys.max_rows)
        ops.cg_backward_raw(cg_cache, dtable, layer.cg_w1, layer.cg_w2, keys.seg_start, layer.d_femb,
                            gv[pre_ + "cg_w1"], gv[pre_ + "cg_b1"], gv[pre_ + "cg_w2"], gv[pre_ + "cg_b2"],
                            gv[pre_ + "feature_embedding"])
        self.kernel_launches += 10 + (1 if need_dx else 0)
        return dx

    # -- input checks (the reference's DimensionError / IndexError, tensor.py:368-400) ---------
    def _checked_inputs(self, x: torch.Tensor, target: torch.Tensor):
        """fp32 contiguous x on this device with d_in columns; int64 labels (CE) or an fp32 target
        with one value per output (MSE).  Label RANGE is checked on the device (no sync): the loss
        kernel flags it and ``read_loss`` raises IndexError."""
        layers = self.model.layers
        if not (isinstance(x, torch.Tensor) and isinstance(target, torch.Tensor)):
            raise TypeError("x and target must be torch tensors on the trainer's device")
        if x.device != self.device or target.device != self.device:
            raise ConfigError(f"x / target must live on {self.device}")
        if x.dim() != 2 or x.shape[1] != layers[0].d_in:
            raise DimensionError(f"x must be [B, {layers[0].d_in}], got {tuple(x.shape)}")
        if x.dtype != torch.float32 or not x.is_contiguous():
            x = x.float().contiguous()
        B = x.shape[0]
        d_last = layers[-1].d_out
        if self.loss_kind == "softmax_cross_entropy":
            if target.dim() != 1 or target.shape[0] != B:
                raise DimensionError(f"labels must be [{B}], got {tuple(target.shape)}")
            if target.dtype.is_floating_point or target.dtype == torch.bool:
                raise DimensionError(f"labels must be integers, got {target.dtype}")
            if target.dtype != torch.int64 or not target.is_contiguous():
                target = target.long().contiguous()
        else:
            if target.numel() != B * d_last:
                raise DimensionError(f"target must hold {B}x{d_last} values, got {tuple(target.shape)}")
            if target.dtype != torch.float32 or not target.is_contiguous():
                target = target.float().contiguous()
        return x, target

    def _global_batch(self, B: int) -> int:
        """Global batch = sum of the shard sizes (uneven shards allowed): all-reduced once per
        local shape and cached, so every rank normalises by the same number."""
        if not self.sync.enabled:
            return B
        cache = self.__dict__.setdefault("_n_global_cache", {})
        if B not in cache:
            t = torch.tensor([B], dtype=torch.int64, device=self.device if dist.get_backend(self.sync.group) == "nccl"
                             else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.sync.group)
            cache[B] = int(t.item())
        return cache[B]

    # -- the step --------------------------------------------------------------------------
    def step(self, x: torch.Tensor, target: torch.Tensor, n_global: int | None = None, lr: float | None = None):
        """One DP training step on this rank's shard (x, target already on the device).
        Returns the device fp64 global loss (read it with ``read_loss``).  ``n_global`` defaults
        to the sum of every rank's shard size."""
        x, target = self._checked_inputs(x, target)
        st = stream_ptr()
        layers = self.model.layers
        B = x.shape[0]
        if n_global is None:
            n_global = self._global_batch(B)
        if getattr(self, "_err", None) is None:
            self._err = torch.zeros(1, device=self.device, dtype=torch.int32)
        else:  # reset the NaN flag with our fill kernel (0.0f has the all-zero bit pattern)
            check(self.lib.ukan_fill_f32(ptr(self._err), 1, 0.0, st), "fill")
            self.kernel_launches += 1
        hs = [x]
        caches = []
        self._pre0 = None
        for li, layer in enumerate(layers):
            self._li = li
            y, cache = self._fwd(layer, hs[-1])
            hs.append(y)
            caches.append(cache)
            if li == 0 and isinstance(layer, KanLayer) and len(layers) > 1:
                self._prep_first_layer(layer, x)
        out = hs[-1]
        if self._loss_buf is None or self._loss_buf.numel() < out.numel() + 1:
            self._loss_buf = torch.empty(out.numel() + 1, device=self.device, dtype=torch.float64)
        gy = torch.empty_like(out)
        if self.loss_kind == "softmax_cross_entropy":
            check(self.lib.ukan_softmax_xent(ptr(out), ptr(target), ptr(self._loss_buf), ptr(gy), B, out.shape[1],
                                             n_global, 1.0, ptr(self._err), st), "softmax_xent")
        else:
            n_el = out.numel()
            check(self.lib.ukan_mse(ptr(out), ptr(target), ptr(self._loss_buf), ptr(gy), n_el,
                                    n_el // B * n_global, st), "mse")
        self.kernel_launches += 2
        loss = self._loss_buf[:1]
        self.sync.allreduce_async(loss)
        for i in range(len(layers) - 1, -1, -1):
            gy = self._bwd(i, layers[i], hs[i], gy, caches[i], need_dx=i > 0)
            lo, hi = self.flat.layer_slice(i, self.model)
            self.sync.allreduce_async(self.flat.grad[lo:hi])
        self.sync.wait()
        self.t += 1  # undone by read_loss if this step's loss diverged (the update is skipped)
        lr = self.lr if lr is None else lr
        n = self.flat.data.numel()
        if self.optimizer == "adam" and self._dev_state is not None:  # graph-replayable form
            t_dev, lr_dev, bc = self._dev_state
            if not torch.cuda.is_current_stream_capturing():
                lr_dev.fill_(lr)  # eager step after capture(): honour lr / self.lr
            check(self.lib.ukan_adam_step_dev(ptr(self.flat.data), ptr(self.flat.grad), ptr(self.m), ptr(self.v), n,
                                              ptr(lr_dev), self.beta1, self.beta2, self.eps, self.wd, ptr(t_dev),
                                              ptr(bc), ptr(loss), st), "adam_dev")
            self.kernel_launches += 1
        elif self.optimizer == "adam":
            check(self.lib.ukan_adam_step(ptr(self.flat.data), ptr(self.flat.grad), ptr(self.m), ptr(self.v), n, lr,
                                          self.beta1, self.beta2, self.eps, self.wd, self.t, ptr(loss), st), "adam")
        else:
            check(self.lib.ukan_sgd_step(ptr(self.flat.data), ptr(self.flat.grad), n, lr, ptr(loss), st), "sgd")
        self.kernel_launches += 1
        self._last_loss = loss
        return loss

    def capture(self, x: torch.Tensor, target: torch.Tensor) -> "CapturedStep":
        """Capture one training step on fixed-shape buffers as a CUDA graph (single process).
        Run at least one eager ``step`` first (lazy buffers); see ``CapturedStep``."""
        return CapturedStep(self, x, target)

    def read_loss(self, loss: torch.Tensor) -> float:
        """Host read of the step's loss; raises DivergedError / IndexError like the reference."""
        # one stream sync for both reads (loss 8 B + NaN flag 4 B into pinned host memory)
        if getattr(self, "_host_rd", None) is None:
            self._host_rd = (torch.empty(1, dtype=torch.float64).pin_memory(),
                             torch.empty(1, dtype=torch.int32).pin_memory())
        hl, he = self._host_rd
        hl.copy_(loss.reshape(1), non_blocking=True)
        err = getattr(self, "_err", None)
        if err is not None:
            he.copy_(err, non_blocking=True)
        else:
            he.zero_()
        torch.cuda.current_stream(self.device).synchronize()
        v = float(hl[0])
        flag = int(he[0])
        if flag or not math.isfinite(v):
            if loss is getattr(self, "_last_loss", None) and self._dev_state is None:
                self.t -= 1  # the guarded optimizer skipped this step (reference: raise before state.t += 1)
        if flag & 2:
            raise IndexError("label out of range for the softmax cross-entropy")
        if flag & 1:
            raise IndexError("non-finite (NaN) input to a bounded-grid KAN layer")
        if not math.isfinite(v):
            raise DivergedError(f"non-finite loss {v}")
        return v

class CapturedStep:
    """A ``SplineTrainer.step`` recorded once as a CUDA graph and replayed per batch: the whole
    step (forward, loss, backward, Adam) costs one graph launch on the host, so a loop that reads
    the loss every step (the reference's train loop, train.py:152-165) no longer exposes the
    per-kernel host overhead.  Inputs go into the static buffers ``x`` / ``target``; the Adam
    step counter, learning rate and bias corrections live on the device (``ukan_adam_step_dev``).
    Capture itself runs no step.  Single process only (NCCL collectives are not captured)."""

    def __init__(self, trainer: "SplineTrainer", x: torch.Tensor, target: torch.Tensor):
        if trainer.sync.enabled:
            raise ConfigError("graph capture covers single-process training")
        if trainer.model.kind != "kan":  # UKAN's key count is data dependent (one host sync per step)
            raise ConfigError("graph capture covers KAN stacks (fixed shapes)")
        dev = trainer.device
        self.trainer = trainer
        self.x = x.detach().clone()
        self.target = target.detach().clone()
        trainer._dev_state = (torch.tensor([trainer.t], dtype=torch.int64, device=dev),
                              torch.tensor([trainer.lr], dtype=torch.float64, device=dev),
                              torch.zeros(2, dtype=torch.float64, device=dev))
        timers, trainer.timers = trainer.timers, None
        t_host = trainer.t
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.loss = trainer.step(self.x, self.target)
        trainer.t = t_host  # capture executed nothing; the device counter advances on replay
        trainer.timers = timers

    def replay(self, x: torch.Tensor | None = None, target: torch.Tensor | None = None) -> torch.Tensor:
        """Copy (x, target) into the static buffers (stream-ordered) and run the step; returns the
        device loss (read it with ``trainer.read_loss``)."""
        if x is not None:
            self.x.copy_(x, non_blocking=True)
        if target is not None:
            self.target.copy_(target, non_blocking=True)
        self.graph.replay()
        return self.loss

    def set_lr(self, lr: float) -> None:
        self.trainer._dev_state[1].fill_(lr)

    def sync_step_count(self) -> int:
        """Copy the device step counter back to the trainer (host read)."""
        self.trainer.t = int(self.trainer._dev_state[0].item())
        return self.trainer.t


class DevicePrefetcher:
    """Host -> device input pipeline for the training loop: while step s runs on the compute
    stream, batch s+1 is copied from pinned host memory on a side stream (the reference loads
    its batches on the host, train.py:152-165; here the copy overlaps the previous step).

    ``host_batches`` yields tuples of (pinned) CPU tensors; iteration yields the same tuples on
    ``device``.  Every batch is still copied host -> device once per step.  Two device buffer
    sets are reused round-robin (no allocation per step); a buffer is refilled only after the
    compute stream has passed the step that read it.  A yielded batch is valid until the
    iteration after next."""

    def __init__(self, host_batches, device):
        self._it = iter(host_batches)
        self._dev = torch.device(device)
        self._side = torch.cuda.Stream(device=self._dev)
        self._bufs = [None, None]
        self._free = [None, None]   # compute-stream event: buffer k no longer read
        self._ready = [None, None]  # side-stream event: buffer k filled
        self._k = 0                 # buffer of the next batch to hand out
        self._have = self._load(0)

    def _load(self, k):
        try:
            batch = next(self._it)
        except StopIteration:
            return False
        buf = self._bufs[k]
        if buf is None or len(buf) != len(batch) or any(b.shape != t.shape or b.dtype != t.dtype
                                                        for b, t in zip(buf, batch)):
            buf = tuple(torch.empty(t.shape, dtype=t.dtype, device=self._dev) for t in batch)
            self._bufs[k] = buf
        with torch.cuda.stream(self._side):
            if self._free[k] is not None:
                self._side.wait_event(self._free[k])
            for b, t in zip(buf, batch):
                b.copy_(t, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self._side)
            self._ready[k] = ev
        return True

    def __iter__(self):
        return self

    def __next__(self):
        if not self._have:
            raise StopIteration
        cur = torch.cuda.current_stream(self._dev)
        k = self._k
        prev = k ^ 1
        if self._bufs[prev] is not None:  # the previous batch's step is enqueued: its buffer frees after it
            ev = torch.cuda.Event()
            ev.record(cur)
            self._free[prev] = ev
        cur.wait_event(self._ready[k])
        batch = self._bufs[k]
        self._have = self._load(prev)
        self._k = prev
        return batch


class LayerTrainer:
    """Data-parallel training step of ONE KAN layer inside a stack (the unit bench.py times at
    cfg3): forward, backward INCLUDING dx (x is a recorded node: the layer below needs it, the
    reference's tape computes it then, tensor.py:455-456), the gradient all-reduce in feature
    buckets that overlap the rest of the backward, and one fused Adam (coupled L2) over the
    layer's flat parameters.  Reference: the layer's share of train.step (train.py:142-150):
    kan_forward's nodes (layers.py:304-318) + T.backward + adam_step (optim.py:31-54).

    ``step(x, gy)`` takes this rank's shard and the upstream gradient dL/dy (already normalised
    by the global batch) and returns (y, dx).  Backward order: records (x only), dx for every
    feature, then the table gradient in ``buckets`` feature slices, each all-reduced (NCCL) as
    soon as it is enqueued, so slice s's all-reduce runs while slice s+1 is computed."""

    def __init__(self, layer: KanLayer, lr: float, weight_decay: float = 0.0, beta1: float = 0.9,
                 beta2: float = 0.999, eps: float = 1e-8, buckets: int = 8, group=None):
        if not isinstance(layer, KanLayer) or layer.base_weight is not None:
            raise ConfigError("LayerTrainer covers KAN layers without the base branch")
        self.lib = _lib.load()
        self.layer = layer
        self.model = Model("kan", [layer])
        self.flat = FlatParams(self.model)
        self.sync = GradSync(group)
        self.lr, self.wd, self.beta1, self.beta2, self.eps = lr, weight_decay, beta1, beta2, eps
        self.m = torch.zeros_like(self.flat.data)
        self.v = torch.zeros_like(self.flat.data)
        self.t = 0
        self.buckets = max(1, int(buckets))
        self.device = self.flat.data.device
        self.timers = None  # optional {phase: [(start, end), ...]}
        self._ws = {}

    def _workspace(self, kind: str, nbytes: int):
        buf = self._ws.get(kind)
        if nbytes <= 0:
            return None, 0
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(nbytes, device=self.device, dtype=torch.uint8)
            self._ws[kind] = buf
        return buf, nbytes

    def _mark(self, name):
        return SplineTrainer._mark(self, name)

    def step(self, x: torch.Tensor, gy: torch.Tensor, lr: float | None = None):
        L = self.layer
        if x.dim() != 2 or x.shape[1] != L.d_in:
            raise DimensionError(f"x must be [B, {L.d_in}], got {tuple(x.shape)}")
        if gy.shape != (x.shape[0], L.d_out):
            raise DimensionError(f"gy must be [{x.shape[0]}, {L.d_out}], got {tuple(gy.shape)}")
        x = x if (x.dtype == torch.float32 and x.is_contiguous()) else x.float().contiguous()
        gy = gy if (gy.dtype == torch.float32 and gy.is_contiguous()) else gy.float().contiguous()
        st = stream_ptr()
        B = x.shape[0]
        args = (B, L.d_in, L.d_out, L.G, L.k)
        grid = (float(L.g_min), float(L.g_max))
        if getattr(self, "_err", None) is None:
            self._err = torch.zeros(1, device=self.device, dtype=torch.int32)
        y = torch.empty((B, L.d_out), device=self.device, dtype=torch.float32)
        dx = torch.empty_like(x)
        gv = self.flat.gviews
        dC, dS = gv["layer0.coeffs"], gv["layer0.scale"]
        with self._mark("forward"):
            wsf, nf = self._workspace("fwd", self.lib.ukan_kan_forward_workspace_size(*args))
            check(self.lib.ukan_kan_forward_ws(ptr(x), ptr(L.coeffs), ptr(L.scale), None, ptr(y), *args, *grid,
                                               ptr(self._err), ptr(wsf), nf, st), "kan_forward")
        wsb, nb = self._workspace("bwd", self.lib.ukan_kan_backward_workspace_size(*args))
        if B > 0 and self.lib.ukan_kan_backward_part_supported(*args):
            with self._mark("backward_prep"):
                prepared = ctypes.c_int32(0)
                check(self.lib.ukan_kan_backward_prep(ptr(x), None, *args, *grid, ptr(wsb), nb, ctypes.byref(prepared),
                                                      st), "kan_backward_prep")
            with self._mark("backward_dx"):
                check(self.lib.ukan_kan_backward_part(ptr(L.coeffs), ptr(L.scale), ptr(gy), ptr(dx), None, None, *args,
                                                      *grid, ptr(wsb), nb, 0, L.d_in, 2, st), "kan_backward_dx")
            bounds = [round(L.d_in * q / self.buckets) for q in range(self.buckets + 1)]
            with self._mark("backward_table"):
                for lo, hi in zip(bounds[:-1], bounds[1:]):
                    if hi <= lo:
                        continue
                    check(self.lib.ukan_kan_backward_part(ptr(L.coeffs), ptr(L.scale), ptr(gy), None, ptr(dC), ptr(dS),
                                                          *args, *grid, ptr(wsb), nb, lo, hi, 1, st),
                          "kan_backward_table")
                    self.sync.allreduce_async(dC[lo:hi])
                    self.sync.allreduce_async(dS[lo:hi])
        else:
            with self._mark("backward"):
                check(self.lib.ukan_kan_backward_ws2(ptr(x), ptr(L.coeffs), ptr(L.scale), None, ptr(gy), ptr(dx),
                                                     ptr(dC), ptr(dS), None, *args, *grid, ptr(wsb), nb, 0, st),
                      "kan_backward")
            self.sync.allreduce_async(self.flat.grad)
        self.sync.wait()
        self.t += 1
        with self._mark("adam"):
            check(self.lib.ukan_adam_step(ptr(self.flat.data), ptr(self.flat.grad), ptr(self.m), ptr(self.v),
                                          self.flat.data.numel(), self.lr if lr is None else lr, self.beta1,
                                          self.beta2, self.eps, self.wd, self.t, None, st), "adam")
        return y, dx

    def check_input(self) -> None:
        """Host read of the NaN flag of the steps so far (the reference raises IndexError)."""
        if getattr(self, "_err", None) is not None and int(self._err.item()):
            raise IndexError("non-finite (NaN) input to a bounded-grid KAN layer")
