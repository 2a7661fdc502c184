"""Drop-in mirror of the reference's layer API (``ukan.layers``, layers.py:1-447) on CUDA.

Same names, constructor arguments, parameter names / shapes / layouts, initial values (the
same NumPy draws, rounded to fp32) and exception types as the reference; tensors are
``torch.Tensor`` on the CUDA device and gradients come from ``loss.backward()``.  Every
spline layer call runs the fused sm_100a kernels of ``libukan_b200.so`` (see ``ops.py``).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import ops
from .errors import ConfigError, DimensionError

_DEFAULT_DEVICE = "cuda"


def _device(device=None):
    return torch.device(device if device is not None else _DEFAULT_DEVICE)


def _param(a: np.ndarray, device) -> torch.Tensor:
    return torch.tensor(np.asarray(a, dtype=np.float64), dtype=torch.float32, device=device).requires_grad_(True)


def as_input(x, device=None) -> torch.Tensor:
    """Accept a torch tensor or array-like; return an fp32 tensor on the CUDA device
    (differentiably, so gradients reach a caller's leaf)."""
    if not isinstance(x, torch.Tensor):
        x = torch.as_tensor(np.asarray(x, dtype=np.float64))
    dev = _device(device) if not x.is_cuda else x.device
    return x.to(device=dev, dtype=torch.float32)


# ---------------------------------------------------------------------------------------
# grid-group helpers (layers.py:112-131)
# ---------------------------------------------------------------------------------------
def positional_encoding(g, d_pe: int) -> torch.Tensor:
    """Sinusoidal encoding of (possibly negative) group indices (layers.py:112-123), float64.
    Host utility mirroring the reference; the kernels evaluate the same formula in fp64."""
    if d_pe % 2 != 0:
        raise ConfigError(f"encoding width must be even, got {d_pe}")
    g = torch.as_tensor(np.asarray(g, dtype=np.float64))
    half = d_pe // 2
    freqs = torch.as_tensor(10000.0 ** (-2.0 * np.arange(half) / d_pe))
    ang = g[..., None] * freqs
    pe = torch.empty(tuple(g.shape) + (d_pe,), dtype=torch.float64)
    pe[..., 0::2] = torch.sin(ang)
    pe[..., 1::2] = torch.cos(ang)
    return pe


def select_window(prev, nxt, g_id: int, K: int):
    """The K coefficients cell g_id consumes out of its group pair (layers.py:126-131)."""
    i = g_id % K
    if isinstance(prev, torch.Tensor):
        both = torch.cat([prev, nxt], dim=-1)
    else:
        both = np.concatenate([np.asarray(prev), np.asarray(nxt)], axis=-1)
    return both[..., i:i + K]


# ---------------------------------------------------------------------------------------
# layers (layers.py:138-229)
# ---------------------------------------------------------------------------------------
@dataclass(eq=False)
class KanLayer:
    d_in: int
    d_out: int
    k: int
    g_min: float
    g_max: float
    G: int
    coeffs: torch.Tensor  # [d_in, G+k, d_out]
    scale: torch.Tensor   # [d_in, d_out]
    base_weight: torch.Tensor | None = None

    def __post_init__(self):
        if not (self.g_min < self.g_max and self.G >= 1):
            raise ConfigError("grid must satisfy g_min < g_max and G >= 1")
        if tuple(self.coeffs.shape) != (self.d_in, self.G + self.k, self.d_out):
            raise ConfigError(f"coefficient table must be [d_in, G+k, d_out], got {tuple(self.coeffs.shape)}")

    @property
    def delta_g(self) -> float:
        return (self.g_max - self.g_min) / self.G

    def parameters(self) -> dict[str, torch.Tensor]:
        p = {"coeffs": self.coeffs, "scale": self.scale}
        if self.base_weight is not None:
            p["base_weight"] = self.base_weight
        return p

    def forward(self, x):
        return kan_forward(self, x)

    def forward_tangent(self, x, tx):
        return kan_forward_tangent(self, x, tx)

    __call__ = forward


@dataclass(eq=False)
class UkanLayer:
    d_in: int
    d_out: int
    k: int
    delta_g: float
    d_pe: int
    d_femb: int
    feature_embedding: torch.Tensor  # [d_in, d_femb]
    cg_w1: torch.Tensor              # [d_femb + d_pe, d_hidden]
    cg_b1: torch.Tensor              # [d_hidden]
    cg_w2: torch.Tensor              # [d_hidden, d_out*K]
    cg_b2: torch.Tensor              # [d_out*K]
    scale: torch.Tensor              # [d_in, d_out]

    def __post_init__(self):
        if self.d_pe % 2 != 0:
            raise ConfigError(f"encoding width must be even, got {self.d_pe}")
        if self.delta_g <= 0:
            raise ConfigError(f"grid spacing must be positive, got {self.delta_g}")
        if self.cg_w2.shape[1] != self.d_out * (self.k + 1):
            raise ConfigError("generator output width must be d_out*(k+1)")

    @property
    def K(self) -> int:
        return self.k + 1

    def parameters(self) -> dict[str, torch.Tensor]:
        return {
            "feature_embedding": self.feature_embedding,
            "cg_w1": self.cg_w1,
            "cg_b1": self.cg_b1,
            "cg_w2": self.cg_w2,
            "cg_b2": self.cg_b2,
            "scale": self.scale,
        }

    def forward(self, x):
        return ukan_forward(self, x)

    def forward_tangent(self, x, tx):
        return ukan_forward_tangent(self, x, tx)

    __call__ = forward


@dataclass(eq=False)
class LinearLayer:
    """MLP baseline layer (layers.py:216-229).  Out of the hot-path scope; plain torch."""
    d_in: int
    d_out: int
    weight: torch.Tensor
    bias: torch.Tensor

    def parameters(self) -> dict[str, torch.Tensor]:
        return {"weight": self.weight, "bias": self.bias}

    def forward(self, x):
        return as_input(x) @ self.weight + self.bias

    __call__ = forward


# ---------------------------------------------------------------------------------------
# fused forward entry points
# ---------------------------------------------------------------------------------------
def kan_forward(layer: KanLayer, x) -> torch.Tensor:
    """Bounded-grid KAN layer (layers.py:304-318) — one fused kernel forward, one fused
    fp64 backward."""
    x = as_input(x, layer.coeffs.device)
    if x.ndim != 2 or x.shape[1] != layer.d_in:
        raise DimensionError(f"expected [batch, {layer.d_in}] input, got {tuple(x.shape)}")
    return ops.KanSplineFn.apply(x, layer.coeffs, layer.scale, layer.base_weight, layer.G, layer.k,
                                 float(layer.g_min), float(layer.g_max))


def naive_kan_forward(layer: KanLayer, x) -> torch.Tensor:
    """Same contract as kan_forward computed the slow way (layers.py:337-370): all G+k basis
    functions per input dotted with the full coefficient table; parameter gradients only.
    The comparison arm of the grid-size benchmark (``bench_arms.run_bench``)."""
    x = as_input(x, layer.coeffs.device)
    if x.ndim != 2 or x.shape[1] != layer.d_in:
        raise DimensionError(f"expected [batch, {layer.d_in}] input, got {tuple(x.shape)}")
    y = ops.NaiveKanFn.apply(x.detach(), layer.coeffs, layer.scale, layer.G, layer.k, float(layer.g_min),
                             float(layer.g_max))
    if layer.base_weight is not None:
        y = y + torch.nn.functional.silu(x) @ layer.base_weight
    return y


def _cg_table(layer: UkanLayer, keys: ops.UkanKeys) -> torch.Tensor:
    return ops.CgMlpFn.apply(layer.feature_embedding, layer.cg_w1, layer.cg_b1, layer.cg_w2, layer.cg_b2,
                             keys.key_f, keys.key_g, keys.seg_start, layer.d_pe)


def ukan_forward(layer: UkanLayer, x, dedup: bool = True) -> torch.Tensor:
    """Unbounded-grid UKAN layer (layers.py:254-291).  ``dedup`` is accepted for API parity;
    the generator always runs once per unique (feature, group) key, which the reference
    shows is bitwise identical to dedup=False (test_layers.py:147-152)."""
    x = as_input(x, layer.scale.device)
    if x.ndim != 2 or x.shape[1] != layer.d_in:
        raise DimensionError(f"expected [batch, {layer.d_in}] input, got {tuple(x.shape)}")
    keys = ops.ukan_build_keys(x.detach(), layer.k, float(layer.delta_g))
    table = _cg_table(layer, keys)
    return ops.UkanSplineFn.apply(x, table, layer.scale, keys.base_row, keys.seg_start, layer.k,
                                  float(layer.delta_g), keys.max_rows)


def kan_forward_tangent(layer: KanLayer, x, tx):
    """kan_forward on x seeded with the tangent direction tx (the reference's
    ``T.seed_tangent(x, tx)`` then ``y.tangent``, tensor.py:411-424): returns (y, ty) with
    ty = (dy/dx) . tx, differentiable in x, tx and the parameters (forward-over-reverse)."""
    x = as_input(x, layer.coeffs.device)
    tx = as_input(tx, layer.coeffs.device)
    if tx.shape != x.shape:
        raise DimensionError(f"tangent seed shape {tuple(tx.shape)} != {tuple(x.shape)}")
    y = kan_forward(layer, x)
    ty = ops.KanJvpFn.apply(x, tx, layer.coeffs, layer.scale, layer.base_weight, layer.G, layer.k,
                            float(layer.g_min), float(layer.g_max))
    return y, ty


def ukan_forward_tangent(layer: UkanLayer, x, tx, dedup: bool = True):
    """ukan_forward on x seeded with the tangent tx: (y, ty), one generated table shared by both."""
    x = as_input(x, layer.scale.device)
    tx = as_input(tx, layer.scale.device)
    if x.ndim != 2 or x.shape[1] != layer.d_in:
        raise DimensionError(f"expected [batch, {layer.d_in}] input, got {tuple(x.shape)}")
    if tx.shape != x.shape:
        raise DimensionError(f"tangent seed shape {tuple(tx.shape)} != {tuple(x.shape)}")
    keys = ops.ukan_build_keys(x.detach(), layer.k, float(layer.delta_g))
    table = _cg_table(layer, keys)
    y = ops.UkanSplineFn.apply(x, table, layer.scale, keys.base_row, keys.seg_start, layer.k, float(layer.delta_g),
                               keys.max_rows)
    ty = ops.UkanJvpFn.apply(x, tx, table, layer.scale, keys.base_row, keys.seg_start, layer.k,
                             float(layer.delta_g))
    return y, ty


def cg_coefficients(layer: UkanLayer, f: int, g: int) -> torch.Tensor:
    """Coefficients of one grid group, shape [d_out, K] (layers.py:246-251)."""
    if not (0 <= f < layer.d_in):
        raise IndexError(f"feature index {f} out of range [0, {layer.d_in})")
    dev = layer.scale.device
    key_f = torch.tensor([f], dtype=torch.int32, device=dev)
    key_g = torch.tensor([g], dtype=torch.int64, device=dev)
    seg = torch.tensor([0] * (f + 1) + [1] * (layer.d_in - f), dtype=torch.int32, device=dev)
    keys = ops.UkanKeys(key_f, key_g, seg, None, 1, layer.K)
    table = _cg_table(layer, keys)
    return table.reshape(layer.K, layer.d_out).transpose(0, 1)


# ---------------------------------------------------------------------------------------
# initialization and model stacking (layers.py:377-447)
# ---------------------------------------------------------------------------------------
def init_layer(kind: str, d_in: int, d_out: int, k: int = 3, *, rng=None, seed=None,
               g_min: float = -1.0, g_max: float = 1.0, G: int = 8,
               delta_g: float = 1.0, d_pe: int = 8, d_femb: int = 8,
               d_hidden: int | None = None, base: bool = False, device=None):
    """Same draws (NumPy default_rng, same order and shapes) as layers.py:377-410, rounded
    to fp32 on the CUDA device."""
    if d_in < 1 or d_out < 1 or k < 0:
        raise ConfigError(f"invalid dims d_in={d_in}, d_out={d_out}, k={k}")
    if rng is None:
        rng = np.random.default_rng(seed)
    dev = _device(device)
    K = k + 1
    if kind == "kan":
        coeffs = _param(rng.normal(0.0, 0.1 / math.sqrt(d_in), (d_in, G + k, d_out)), dev)
        scale = _param(np.ones((d_in, d_out)), dev)
        base_w = _param(rng.normal(0.0, 0.1 / math.sqrt(d_in), (d_in, d_out)), dev) if base else None
        return KanLayer(d_in, d_out, k, g_min, g_max, G, coeffs, scale, base_w)
    if kind == "ukan":
        if d_hidden is None:
            d_hidden = 2 * (d_pe + d_femb)
        d_cg_in = d_femb + d_pe
        return UkanLayer(
            d_in, d_out, k, delta_g, d_pe, d_femb,
            feature_embedding=_param(rng.normal(0.0, 1.0, (d_in, d_femb)), dev),
            cg_w1=_param(rng.normal(0.0, 0.1 / math.sqrt(d_cg_in), (d_cg_in, d_hidden)), dev),
            cg_b1=_param(np.zeros(d_hidden), dev),
            cg_w2=_param(rng.normal(0.0, 0.1 / math.sqrt(d_hidden), (d_hidden, d_out * K)), dev),
            cg_b2=_param(np.zeros(d_out * K), dev),
            scale=_param(np.ones((d_in, d_out)), dev),
        )
    if kind == "linear":
        return LinearLayer(
            d_in, d_out,
            weight=_param(rng.normal(0.0, 1.0 / math.sqrt(d_in), (d_in, d_out)), dev),
            bias=_param(np.zeros(d_out), dev),
        )
    raise ConfigError(f"unknown layer kind {kind!r}")


@dataclass(eq=False)
class Model:
    """A stack of layers; spline layers connect directly, 'mlp' inserts SiLU (layers.py:413-435)."""
    kind: str
    layers: list = field(default_factory=list)

    def forward_tangent(self, x, tx):
        """(f(x), df/dx . tx) through the spline stack (the reference's seed_tangent +
        Model.forward, tensor.py:411-424, layers.py:420-426)."""
        if self.kind == "mlp":
            raise ConfigError("forward_tangent covers spline stacks (kan / ukan)")
        h, th = x, tx
        for layer in self.layers:
            h, th = layer.forward_tangent(h, th)
        return h, th

    def forward(self, x):
        h = x
        for i, layer in enumerate(self.layers):
            h = layer(h)
            if self.kind == "mlp" and i < len(self.layers) - 1:
                h = torch.nn.functional.silu(h)
        return h

    __call__ = forward

    def parameters(self) -> dict[str, torch.Tensor]:
        out = {}
        for i, layer in enumerate(self.layers):
            for name, p in layer.parameters().items():
                out[f"layer{i}.{name}"] = p
        return out


def build_model(kind: str, widths: list[int], k: int = 3, *, seed=None, device=None, **layer_kw) -> Model:
    if len(widths) < 2:
        raise ConfigError("need at least input and output widths")
    rng = np.random.default_rng(seed)
    layer_kind = "linear" if kind == "mlp" else kind
    layers = [init_layer(layer_kind, widths[i], widths[i + 1], k, rng=rng, device=device, **layer_kw)
              for i in range(len(widths) - 1)]
    return Model(kind=kind, layers=layers)
