"""Physics-informed loss over the forward tangent — the caller of the F2 path.

Mirrors ``PinnProblem`` / ``pinn_loss`` (tasks.py:133-166): logistic growth df/dt = R f (1 - f)
with f(0) = 1/2; df/dt comes from the layer's forward tangent (``Model.forward_tangent`` ->
``KanJvpFn`` / ``UkanJvpFn``), so the loss stays differentiable in the model parameters.  The
residual arithmetic on the [n, 1] outputs is a handful of elementwise torch ops (float64, as
the reference); every spline evaluation and its derivatives run in ``libukan_b200.so``.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .errors import ConfigError
from .layers import as_input


@dataclass(frozen=True)
class PinnProblem:
    """Logistic growth df/dt = R f (1 - f) with f(0) = 0.5 (tasks.py:133-149)."""
    growth_rate: float = 1.0
    t_lo: float = -5.0
    t_hi: float = 5.0
    n_collocation: int = 128

    def __post_init__(self):
        if not (self.t_lo < self.t_hi and self.n_collocation >= 1):
            raise ConfigError("need t_lo < t_hi and at least one collocation point")

    def analytic(self, t: np.ndarray) -> np.ndarray:
        return 1.0 / (1.0 + np.exp(-self.growth_rate * t))

    def sample_collocation(self, rng) -> np.ndarray:
        return rng.uniform(self.t_lo, self.t_hi, (self.n_collocation, 1))


def _tangent_fn(model):
    for obj in (model, getattr(model, "__self__", None)):
        if obj is not None and hasattr(obj, "forward_tangent"):
            return obj.forward_tangent, obj
    raise ConfigError("pinn_loss needs a spline model (or its bound forward) with a forward tangent")


def pinn_loss(model, problem: PinnProblem, collocation) -> torch.Tensor:
    """mean((df/dt - R f (1 - f))^2) + (f(0) - 0.5)^2 (tasks.py:153-166), float64 scalar."""
    fwd_tan, obj = _tangent_fn(model)
    dev = next(iter(obj.parameters().values())).device
    t = as_input(collocation, dev)
    fv, df = fwd_tan(t, torch.ones_like(t))
    if fv.ndim != 2 or fv.shape[1] != 1:
        raise ConfigError(f"model must map scalar t to scalar f, got output {tuple(fv.shape)}")
    f64, df64 = fv.double(), df.double()
    r = problem.growth_rate
    residual = df64 - r * (f64 * (1.0 - f64))
    f0 = obj.forward(as_input([[0.0]], dev)).double()
    return (residual * residual).mean() + ((f0 - 0.5) ** 2).mean()
