"""B200-native (sm_100a) matrix-form B-spline KAN / UKAN layers — a drop-in for the hot path
of arXiv 2408.11200's reference package ``ukan`` (layers.py), with fused CUDA kernels behind a
C ABI (``include/ukan_b200.h``, ``libukan_b200.so``) and a data-parallel training step."""

from .bspline import BasisMatrix, basis_matrix
from .errors import (ConfigError, ContractError, DimensionError, DivergedError, DomainError,
                     FormatError, UkanError)
from .layers import (KanLayer, LinearLayer, Model, UkanLayer, build_model, cg_coefficients,
                     init_layer, kan_forward, kan_forward_tangent, naive_kan_forward, positional_encoding, select_window,
                     ukan_forward, ukan_forward_tangent)
from .optim import AdamState, LrSchedule, adam_step, lr_at, sgd_step
from .ops import flush_checks, set_check_mode
from .pinn import PinnProblem, pinn_loss
from .train import CapturedStep, DevicePrefetcher, GradSync, LayerTrainer, SplineTrainer, shard_bounds

__all__ = [name for name in dir() if not name.startswith("_")]
__version__ = "0.1.0"
