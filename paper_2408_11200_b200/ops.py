"""Fused spline ops as ``torch.autograd.Function``s over the C ABI.

Each op replaces a fused group of the reference's graph ops (``ukan.layers``) and records one
node on torch's tape, the way the reference records one ``make_node`` per op
(tensor.py:96-103).  The backward computes dx only when x needs a gradient — the reference
computes dx only when x is a recorded node (tensor.py:455-456).

All arithmetic happens in ``libukan_b200.so``; these classes allocate outputs / workspaces
with torch's caching allocator and pass raw pointers plus the current stream.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import check, ptr, stream_ptr
from .errors import DomainError

# ---------------------------------------------------------------------------------------
# Input checks.  The KAN reference raises IndexError on NaN input (SURVEY gotcha 10: NaN
# survives np.clip and breaks the gather).  Detecting it needs a device->host read; in
# "eager" mode (the drop-in default) it happens inside kan_forward, in "deferred" mode the
# flags are kept on the device and checked by flush_checks() (the trainer calls it when it
# reads the loss, i.e. at a point that synchronises anyway).
# ---------------------------------------------------------------------------------------
_check_mode = "eager"
_pending: list[torch.Tensor] = []


def set_check_mode(mode: str) -> None:
    global _check_mode
    if mode not in ("eager", "deferred"):
        raise ValueError(mode)
    _check_mode = mode


def flush_checks() -> None:
    global _pending
    flags, _pending = _pending, []
    if flags and int(torch.stack(flags).max().item()):
        raise IndexError("non-finite (NaN) input to a bounded-grid KAN layer")


def _nan_check(err: torch.Tensor) -> None:
    if _check_mode == "eager":
        if int(err.item()):
            raise IndexError("non-finite (NaN) input to a bounded-grid KAN layer")
    else:
        _pending.append(err)


def _f32(t: torch.Tensor) -> torch.Tensor:
    if t.dtype != torch.float32:
        t = t.float()
    return t.contiguous()


# ---------------------------------------------------------------------------------------
# KAN spline layer
# ---------------------------------------------------------------------------------------
class KanSplineFn(torch.autograd.Function):
    """y = kan_forward(x) for coeffs [d_in, G+k, d_out] (layers.py:304-318)."""

    @staticmethod
    def forward(ctx, x, coeffs, scale, base_weight, G: int, k: int, g_min: float, g_max: float):
        lib = _lib.load()
        _lib.require_cuda(x, coeffs, scale, base_weight)
        _lib.require_params(x.device, coeffs, scale, base_weight)
        x = _f32(x)
        B, d_in = x.shape
        d_out = coeffs.shape[2]
        y = torch.empty((B, d_out), device=x.device, dtype=torch.float32)
        err = torch.zeros(1, device=x.device, dtype=torch.int32)
        nbytes = 0 if base_weight is not None else lib.ukan_kan_forward_workspace_size(B, d_in, d_out, G, k)
        ws = torch.empty(nbytes, device=x.device, dtype=torch.uint8) if nbytes > 0 else None
        check(lib.ukan_kan_forward_ws(ptr(x), ptr(coeffs), ptr(scale), ptr(base_weight), ptr(y), B, d_in,
                                      d_out, G, k, g_min, g_max, ptr(err), ptr(ws), nbytes, stream_ptr()),
              "kan_forward")
        _nan_check(err)
        ctx.save_for_backward(x, coeffs, scale, base_weight)
        ctx.meta = (G, k, float(g_min), float(g_max))
        return y

    @staticmethod
    def backward(ctx, gy):
        lib = _lib.load()
        x, coeffs, scale, bw = ctx.saved_tensors
        G, k, g_min, g_max = ctx.meta
        gy = _f32(gy)
        B, d_in = x.shape
        d_out = coeffs.shape[2]
        dx = torch.empty_like(x) if ctx.needs_input_grad[0] else None
        dC = torch.empty_like(coeffs)
        ds = torch.empty_like(scale)
        dbw = torch.empty_like(bw) if bw is not None else None
        nbytes = lib.ukan_kan_backward_workspace_size(B, d_in, d_out, G, k)
        ws = torch.empty(nbytes, device=x.device, dtype=torch.uint8) if nbytes > 0 else None
        check(lib.ukan_kan_backward_ws(ptr(x), ptr(coeffs), ptr(scale), ptr(bw), ptr(gy), ptr(dx), ptr(dC),
                                       ptr(ds), ptr(dbw), B, d_in, d_out, G, k, g_min, g_max, ptr(ws),
                                       nbytes, stream_ptr()), "kan_backward")
        return dx, dC, ds, dbw, None, None, None, None


class NaiveKanFn(torch.autograd.Function):
    """naive_kan_forward (layers.py:337-370): all G+k bases by Cox-de Boor, dotted with the whole
    coefficient table (the grid-size benchmark's comparison arm).  Backward covers the parameters
    only, as the reference."""

    @staticmethod
    def forward(ctx, x, coeffs, scale, G: int, k: int, g_min: float, g_max: float):
        lib = _lib.load()
        _lib.require_cuda(x, coeffs, scale)
        x = _f32(x)
        B, d_in = x.shape
        d_out = coeffs.shape[2]
        y = torch.empty((B, d_out), device=x.device, dtype=torch.float32)
        tmp = torch.empty((B, d_in, d_out), device=x.device, dtype=torch.float32)
        check(lib.ukan_kan_naive_forward(ptr(x), ptr(coeffs), ptr(scale), ptr(y), ptr(tmp), B, d_in, d_out, G, k,
                                         g_min, g_max, stream_ptr()), "naive_kan_forward")
        ctx.save_for_backward(x, scale, tmp)
        ctx.meta = (G, k, float(g_min), float(g_max), tuple(coeffs.shape))
        return y

    @staticmethod
    def backward(ctx, gy):
        lib = _lib.load()
        x, scale, tmp = ctx.saved_tensors
        G, k, g_min, g_max, cshape = ctx.meta
        gy = _f32(gy)
        B, d_in = x.shape
        d_out = cshape[2]
        dC = torch.empty(cshape, device=x.device, dtype=torch.float32)
        ds = torch.empty_like(scale)
        check(lib.ukan_kan_naive_backward(ptr(x), ptr(scale), ptr(tmp), ptr(gy), ptr(dC), ptr(ds), B, d_in, d_out, G,
                                          k, g_min, g_max, stream_ptr()), "naive_kan_backward")
        return None, dC, ds, None, None, None, None


def kan_locate(x: torch.Tensor, G: int, g_min: float, g_max: float):
    """(cell int32, u float64) exactly as layers.py:296-300 — for parity tooling."""
    lib = _lib.load()
    _lib.require_cuda(x)
    x = _f32(x)
    cell = torch.empty(x.shape, device=x.device, dtype=torch.int32)
    u = torch.empty(x.shape, device=x.device, dtype=torch.float64)
    check(lib.ukan_kan_locate(ptr(x), ptr(cell), ptr(u), x.shape[0], x.shape[1], G, g_min, g_max,
                              stream_ptr()), "kan_locate")
    return cell, u


# ---------------------------------------------------------------------------------------
# UKAN: keys, coefficient generator, spline over the generated table
# ---------------------------------------------------------------------------------------
class UkanKeys:
    """Unique (feature, group) keys of one batch, feature-major (see ukan_b200.h)."""

    __slots__ = ("key_f", "key_g", "seg_start", "base_row", "n_u", "max_rows")

    def __init__(self, key_f, key_g, seg_start, base_row, n_u, max_rows):
        self.key_f, self.key_g, self.seg_start, self.base_row = key_f, key_g, seg_start, base_row
        self.n_u, self.max_rows = n_u, max_rows


def ukan_build_keys(x: torch.Tensor, k: int, delta_g: float, max_keys: int | None = None) -> UkanKeys:
    """layers.py:261-287: locate, key generation, dedup (np.unique) and window rows."""
    lib = _lib.load()
    _lib.require_cuda(x)
    x = _f32(x)
    B, d_in = x.shape
    dev = x.device
    limit = max(2 * B * d_in, 1)
    cap = min(limit, max_keys or (1 << 20))
    seg_start = torch.empty(d_in + 1, device=dev, dtype=torch.int32)
    base_row = torch.empty((B, d_in), device=dev, dtype=torch.int32)
    while True:
        key_f = torch.empty(cap, device=dev, dtype=torch.int32)
        key_g = torch.empty(cap, device=dev, dtype=torch.int64)
        nbytes = lib.ukan_ukan_keys_workspace_size(B, d_in, cap)
        ws = torch.empty(nbytes, device=dev, dtype=torch.uint8)
        n_u = ctypes.c_int64(0)
        max_rows = ctypes.c_int64(0)
        nonfinite = ctypes.c_int32(0)
        rc = lib.ukan_ukan_build_keys(ptr(x), B, d_in, k, delta_g, ptr(key_f), ptr(key_g), ptr(seg_start),
                                      ptr(base_row), cap, ptr(ws), nbytes, ctypes.byref(n_u),
                                      ctypes.byref(max_rows), ctypes.byref(nonfinite), stream_ptr())
        if nonfinite.value == 1:
            raise DomainError("non-finite input")
        if nonfinite.value == 2:
            raise DomainError("input magnitude exceeds the supported grid-index range (|x/delta_g| >= 2^42)")
        if rc == _lib.UKAN_E_CAPACITY and cap < limit:
            cap = min(limit, cap * 4)
            continue
        check(rc, "ukan_build_keys")
        break
    n = int(n_u.value)
    return UkanKeys(key_f[:n], key_g[:n], seg_start, base_row, n, int(max_rows.value))


def cg_forward_raw(key_f, key_g, emb, w1, b1, w2, b2, d_pe: int, table_out=None):
    """_cg_eval (layers.py:232-243) on raw buffers, fp64 between the GEMMs:
    inp64 = [emb[f] || PE(g)] (fp64 PE), pre64 = inp64 @ W1 + b1 and H64 = silu(pre64) on the FP64
    tensor cores, H32 = (float)H64, table = H32 @ W2 + b2 on tcgen05 (tf32 pieces, fp32-exact
    products).  Returns (table [n_u, K*d_out] fp32, cache for ``cg_backward_raw``)."""
    lib = _lib.load()
    n_u = key_f.shape[0]
    d_femb = emb.shape[1]
    d_cg_in, d_h = w1.shape
    n_out = w2.shape[1]
    dev = emb.device
    st = stream_ptr()
    inp = torch.empty((n_u, d_cg_in), device=dev, dtype=torch.float64)
    pre = torch.empty((n_u, d_h), device=dev, dtype=torch.float64)
    H64 = torch.empty((n_u, d_h), device=dev, dtype=torch.float64)
    H32 = torch.empty((n_u, d_h), device=dev, dtype=torch.float32)
    table = table_out if table_out is not None else torch.empty((n_u, n_out), device=dev, dtype=torch.float32)
    if n_u > 0:
        check(lib.ukan_ukan_cg_input(ptr(key_f), ptr(key_g), ptr(emb), ptr(inp), n_u, d_femb, d_pe, st), "cg_input")
        check(lib.ukan_gemm_f64(0, ptr(inp), _lib.UKAN_F64, ptr(w1), _lib.UKAN_F32, ptr(b1), 1, ptr(pre), ptr(H32),
                                ptr(H64), None, n_u, d_h, d_cg_in, st), "cg_gemm1")
        check(lib.ukan_gemm_bias_act(ptr(H32), ptr(w2), ptr(b2), ptr(table), None, n_u, n_out, d_h, 0, st),
              "cg_gemm2")
    return table, (inp, pre, H64)


def cg_backward_raw(cache, dtable, w1, w2, seg_start, d_femb: int, dw1, db1, dw2, db2, demb):
    """Tape backward of _cg_eval (matmul / silu / gather_rows / concat_last, tensor.py:189-197,
    228-233, 257-268, 276-285) given dtable [n_u, K*d_out]: every GEMM on the FP64 tensor cores
    with fp64 intermediates (dH, dpre, dinp); gradients WRITTEN into dw1, db1, dw2, db2 and (if
    not None) demb."""
    lib = _lib.load()
    inp, pre, H64 = cache
    n_u, d_cg_in = inp.shape
    d_h = H64.shape[1]
    n_out = w2.shape[1]
    d_in = seg_start.shape[0] - 1
    dev = inp.device
    st = stream_ptr()
    if n_u == 0:
        for t in (dw1, db1, dw2, db2, demb):
            if t is not None:
                t.zero_()
        return
    F32, F64 = _lib.UKAN_F32, _lib.UKAN_F64
    check(lib.ukan_gemm_f64(2, ptr(H64), F64, ptr(dtable), F32, None, 0, None, ptr(dw2), None, ptr(db2), d_h, n_out,
                            n_u, st), "cg_dW2")
    dH = torch.empty((n_u, d_h), device=dev, dtype=torch.float64)
    check(lib.ukan_gemm_f64(1, ptr(dtable), F32, ptr(w2), F32, None, 0, None, None, ptr(dH), None, n_u, d_h, n_out,
                            st), "cg_dH")
    dpre = torch.empty_like(dH)
    check(lib.ukan_silu_backward(ptr(pre), ptr(dH), ptr(dpre), dH.numel(), st), "cg_dsilu")
    check(lib.ukan_gemm_f64(2, ptr(inp), F64, ptr(dpre), F64, None, 0, None, ptr(dw1), None, ptr(db1), d_cg_in, d_h,
                            n_u, st), "cg_dW1")
    if demb is not None:
        dinp = torch.empty_like(inp)
        check(lib.ukan_gemm_f64(1, ptr(dpre), F64, ptr(w1), F32, None, 0, None, None, ptr(dinp), None, n_u, d_cg_in,
                                d_h, st), "cg_dinp")
        check(lib.ukan_ukan_emb_backward(ptr(seg_start), ptr(dinp), ptr(demb), d_in, d_femb, d_cg_in, st), "cg_demb")


class CgMlpFn(torch.autograd.Function):
    """Coefficient generator over unique keys (layers.py:232-243):
    table = silu([emb[f] || PE(g)] @ W1 + b1) @ W2 + b2  ->  [n_u, K*d_out] (slot-major)."""

    @staticmethod
    def forward(ctx, emb, w1, b1, w2, b2, key_f, key_g, seg_start, d_pe: int):
        _lib.require_cuda(emb, w1, b1, w2, b2)
        _lib.require_params(emb.device, emb, w1, b1, w2, b2)
        table, cache = cg_forward_raw(key_f, key_g, emb, w1, b1, w2, b2, d_pe)
        ctx.save_for_backward(*cache, w1, w2, seg_start)
        ctx.d_femb = emb.shape[1]
        return table

    @staticmethod
    def backward(ctx, dtable):
        inp, pre, H64, w1, w2, seg_start = ctx.saved_tensors
        dtable = _f32(dtable)
        dev = inp.device
        d_femb = ctx.d_femb
        d_in = seg_start.shape[0] - 1
        dw1, dw2 = torch.empty_like(w1), torch.empty_like(w2)
        db1 = torch.empty(w1.shape[1], device=dev, dtype=torch.float32)
        db2 = torch.empty(w2.shape[1], device=dev, dtype=torch.float32)
        demb = torch.empty((d_in, d_femb), device=dev, dtype=torch.float32) if ctx.needs_input_grad[0] else None
        cg_backward_raw((inp, pre, H64), dtable, w1, w2, seg_start, d_femb, dw1, db1, dw2, db2, demb)
        return demb, dw1, db1, dw2, db2, None, None, None, None


class UkanSplineFn(torch.autograd.Function):
    """Spline evaluation over the generated table (layers.py:284-291)."""

    @staticmethod
    def forward(ctx, x, table, scale, base_row, seg_start, k: int, delta_g: float, max_rows: int = 0):
        lib = _lib.load()
        _lib.require_cuda(x, table, scale)
        _lib.require_params(x.device, table, scale)
        x = _f32(x)
        B, d_in = x.shape
        d_out = scale.shape[1]
        y = torch.empty((B, d_out), device=x.device, dtype=torch.float32)
        ukan_forward_into(x, base_row, seg_start, table, scale, y, k, delta_g, max_rows)
        ctx.save_for_backward(x, table, scale, base_row, seg_start)
        ctx.meta = (k, float(delta_g), int(max_rows))
        return y

    @staticmethod
    def backward(ctx, gy):
        x, table, scale, base_row, seg_start = ctx.saved_tensors
        k, delta_g, max_rows = ctx.meta
        gy = _f32(gy)
        dx = torch.empty_like(x) if ctx.needs_input_grad[0] else None
        dtable = torch.empty_like(table)
        ds = torch.empty_like(scale)
        ukan_backward_into(x, base_row, seg_start, table, scale, gy, dx, dtable, ds, k, delta_g, max_rows)
        return dx, dtable, ds, None, None, None, None, None


def ukan_forward_into(x, base_row, seg_start, table, scale, y, k: int, delta_g: float, max_rows: int = 0) -> None:
    """y of the UKAN spline over the generated table (layers.py:284-291).  Dense layers (every
    feature's segment <= 67 rows, d_out >= 128) take the TMEM-gather forward
    (ukan_ukan_forward_dense); the others the gather kernel (ukan_ukan_forward)."""
    lib = _lib.load()
    B, d_in = x.shape
    d_out = scale.shape[1]
    st = stream_ptr()
    nbytes = lib.ukan_ukan_forward_dense_workspace_size(B, d_in, d_out, max_rows, k) if max_rows > 0 else 0
    if nbytes > 0:
        ws = torch.empty(nbytes, device=x.device, dtype=torch.uint8)
        check(lib.ukan_ukan_forward_dense(ptr(x), ptr(base_row), ptr(seg_start), ptr(table), ptr(scale), ptr(y), B,
                                          d_in, d_out, max_rows, k, delta_g, ptr(ws), nbytes, st), "ukan_forward_dense")
        return
    check(lib.ukan_ukan_forward(ptr(x), ptr(base_row), ptr(table), ptr(scale), ptr(y), B, d_in, d_out, k, delta_g, st),
          "ukan_forward")


def ukan_backward_into(x, base_row, seg_start, table, scale, gy, dx, dtable, dscale, k: int, delta_g: float,
                       max_rows: int = 0) -> None:
    """dx (optional), dtable, dscale of the UKAN spline (layers.py:284-291 backward).  Dense layers
    (every feature's virtual table <= 67 rows: max_rows from ukan_build_keys) take the KAN FP64
    tensor-core backward (ukan_ukan_backward_dense); the others the sorted-merge sweep."""
    lib = _lib.load()
    B, d_in = x.shape
    d_out = scale.shape[1]
    n_u = table.shape[0]
    st = stream_ptr()
    if max_rows > 0:  # dense layers on the tensor-core path; max_rows also bounds the sorted sweep's histogram
        nbytes = lib.ukan_ukan_backward2_workspace_size(B, d_in, d_out, n_u, max_rows, k)
        ws = torch.empty(max(nbytes, 8), device=x.device, dtype=torch.uint8)
        check(lib.ukan_ukan_backward2(ptr(x), ptr(base_row), ptr(seg_start), ptr(table), ptr(scale), ptr(gy), ptr(dx),
                                      ptr(dtable), ptr(dscale), B, d_in, d_out, n_u, max_rows, k, delta_g, ptr(ws),
                                      nbytes, st), "ukan_backward2")
        return
    nbytes = lib.ukan_ukan_backward_workspace_size(B, d_in, d_out, n_u, k)
    ws = torch.empty(max(nbytes, 8), device=x.device, dtype=torch.uint8)
    check(lib.ukan_ukan_backward(ptr(x), ptr(base_row), ptr(seg_start), ptr(table), ptr(scale), ptr(gy), ptr(dx),
                                 ptr(dtable), ptr(dscale), B, d_in, d_out, n_u, k, delta_g, ptr(ws), nbytes, st),
          "ukan_backward")


class KanJvpFn(torch.autograd.Function):
    """Forward tangent ty = (dy/dx) . tx of kan_forward — the tangent channel of basis_features /
    edge_combine / clamp / silu (layers.py:49-53, 91-104; tensor.py:236-241, 336-337).  Its
    backward is the reverse pass through that tangent graph (forward-over-reverse, as pinn_loss
    needs, tasks.py:153-166): dx (tangent share), dtx, dcoeffs, dscale, dbase_weight."""

    @staticmethod
    def forward(ctx, x, tx, coeffs, scale, base_weight, G: int, k: int, g_min: float, g_max: float):
        lib = _lib.load()
        _lib.require_cuda(x, tx, coeffs, scale, base_weight)
        _lib.require_params(x.device, coeffs, scale, base_weight)
        x, tx = _f32(x), _f32(tx)
        B, d_in = x.shape
        d_out = coeffs.shape[2]
        ty = torch.empty((B, d_out), device=x.device, dtype=torch.float32)
        check(lib.ukan_kan_jvp_forward(ptr(x), ptr(tx), ptr(coeffs), ptr(scale), ptr(base_weight), ptr(ty), B, d_in,
                                       d_out, G, k, g_min, g_max, stream_ptr()), "kan_jvp_forward")
        ctx.save_for_backward(x, tx, coeffs, scale, base_weight)
        ctx.meta = (G, k, float(g_min), float(g_max))
        return ty

    @staticmethod
    def backward(ctx, gt):
        lib = _lib.load()
        x, tx, coeffs, scale, bw = ctx.saved_tensors
        G, k, g_min, g_max = ctx.meta
        gt = _f32(gt)
        B, d_in = x.shape
        d_out = coeffs.shape[2]
        dx = torch.empty_like(x) if ctx.needs_input_grad[0] else None
        dtx = torch.empty_like(tx) if ctx.needs_input_grad[1] else None
        dC = torch.empty_like(coeffs)
        ds = torch.empty_like(scale)
        dbw = torch.empty_like(bw) if bw is not None else None
        check(lib.ukan_kan_jvp_backward(ptr(x), ptr(tx), ptr(coeffs), ptr(scale), ptr(bw), ptr(gt), ptr(dx), ptr(dtx),
                                        ptr(dC), ptr(ds), ptr(dbw), B, d_in, d_out, G, k, g_min, g_max,
                                        stream_ptr()), "kan_jvp_backward")
        return dx, dtx, dC, ds, dbw, None, None, None, None


class UkanJvpFn(torch.autograd.Function):
    """Forward tangent of the UKAN spline over the generated table (u = x/dg - g_id carries
    tx/dg, layers.py:264; the table itself has no tangent) and its reverse pass: dx (tangent
    share), dtx, dtable (flows on into the CG backward), dscale."""

    @staticmethod
    def forward(ctx, x, tx, table, scale, base_row, seg_start, k: int, delta_g: float):
        lib = _lib.load()
        _lib.require_cuda(x, tx, table, scale)
        _lib.require_params(x.device, table, scale)
        x, tx = _f32(x), _f32(tx)
        B, d_in = x.shape
        d_out = scale.shape[1]
        ty = torch.empty((B, d_out), device=x.device, dtype=torch.float32)
        check(lib.ukan_ukan_jvp_forward(ptr(x), ptr(tx), ptr(base_row), ptr(table), ptr(scale), ptr(ty), B, d_in,
                                        d_out, k, delta_g, stream_ptr()), "ukan_jvp_forward")
        ctx.save_for_backward(x, tx, table, scale, base_row, seg_start)
        ctx.meta = (k, float(delta_g))
        return ty

    @staticmethod
    def backward(ctx, gt):
        lib = _lib.load()
        x, tx, table, scale, base_row, seg_start = ctx.saved_tensors
        k, delta_g = ctx.meta
        gt = _f32(gt)
        B, d_in = x.shape
        d_out = scale.shape[1]
        n_u = table.shape[0]
        dx = torch.empty_like(x) if ctx.needs_input_grad[0] else None
        dtx = torch.empty_like(tx) if ctx.needs_input_grad[1] else None
        dtable = torch.empty_like(table)
        ds = torch.empty_like(scale)
        check(lib.ukan_ukan_jvp_backward(ptr(x), ptr(tx), ptr(base_row), ptr(seg_start), ptr(table), ptr(scale),
                                         ptr(gt), ptr(dx), ptr(dtx), ptr(dtable), ptr(ds), B, d_in, d_out, n_u, k,
                                         delta_g, stream_ptr()), "ukan_jvp_backward")
        return dx, dtx, dtable, ds, None, None, None, None
