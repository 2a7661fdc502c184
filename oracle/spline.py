"""Float64 NumPy restatement of the reference hot path — TEST INFRASTRUCTURE ONLY.

Every function names the reference file:line (under /root/reference/pkg/src/ukan/) it
restates.  Gradients are written out explicitly (the reference obtains the same quantities
from its tape: tensor.py:427-474 over the bwd closures in layers.py:44-46, 67-70, 84-88).
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

_M_CACHE: dict[int, np.ndarray] = {}


def basis_matrix(k: int) -> np.ndarray:
    """Exact K x K basis matrix rounded to float64 (bspline.py:24-80)."""
    if k in _M_CACHE:
        return _M_CACHE[k]
    polys = {0: [Fraction(1)]}
    for kk in range(1, k + 1):
        nxt = {}
        for j in range(-kk, 1):
            c = [Fraction(0)] * (kk + 1)
            left, right = polys.get(j), polys.get(j + 1)
            if left is not None:
                for i, a in enumerate(left):
                    c[i + 1] += a / kk
                    c[i] += a * Fraction(-j, kk)
            if right is not None:
                for i, a in enumerate(right):
                    c[i] += a * Fraction(j + kk + 1, kk)
                    c[i + 1] -= a / kk
            nxt[j] = c
        polys = nxt
    cols = [polys[j - k] for j in range(k + 1)]
    M = np.array([[float(cols[j][i]) for j in range(k + 1)] for i in range(k + 1)])
    _M_CACHE[k] = M
    return M


def basis_values(u: np.ndarray, k: int, d: int = 0) -> np.ndarray:
    """Rows of U^(d) . M (layers.py:29-37)."""
    if d > k:
        return np.zeros(u.shape + (k + 1,))
    U = np.zeros(u.shape + (k + 1,))
    for j in range(d, k + 1):
        U[..., j] = math.perm(j, d) * u ** (j - d)
    return U @ basis_matrix(k)


def kan_locate(x: np.ndarray, g_min: float, g_max: float, G: int):
    """layers.py:294-301 with the clamp of tensor.py:327-338.  Returns (cell int64, u, mask)."""
    x = np.asarray(x, dtype=np.float64)
    hi = np.nextafter(g_max, g_min)
    xc = np.clip(x, g_min, hi)
    mask = ((x >= g_min) & (x <= hi)).astype(np.float64)
    dg = (g_max - g_min) / G
    cell = np.clip(np.floor((xc - g_min) / dg), 0, G - 1).astype(np.int64)
    u = xc * (1.0 / dg) - (cell.astype(np.float64) + g_min / dg)
    return cell, u, mask


def _silu(x):
    s = 1.0 / (1.0 + np.exp(-x))
    return x * s, s + x * s * (1.0 - s)


def _spline_fwd_bwd(table, rows, cols, u, scale, gy, k, need_dx):
    """span_gather (layers.py:57-75) + basis_features (40-54) + edge_combine (78-105) and
    their bwd closures.  table [P, C, d_out]; rows/cols [B, f, K]."""
    windows = table[rows, cols]                               # layers.py:65
    basis = basis_values(u, k)                                # layers.py:42
    tmp = np.einsum("bfj,bfjo->bfo", basis, windows)          # layers.py:81
    y = np.einsum("bfo,fo->bo", tmp, scale)                   # layers.py:82
    if gy is None:
        return y, None
    dtmp = gy[:, None, :] * scale[None, :, :]                 # layers.py:85
    dscale = np.einsum("bo,bfo->fo", gy, tmp)                 # layers.py:86
    dbasis = np.einsum("bfo,bfjo->bfj", dtmp, windows)        # layers.py:87
    dwin = basis[..., None] * dtmp[:, :, None, :]             # layers.py:88
    dtable = np.zeros_like(table)
    np.add.at(dtable, (rows, cols), dwin)                     # layers.py:67-70
    du = (dbasis * basis_values(u, k, 1)).sum(axis=-1) if need_dx else None  # layers.py:44-46
    return y, dict(dtable=dtable, dscale=dscale, du=du)


def kan_forward_backward(x, coeffs, scale, gy=None, *, k, g_min, g_max, G, base_weight=None,
                         need_dx=True):
    """kan_forward (layers.py:304-318) and, given gy = dL/dy, every gradient the reference's
    tape produces (dx only matters when x is a recorded node, tensor.py:455-456)."""
    x = np.asarray(x, dtype=np.float64)
    B, f = x.shape
    K = k + 1
    cell, u, mask = kan_locate(x, g_min, g_max, G)
    rows = np.broadcast_to(np.arange(f)[None, :, None], (B, f, K))      # layers.py:311
    cols = cell[..., None] + np.arange(K)                                # layers.py:312
    y, g = _spline_fwd_bwd(coeffs, rows, cols, u, scale, gy, k, need_dx)
    out = dict(y=y, cell=cell, u=u)
    if base_weight is not None:                                          # layers.py:316-317
        sx, dsx = _silu(x)
        y = y + sx @ base_weight
        out["y"] = y
    if gy is None:
        return out
    out.update(dcoeffs=g["dtable"], dscale=g["dscale"])
    if need_dx:
        dx = g["du"] * (1.0 / ((g_max - g_min) / G)) * mask              # mul/sub + clamp bwd
        if base_weight is not None:
            dx = dx + dsx * (gy @ base_weight.T)
        out["dx"] = dx
    if base_weight is not None:
        out["dbase_weight"] = sx.T @ gy
    return out


def ukan_locate(x: np.ndarray, delta_g: float, k: int):
    """layers.py:261-267: g_id = floor(x*(1/dg)), u = x*(1/dg) - g_id, Euclidean group/offset."""
    x = np.asarray(x, dtype=np.float64)
    inv = 1.0 / delta_g
    g_id = np.floor(x * inv).astype(np.int64)
    u = x * inv - g_id.astype(np.float64)
    K = k + 1
    return g_id, u, g_id // K, g_id % K


def ukan_keys(x, delta_g, k):
    """layers.py:268-278: keys (group*d_in + f, (group+1)*d_in + f) and np.unique."""
    B, f = x.shape
    g_id, u, group, offset = ukan_locate(x, delta_g, k)
    feat = np.broadcast_to(np.arange(f, dtype=np.int64)[None, :], (B, f))
    all_keys = np.concatenate([(group * f + feat).ravel(), ((group + 1) * f + feat).ravel()])
    uniq, inverse = np.unique(all_keys, return_inverse=True)
    return uniq, inverse, g_id, u, offset


def positional_encoding(g, d_pe: int) -> np.ndarray:
    """layers.py:112-123."""
    g = np.asarray(g, dtype=np.float64)
    half = d_pe // 2
    freqs = 10000.0 ** (-2.0 * np.arange(half) / d_pe)
    ang = g[..., None] * freqs
    pe = np.empty(g.shape + (d_pe,))
    pe[..., 0::2] = np.sin(ang)
    pe[..., 1::2] = np.cos(ang)
    return pe


def cg_forward(keys, d_in, emb, w1, b1, w2, b2, d_pe, K, d_out):
    """_cg_eval (layers.py:232-243): returns (table [n, K, d_out], cache for backward)."""
    f_idx = keys % d_in
    groups = keys // d_in
    inp = np.concatenate([emb[f_idx], positional_encoding(groups, d_pe)], axis=-1)
    pre = inp @ w1 + b1
    s = 1.0 / (1.0 + np.exp(-pre))
    H = pre * s
    out = H @ w2 + b2
    return out.reshape(keys.shape[0], K, d_out), dict(f_idx=f_idx, inp=inp, pre=pre, s=s, H=H)


def _cg_backward(c, p, dtable):
    """Tape backward of _cg_eval (layers.py:232-243) through matmul/silu/gather_rows/concat_last
    (tensor.py:189-197, 228-233, 257-268, 276-285), given dL/dtable [n, K, d_out]."""
    dout = dtable.reshape(dtable.shape[0], -1)                            # reshape bwd
    dw2 = c["H"].T @ dout
    db2 = dout.sum(axis=0)
    dH = dout @ p["cg_w2"].T
    dpre = dH * (c["s"] + c["pre"] * c["s"] * (1.0 - c["s"]))            # tensor.py:233
    dw1 = c["inp"].T @ dpre
    db1 = dpre.sum(axis=0)
    dinp = dpre @ p["cg_w1"].T
    demb = np.zeros_like(p["feature_embedding"])
    np.add.at(demb, c["f_idx"], dinp[:, :p["feature_embedding"].shape[1]])  # tensor.py:265-268
    return dict(dcg_w1=dw1, dcg_b1=db1, dcg_w2=dw2, dcg_b2=db2, dfeature_embedding=demb)


def ukan_forward_backward(x, p, gy=None, *, k, delta_g, d_pe, need_dx=True):
    """ukan_forward (layers.py:254-291) + the tape backward through span_gather, the CG MLP
    (matmul/silu/gather_rows/concat_last, tensor.py:189-197, 228-233, 257-268, 276-285).
    p: dict with feature_embedding, cg_w1, cg_b1, cg_w2, cg_b2, scale (float64)."""
    x = np.asarray(x, dtype=np.float64)
    B, f = x.shape
    K = k + 1
    d_out = p["scale"].shape[1]
    uniq, inverse, g_id, u, offset = ukan_keys(x, delta_g, k)
    n = B * f
    table, c = cg_forward(uniq, f, p["feature_embedding"], p["cg_w1"], p["cg_b1"], p["cg_w2"],
                          p["cg_b2"], d_pe, K, d_out)
    idx_prev = inverse[:n].reshape(B, f)
    idx_next = inverse[n:].reshape(B, f)
    col = offset[..., None] + np.arange(K)                                # layers.py:285
    rows = np.where(col < K, idx_prev[..., None], idx_next[..., None])    # layers.py:286
    cols = col % K                                                        # layers.py:287
    y, g = _spline_fwd_bwd(table, rows, cols, u, p["scale"], gy, k, need_dx)
    out = dict(y=y, g_id=g_id, uniq=uniq)
    if gy is None:
        return out
    out.update(dscale=g["dscale"], table=table, **_cg_backward(c, p, g["dtable"]))
    if need_dx:
        out["dx"] = g["du"] * (1.0 / delta_g)                            # T.mul(x, inv_dg) bwd
    return out


def _silu2(x):
    """Second derivative of silu, d/dx [s + x s (1 - s)] (the tape derivative of the silu
    tangent, tensor.py:236-241)."""
    s = 1.0 / (1.0 + np.exp(-x))
    return s * (1.0 - s) * (2.0 + x * (1.0 - 2.0 * s))


def _spline_tangent(table, rows, cols, u, tu, scale, gt, k):
    """Forward tangent of span_gather + basis_features + edge_combine when only u carries a
    tangent tu (basis.tangent = w'(u) * u.tangent, layers.py:49-53; edge_combine of the tangent
    basis, layers.py:91-104), and the tape backward of sum(ty * gt) through that tangent graph."""
    windows = table[rows, cols]
    d1 = basis_values(u, k, 1)
    bt = d1 * tu[..., None]                                   # layers.py:51-52
    tmp = np.einsum("bfj,bfjo->bfo", bt, windows)             # layers.py:81 on the tangent basis
    ty = np.einsum("bfo,fo->bo", tmp, scale)
    if gt is None:
        return ty, None
    dtmp = gt[:, None, :] * scale[None, :, :]
    dscale = np.einsum("bo,bfo->fo", gt, tmp)
    dbt = np.einsum("bfo,bfjo->bfj", dtmp, windows)
    dwin = bt[..., None] * dtmp[:, :, None, :]
    dtable = np.zeros_like(table)
    np.add.at(dtable, (rows, cols), dwin)
    dtu = (dbt * d1).sum(axis=-1)                             # mul bwd into u.tangent
    du = (dbt * tu[..., None] * basis_values(u, k, 2)).sum(axis=-1)  # basis_features(d=1) bwd
    return ty, dict(dtable=dtable, dscale=dscale, dtu=dtu, du=du)


def kan_tangent_forward_backward(x, tx, coeffs, scale, gy, gt, *, k, g_min, g_max, G, base_weight=None):
    """kan_forward (layers.py:304-318) on x seeded with the tangent tx (tensor.py:411-424):
    returns y, ty = dy/dx . tx and the gradients of L = sum(y * gy) + sum(ty * gt) with respect
    to x, tx, coeffs, scale (and base_weight), as the reference's tape produces them through the
    tangent graph (clamp tangent tensor.py:336-337, mul(xc, 1/dg) layers.py:300, silu tangent
    tensor.py:236-241)."""
    x = np.asarray(x, dtype=np.float64)
    tx = np.asarray(tx, dtype=np.float64)
    B, f = x.shape
    K = k + 1
    prim = kan_forward_backward(x, coeffs, scale, gy, k=k, g_min=g_min, g_max=g_max, G=G,
                                base_weight=base_weight, need_dx=True)
    cell, u, mask = kan_locate(x, g_min, g_max, G)
    inv = 1.0 / ((g_max - g_min) / G)
    tu = tx * mask * inv
    rows = np.broadcast_to(np.arange(f)[None, :, None], (B, f, K))
    cols = cell[..., None] + np.arange(K)
    ty, t = _spline_tangent(coeffs, rows, cols, u, tu, scale, gt, k)
    dx = prim["dx"] + t["du"] * mask * inv
    dtx = t["dtu"] * mask * inv
    out = dict(y=prim["y"], cell=cell, dcoeffs=prim["dcoeffs"] + t["dtable"], dscale=prim["dscale"] + t["dscale"])
    if base_weight is not None:
        _, dsx = _silu(x)
        ty = ty + (dsx * tx) @ base_weight
        gb = gt @ base_weight.T
        dx = dx + gb * tx * _silu2(x)
        dtx = dtx + gb * dsx
        out["dbase_weight"] = prim["dbase_weight"] + (dsx * tx).T @ gt
    out.update(ty=ty, dx=dx, dtx=dtx)
    return out


def ukan_tangent_forward_backward(x, tx, p, gy, gt, *, k, delta_g, d_pe):
    """ukan_forward (layers.py:254-291) on x seeded with the tangent tx: u = x*(1/dg) - g_id
    carries tu = tx/dg (mul tangent, tensor.py:166-177); the generated table has no tangent.
    Returns y, ty and the gradients of L = sum(y * gy) + sum(ty * gt) for x, tx, scale and the
    CG parameters (the table gradient of both paths flows through one CG backward)."""
    x = np.asarray(x, dtype=np.float64)
    tx = np.asarray(tx, dtype=np.float64)
    B, f = x.shape
    K = k + 1
    d_out = p["scale"].shape[1]
    uniq, inverse, g_id, u, offset = ukan_keys(x, delta_g, k)
    n = B * f
    table, c = cg_forward(uniq, f, p["feature_embedding"], p["cg_w1"], p["cg_b1"], p["cg_w2"],
                          p["cg_b2"], d_pe, K, d_out)
    idx_prev = inverse[:n].reshape(B, f)
    idx_next = inverse[n:].reshape(B, f)
    col = offset[..., None] + np.arange(K)
    rows = np.where(col < K, idx_prev[..., None], idx_next[..., None])
    cols = col % K
    inv = 1.0 / delta_g
    y, g = _spline_fwd_bwd(table, rows, cols, u, p["scale"], gy, k, True)
    ty, t = _spline_tangent(table, rows, cols, u, tx * inv, p["scale"], gt, k)
    out = dict(y=y, ty=ty, g_id=g_id, dscale=g["dscale"] + t["dscale"], dx=(g["du"] + t["du"]) * inv,
               dtx=t["dtu"] * inv)
    out.update(_cg_backward(c, p, g["dtable"] + t["dtable"]))
    return out


def softmax_xent(logits, labels):
    """tensor.py:377-400: mean CE and its gradient."""
    n = logits.shape[0]
    z = logits - logits.max(axis=1, keepdims=True)
    logp = z - np.log(np.exp(z).sum(axis=1, keepdims=True))
    loss = -logp[np.arange(n), labels].mean()
    p = np.exp(logp)
    p[np.arange(n), labels] -= 1.0
    return loss, p / n


def mse(pred, target):
    """tensor.py:368-374."""
    d = pred - target
    return float((d * d).mean()), 2.0 * d / d.size


def adam_step(params, grads, m, v, t, lr, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0):
    """optim.py:31-54 (coupled L2); updates params / m / v in place."""
    bc1 = 1.0 - beta1 ** t
    bc2 = 1.0 - beta2 ** t
    for i, (p, g) in enumerate(zip(params, grads)):
        if weight_decay:
            g = g + weight_decay * p
        m[i] *= beta1
        m[i] += (1.0 - beta1) * g
        v[i] *= beta2
        v[i] += (1.0 - beta2) * g * g
        p -= lr * (m[i] / bc1) / (np.sqrt(v[i] / bc2) + eps)


def model_step(kind, layer_params, layer_cfgs, x, target, loss_kind, lr, t=1, weight_decay=0.0,
               m=None, v=None):
    """One training step of a spline stack (train.py:142-150): forward through the layers
    (no activation between spline layers, layers.py:420-426), loss, backward, Adam.
    Returns (loss, grads per layer, updated params per layer)."""
    hs = [np.asarray(x, dtype=np.float64)]
    for lp, cfg in zip(layer_params, layer_cfgs):
        if kind == "kan":
            hs.append(kan_forward_backward(hs[-1], lp["coeffs"], lp["scale"], None, **cfg)["y"])
        else:
            hs.append(ukan_forward_backward(hs[-1], lp, None, **cfg)["y"])
    if loss_kind == "softmax_cross_entropy":
        loss, g = softmax_xent(hs[-1], target)
    else:
        loss, g = mse(hs[-1], target)
    grads = [None] * len(layer_params)
    for li in range(len(layer_params) - 1, -1, -1):
        lp, cfg = layer_params[li], layer_cfgs[li]
        need_dx = li > 0
        if kind == "kan":
            r = kan_forward_backward(hs[li], lp["coeffs"], lp["scale"], g, need_dx=need_dx, **cfg)
            grads[li] = {"coeffs": r["dcoeffs"], "scale": r["dscale"]}
        else:
            r = ukan_forward_backward(hs[li], lp, g, need_dx=need_dx, **cfg)
            grads[li] = {n: r["d" + n] for n in lp}
        g = r.get("dx")
    flat_p = [lp[n] for lp in layer_params for n in lp]
    flat_g = [gr[n] for gr, lp in zip(grads, layer_params) for n in lp]
    if m is None:
        m = [np.zeros_like(a) for a in flat_p]
        v = [np.zeros_like(a) for a in flat_p]
    new_p = [a.copy() for a in flat_p]
    adam_step(new_p, flat_g, m, v, t, lr, weight_decay=weight_decay)
    return loss, grads, new_p, m, v


# ---------------------------------------------------------------------------------------
# Memory-bounded forms for parity at the benchmarked (full) shapes.  The reference
# materialises windows [B, d_in, K, d_out] (layers.py:65) and a full zeros_like(table)
# (layers.py:68), which is 35 PB at cfg3; the two functions below compute the SAME float64
# quantities on a subset: per-sample rows (y, dx of a few samples need only those samples) and
# per-feature gradients (dC[i], dscale[i] need only column i of x and the whole upstream g).
# Only the float64 summation order differs from the reference (~1e-16 relative).
# ---------------------------------------------------------------------------------------
def kan_rows(x_rows, coeffs, scale, gy_rows, *, k, g_min, g_max, G, feat_block=256):
    """y and dx of the given sample rows (layers.py:304-318 forward; basis_features /
    edge_combine / clamp bwd, layers.py:44-46, 84-88, tensor.py:327-338), features in blocks so
    the windows of one block stay small.  Returns dict(y [n, d_out], dx [n, d_in], cell)."""
    x_rows = np.asarray(x_rows, dtype=np.float64)
    n, f = x_rows.shape
    y = np.zeros((n, coeffs.shape[2]))
    dx = np.zeros((n, f))
    cells = np.zeros((n, f), dtype=np.int64)
    for i0 in range(0, f, feat_block):
        sl = slice(i0, min(f, i0 + feat_block))
        K = k + 1
        cell, u, mask = kan_locate(x_rows[:, sl], g_min, g_max, G)
        cells[:, sl] = cell
        fi = np.arange(sl.start, sl.stop)
        win = coeffs[fi[None, :, None], cell[..., None] + np.arange(K)]        # layers.py:65
        basis = basis_values(u, k)
        tmp = np.einsum("bfj,bfjo->bfo", basis, win)                           # layers.py:81
        y += np.einsum("bfo,fo->bo", tmp, scale[sl])                           # layers.py:82
        dtmp = gy_rows[:, None, :] * scale[None, sl, :]                        # layers.py:85
        dbasis = np.einsum("bfo,bfjo->bfj", dtmp, win)                         # layers.py:87
        du = (dbasis * basis_values(u, k, 1)).sum(axis=-1)                     # layers.py:44-46
        dx[:, sl] = du * (1.0 / ((g_max - g_min) / G)) * mask
    return dict(y=y, dx=dx, cell=cells)


def kan_feature_grads(x_col, coeffs_i, scale_i, gy, *, k, g_min, g_max, G):
    """dC[i] [G+k, d_out] and dscale[i] [d_out] of ONE feature over the whole batch: the
    np.add.at scatter of layers.py:67-70 written as the equivalent dense product
    W[r, b] @ g[b, o] with W[c_b + j, b] = w_j(u_b) (float64), then edge_combine's bwd
    (layers.py:84-88): dC = scale * A, dscale = sum_b g * tmp = sum_r C * A."""
    x_col = np.asarray(x_col, dtype=np.float64)
    B = x_col.shape[0]
    K = k + 1
    R = G + k
    cell, u, _ = kan_locate(x_col, g_min, g_max, G)
    basis = basis_values(u, k)                                                  # [B, K]
    W = np.zeros((R, B))
    for j in range(K):
        W[cell + j, np.arange(B)] = basis[:, j]
    A = W @ np.asarray(gy, dtype=np.float64)                                    # [R, d_out]
    return dict(dcoeffs=scale_i[None, :] * A, dscale=(coeffs_i * A).sum(axis=0))
