"""Pin the CPU oracle (oracle/, a float64 NumPy restatement) against golden vectors produced by
the reference implementation itself (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from conftest import golden_names, load_golden

import oracle


@pytest.mark.parametrize("name", golden_names("kan_"))
def test_kan_oracle_matches_reference(name):
    g = load_golden(name)
    k, G, gmin, gmax = int(g["k"]), int(g["G"]), float(g["g_min"]), float(g["g_max"])
    r = oracle.kan_forward_backward(g["x"], g["coeffs"], g["scale"], g["g_up"], k=k, g_min=gmin, g_max=gmax, G=G,
                                    base_weight=g.get("base_weight"))
    np.testing.assert_array_equal(r["cell"], g["cell"])
    for key, ref in (("y", "y"), ("dx", "dx"), ("dcoeffs", "dcoeffs"), ("dscale", "dscale"),
                     ("dbase_weight", "dbase_weight")):
        if ref in g:
            np.testing.assert_allclose(r[key], g[ref], rtol=1e-12, atol=1e-13, err_msg=f"{name}.{key}")


@pytest.mark.parametrize("name", golden_names("ukan_"))
def test_ukan_oracle_matches_reference(name):
    g = load_golden(name)
    names = ["feature_embedding", "cg_w1", "cg_b1", "cg_w2", "cg_b2", "scale"]
    p = {n: g[n] for n in names}
    r = oracle.ukan_forward_backward(g["x"], p, g["g_up"], k=int(g["k"]), delta_g=float(g["delta_g"]),
                                     d_pe=int(g["d_pe"]))
    np.testing.assert_array_equal(r["g_id"], g["g_id"])
    np.testing.assert_array_equal(r["uniq"], g["keys"])
    np.testing.assert_allclose(r["y"], g["y"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(r["dx"], g["dx"], rtol=1e-10, atol=1e-12)
    for n in names:
        np.testing.assert_allclose(r["d" + n], g["d" + n], rtol=1e-10, atol=1e-12, err_msg=n)


@pytest.mark.parametrize("name", golden_names("step_"))
def test_training_step_oracle_matches_reference(name):
    g = load_golden(name)
    kind = str(g["kind"])
    widths = [int(w) for w in g["widths"]]
    k = int(g["k"])
    names = [n[len("init."):] for n in g if n.startswith("init.")]
    per_layer = [dict() for _ in range(len(widths) - 1)]
    for n in names:
        li, pn = n.split(".", 1)
        per_layer[int(li[len("layer"):])][pn] = g["init." + n].copy()
    if kind == "kan":
        cfgs = [dict(k=k, g_min=float(g["kw_g_min"]), g_max=float(g["kw_g_max"]), G=int(g["kw_G"]))] * len(per_layer)
    else:
        cfgs = [dict(k=k, delta_g=float(g["kw_delta_g"]), d_pe=int(g["kw_d_pe"]))] * len(per_layer)
    m = v = None
    params = per_layer
    for s in range(int(g["steps"])):
        loss, grads, new_p, m, v = oracle.model_step(kind, params, cfgs, g["x"], g["target"], str(g["loss_kind"]),
                                                     float(g["lr"]), t=s + 1, weight_decay=float(g["wd"]), m=m, v=v)
        assert abs(loss - g["losses"][s]) < 1e-12
        if s == 0:
            for li, gr in enumerate(grads):
                for pn, a in gr.items():
                    np.testing.assert_allclose(a, g[f"grad0.layer{li}.{pn}"], rtol=1e-10, atol=1e-13)
        it = iter(new_p)
        params = [{pn: next(it) for pn in lp} for lp in params]
    for li, lp in enumerate(params):
        for pn, a in lp.items():
            np.testing.assert_allclose(a, g[f"final.layer{li}.{pn}"], rtol=1e-10, atol=1e-12)


def test_basis_matrix_eq3():
    M = oracle.basis_matrix(3) * 6
    np.testing.assert_array_equal(M, [[1, 4, 1, 0], [-3, 0, 3, 0], [3, -6, 3, 0], [-1, 3, -3, 1]])


def _tangent_single(name):
    return [n for n in golden_names("tan_") if "stack" not in n]


@pytest.mark.parametrize("name", _tangent_single("tan_"))
def test_tangent_oracle_matches_reference(name):
    """F2: the forward tangent (x seeded with tx) and the gradients of sum(y gup) + sum(ty gt)
    through the reference's tangent graph, single layer."""
    g = load_golden(name)
    k = int(g["k"])
    if str(g["kind"]) == "kan":
        r = oracle.kan_tangent_forward_backward(
            g["x"], g["tx"], g["layer0.coeffs"], g["layer0.scale"], g["g_up"], g["g_tan"], k=k,
            g_min=float(g["kw_g_min"]), g_max=float(g["kw_g_max"]), G=int(g["kw_G"]),
            base_weight=g.get("layer0.base_weight"))
        pairs = [("dcoeffs", "dlayer0.coeffs"), ("dscale", "dlayer0.scale"), ("dbase_weight", "dlayer0.base_weight")]
    else:
        names = ["feature_embedding", "cg_w1", "cg_b1", "cg_w2", "cg_b2", "scale"]
        p = {n: g["layer0." + n] for n in names}
        r = oracle.ukan_tangent_forward_backward(g["x"], g["tx"], p, g["g_up"], g["g_tan"], k=k,
                                                 delta_g=float(g["kw_delta_g"]), d_pe=int(g["kw_d_pe"]))
        pairs = [("d" + n, "dlayer0." + n) for n in names]
    for key, ref in [("y", "y"), ("ty", "ty"), ("dx", "dx")] + pairs:
        if ref in g:
            np.testing.assert_allclose(r[key], g[ref], rtol=1e-10, atol=1e-12, err_msg=f"{name}.{key}")
