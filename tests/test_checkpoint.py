"""UKANCKP1 interop: read a checkpoint written by the reference's own
save_checkpoint, and write byte-identical files."""
import os

import numpy as np
import pytest

from conftest import GOLDEN

import paper_2408_11200_b200 as P
from paper_2408_11200_b200 import checkpoint as ck
from paper_2408_11200_b200.errors import FormatError

REF_CKPT = os.path.join(GOLDEN, "ref_checkpoint.ukanckp")


def test_reads_reference_checkpoint_and_rewrites_identically(tmp_path):
    cfg, tensors, meta = ck.load_checkpoint(REF_CKPT)
    assert meta == {"adam_t": 3, "epoch": 7}
    assert "model = kan" in cfg and "widths = 3,4,2" in cfg
    assert list(tensors) == ["layer0.coeffs", "layer0.scale", "layer1.coeffs", "layer1.scale"]
    out = tmp_path / "again.ukanckp"
    ck.save_checkpoint(str(out), cfg, tensors, meta)
    assert out.read_bytes() == open(REF_CKPT, "rb").read()


def test_model_roundtrip_through_reference_format(tmp_path):
    _, tensors, _ = ck.load_checkpoint(REF_CKPT)
    model = P.build_model("kan", [3, 4, 2], 3, seed=0, G=6, device="cpu")
    ck.load_model_state(model, tensors)
    state = ck.model_state(model)
    for n in tensors:
        np.testing.assert_array_equal(state[n], tensors[n])   # values are fp32-representable
    p = tmp_path / "m.ukanckp"
    ck.save_checkpoint(str(p), model, state, {"epoch": 1})
    cfg2, t2, m2 = ck.load_checkpoint(str(p))
    assert m2 == {"epoch": 1} and all(np.array_equal(t2[n], state[n]) for n in state)
    # the echo rebuilds the same architecture in the reference's config format
    assert "model = kan\n" in cfg2 and "widths = 3,4,2\n" in cfg2 and "grid_size = 6\n" in cfg2
    assert "degree = 3\n" in cfg2 and cfg2.startswith("task = ")
    with pytest.raises(P.ConfigError):
        ck.save_checkpoint(str(p), None, state, {})


def test_format_errors(tmp_path):
    bad = tmp_path / "bad"
    bad.write_bytes(b"NOTACKPT" + b"\x01")
    with pytest.raises(FormatError):
        ck.load_checkpoint(str(bad))
    data = open(REF_CKPT, "rb").read()
    (tmp_path / "trunc").write_bytes(data[:-5])
    with pytest.raises(FormatError):
        ck.load_checkpoint(str(tmp_path / "trunc"))
    (tmp_path / "trail").write_bytes(data + b"x")
    with pytest.raises(FormatError):
        ck.load_checkpoint(str(tmp_path / "trail"))
    model = P.build_model("kan", [3, 5, 2], 3, seed=0, G=6, device="cpu")
    _, tensors, _ = ck.load_checkpoint(REF_CKPT)
    with pytest.raises(FormatError):
        ck.load_model_state(model, tensors)
    model = P.build_model("kan", [3, 4, 2], 3, seed=0, G=6, device="cpu")
    with pytest.raises(FormatError):  # extra names are rejected, as the reference does
        ck.load_model_state(model, {**tensors, "layer2.coeffs": tensors["layer0.coeffs"]})


def test_config_echo_for_ukan_model_and_runconfig_like(tmp_path):
    model = P.build_model("ukan", [2, 3, 1], 3, seed=0, delta_g=0.5, d_pe=6, d_femb=4, device="cpu")
    text = ck.config_text(model)
    assert "model = ukan\n" in text and "widths = 2,3,1\n" in text and "delta_g = 0.5\n" in text
    assert "d_pe = 6\n" in text and "d_femb = 4\n" in text and text.endswith("out_dir = .\n")
    from dataclasses import dataclass, field

    @dataclass
    class RunConfigLike:  # field order and widths rendering as config_to_text (config.py:130-137)
        task: str = "regression_II"
        model: str = "kan"
        widths: list = field(default_factory=lambda: [2, 5, 1])

    assert ck.config_text(RunConfigLike()) == "task = regression_II\nmodel = kan\nwidths = 2,5,1\n"
    p = tmp_path / "u.ukanckp"
    ck.save_checkpoint(str(p), model, ck.model_state(model), {"epoch": 0})
    cfg, tensors, meta = ck.load_checkpoint(str(p))
    assert cfg == text and list(tensors) == list(model.parameters())
