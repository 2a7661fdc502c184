"""compat.install / uninstall patch exactly the reference's two layer functions (CPU only: no
kernel is called).  The numerics through the patched functions are in test_compat_gpu.py."""
import os
import sys

import pytest

from conftest import ROOT

REF = os.path.join(ROOT, "baseline", "_ref")


def test_install_routes_reference_layer_functions():
    if not os.path.isdir(os.path.join(REF, "ukan")):
        pytest.skip("baseline/_ref not installed (needs /root/reference; __graft_entry__.build() installs it)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import ukan
    from paper_2408_11200_b200 import compat
    orig_k, orig_u = ukan.layers.kan_forward, ukan.layers.ukan_forward
    compat.install(ukan)
    try:
        assert ukan.layers.kan_forward is compat.kan_forward and ukan.kan_forward is compat.kan_forward
        assert ukan.layers.ukan_forward is compat.ukan_forward and ukan.ukan_forward is compat.ukan_forward
        compat.install(ukan)  # idempotent: the saved originals stay the reference's
    finally:
        compat.uninstall()
    assert ukan.layers.kan_forward is orig_k and ukan.layers.ukan_forward is orig_u
    assert ukan.kan_forward is orig_k
