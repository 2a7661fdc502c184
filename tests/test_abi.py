"""The C-ABI library loads and exports every symbol include/ukan_b200.h declares; host-only
entry points work without a GPU.  CPU only (no compute calls)."""
import ctypes
import os
import re

import numpy as np

from conftest import ROOT

from paper_2408_11200_b200 import _lib
from paper_2408_11200_b200.bspline import basis_matrix

import oracle

HEADER = os.path.join(ROOT, "include", "ukan_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t)\s+(ukan_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_api():
    fns = declared_functions()
    assert "ukan_kan_forward" in fns and "ukan_ukan_build_keys" in fns and len(fns) >= 20


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for fn in declared_functions():
        assert hasattr(lib, fn), fn


def test_binding_covers_header_exactly():
    assert sorted(_lib.SIGNATURES) == declared_functions()


def test_version():
    assert _lib.load().ukan_version() >= 100


def test_basis_matrix_abi_matches_oracle_all_degrees():
    for k in range(0, 11):
        bm = basis_matrix(k)
        np.testing.assert_array_equal(bm.floats, oracle.basis_matrix(k))
        # partition of unity: rows of M sum to (1, 0, ..., 0)
        np.testing.assert_allclose(bm.floats.sum(axis=1), np.eye(k + 1)[0], atol=1e-14)


def test_basis_matrix_rejects_bad_degree():
    buf = (ctypes.c_double * 4)()
    assert _lib.load().ukan_basis_matrix(11, ctypes.cast(buf, ctypes.c_void_p)) == _lib.UKAN_E_DEGREE
    assert _lib.load().ukan_basis_matrix(-1, ctypes.cast(buf, ctypes.c_void_p)) == _lib.UKAN_E_DEGREE


def test_workspace_queries():
    lib = _lib.load()
    assert lib.ukan_kan_backward_workspace_size(1024, 64, 64, 10, 3) >= 0
    # G beyond the register path: chunk records (256 samples: keys, u, 32-row tile starts) + dscale partials
    n_rt = (4099 + 31) // 32
    recb = 256 * 12 + (n_rt + 1 + 3) // 4 * 4 * 4
    assert lib.ukan_kan_backward_workspace_size(4096, 32, 32, 4096, 3) == 32 * 16 * recb + 8 * 32 * n_rt * 32
    assert lib.ukan_ukan_keys_workspace_size(100, 10, 1000) > 2 * 1000 * 8
    # segmented sweep: sorted chunk records (256 x 12 B per feature and chunk) + tile starts + fp64
    # dscale partials per 32-row tile (n_u*K rows, plus one partial tile per feature)
    rec, ts, tiles = 4 * 1 * 256 * 12, 256, (10 * 4 + 31) // 32 + 4
    # + per-feature sorted order (sample 4 B + u 8 B per (feature, sample)) and row starts
    al = lambda n: (n + 255) // 256 * 256  # noqa: E731
    seg = rec + ts + al(8 * tiles * 3) + al(12 * 4 * 8) + al(4 * (10 * 4 + 4 + 1))
    # + g and scale widened to fp64 for the dx kernel
    assert lib.ukan_ukan_backward_workspace_size(8, 4, 3, 10, 3) == (seg + 255) // 256 * 256 + 8 * (8 * 3 + 4 * 3)


def test_argument_errors_without_gpu():
    lib = _lib.load()
    # degree / grid validation happens before any CUDA call
    assert lib.ukan_kan_forward(None, None, None, None, None, 1, 1, 1, 8, 11, -1.0, 1.0, None, None) == _lib.UKAN_E_DEGREE
    assert lib.ukan_kan_forward(None, None, None, None, None, 1, 1, 1, 8, 3, 1.0, -1.0, None, None) == _lib.UKAN_E_GRID
    assert lib.ukan_kan_forward(None, None, None, None, None, 1, 1, 1, 8, 3, -1.0, 1.0, None, None) == _lib.UKAN_E_ARG
