"""CPU checks of the drop-in boundary: libqdwhg.so loads, exports every symbol
include/qdwhg.h declares, the ctypes struct layouts match the header, and the
host-scalar entry points (no GPU needed) are bit-identical to the reference."""
import ctypes
import re

import numpy as np
import pytest

from conftest import golden
from paper_2104_14186_b200 import _lib, matgen, qdwh

EPS = np.finfo(float).eps


def header_functions():
    src = open(_lib.HEADER_PATH).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qdwhg_[a-z_0-9]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert header_functions() == sorted(_lib.SIGNATURES)


def test_library_exports_every_symbol():
    lib = _lib.load()
    for name in header_functions():
        assert hasattr(lib, name), name


def test_struct_sizes():
    # field-by-field layout of the info structs (checked against offsets in the header order)
    assert ctypes.sizeof(_lib.EigInfo) == 4 * 8 + 7 * 8 + 4 * 4 + 64 * 8 + 2 * 8 + 8 * 8
    assert ctypes.sizeof(_lib.SvdInfo) == 4 * 8 + 6 * 8 + 4 * 4 + 64 * 8 + 2 * 8 + 8 * 8
    assert ctypes.sizeof(_lib.EigRequest) == 48
    assert ctypes.sizeof(_lib.SvdRequest) == 40


def test_host_scalars_bit_exact_with_reference():
    g = golden("scalars")
    for ell, w, it in zip(g["ells"], g["weights"], g["iters"]):
        ws = qdwh.halley_weights(float(ell))
        assert [ws.a, ws.b, ws.c, ws.ell_in, ws.ell_out] == list(w)
        assert qdwh.iterations_to_converge(float(ell), 5 * EPS) == it


def test_host_scalar_errors():
    with pytest.raises(ValueError):
        qdwh.halley_weights(0.0)
    with pytest.raises(ValueError):
        qdwh.halley_weights(-0.1)
    with pytest.raises(ValueError):
        qdwh.halley_weights(1.5)
    with pytest.raises(ValueError):
        qdwh.choose_shift(4)
    with pytest.raises(ValueError):
        qdwh.choose_shift(1)
    assert qdwh.choose_shift(3).s == 0.2 and qdwh.choose_shift(2).s == 0.875
    with pytest.raises(qdwh.NotConverged):
        qdwh.iterations_to_converge(1e-15, 5 * EPS, 2)


def test_detect_deficiency_index():
    # test_partial.cpp:44-49
    assert qdwh.detect_deficiency_index(np.diag([5.0, 3.0, 0.5, 1e-8])) == 4
    assert qdwh.detect_deficiency_index(np.diag([2.0, 1.5, 1.1])) is None
    assert qdwh.detect_deficiency_index(np.diag([0.005, 3.0, 2.0])) == 1
    assert qdwh.detect_deficiency_index(np.diag([-0.5, 0.02, 1.0]), 0.1) == 2


def test_matgen_hash_matches_reference_generator():
    from oracle import qdwh_oracle as O
    i = np.arange(100)
    h = matgen.hash64_np(42, i)
    assert all(int(h[j]) == O.hash64(42, j) for j in range(100))
    u = matgen.to_unit_np(h)
    assert all(u[j] == O.to_unit(O.hash64(42, j)) for j in range(100))


def test_config_spectra():
    lam = matgen.config_eigenvalues("uniform", 1024)
    assert lam.min() > -1 and lam.max() <= 1
    c = matgen.largest_k_shift(lam, 103)
    assert np.sum(lam > c) == 103
    lam2 = matgen.config_eigenvalues("logsigned", 4096)
    assert np.allclose(np.sort(np.abs(lam2)), np.logspace(-8, 0, 4096))
    c2 = matgen.largest_k_shift(lam2, 41)
    assert np.sum(lam2 > c2) == 41
    sig = matgen.config_singular_values("log16", 8192)
    assert np.sum(sig > matgen.sigma_cut(sig, 410)) == 410
    sig5 = matgen.config_singular_values("inv", 8192)
    assert np.sum(sig5 > matgen.sigma_cut(sig5, 819)) == 819
