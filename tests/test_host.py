"""Host-side logic of the drop-in (no GPU compute): configuration objects,
value types, seeded generation, slot-order assembly, and the C ABI library
(loads, exports every symbol of include/kapsm_b200.h, signatures bound)."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2201_05024_b200 as K
from paper_2201_05024_b200 import _lib
from paper_2201_05024_b200.apsm import _assemble, _qtab_host
from oracle import kapsm_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def header_symbols():
    src = open(os.path.join(ROOT, "include", "kapsm_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kapsm_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, f"{s} not bound in _lib.SIGNATURES"
    assert lib.kapsm_abi_version() == 100
    assert lib.kapsm_max_window() >= 20
    assert lib.kapsm_max_samples() >= 1370
    assert lib.kapsm_strerror(0) == b"ok"
    assert lib.kapsm_strerror(3).startswith(b"configuration")


def test_library_is_sm100a():
    path = _lib.LIB_PATH
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_argument_validation_without_gpu():
    """Invalid arguments are rejected before any launch (no device needed)."""
    lib = _lib.load()
    kp = _lib.KernelParamsC(0.5, 0.5, 0.05)
    nul = ctypes.c_void_p(None)
    assert lib.kapsm_pilot_gram_f32(nul, 0, 1, 4, 2, kp, nul, 8, 64, nul) == _lib.KAPSM_ERR_INVALID
    assert lib.kapsm_train_f32(nul, 8, 64, nul, 0, nul, 0, 4, nul, 1, 1, 8, 20, 0.01, kp, nul,
                               nul, nul, nul, nul, nul, nul, nul, nul) == _lib.KAPSM_ERR_INVALID
    assert lib.kapsm_demap_f32(nul, 4, nul, 4, nul, nul) == _lib.KAPSM_ERR_INVALID
    assert lib.kapsm_count_mismatch(nul, nul, 0, 8, nul, nul) == _lib.KAPSM_ERR_INVALID


def test_config_validation_mirrors_reference():
    with pytest.raises(ValueError):
        K.KernelParams(sigma_sq=0.0)
    with pytest.raises(ValueError):
        K.KernelParams(w_l=-1.0)
    with pytest.raises(ValueError):
        K.KernelParams(0.0, 0.0, 0.05)
    with pytest.raises(ValueError):
        K.ApsmConfig(window=0)
    with pytest.raises(ValueError):
        K.ApsmConfig(epsilon=0.0)
    with pytest.raises(ValueError):
        K.ApsmConfig(weight_scheme="adaptive")
    with pytest.raises(ValueError):
        K.ApsmConfig(max_atoms=0)
    with pytest.raises(ValueError):
        K.EngineConfig(stage="warp")
    with pytest.raises(ValueError):
        K.EngineConfig(tile_atoms=0)
    with pytest.raises(ValueError):
        K.EngineConfig(precision="f16")
    with pytest.raises(ValueError):
        K.FrameSpec(-1, 10)
    with pytest.raises(ValueError):
        K.FrameSpec(10, 10, scheme="APSK")
    cfg = K.ApsmConfig()
    assert (cfg.window, cfg.epsilon, cfg.params.sigma_sq) == (20, 0.01, 0.05)
    assert K.EngineConfig().precision == "f64"


def test_filter_state_and_expansion():
    f = K.zero_filter(4)
    assert f.dim == 4 and f.n_atoms == 0
    with pytest.raises(ValueError):
        K.FilterState(np.zeros(3), np.zeros((2, 4)), np.zeros(2))
    with pytest.raises(ValueError):
        K.FilterState(np.zeros(4), np.zeros((2, 4)), np.zeros(3))
    p = K.KernelParams()
    g = K.from_expansion([1.0, 2.0], [[1.0, 0.0], [0.0, 1.0]], p)
    assert np.allclose(g.theta, [0.5, 1.0])
    assert K.self_kernel(np.array([1.0, 0.0]), p) == 1.0


def test_window_and_weights():
    assert list(K.window_indices(0, 20)) == [0]
    assert list(K.window_indices(25, 20)) == list(range(6, 26))
    g = np.load(os.path.join(GOLDEN, "uniform_weights.npz"))
    for n in (1, 7, 20, 64, 128):
        assert np.array_equal(K.uniform_weights(n), g[f"w{n}"])
    q = _qtab_host(20)
    for j in range(1, 21):
        w = g[f"w{j}"]
        assert q[2 * (j - 1)] == w[0] and q[2 * (j - 1) + 1] == w[-1]


def test_realify_and_pairs():
    s1, s2 = K.complex_to_real_pair(np.array([1 + 2j]), 3 + 4j)
    assert np.array_equal(s1.r, [1.0, 2.0]) and s1.b == 3.0
    assert np.array_equal(s2.r, [2.0, -1.0]) and s2.b == 4.0
    rng = np.random.default_rng(1)
    rx = rng.standard_normal((6, 3)) + 1j * rng.standard_normal((6, 3))
    assert np.array_equal(K.realify_batch(rx), O.realify(rx))


def test_constellations_and_labels():
    for scheme in K.SCHEMES:
        pts = K.get_constellation(scheme).points
        ref, _ = O.constellation(scheme)
        assert np.array_equal(pts, ref)
    bits = np.array([[0, 1, 1, 1, 1, 0, 0, 0]])
    assert list(K.symbol_labels(bits, 2)[0]) == [1, 3, 2, 0]


@pytest.mark.parametrize("name", ["small_s1_K6_M3_QPSK.npz", "small_s2_K4_M8_QAM16.npz"])
def test_seeded_generation_bit_identical(name):
    g = np.load(os.path.join(GOLDEN, name))
    fr = K.seeded_frame(int(g["seed"]), int(g["K"]), int(g["M"]), int(g["n_train"]),
                        int(g["n_data"]), str(g["scheme"]))
    assert np.array_equal(fr["rx"], g["rx"])
    assert np.array_equal(fr["bits"], g["bits"])


def test_assemble_slot_order_and_cap():
    """Device outputs (coeff, first_step per sample) -> reference slot order:
    sort by (first activation step, index) (apsm.py:341-358)."""
    rows = np.arange(12, dtype=float).reshape(6, 2)
    coeff = np.array([0.1, 0.0, 0.3, 0.4, 0.5, 0.6])
    fs = np.array([0, -1, 3, 2, 2, 5])
    cfg = K.ApsmConfig()
    f = _assemble(cfg, rows, np.zeros(2), coeff, fs, 0, None)
    assert np.array_equal(f.atoms, rows[[0, 3, 4, 2, 5]])
    assert np.array_equal(f.coeffs, coeff[[0, 3, 4, 2, 5]])
    with pytest.raises(K.DictionaryCapacityError):
        _assemble(K.ApsmConfig(max_atoms=4), rows, np.zeros(2), coeff, fs, 0, None)
    with pytest.raises(K.DegenerateSampleError):
        _assemble(cfg, rows, np.zeros(2), coeff, fs, _lib.TRAIN_DEGENERATE, None)
    lin = _assemble(K.ApsmConfig(params=K.KernelParams(1.0, 0.0, 0.05)), rows, np.ones(2), coeff,
                    fs, 0, None)
    assert lin.n_atoms == 0


def test_oracle_not_imported_by_product():
    import sys
    import importlib
    for mod in list(sys.modules):
        if mod.startswith("paper_2201_05024_b200"):
            m = sys.modules[mod]
            src = getattr(m, "__file__", "") or ""
            if src.endswith(".py"):
                text = open(src).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", text, re.M), mod


def test_inner_product_error_rules():
    """Zero weights / dimension mismatch raise like kernels.py:209-248 (host-side, no GPU)."""
    import paper_2201_05024_b200 as K
    p_lin = K.KernelParams(1.0, 0.0, 0.05)
    f = K.FilterState(np.array([1.0, 2.0]), np.array([[0.1, 0.2]]), np.array([0.5]))
    with pytest.raises(ValueError):
        K.inner_product(f, f, p_lin)                    # Gaussian weight zero, Gaussian part
    g = K.FilterState(np.array([1.0, 2.0]), np.empty((0, 2)), np.empty(0))
    assert K.inner_product(g, g, p_lin) == 5.0
    with pytest.raises(ValueError):
        K.inner_product(K.zero_filter(4), K.zero_filter(6), p_lin)
    with pytest.raises(ValueError):
        K.inner_product(g, g, K.KernelParams(0.0, 1.0, 0.05))   # linear weight zero
