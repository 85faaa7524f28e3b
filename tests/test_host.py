"""CPU-only checks of the host side: the C-ABI library loads and exports every symbol the
public header declares, configuration validation, error mapping, and block geometry."""

import ctypes
import math

import pytest

from paper_2602_13515_b200 import _lib
from paper_2602_13515_b200 import masker as mk
from paper_2602_13515_b200.numerics import num_blocks


def test_library_exports_every_header_symbol():
    names = _lib.header_symbols()
    assert len(names) >= 9
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in names:
        assert hasattr(lib, name), name
    assert set(_lib.SIGNATURES) == set(names)
    assert _lib.load().spa2_version().startswith(b"spa2")
    assert not any(n.startswith("spa2_probe") for n in names)  # diagnostics live in libspa2_diag.so


def test_diag_library_exports_every_diag_header_symbol():
    names = _lib.header_symbols(_lib.DIAG_HEADER_PATH)
    lib = ctypes.CDLL(_lib.DIAG_LIB_PATH)
    for name in names:
        assert hasattr(lib, name), name
    assert set(_lib.DIAG_SIGNATURES) == set(names)
    assert not hasattr(ctypes.CDLL(_lib.LIB_PATH), "spa2_probe_gemm")


def test_error_mapping():
    with pytest.raises(ValueError):
        _lib.check(_lib.SPA2_ERR_VALUE, "x")
    with pytest.raises(ValueError):
        _lib.check(_lib.SPA2_ERR_UNSUPPORTED, "x")
    with pytest.raises(FloatingPointError):
        _lib.check(_lib.SPA2_ERR_NONFINITE, "x")
    with pytest.raises(RuntimeError):
        _lib.check(_lib.SPA2_ERR_CUDA, "x")
    _lib.check(_lib.SPA2_OK, "x")


def test_argument_errors_need_no_gpu():
    lib = _lib.load()
    assert lib.spa2_select(None, 0, 4, 1, 0.5, None, None, None) == _lib.SPA2_ERR_VALUE
    assert "empty" in _lib.last_error()
    assert lib.spa2_select(None, 3, 4, 0, 0.5, None, None, None) == _lib.SPA2_ERR_VALUE
    assert lib.spa2_build_lists(None, 0, 1, 1, *([None] * 7), None) == _lib.SPA2_ERR_VALUE
    diag = _lib.load_diag()
    assert diag.spa2_probe_gemm(None, None, None, 32, 64, 64, 0, 0, 0, None) == _lib.SPA2_ERR_UNSUPPORTED


def test_sparsity_config_validation():
    mk.SparsityConfig(0.0, 1.0, 1, 1)  # test_masker.py:22-29
    for bad in ((-0.1, 0.5, 4, 4), (0.5, 1.5, 4, 4), (0.5, 0.5, 0, 4), (0.5, 0.5, 4, 0)):
        with pytest.raises(ValueError):
            mk.SparsityConfig(*bad)


def test_top_k_count_ieee():
    assert mk.top_k_count(0.07, 100) == 8  # 0.07*100 = 7.000000000000001
    assert mk.top_k_count(0.0, 512) == 1
    assert mk.top_k_count(0.03, 512) == math.ceil(0.03 * 512) == 16
    assert mk.top_k_count(1.0, 7) == 7


def test_geometry():
    assert num_blocks(32760, 128) == 256 and num_blocks(32760, 64) == 512
    assert num_blocks(75600, 128) == 591 and num_blocks(75600, 64) == 1182


def test_require_device_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        mk.pooled_map([[0.0, 1.0]], [[0.0, 1.0]], mk.SparsityConfig(0.5, 0.5, 1, 1))


def test_mask_device_placement():
    """Masks follow the inputs' device: a host (numpy) mask is uploaded to it once per device;
    a device mask on another device than the inputs is an error, not a silent copy."""
    import types

    import torch

    from paper_2602_13515_b200 import attention as at

    keep = torch.ones((2, 4), dtype=torch.bool)
    host = types.SimpleNamespace(dev=keep, on_host=True, _cache={})
    moved = at._mask_on(host, torch.device("meta"))
    assert moved.device.type == "meta"
    assert at._mask_on(host, torch.device("meta")) is moved  # cached per device
    assert at._mask_on(host, torch.device("cpu")) is keep
    dev_mask = types.SimpleNamespace(dev=keep, on_host=False, _cache={})
    with pytest.raises(ValueError, match="inputs are on"):
        at._mask_on(dev_mask, torch.device("meta"))
