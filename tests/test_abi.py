"""C-ABI boundary: the library loads and exports every entry point include/dp_b200.h declares."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2201_01446_b200 as dp

HEADER = Path(__file__).resolve().parent.parent / "include" / "dp_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dp_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    lib = ctypes.CDLL(str(dp.library_path()))
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_error_codes_match_reference_cli():
    text = HEADER.read_text()
    assert "#define DP_NUMERICAL_ERROR 1" in text
    assert "#define DP_INPUT_ERROR 2" in text


def test_version_string():
    assert b"sm_100a" in dp._lib().dp_version()


def test_generator_errors_map_to_input_error():
    with pytest.raises(dp.InputError):
        dp.get_preset("no-such-preset")
    with pytest.raises(dp.InputError):
        dp.make_test_model(1, 4, 0, 12, 2, [8], 6.0, 5.0, 1)  # m_lt out of range
    with pytest.raises(dp.InputError):
        dp.make_test_model(1, 4, 4, 12, 2, [8], 5.0, 6.0, 1)  # r_smooth >= r_cut


def test_no_gpu_means_loud_failure_not_fallback():
    """Without a device dp_create must fail (runtime error), never compute on the CPU."""
    from conftest import gpu_available
    if gpu_available():
        pytest.skip("GPU present")
    m = dp.make_test_model(1, 4, 4, 12, 2, [16], 5.0, 4.0, 1)
    t = dp.build_tables(m, 0.05)
    with pytest.raises(dp.DPRuntimeError):
        dp.DeepPot(m, t)
