"""C-ABI library checks that need no GPU: it loads and exports every symbol
include/swe_b200.h declares, and the Python mirror rejects bad input the way
the reference does (ValueError) before touching the device."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "swe_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(swe_[a-z_]+)\s*\(", text)))


def test_header_declares_what_the_binding_lists():
    from paper_2306_09497_b200 import _lib
    assert header_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_symbol():
    from paper_2306_09497_b200 import _lib, build
    build.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for sym in header_symbols():
        assert getattr(lib, sym) is not None, sym
    _lib.load()
    assert _lib.kernel_launches() >= 0
    assert isinstance(_lib.last_error(), str)


def test_option_switches_validate():
    from paper_2306_09497_b200 import _lib
    _lib.set_option("fft_path", 0)
    with pytest.raises(ValueError):
        _lib.set_option("no_such_option", 1)
    with pytest.raises(ValueError):
        _lib.set_option("fft_path", 7)


def test_config_validation_mirrors_reference():
    from paper_2306_09497_b200 import dynamics, spharm, steppers
    with pytest.raises(ValueError):
        spharm.Truncation(M=0, nlat=1, nlon=2)
    with pytest.raises(ValueError):
        spharm.SphereGeometry(radius_a=-1.0)
    with pytest.raises(ValueError):
        dynamics.ViscositySpec(order_q=3)
    with pytest.raises(ValueError):
        steppers.StepperConfig(dt=0.0)
    with pytest.raises(ValueError):
        steppers.StepperConfig(coriolis_treatment="sideways")
    t = spharm.Truncation.for_wavenumber(256)
    assert (t.nlat, t.nlon, t.n_modes) == (385, 770, 33153)
