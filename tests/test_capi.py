"""C-ABI library: it loads, exports exactly what include/hlbm.h declares, and the Python
host layer validates like the reference (no compute calls here: CPU-only)."""

import re
from pathlib import Path

import numpy as np
import pytest

from paper_2602_05295_b200 import QuantSpec, SimGrid, SolverConfig, _lib

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "hlbm.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hlbm_[a-z_]+)\s*\(", text)))


def test_library_loads_and_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for name in syms:
        assert hasattr(lib, name), name
    assert sorted(_lib.SIGNATURES) == syms      # the ctypes binding covers the whole ABI
    assert b"sm_100a" in lib.hlbm_version()


def test_library_is_an_sm100a_binary():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    assert out.returncode == 0
    assert "sm_100a" in out.stdout


def test_config_validation_mirrors_reference_errors():
    with pytest.raises(ValueError):
        SolverConfig(nu=-0.01)                    # tau <= 1/2 (collision.py:102-103)
    with pytest.raises(ValueError):
        SolverConfig(lattice="D2Q9")
    with pytest.raises(ValueError):
        SolverConfig(precision="fp8")
    with pytest.raises(ValueError):
        SolverConfig(bc={"y": ("inflow", "outflow")})
    with pytest.raises(ValueError):
        SimGrid((8, 8, 6))                         # nz % 4
    with pytest.raises(ValueError):
        SimGrid((8, 8, 8), mask=np.zeros((8, 8, 4)))
    with pytest.raises(ValueError):
        QuantSpec(bits=(17,) * 10)
    assert SolverConfig(nu=0.01).tau == pytest.approx(0.53)    # tau = 0.5 + 3 nu (collision.py:30-31)
    q = QuantSpec.preset("16/15")
    assert q.bits == (16,) * 4 + (15,) * 6 and q.words_per_node == 5


def test_create_without_gpu_fails_loudly():
    import ctypes as C
    lib = _lib.load()
    if lib.hlbm_device_count() > 0:
        pytest.skip("a GPU is visible")
    c = _lib.HlbmConfig()
    c.nx = c.ny = c.nz = 8
    c.tau = 0.6
    ctx = C.c_void_p()
    rc = lib.hlbm_create(C.byref(c), C.byref(ctx))
    assert rc != _lib.HLBM_OK                      # no silent CPU path
    if ctx.value:
        assert lib.hlbm_last_error(ctx)
        lib.hlbm_destroy(ctx)


def test_invalid_grid_rejected_by_the_library():
    import ctypes as C
    lib = _lib.load()
    c = _lib.HlbmConfig()
    c.nx, c.ny, c.nz = 8, 8, 6
    c.tau = 0.6
    ctx = C.c_void_p()
    assert lib.hlbm_create(C.byref(c), C.byref(ctx)) == _lib.HLBM_EINVAL
    assert b"multiple of 4" in lib.hlbm_last_error(ctx)
    lib.hlbm_destroy(ctx)
    c.nz = 8
    c.tau = 0.5
    ctx = C.c_void_p()
    assert lib.hlbm_create(C.byref(c), C.byref(ctx)) == _lib.HLBM_EINVAL
    assert b"tau" in lib.hlbm_last_error(ctx)
    lib.hlbm_destroy(ctx)


def test_lattice_choice_validation():
    assert SolverConfig(lattice="D3Q19").lattice == "D3Q19"
    with pytest.raises(ValueError):
        SolverConfig(lattice="D3Q15")
