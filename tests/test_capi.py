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
    lib.hlbm_config_init(C.byref(c))
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
    lib.hlbm_config_init(C.byref(c))
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


def test_config_struct_size_guard():
    """hlbm_config carries its own size: a binding built against another layout (the round-1
    INTEGRATION.md struct without `q`, 8 bytes short) is rejected before any field is read."""
    import ctypes as C
    lib = _lib.load()
    c = _lib.HlbmConfig()
    lib.hlbm_config_init(C.byref(c))
    assert c.struct_size == C.sizeof(_lib.HlbmConfig) == 352
    assert c.q == 27 and list(c.bits) == [16] * 10 and c.qmax[0] == 1.5
    c.nx = c.ny = c.nz = 8
    c.tau = 0.6
    c.struct_size = 344
    ctx = C.c_void_p()
    assert lib.hlbm_create(C.byref(c), C.byref(ctx)) == _lib.HLBM_EINVAL
    assert b"struct_size is 344" in lib.hlbm_last_error(ctx)
    lib.hlbm_destroy(ctx)


def test_ctypes_layout_matches_the_c_header(tmp_path):
    """Field offsets of the ctypes structs equal offsetof() of include/hlbm.h compiled by gcc."""
    import ctypes as C
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    src = ['#include <stdio.h>', '#include <stddef.h>', '#include "hlbm.h"', "int main(void){"]
    for st, cname in ((_lib.HlbmConfig, "hlbm_config"), (_lib.HlbmStats, "hlbm_stats")):
        src.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in st._fields_:
            src.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    src.append("return 0;}")
    (tmp_path / "l.c").write_text("\n".join(src))
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(tmp_path / "l.c"), "-o", str(tmp_path / "l")], check=True)
    got = subprocess.run([str(tmp_path / "l")], capture_output=True, text=True, check=True).stdout.split("\n")
    want = []
    for st, cname in ((_lib.HlbmConfig, "hlbm_config"), (_lib.HlbmStats, "hlbm_stats")):
        want.append(f"{cname} size {C.sizeof(st)}")
        want += [f"{cname} {f} {getattr(st, f).offset}" for f, _ in st._fields_]
    assert [g for g in got if g] == want


# ---- a plain-C host of the C-ABI (examples/tgv_c.c): the header is C99, the program links
def _build_c_example(tmp_path):
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    root = Path(__file__).resolve().parents[1]
    exe = tmp_path / "tgv_c"
    libdir = root / "paper_2602_05295_b200"
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", f"-I{root / 'include'}",
           str(root / "examples" / "tgv_c.c"), f"-L{libdir}", "-lhlbm", f"-Wl,-rpath,{libdir}", "-lm",
           "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_example_compiles_and_links(tmp_path):
    assert _build_c_example(tmp_path).exists()


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp32", "q16"])
def test_c_example_matches_python_host(tmp_path, precision):
    """The same TGV 32^3 x 10 steps through the C host and through the Python host agree (the
    inputs are built with C libm and with NumPy, so to rounding of the float64 inputs)."""
    import subprocess
    from paper_2602_05295_b200 import SimGrid, Solver, SolverConfig
    from paper_2602_05295_b200.geometry import taylor_green_fields
    exe = _build_c_example(tmp_path)
    out = tmp_path / "rho.bin"
    r = subprocess.run([str(exe), "32", "10", precision, str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert "finite 1" in r.stdout
    rho_c = np.fromfile(out, dtype=np.float64).reshape(32, 32, 32)
    with Solver(SimGrid((32, 32, 32)), SolverConfig(nu=0.01, precision=precision)) as s:
        s.set_equilibrium(*taylor_green_fields(32))
        s.step(10)
        rho_py = s.moments()[0]
    tol = 1e-9 if precision == "fp32" else 2.2e-5      # q16: 2 LSB of rho (0.7 / 65535)
    assert np.max(np.abs(rho_c - rho_py)) <= tol
