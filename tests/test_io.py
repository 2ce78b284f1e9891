"""On-disk formats: round trips on CPU; exact resume on GPU."""

import numpy as np
import pytest

from oracle import codec
from oracle import step as OS
from oracle.moments import neq_decompose
from paper_2602_05295_b200 import io as hio


def test_packed_dump_round_trip(tmp_path):
    r, m, s = OS.random_state((6, 5, 8), seed=1)
    w, _ = codec.encode_state(r, m, neq_decompose(r, m, s))
    hio.write_packed(tmp_path / "a.hlbm", w, [16] * 10, codec.DEFAULT_MIN, codec.DEFAULT_MAX, step=7)
    d = hio.read_packed(tmp_path / "a.hlbm")
    assert d["dims"] == (6, 5, 8) and d["step"] == 7 and np.array_equal(d["words"], w)
    raw = (tmp_path / "a.hlbm").read_bytes()
    # node-major, little-endian: the first node's 5 words follow the header
    hdr = 8 + 12 + 4 + 40 + 80 + 80 + 8
    first = np.frombuffer(raw[hdr:hdr + 20], dtype="<u4")
    assert np.array_equal(first, w[:, 0, 0, 0])


def test_snapshot_round_trip(tmp_path):
    r, m, s = OS.random_state((4, 6, 8), seed=2)
    hio.write_snapshot(tmp_path / "s.snap", r, m, s, step=3)
    d = hio.read_snapshot(tmp_path / "s.snap")
    assert d["step"] == 3
    np.testing.assert_allclose(d["rho"], r, rtol=1e-7)
    np.testing.assert_allclose(d["stress"], s, atol=1e-8)


def test_stats_csv(tmp_path):
    from paper_2602_05295_b200.solver import StepStats
    st = StepStats(step=5, t_fluid_ms=1.0, t_copy_ms=0.0, t_solid_ms=0.1, mass=10.5,
                   momentum=np.array([1.0, 2.0, 3.0]), max_u=0.1, saturation=np.zeros(10, int), n_fluid=10)
    with hio.StatsCSV(tmp_path / "s.csv") as f:
        f.write(st)
    lines = (tmp_path / "s.csv").read_text().splitlines()
    assert lines[0].startswith("step,t_fluid_ms") and lines[1].startswith("5,")


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp32", "q16"])
def test_checkpoint_resume_bitwise(tmp_path, precision):
    from paper_2602_05295_b200 import QuantSpec, SimGrid, Solver, SolverConfig
    shape = (20, 16, 32)
    state = OS.random_state(shape, seed=4, drho=0.05, umax=0.05, sneq=0.005)
    cfg = SolverConfig(nu=0.02, precision=precision, quant=QuantSpec(dither=True), seed=9)
    with Solver(SimGrid(shape), cfg) as a:
        a.set_moments(*state)
        a.step(4)
        hio.save_checkpoint(tmp_path / "c.hlbm", a)
        a.step(5)
        ref = a.get_state()
    with Solver(SimGrid(shape), cfg) as b:
        assert hio.load_checkpoint(tmp_path / "c.hlbm", b) == 4
        b.step(5)
        assert np.array_equal(b.get_state(), ref)


def test_vorticity_pgm(tmp_path):
    from paper_2602_05295_b200.io import vorticity_z, write_vorticity_pgm
    n = 32
    k = 2 * np.pi / n
    x = np.arange(n)[:, None, None]
    y = np.arange(n)[None, :, None]
    u = np.zeros((3, n, n, 4))
    u[0] = np.sin(k * y) * np.ones((1, 1, 4))          # shear u_x(y): omega_z = -du_x/dy = -k cos(ky)
    w = vorticity_z(u)
    np.testing.assert_allclose(w, -np.sin(k) * np.cos(k * y[:, :, 0]) * np.ones((n, 1)), atol=1e-12)
    p = tmp_path / "w.pgm"
    write_vorticity_pgm(p, u, vrange=2 * np.sin(k))
    data = p.read_bytes()
    assert data.startswith(b"P5\n32 32\n255\n") and len(data) == len(b"P5\n32 32\n255\n") + n * n
    img = np.frombuffer(data[len(b"P5\n32 32\n255\n"):], dtype=np.uint8).reshape(n, n)
    assert img.min() >= 63 and img.max() <= 192          # |omega| <= vrange / 2 -> the middle half
