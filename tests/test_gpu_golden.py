"""The CUDA path against SURVEY.md §8c's golden vectors generated from the reference package
(tests/golden/gen_golden.py --extra: the reference's collide / reconstruct / moments functions,
np.roll streaming, and the SPEC codec and boundary-list definitions written out in the generator)."""

from pathlib import Path

import numpy as np
import pytest

from oracle import codec
from paper_2602_05295_b200 import QuantSpec, SimGrid, Solver, SolverConfig
from paper_2602_05295_b200.geometry import taylor_green_fields

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"


def test_q16_one_step_codes_within_1_lsb_of_reference():
    z = np.load(G / "q16_step16.npz")
    tau = float(z["tau"])
    with Solver(SimGrid((16, 16, 16)), SolverConfig(nu=(tau - 0.5) / 3, precision="q16",
                                                    quant=QuantSpec(dither=False))) as s:
        s.codes = codec.pack(z["codes0"].astype(np.uint32))
        s.step(1)
        got = codec.unpack(s.codes)
    d = np.abs(got.astype(np.int64) - z["codes1"].astype(np.int64))
    assert d.max() <= 1
    assert (d > 0).mean() < 0.01          # fp32 arithmetic: 1-LSB flips only at rounding boundaries


def test_sphere_lists_bit_exact_with_reference_directions():
    z = np.load(G / "sphere32.npz")
    with Solver(SimGrid((32, 32, 32), z["mask"]), SolverConfig(nu=0.02)) as s:
        assert np.array_equal(s.boundary_cells, z["boundary_cells"])
        assert np.array_equal(s.link_masks, z["link_masks"])


PAIRS = ((0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2))


def _rel(a, b):
    return np.sqrt(((a - b) ** 2).sum()) / max(np.sqrt((b ** 2).sum()), 1e-30)


def test_tgv64_200_steps_against_reference():
    """SURVEY config 1 end to end: fp32 state, 200 steps; per-moment relative error of two full
    x-planes after 1, 10 and 200 steps <= 1e-5 (BASELINE north_star) and the kinetic energy."""
    z = np.load(G / "tgv64.npz")
    tau = float(z["tau"])
    rho, u = taylor_green_fields(64)
    with Solver(SimGrid((64, 64, 64)), SolverConfig(nu=(tau - 0.5) / 3)) as s:
        s.set_equilibrium(rho, u)
        done = 0
        for k in (1, 10, 200):
            s.step(k - done)
            done = k
            r, m, st = s.moments()
            ref = z[f"planes{k}"]                    # (rho, rho u, sneq) on planes x = 0, 21
            rr, rm = ref[0], ref[1:4]
            rst = ref[4:] + np.stack([rm[a] * rm[b] / rr for a, b in PAIRS])
            errs = [_rel(r[[0, 21]], rr), _rel(m[:, [0, 21]], rm), _rel(st[:, [0, 21]], rst)]
            assert max(errs) <= 1e-5, (k, errs)     # rho, mom, stress (test_gpu_parity.moment_errors)
            ke = 0.5 * float((m ** 2 / r).sum())
            assert ke == pytest.approx(float(z["ke"][k - 1]), rel=1e-5)
