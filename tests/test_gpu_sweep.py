"""Quantization accuracy-memory sweep (SPEC.md:541-544 cmd_quant_sweep; Fig. 11) on the
GPU path, against the float64 oracle's run of the same scenario."""

import numpy as np
import pytest

from oracle import step as OS
from paper_2602_05295_b200.sweep import DEFAULT_PRESETS, Scenario, quant_sweep, to_csv


def test_sweep_cpu_pieces():
    sc = Scenario(n=16, steps=1)
    rho, u = sc.initial()
    assert rho.shape == (16, 16, 4) and u.shape == (3, 16, 16, 4)
    assert np.allclose(u[:, :, :, 0], u[:, :, :, 3]) and np.abs(u).max() <= sc.u0 + 1e-12
    with pytest.raises(ValueError):
        quant_sweep(sc, presets=("16/9",))
    assert to_csv([{"config": "a", "l2_rel_error": 0.5}]) == "config,l2_rel_error\na,0.5\n"


@pytest.mark.gpu
def test_quant_sweep_against_fp64_oracle():
    sc = Scenario(n=32, steps=120, re=2000.0)
    rho, u = sc.initial()
    mom = rho * u
    stress = np.stack([mom[a] * u[b] for a, b in ((0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2))])
    r, m, _ = OS.run(rho, mom, stress, 0.5 + 3 * sc.nu, sc.steps)
    ref = m / r
    rows = quant_sweep(sc, reference=ref, reference_label="fp64")
    err = {row["config"]: row["l2_rel_error"] for row in rows}
    assert err["fp64"] == 0.0 and err["fp32"] < 1e-5
    e = [err[p] for p in DEFAULT_PRESETS]
    assert e[0] < 1e-3                                    # 16/16 resolves the flow
    assert all(b >= a * 0.9 for a, b in zip(e, e[1:]))    # fewer bits, no better (10% noise band)
    assert e[-1] > 4 * e[0]                               # 12/11 visibly degraded (Fig. 11 trend)
    pay = [row["bytes_payload"] for row in rows if row["config"] in DEFAULT_PRESETS]
    assert pay == sorted(pay, reverse=True) and pay[0] == 20
