"""Quantization accuracy-memory sweep (SPEC.md:541-544 ``cmd_quant_sweep``; Fig. 11).

Runs one scenario at a reference precision and then once per bit-allocation preset
(``QuantSpec.preset``), and reports the l2 relative error of the final velocity
field, ||u_preset - u_ref||_2 / ||u_ref||_2, beside the bytes per node.

The paper's Fig. 11 scenario is a 2-D double-layer vortex on D2Q9.  The B200 step is 3-D, so the
scenario here is the same double shear layer made z-invariant on a thin periodic slab
(n x n x 4 cells): a 3-D lattice carrying a 2-D flow.  The reference is whatever field the
caller passes (the tests pass the float64 oracle's); by default it is this library's own fp32
run, labelled ``fp32`` -- the only 64-bit path in the repository is the CPU test oracle, which
product code does not call.

Bytes per node: ``stored`` is what the state layout holds (fp64 reference 80 B, fp32 40 B, every
16-bit preset 20 B -- 16-bit slots); ``payload`` is the preset's own bit budget,
(4 b_rho_u + 6 b_S) / 8 bytes, the memory axis of Fig. 11.
"""

from __future__ import annotations

import csv
import io
from dataclasses import dataclass
from typing import Iterable, Optional, Sequence

import numpy as np

from .quantization import PRESETS, QuantSpec
from .solver import SimGrid, Solver, SolverConfig

DEFAULT_PRESETS = ("16/16", "16/15", "15/14", "14/13", "13/12", "12/11")


@dataclass(frozen=True)
class Scenario:
    """Double shear layer (z-invariant): u_x = U0 tanh(k (y - 1/4)) for y <= 1/2 and
    U0 tanh(k (3/4 - y)) above, u_y = U0 delta sin(2 pi (x + 1/4)), rho = 1, sneq = 0."""
    n: int = 64
    nz: int = 4
    u0: float = 0.05
    k: float = 80.0
    delta: float = 0.05
    re: float = 10000.0
    steps: int = 200

    @property
    def nu(self) -> float:
        return self.u0 * self.n / self.re

    def initial(self):
        n = self.n
        x = (np.arange(n) + 0.5) / n
        X, Y = np.meshgrid(x, x, indexing="ij")
        ux = np.where(Y <= 0.5, np.tanh(self.k * (Y - 0.25)), np.tanh(self.k * (0.75 - Y)))
        uy = self.delta * np.sin(2 * np.pi * (X + 0.25))
        u = np.zeros((3, n, n, self.nz))
        u[0] = self.u0 * ux[:, :, None]
        u[1] = self.u0 * uy[:, :, None]
        rho = np.ones((n, n, self.nz))
        return rho, u


def run_scenario(sc: Scenario, precision: str, quant: Optional[QuantSpec] = None) -> np.ndarray:
    """Final velocity field (3, n, n, nz) of one run on the GPU."""
    cfg = SolverConfig(nu=sc.nu, precision=precision, quant=quant or QuantSpec())
    rho, u = sc.initial()
    with Solver(SimGrid((sc.n, sc.n, sc.nz)), cfg) as s:
        s.set_equilibrium(rho, u)
        s.step(sc.steps)
        return s.velocity


def l2_relative(u: np.ndarray, ref: np.ndarray) -> float:
    den = float(np.linalg.norm(ref))
    return float(np.linalg.norm(u - ref)) / den if den > 0 else float(np.linalg.norm(u))


def quant_sweep(sc: Scenario = Scenario(), presets: Sequence[str] = DEFAULT_PRESETS,
                reference: Optional[np.ndarray] = None, reference_label: str = "fp64",
                dither: bool = False) -> list:
    """Rows (config, l2 relative error, stored bytes per node, payload bytes per node)."""
    for p in presets:
        if p not in PRESETS:
            raise ValueError(f"unknown preset {p!r} (known: {', '.join(PRESETS)})")
    rows = []
    fp32 = run_scenario(sc, "fp32")
    if reference is None:
        reference, reference_label = fp32, "fp32"
    ref_bytes = 80 if reference_label == "fp64" else 40
    rows.append({"config": reference_label, "l2_rel_error": 0.0, "bytes_stored": ref_bytes,
                 "bytes_payload": ref_bytes})
    if reference_label != "fp32":
        rows.append({"config": "fp32", "l2_rel_error": l2_relative(fp32, reference), "bytes_stored": 40,
                     "bytes_payload": 40})
    for p in presets:
        b_ru, b_s = PRESETS[p]
        u = run_scenario(sc, "q16", QuantSpec.preset(p, dither=dither))
        rows.append({"config": p, "l2_rel_error": l2_relative(u, reference), "bytes_stored": 20,
                     "bytes_payload": (4 * b_ru + 6 * b_s) / 8})
    return rows


def to_csv(rows: Iterable[dict]) -> str:
    rows = list(rows)
    out = io.StringIO()
    w = csv.DictWriter(out, fieldnames=list(rows[0]), lineterminator="\n")
    w.writeheader()
    for r in rows:
        w.writerow(r)
    return out.getvalue()


if __name__ == "__main__":   # python -m paper_2602_05295_b200.sweep [n] [steps]
    import sys
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    print(to_csv(quant_sweep(Scenario(n=n, steps=steps))), end="")
