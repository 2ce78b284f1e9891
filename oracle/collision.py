"""ORACLE (test infrastructure only) -- moment-space collision, float64.

Restates ``/root/reference/pkg/src/momentlbm/collision.py``:
  * ``tau_from_viscosity`` -- collision.py:30-31 (tau = 0.5 + nu/cs2)
  * ``collide_moments``    -- collision.py:137-194, 3D branch (174-192)
"""

from __future__ import annotations

import numpy as np

from .lattice import CS2


def tau_from_viscosity(nu: float) -> float:
    return 0.5 + nu / CS2


def collide_moments(rho, mom, stress, force, tau):
    """Post-collision (rho, mom, stress); collision.py:137-194 (dims=3).

    u = mom/rho (pre-kick, :158); mom+ = mom + F/2 (:160); coupled
    diagonal update with cd = (tau-1)/(3 tau) (:176-188); off-diagonal
    relaxation with cxy = (2 tau - 1)/(2 tau) (:189-191)."""
    rho = np.asarray(rho, dtype=np.float64)
    mom = np.asarray(mom, dtype=np.float64)
    stress = np.asarray(stress, dtype=np.float64)
    if force is None:
        force = np.zeros((3,) + (1,) * rho.ndim)
    else:
        force = np.asarray(force, dtype=np.float64)
        force = force.reshape((3,) + (1,) * rho.ndim) if force.ndim == 1 else force

    u = mom / rho
    s = 1.0 / tau
    mom_new = mom + 0.5 * force
    fu = {(a, b): force[a] * u[b] for a in range(3) for b in range(3)}

    ux, uy, uz = u
    cxy = (2 * tau - 1) / (2 * tau)
    cd = (tau - 1) / (3 * tau)
    u2 = (ux * ux, uy * uy, uz * uz)
    diag = (stress[0], stress[3], stress[5])
    new_diag = []
    for a in range(3):
        b, g = [i for i in range(3) if i != a]
        val = (cd * (2 * diag[a] - diag[b] - diag[g])
               + rho * (u2[0] + u2[1] + u2[2]) / 3.0
               + rho * (2 * u2[a] - u2[b] - u2[g]) / (3 * tau)
               + fu[(a, a)]
               + cd * (2 * fu[(a, a)] - fu[(b, b)] - fu[(g, g)]))
        new_diag.append(val)
    sxy = (1 - s) * stress[1] + s * rho * ux * uy + cxy * (fu[(0, 1)] + fu[(1, 0)])
    sxz = (1 - s) * stress[2] + s * rho * ux * uz + cxy * (fu[(0, 2)] + fu[(2, 0)])
    syz = (1 - s) * stress[4] + s * rho * uy * uz + cxy * (fu[(1, 2)] + fu[(2, 1)])
    stress_new = np.stack([new_diag[0], sxy, sxz, new_diag[1], syz, new_diag[2]])
    return rho.copy(), mom_new, stress_new
