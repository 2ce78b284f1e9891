"""ORACLE (test infrastructure only) -- moment algebra, float64 NumPy.

Restates ``/root/reference/pkg/src/momentlbm/moments.py`` for the D3Q27
lattice; arrays put the component/direction axis first and accept any grid
shape after it (moments.py:11-13).

  * ``moments_from_distributions``  -- moments.py:25-39
  * ``_third_order_tensor``         -- moments.py:42-52
  * ``reconstruct_distributions``   -- moments.py:64-90
  * ``neq_decompose/neq_recompose`` -- moments.py:93-102
  * ``_outer_voigt``                -- moments.py:124-133
"""

from __future__ import annotations

import numpy as np

from . import lattice as L


def moments_from_distributions(f, lat=None):
    """rho = sum f, mom = c^T f, stress = h2^T f (moments.py:25-39).

    No F/2 term: the body-force half step belongs to the collision
    (moments.py:31-32).  ``lat``: an ``oracle.lattice.Lat`` (default D3Q27)."""
    lat = lat or L.D3Q27
    if f.shape[0] != lat.Q:
        raise ValueError(f"expected {lat.Q} distributions, got {f.shape[0]}")
    c = lat.C.astype(np.float64)
    rho = f.sum(axis=0)
    mom = np.tensordot(c.T, f, axes=1)
    stress = np.tensordot(lat.H2.T, f, axes=1)
    return rho, mom, stress


def _third_order_tensor(u, s, labels=L.H3_LABELS):
    """T_abg = S_ab u_g + S_ag u_b + S_bg u_a - 2 u_a u_b u_g (moments.py:42-52)."""
    vidx = L.voigt_index()
    out = []
    for label in labels:
        a, b, g = (L._AXIS[ch] for ch in label)
        t = (s[vidx[tuple(sorted((a, b)))]] * u[g]
             + s[vidx[tuple(sorted((a, g)))]] * u[b]
             + s[vidx[tuple(sorted((b, g)))]] * u[a]
             - 2.0 * u[a] * u[b] * u[g])
        out.append(t)
    return np.stack(out, axis=0)


def reconstruct_distributions(rho, mom, stress, lat=None):
    """f_i = rho w_i [1 + c.u/cs2 + H2:S/(2cs4) + sum_l H3_l T_l/(2cs6)] (moments.py:64-90).

    Each H3 label (including xyz on D3Q27) enters once with 1/(2 cs^6), exactly as
    the reference does (moments.py:86); D3Q19 drops xyz (moments.py:74-76)."""
    lat = lat or L.D3Q27
    rho = np.asarray(rho, dtype=np.float64)
    mom = np.asarray(mom, dtype=np.float64)
    stress = np.asarray(stress, dtype=np.float64)
    cs2 = L.CS2
    cs4, cs6 = cs2 ** 2, cs2 ** 3
    u = mom / rho
    s = stress / rho
    h2_term = np.tensordot(lat.H2C, s, axes=1) / (2 * cs4)
    t = _third_order_tensor(u, s, lat.H3_LABELS)
    h3_term = np.tensordot(lat.H3, t, axes=1) / (2 * cs6)
    cu = np.tensordot(lat.C.astype(np.float64), u, axes=1)
    w = lat.W.reshape((lat.Q,) + (1,) * rho.ndim)
    return rho * w * (1.0 + cu / cs2 + h2_term + h3_term)


def outer_voigt(mom):
    """Voigt-ordered mom_a mom_b (moments.py:124-133)."""
    mom = np.asarray(mom, dtype=np.float64)
    rows = []
    for name in L.VOIGT:
        a, b = L._AXIS[name[0]], L._AXIS[name[1]]
        rows.append(mom[a] * mom[b])
    return np.stack(rows, axis=0)


def neq_decompose(rho, mom, stress):
    """sneq = stress - mom mom / rho (moments.py:93-96), Eq.-5 convention."""
    return np.asarray(stress, dtype=np.float64) - outer_voigt(mom) / rho


def neq_recompose(rho, mom, sneq):
    """Exact inverse of neq_decompose (moments.py:99-102)."""
    return np.asarray(sneq, dtype=np.float64) + outer_voigt(mom) / rho
