"""ORACLE (test infrastructure only) -- D3Q27 (and D3Q19) lattice tables.

CPU restatement of the reference's lattice construction, used ONLY by
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
leg as the checker.  The product path never imports this package.

Restates ``/root/reference/pkg/src/momentlbm/lattice.py``:
  * direction order            -- ``_d3_velocities`` (lattice.py:99-116)
  * weights by |c|^2           -- ``_WEIGHT_BY_SPEED2["D3Q27"]`` (lattice.py:119-124)
  * opposite table             -- ``make_lattice`` (lattice.py:198-201)
  * Hermite tables h2 / h2c / h3 -- ``hermite2``/``hermite3``/``_build_hermite``
    (lattice.py:142-169); Voigt order xx,xy,xz,yy,yz,zz (lattice.py:23);
    third-order labels xxy,xyy,xxz,xzz,yzz,yyz,xyz (lattice.py:30).
  * D3Q19 -- the first 19 directions of the same order (no corners, lattice.py:99-116),
    weights 1/3, 1/18, 1/36 (``_WEIGHT_BY_SPEED2["D3Q19"]``, lattice.py:121), no xyz label
    (lattice.py:166-167).  The module-level names are the D3Q27 tables; ``D3Q19`` / ``D3Q27``
    / ``get(q)`` return the same tables as a ``Lat`` record.
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np

CS2 = 1.0 / 3.0  # lattice.py:17

VOIGT = ("xx", "xy", "xz", "yy", "yz", "zz")          # lattice.py:23
H3_LABELS = ("xxy", "xyy", "xxz", "xzz", "yzz", "yyz", "xyz")  # lattice.py:30
_AXIS = {"x": 0, "y": 1, "z": 2}                       # lattice.py:19


def d3q27_velocities() -> np.ndarray:
    """Rest, axis (+/-), face diagonals, corners -- lattice.py:99-116."""
    vels = [(0, 0, 0)]
    for a in range(3):
        for s in (1, -1):
            v = [0, 0, 0]
            v[a] = s
            vels.append(tuple(v))
    for a, b in ((0, 1), (0, 2), (1, 2)):
        for sa, sb in ((1, 1), (-1, -1), (1, -1), (-1, 1)):
            v = [0, 0, 0]
            v[a], v[b] = sa, sb
            vels.append(tuple(v))
    for corner in ((1, 1, 1), (-1, -1, -1), (1, 1, -1), (-1, -1, 1),
                   (1, -1, 1), (-1, 1, -1), (1, -1, -1), (-1, 1, 1)):
        vels.append(corner)
    return np.array(vels, dtype=np.int64)


C = d3q27_velocities()
Q = 27
_W_EXACT = {0: Fraction(8, 27), 1: Fraction(2, 27), 2: Fraction(1, 54), 3: Fraction(1, 216)}
W_EXACT = tuple(_W_EXACT[int((v * v).sum())] for v in C)
W = np.array([float(x) for x in W_EXACT])
OPP = np.array([[int(j) for j in range(Q) if (C[j] == -C[i]).all()][0] for i in range(Q)],
               dtype=np.int64)


def _h2(c, a, b):
    # H2_ab(c) = c_a c_b - cs2 d_ab  (lattice.py:142-145)
    return c[:, a] * c[:, b] - (CS2 if a == b else 0.0)


def _h3(c, label):
    # lattice.py:148-153
    a, b, g = (_AXIS[ch] for ch in label)
    ca, cb, cg = c[:, a], c[:, b], c[:, g]
    d = lambda i, j: 1.0 if i == j else 0.0
    return ca * cb * cg - CS2 * (ca * d(b, g) + cb * d(a, g) + cg * d(a, b))


_CF = C.astype(np.float64)
H2 = np.stack([_h2(_CF, _AXIS[l[0]], _AXIS[l[1]]) for l in VOIGT], axis=1)   # (27, 6)
H2C = H2.copy()
for _j, _l in enumerate(VOIGT):
    if _l[0] != _l[1]:
        H2C[:, _j] *= 2.0                                                   # lattice.py:159-162
H3 = np.stack([_h3(_CF, l) for l in H3_LABELS], axis=1)                     # (27, 7)


class Lat:
    """One velocity set: C, Q, W, OPP, H2, H2C, H3, H3_LABELS."""

    def __init__(self, q: int):
        c = d3q27_velocities()[:q]
        self.Q = q
        self.C = c
        wex = {27: _W_EXACT, 19: {0: Fraction(1, 3), 1: Fraction(1, 18), 2: Fraction(1, 36)}}[q]
        self.W_EXACT = tuple(wex[int((v * v).sum())] for v in c)
        self.W = np.array([float(x) for x in self.W_EXACT])
        self.OPP = np.array([[int(j) for j in range(q) if (c[j] == -c[i]).all()][0] for i in range(q)],
                            dtype=np.int64)
        cf = c.astype(np.float64)
        self.H2 = np.stack([_h2(cf, _AXIS[l[0]], _AXIS[l[1]]) for l in VOIGT], axis=1)
        self.H2C = self.H2.copy()
        for j, l in enumerate(VOIGT):
            if l[0] != l[1]:
                self.H2C[:, j] *= 2.0
        self.H3_LABELS = H3_LABELS if q == 27 else tuple(l for l in H3_LABELS if l != "xyz")
        self.H3 = np.stack([_h3(cf, l) for l in self.H3_LABELS], axis=1)


D3Q27 = Lat(27)
D3Q19 = Lat(19)


def get(q=None) -> Lat:
    return D3Q19 if q == 19 else D3Q27


def voigt_index():
    """(a,b) sorted -> Voigt slot (moments.py:55-61)."""
    idx = {}
    for j, name in enumerate(VOIGT):
        a, b = _AXIS[name[0]], _AXIS[name[1]]
        idx[tuple(sorted((a, b)))] = j
    return idx


def check_isotropy() -> bool:
    """Exact rational check of the 0th..4th order identities (lattice.py:127-139)."""
    cs2 = Fraction(1, 3)
    if sum(W_EXACT) != 1:
        return False
    for a in range(3):
        if sum(w * v[a] for v, w in zip(C.tolist(), W_EXACT)) != 0:
            return False
        for b in range(3):
            s = sum(w * v[a] * v[b] for v, w in zip(C.tolist(), W_EXACT))
            if s != (cs2 if a == b else 0):
                return False
    for a in range(3):
        for b in range(3):
            for c in range(3):
                for d in range(3):
                    tot = sum(w * v[a] * v[b] * v[c] * v[d] for v, w in zip(C.tolist(), W_EXACT))
                    dd = lambda i, j: 1 if i == j else 0
                    exp = cs2 * cs2 * (dd(a, b) * dd(c, d) + dd(a, c) * dd(b, d) + dd(a, d) * dd(b, c))
                    if tot != exp:
                        return False
    return True
