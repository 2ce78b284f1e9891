"""ORACLE (test infrastructure only) -- D3Q27 lattice tables.

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
