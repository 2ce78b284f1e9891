"""Triangle-mesh oracle: link-triangle intersection known answers and an
independent signed-volume cross-check ('agrees with the orientation-sign
brute-force oracle')."""

import numpy as np

from oracle import mesh as M
from oracle import step as OS


def one(o, d, v0, v1, v2):
    hit, t = M.segment_triangle(tuple(np.array([x]) for x in o), tuple(np.array([x]) for x in d), v0, v1, v2)
    return bool(hit[0]), float(t[0])


def test_axis_link_through_perpendicular_triangle_midpoint():
    hit, t = one((5.0, 5.0, 5.0), (1.0, 0.0, 0.0), (5.5, 4.0, 4.0), (5.5, 7.0, 4.0), (5.5, 4.0, 7.0))
    assert hit and t == 0.5


def test_parallel_coplanar_link_never_hits():
    hit, _ = one((5.0, 5.0, 5.0), (0.0, 1.0, 0.0), (5.0, 4.0, 4.0), (5.0, 7.0, 4.0), (5.0, 4.0, 7.0))
    assert not hit


def test_miss_beyond_segment():
    hit, _ = one((5.0, 5.0, 5.0), (1.0, 0.0, 0.0), (6.5, 4.0, 4.0), (6.5, 7.0, 4.0), (6.5, 4.0, 7.0))
    assert not hit


def _orient(a, b, c, d):
    return np.linalg.det(np.stack([b - a, c - a, d - a]))


def test_against_signed_volume_oracle():
    rng = np.random.default_rng(3)
    n_agree = n = 0
    for _ in range(20000):
        o = rng.uniform(0, 2, 3)
        d = rng.choice([-1.0, 0.0, 1.0], 3)
        if not d.any():
            continue
        tri = rng.uniform(0, 2, (3, 3))
        hit, t = one(tuple(o), tuple(d), tuple(tri[0]), tuple(tri[1]), tuple(tri[2]))
        e = o + d
        # segment crosses the triangle iff the endpoints are on opposite sides of its plane and
        # the segment passes inside all three edges (same-sign orientations)
        s1, s2 = _orient(tri[0], tri[1], tri[2], o), _orient(tri[0], tri[1], tri[2], e)
        a1 = _orient(o, e, tri[0], tri[1])
        a2 = _orient(o, e, tri[1], tri[2])
        a3 = _orient(o, e, tri[2], tri[0])
        ref = (s1 * s2 < 0) and ((a1 > 0 and a2 > 0 and a3 > 0) or (a1 < 0 and a2 < 0 and a3 < 0))
        margin = min(abs(s1), abs(s2), abs(a1), abs(a2), abs(a3))
        if margin < 1e-6:
            continue   # inside the eps band: policy-dependent
        n += 1
        n_agree += hit == ref
    assert n > 10000 and n_agree == n


def test_cut_links_earliest_hit_and_tie_break():
    # two parallel triangles crossing the same links: the nearer one (smaller t) wins; a duplicated
    # triangle ties and the lower index wins
    V = np.array([[5.3, 3, 3], [5.3, 8, 3], [5.3, 3, 8], [5.7, 3, 3], [5.7, 8, 3], [5.7, 3, 8]], dtype=float)
    F = np.array([[3, 4, 5], [0, 1, 2], [0, 1, 2]])
    cells, masks, t, tri = M.cut_links(V, F, (10, 10, 12))
    x, y, z = 5, 4, 4
    n = np.searchsorted(cells, (x * 10 + y) * 12 + z)
    i = 2   # c = (-1,0,0): link 5 -> 6 crosses x = 5.3 first (t = 0.3)
    assert t[n, i] == np.float64(5.3) - 5.0 or abs(t[n, i] - 0.3) < 1e-15
    assert tri[n, i] == 1


def test_mesh_step_conserves_mass_closed_sphere_at_rest():
    V, F = M.icosphere((8, 8, 8), 3.0, 1)
    cells, masks, t, tri = M.cut_links(V, F, (16, 16, 16))
    shape = (16, 16, 16)
    rho = np.ones(shape)
    mom = np.zeros((3,) + shape)
    st = np.zeros((6,) + shape)
    r, m, s, Fs, Ts = M.step_with_mesh(rho, mom, st, 0.6, cells, t)
    assert np.abs(r - 1).max() < 1e-14 and np.abs(m).max() < 1e-14 and np.abs(Fs).max() < 1e-14
