"""SPEC.md:404-407 load_mesh: Wavefront OBJ parsing (v / f records), affine transform, errors with line
numbers / face indices."""

import numpy as np
import pytest

from oracle import mesh as M
from paper_2602_05295_b200.geometry import load_obj, save_obj


def test_unit_right_triangle(tmp_path):
    p = tmp_path / "t.obj"
    p.write_text("# unit right triangle\nv 0 0 0\nv 1 0 0\nv 0 1 0\nvn 0 0 1\nf 1//1 2//1 3//1\n")
    V, F = load_obj(p)
    assert V.shape == (3, 3) and F.tolist() == [[0, 1, 2]]


def test_polygons_negative_indices_and_transform(tmp_path):
    p = tmp_path / "q.obj"
    p.write_text("o quad\nv 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nf -4/1 -3/2 -2/3 -1/4\n")
    V, F = load_obj(p, transform=[[2, 0, 0, 10], [0, 2, 0, 20], [0, 0, 2, 30]])
    assert F.tolist() == [[0, 1, 2], [0, 2, 3]]
    assert V[2].tolist() == [12.0, 22.0, 30.0]


def test_round_trip_matches_independent_counts(tmp_path):
    V0, F0 = M.icosphere((10.0, 11.0, 12.0), 5.0, 3)
    p = tmp_path / "s.obj"
    save_obj(p, V0, F0)
    text = p.read_text().splitlines()
    assert sum(l.startswith("v ") for l in text) == len(V0) and sum(l.startswith("f ") for l in text) == len(F0)
    V, F = load_obj(p)
    assert np.array_equal(V, V0) and np.array_equal(F, F0)


@pytest.mark.parametrize("body,msg", [("v 0 0\n", ":1: vertex record"), ("v 0 0 0\nv 1 0 0\nf 1 2\n", ":3: face record"),
                                      ("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 x\n", ":4: malformed face"),
                                      ("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 7\n", ":4: face index"),
                                      ("v 0 0 0\nv 1 0 0\nv 0 1 0\nv 2 0 0\nf 1 2 3\nf 1 2 4\n", "degenerate face 1")])
def test_malformed_records(tmp_path, body, msg):
    p = tmp_path / "bad.obj"
    p.write_text(body)
    with pytest.raises(ValueError, match=msg):
        load_obj(p)


def test_scene_helpers_match_the_oracle_inputs():
    """geometry.icosphere / taylor_green_fields (the tools' scene inputs) equal the oracle's."""
    from oracle import mesh as M
    from oracle import step as OS
    from paper_2602_05295_b200.geometry import icosphere, taylor_green_fields
    V, F = icosphere((3.0, 4.0, 5.0), 2.5, 2)
    V0, F0 = M.icosphere((3.0, 4.0, 5.0), 2.5, 2)
    assert np.array_equal(F, F0) and np.allclose(V, V0, rtol=0, atol=1e-13)
    rho, u = taylor_green_fields(16)
    r0, m0, _ = OS.taylor_green(16)
    assert np.allclose(rho, r0, rtol=0, atol=1e-15) and np.allclose(rho * u, m0, rtol=0, atol=1e-15)
