"""The CPU oracle (oracle/) pinned against outputs of the reference package itself.

Fixtures in tests/golden/ were produced by tests/golden/gen_golden.py, which runs
/root/reference/pkg/src/momentlbm (lattice.py, moments.py, collision.py)."""

from pathlib import Path

import numpy as np

from oracle import collision as OC
from oracle import lattice as OL
from oracle import moments as OM
from oracle import step as OS

G = Path(__file__).resolve().parent / "golden"


def load(name):
    return np.load(G / name)


def test_lattice_tables_exact():
    z = load("lattice.npz")
    assert np.array_equal(z["velocities"], OL.C)
    assert np.array_equal(z["weights"], OL.W)
    assert np.array_equal(z["opposite"], OL.OPP)
    assert np.array_equal(z["h2"], OL.H2)
    assert np.array_equal(z["h2c"], OL.H2C)
    assert np.array_equal(z["h3"], OL.H3)


def test_lattice_isotropy_exact():
    # SPEC.md:567 acceptance 1 (rational check), lattice.py:127-139
    assert OL.check_isotropy()
    assert OL.W_EXACT[0] == OL.Fraction(8, 27) if hasattr(OL, "Fraction") else True


def test_moments_against_reference():
    z = load("moments.npz")
    f = OM.reconstruct_distributions(z["rho"], z["mom"], z["stress"])
    assert np.array_equal(f, z["f"])
    r, m, s = OM.moments_from_distributions(z["f_rand"])
    assert np.array_equal(r, z["rho_of_f"])
    assert np.array_equal(m, z["mom_of_f"])
    assert np.array_equal(s, z["stress_of_f"])
    assert np.array_equal(OM.neq_decompose(z["rho"], z["mom"], z["stress"]), z["sneq"])


def test_collision_against_reference():
    z = load("collision.npz")
    for k, force in ((0, None), (1, z["force"])):
        r, m, s = OC.collide_moments(z["rho"], z["mom"], z["stress"], force, float(z[f"tau{k}"]))
        assert np.array_equal(r, z[f"rho{k}"])
        assert np.array_equal(m, z[f"mom{k}"])
        assert np.array_equal(s, z[f"stress{k}"])


def test_periodic_step_against_reference_composition():
    z = load("step16.npz")
    r, m, s = OS.fluid_step(z["rho"], z["mom"], z["stress"], float(z["tau"]))
    np.testing.assert_allclose(r, z["rho1"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(m, z["mom1"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(s, z["stress1"], rtol=0, atol=1e-15)


def test_tgv32_ten_steps_against_reference_composition():
    z = load("tgv32.npz")
    r, m, s = OS.run(z["rho0"], z["mom0"], z["stress0"], float(z["tau"]), int(z["steps"]))
    np.testing.assert_allclose(r, z["rho"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(m, z["mom"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(s, z["stress"], rtol=0, atol=1e-14)
    # and the oracle's own TGV initialisation is the fixture's
    r0, m0, s0 = OS.taylor_green(32)
    np.testing.assert_allclose(r0, z["rho0"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(m0, z["mom0"], rtol=0, atol=1e-15)


def test_oracle_d3q19_matches_reference():
    """D3Q19 lattice tables and 1 / 3 periodic steps (reference composition, tests/golden/d3q19.npz)."""
    z = np.load(G / "d3q19.npz")
    lat = OL.D3Q19
    assert np.array_equal(lat.C, z["velocities"])
    np.testing.assert_array_equal(lat.W, z["weights"])
    assert np.array_equal(lat.OPP, z["opposite"])
    np.testing.assert_allclose(lat.H2C, z["h2c"], rtol=0, atol=0)
    np.testing.assert_allclose(lat.H3, z["h3"], rtol=0, atol=1e-15)
    tau = float(z["tau"])
    got1 = OS.run(z["rho"], z["mom"], z["stress"], tau, 1, lat=lat)
    got3 = OS.run(z["rho"], z["mom"], z["stress"], tau, 3, lat=lat)
    for g, r in zip(got1, (z["rho1"], z["mom1"], z["stress1"])):
        np.testing.assert_allclose(g, r, rtol=0, atol=1e-15)
    for g, r in zip(got3, (z["rho3"], z["mom3"], z["stress3"])):
        np.testing.assert_allclose(g, r, rtol=0, atol=1e-14)


# ---- SURVEY.md §8c's remaining golden vectors (gen_golden.py --extra: reference functions + SPEC
# codec / list definitions written out in the generator, independent of oracle/)
def test_oracle_q16_step_matches_reference_composition():
    from oracle import codec
    z = load("q16_step16.npz")
    words = codec.pack(z["codes0"].astype(np.uint32))
    got = codec.unpack(OS.fluid_step_q16(words, float(z["tau"]), 0)[0])
    assert np.array_equal(got, z["codes1"].astype(np.uint32))   # float64 both sides: bit-exact


def test_oracle_boundary_lists_match_reference_directions():
    z = load("sphere32.npz")
    cells, masks = OS.boundary_lists(z["mask"], OS.BC())
    assert np.array_equal(cells, z["boundary_cells"])
    assert np.array_equal(masks, z["link_masks"])
    assert np.array_equal(OS.solid_cells(z["mask"]), z["solid_cells"])


def test_oracle_tgv64_ten_steps():
    z = load("tgv64.npz")
    r, m, s = OS.taylor_green(64)
    for _ in range(10):
        r, m, s = OS.fluid_step(r, m, s, float(z["tau"]))
    got = np.concatenate([r[None], m, OM.neq_decompose(r, m, s)])[:, [0, 21]]
    np.testing.assert_allclose(got, z["planes10"], rtol=0, atol=1e-13)
    assert 0.5 * float((m ** 2 / r).sum()) == __import__("pytest").approx(z["ke"][9], rel=1e-12)
