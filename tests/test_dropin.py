"""The drop-in: ``momentlbm.solver`` inside the reference package's namespace (the reference ships
lattice / moments / collision / stability but not the solver its layout names).  CPU tests cover the
import, the SPEC types and their validation; GPU tests run TGV 64^3 (BASELINE config 1) and the split
two-phase step through it against the oracle."""

import numpy as np
import pytest

from paper_2602_05295_b200 import dropin


def _mods():
    pkg = dropin.install()
    import momentlbm.solver as S
    return pkg, S


def test_solver_module_lives_in_the_reference_namespace():
    pkg, S = _mods()
    import momentlbm.moments as RM
    assert S.__name__ == "momentlbm.solver"
    assert S.__file__.endswith("overlay/momentlbm/solver.py")
    assert "baseline" in pkg.__file__ or "reference" in pkg.__file__     # the unmodified reference package
    assert S.MomentSet is RM.MomentSet                                   # the reference's own value type
    for name in ("SimGrid", "SolverConfig", "StepStats", "fused_step", "fluid_update_step",
                 "solid_correction_step", "run"):
        assert hasattr(S, name)


def test_spec_types_validate_like_the_reference():
    _, S = _mods()
    with pytest.raises(ValueError):
        S.SolverConfig(lattice="D3Q15")           # make_lattice rejects it (lattice.py:172-211)
    with pytest.raises(ValueError):
        S.SolverConfig(nu=0.0)                    # tau <= 1/2 (collision.py:102-103)
    with pytest.raises(ValueError):
        S.SolverConfig(bc={"x-": "slip"})
    with pytest.raises(ValueError):
        S.SolverConfig(bc={"q+": "wall"})
    cfg = S.SolverConfig(nu=0.01, bc={"x-": ("inflow", (0.05, 0, 0)), "x+": "outflow"}, quantization="16/15")
    assert cfg.tau == pytest.approx(0.53)
    b = cfg._b200()
    assert b.precision == "q16" and b.bc["x"] == ("inflow", "outflow") and tuple(b.u_in) == (0.05, 0, 0)
    assert b.quant.bits == (16,) * 4 + (15,) * 6
    g = S.SimGrid((8, 8, 8))
    r = np.full((8, 8, 8), 1.01)
    g.set_moments(r, np.zeros((3, 8, 8, 8)), np.zeros((6, 8, 8, 8)))
    ms = g.moment_set(1, 2, 3)                    # before any device state: the pending moments
    assert ms.rho == pytest.approx(1.01) and type(ms).__module__ == "momentlbm.moments"
    with pytest.raises(ValueError):
        S.SimGrid((8, 8, 8), mask=np.zeros((8, 8, 4)))


@pytest.mark.gpu
def test_tgv64_through_momentlbm_solver():
    """BASELINE config 1 via the drop-in: run(config, 200) on TGV 64^3 vs the oracle (<= 1e-5)."""
    from oracle import step as OS
    _, S = _mods()
    state = OS.taylor_green(64)
    cfg = S.SolverConfig(nu=0.01, dims=(64, 64, 64), initial=state)
    res = S.run(cfg, 200, snapshot_every=100)
    assert [sn.step for sn in res.snapshots] == [0, 100, 200]
    assert len(res.stats) == 200
    got = res.grid.moments()
    ref = OS.run(*state, cfg.tau, 200)
    err = [float(np.linalg.norm(g - r) / np.linalg.norm(r)) for g, r in zip(got, ref)]
    print("momentlbm.solver TGV64 x 200:", err)
    assert max(err) <= 1e-5
    m0 = res.stats[0].mass
    assert all(abs(st.mass - m0) / m0 < 1e-7 for st in res.stats)      # mass conservation (fp32 state)
    res.grid.close()


@pytest.mark.gpu
def test_two_phase_split_step_equals_solver_step():
    from oracle import step as OS
    from paper_2602_05295_b200 import SimGrid, Solver
    from paper_2602_05295_b200.geometry import sphere_mask
    _, S = _mods()
    shape = (24, 20, 28)
    mask = sphere_mask(shape, (10, 9.5, 13.5), 4)
    cfg = S.SolverConfig(nu=0.02, bc={"x-": ("inflow", (0.05, 0, 0)), "x+": "outflow", "z-": "wall", "z+": "wall"},
                         obstacles=[mask])
    state = OS.random_state(shape, seed=3, drho=0.04, umax=0.05, sneq=0.004)
    g = S.SimGrid(shape)
    g.set_moments(*state)
    for _ in range(3):
        S.fluid_update_step(g, cfg)
        S.solid_correction_step(g, cfg)
    assert g.last_stats.t_solid_ms > 0 and g.step_count == 3
    S.fluid_update_step(g, cfg)          # left uncommitted: the accessor finishes it
    got = g.solver.get_state()
    with Solver(SimGrid(shape, mask), cfg._b200()) as s:
        s.set_moments(*state)
        s.step(4)
        ref = s.get_state()
    assert np.array_equal(got, ref)
    # solid_correction_step without a pending update, and without obstacles: identity
    before = g.solver.get_state()
    S.solid_correction_step(g, cfg)
    assert np.array_equal(g.solver.get_state(), before)
    g.close()


@pytest.mark.gpu
def test_fused_step_and_alignment():
    from oracle import step as OS
    _, S = _mods()
    shape = (16, 16, 24)
    cfg = S.SolverConfig(nu=0.02)
    state = OS.random_state(shape, seed=4, drho=0.04, umax=0.05, sneq=0.004)
    g = S.SimGrid(shape)
    g.set_moments(*state)
    for _ in range(4):
        S.fused_step(g, cfg)
    S.align_to_split(g, cfg)
    ref = state
    for _ in range(4):
        ref = OS.alg1_step(*ref, cfg.tau)
    ref = OS.stream_step(*ref)
    err = [float(np.linalg.norm(a - b) / np.linalg.norm(b)) for a, b in zip(g.moments(), ref)]
    assert max(err) <= 1e-5, err
    g.close()


@pytest.mark.gpu
def test_run_divergence_restores_last_good_snapshot():
    from oracle.moments import neq_recompose
    _, S = _mods()
    shape = (8, 8, 8)
    rho = np.ones(shape)
    mom = np.zeros((3,) + shape)
    mom[0] = 0.85                            # uniform flow accelerated by a body force past 0.9
    st = neq_recompose(rho, mom, np.zeros((6,) + shape))
    cfg = S.SolverConfig(nu=0.01, force=(0.002, 0.0, 0.0), dims=shape, initial=(rho, mom, st))
    with pytest.raises(S.SolverDiverged) as ei:
        S.run(cfg, 500, checkpoint_every=1)
    e = ei.value
    assert isinstance(e, FloatingPointError)
    assert 40 <= e.step <= 60 and e.last_good.step == e.step - 1   # +F/2 per step (collision.py:160)
    assert np.all(np.isfinite(e.last_good.rho)) and np.abs(e.last_good.mom[0]).max() < 0.9


@pytest.mark.gpu
def test_run_zero_steps_is_the_initial_snapshot():
    _, S = _mods()
    res = S.run(S.SolverConfig(dims=(8, 8, 8)), 0)
    assert len(res.snapshots) == 1 and res.snapshots[0].step == 0 and res.stats == []
    assert np.all(res.snapshots[0].rho == 1.0)
    res.grid.close()


def test_geometry_module_in_the_reference_namespace(tmp_path):
    """momentlbm.geometry: load_mesh, link_intersect, voxelize_surface, with the
    SPEC examples, and the surface mask covers every node the GPU cut-link finder (same test) cuts."""
    dropin.install()
    import momentlbm.geometry as G
    from oracle import mesh as M
    p = tmp_path / "tri.obj"
    p.write_text("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n")
    m = G.load_mesh(p)
    assert m.vertices.shape == (3, 3) and m.faces.tolist() == [[0, 1, 2]]
    # axis link crossing a perpendicular triangle at its midpoint -> t = 0.5
    tri = np.array([[0.5, -1.0, -1.0], [0.5, 3.0, -1.0], [0.5, -1.0, 3.0]])
    t, hit = G.link_intersect((1.0, 0.0, 0.0), (1, 0, 0), tri)
    assert t == pytest.approx(0.5) and np.allclose(hit, (0.5, 0, 0))
    # parallel / coplanar link -> no hit
    assert G.link_intersect((0.5, 0.0, 0.0), (0, 1, 0), tri) is None
    # SurfaceMask covers the nodes with cut links
    V, F = M.icosphere((10.3, 9.7, 11.1), 4.2, 2)
    dims = (22, 20, 24)
    mask = G.voxelize_surface(G.TriangleMesh(V, F), dims)
    cells, _, _, _ = M.cut_links(V, F, dims)
    x, r = np.divmod(cells, dims[1] * dims[2])
    y, z = np.divmod(r, dims[2])
    assert mask[x, y, z].all()
    assert mask.sum() < 0.25 * mask.size


@pytest.mark.gpu
def test_solver_with_mesh_obstacle_and_solid_state():
    """A TriangleMesh with a SolidState as a momentlbm.solver obstacle: the step applies Eq. 8 with
    the body's velocity (oracle mesh step with the same motion)."""
    from oracle import mesh as M
    from oracle import step as OS
    _, S = _mods()
    import momentlbm.geometry as G
    shape = (24, 20, 28)
    V, F = M.icosphere((11.3, 9.7, 13.9), 5.2, 2)
    motion = ((0.01, -0.005, 0.0), (0.0, 0.002, 0.001), (11.3, 9.7, 13.9))
    mesh = G.TriangleMesh(V, F, G.SolidState(*motion))
    cfg = S.SolverConfig(nu=0.02, obstacles=[mesh])
    state = OS.random_state(shape, seed=5, drho=0.02, umax=0.04, sneq=0.002)
    g = S.SimGrid(shape)
    g.set_moments(*state)
    S.fluid_update_step(g, cfg)
    S.solid_correction_step(g, cfg)
    got = g.moments()
    cells, _, t, _ = M.cut_links(V, F, shape)
    r, m, sx, Fs, _ = M.step_with_mesh(*state, cfg.tau, cells, t, solid=motion)
    for a, b in zip(got, (r, m, sx)):
        assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-5
    np.testing.assert_allclose(g.last_stats.force, Fs, rtol=1e-4, atol=1e-7)
    g.close()
