"""Triangle-mesh solid coupling on the GPU vs the oracle (oracle/mesh.py): bit-exact cut-link
table (cells, masks, t, triangle), fp32 step parity (per-moment <= 1e-5), momentum-exchange
force/torque, a moving (rotating) solid, q16, and slab decomposition (bitwise)."""

import numpy as np
import pytest

from oracle import codec
from oracle import mesh as M
from oracle import step as OS
from oracle.moments import neq_decompose
from paper_2602_05295_b200 import QuantSpec, SimGrid, Slab, Solver, SolverConfig
from paper_2602_05295_b200.distributed import device_view, partition

pytestmark = pytest.mark.gpu


def _scene(shape=(24, 20, 28), seed=5):
    V, F = M.icosphere((11.3, 9.7, 13.9), 5.2, 2)
    state = OS.random_state(shape, seed=seed, drho=0.02, umax=0.04, sneq=0.002)
    return V, F, state


def test_cut_link_table_bit_exact():
    shape = (24, 20, 28)
    V, F, _ = _scene(shape)
    cells, masks, t, tri = M.cut_links(V, F, shape)
    with Solver(SimGrid(shape), SolverConfig(nu=0.02)) as s:
        s.set_mesh(V, F)
        gc, gm, gt, gtri = s.cut_links()
    assert np.array_equal(gc, cells)
    assert np.array_equal(gm, masks)
    assert np.array_equal(np.isnan(gt), np.isnan(t))
    assert np.array_equal(gt[~np.isnan(gt)], t[~np.isnan(t)])
    assert np.array_equal(gtri[~np.isnan(gt)], tri[~np.isnan(t)])


@pytest.mark.parametrize("motion", [None, ((0.01, -0.005, 0.0), (0.0, 0.002, 0.001), (11.3, 9.7, 13.9))])
def test_mesh_step_parity_and_force(motion):
    shape = (24, 20, 28)
    V, F, state = _scene(shape)
    cells, masks, t, _ = M.cut_links(V, F, shape)
    cfg = SolverConfig(nu=0.02)
    with Solver(SimGrid(shape), cfg) as s:
        if motion is None:
            s.set_mesh(V, F)
        else:
            s.set_mesh(V, F, *motion)
        s.set_moments(*state)
        st = s.step(1)
        got = s.moments()
    r, m, sx, Fs, Ts = M.step_with_mesh(*state, cfg.tau, cells, t, solid=motion)
    for g, ref in zip(got, (r, m, sx)):
        assert np.linalg.norm(g - ref) / np.linalg.norm(ref) <= 1e-5
    np.testing.assert_allclose(st.force, Fs, rtol=1e-4, atol=1e-7)
    np.testing.assert_allclose(st.torque, Ts, rtol=1e-4, atol=1e-6)


def test_mesh_q16_one_step_within_1_lsb():
    shape = (24, 20, 28)
    V, F, state = _scene(shape)
    cells, masks, t, _ = M.cut_links(V, F, shape)
    w0, _ = codec.encode_state(state[0], state[1], neq_decompose(*state))
    cfg = SolverConfig(nu=0.02, precision="q16", quant=QuantSpec())
    with Solver(SimGrid(shape), cfg) as s:
        s.set_mesh(V, F)
        s.codes = w0
        s.step(1)
        got = codec.unpack(s.codes)
    rho, mom, sn = codec.decode_state(w0)
    from oracle.moments import neq_recompose
    r, m, sx, _, _ = M.step_with_mesh(rho, mom, neq_recompose(rho, mom, sn), cfg.tau, cells, t)
    ref = codec.unpack(codec.encode_state(r, m, neq_decompose(r, m, sx))[0])
    assert np.abs(got.astype(np.int64) - ref.astype(np.int64)).max() <= 1


def test_mesh_slabs_bitwise():
    import torch
    shape = (40, 20, 28)
    V, F = M.icosphere((19.5, 9.7, 13.9), 6.0, 2)
    state = OS.random_state(shape, seed=7, drho=0.02, umax=0.04, sneq=0.002)
    cfg = SolverConfig(nu=0.02)
    with Solver(SimGrid(shape), cfg) as s:
        s.set_mesh(V, F)
        s.set_moments(*state)
        s.step(3)
        ref = s.moments()
    plans = partition(shape[0], 3, True)
    solvers = []
    for p in plans:
        sl = slice(p.x0, p.x0 + p.nx)
        sv = Solver(SimGrid((p.nx,) + shape[1:]), cfg, slab=Slab(p.x0, shape[0], True, True))
        sv.set_mesh(V, F)
        sv.set_moments(state[0][sl], state[1][:, sl], state[2][:, sl])
        solvers.append(sv)
    for _ in range(3):
        views = []
        for sv in solvers:
            ptrs, nb = sv.halo_planes()
            views.append([device_view(q, nb) for q in ptrs])
        for p, v in zip(plans, views):
            v[2].copy_(views[p.lo][1])
            v[3].copy_(views[p.hi][0])
        torch.cuda.synchronize()
        for sv in solvers:
            sv.step(1)
    got = [sv.moments() for sv in solvers]
    for sv in solvers:
        sv.close()
    for k in range(3):
        assert np.array_equal(np.concatenate([g[k] for g in got], axis=-3), ref[k])


@pytest.mark.parametrize("precision", ["fp32", "q16"])
def test_d3q19_mesh_links_and_step(precision):
    """D3Q19 with a triangle mesh (the paper's Fig. 3 D3Q19 / D3Q27 comparison): the cut-link table
    tests the 18 D3Q19 links only (bit-exact vs the oracle), and one step with the Eq.-8 boundary
    populations (D3Q19 weights) matches the oracle: fp32 per-moment <= 1e-5, q16 within 1 LSB."""
    from oracle import lattice as OL
    shape = (24, 20, 28)
    V, F, state = _scene(shape)
    cells, masks, t, tri = M.cut_links(V, F, shape, OL.D3Q19)
    assert masks.max() < (1 << 19)
    cfg = SolverConfig(nu=0.02, lattice="D3Q19", precision=precision)
    with Solver(SimGrid(shape), cfg) as s:
        s.set_mesh(V, F)
        gc, gm, gt, gtri = s.cut_links()
        assert np.array_equal(gc, cells) and np.array_equal(gm, masks)
        assert np.array_equal(np.isnan(gt), np.isnan(t)) and np.array_equal(gt[~np.isnan(gt)], t[~np.isnan(t)])
        if precision == "fp32":
            s.set_moments(*state)
            st = s.step(1)
            got = s.moments()
        else:
            w0, _ = codec.encode_state(state[0], state[1], neq_decompose(*state))
            s.codes = w0
            s.step(1)
            got = codec.unpack(s.codes)
    if precision == "fp32":
        r, m, sx, Fs, Ts = M.step_with_mesh(*state, cfg.tau, cells, t, lat=OL.D3Q19)
        for g, ref in zip(got, (r, m, sx)):
            assert np.linalg.norm(g - ref) / np.linalg.norm(ref) <= 1e-5
        np.testing.assert_allclose(st.force, Fs, rtol=1e-4, atol=1e-7)
    else:
        from oracle.moments import neq_recompose
        rho, mom, sn = codec.decode_state(w0)
        r, m, sx, _, _ = M.step_with_mesh(rho, mom, neq_recompose(rho, mom, sn), cfg.tau, cells, t, lat=OL.D3Q19)
        ref = codec.unpack(codec.encode_state(r, m, neq_decompose(r, m, sx))[0])
        assert np.abs(got.astype(np.int64) - ref.astype(np.int64)).max() <= 1


@pytest.mark.parametrize("precision", ["fp32", "q16"])
def test_mesh_with_wall_faces(precision):
    """A triangle mesh next to wall faces (a body near the floor of a channel): the cut-link list is
    the union of the mesh-cut and the wall-adjacent cells; wall links bounce back (and win over a
    mesh hit on the same link), mesh links take Eq. 8.  fp32 per-moment <= 1e-5 with the momentum
    exchange on the mesh; q16 within 1 LSB (round 1 dropped the wall links silently here)."""
    shape = (24, 20, 28)
    V, F = M.icosphere((11.3, 9.7, 3.9), 4.2, 2)          # the sphere's bottom 0.3 cell above the z = 0 layer
    state = OS.random_state(shape, seed=6, drho=0.02, umax=0.04, sneq=0.002)
    bc = {"x": ("periodic", "periodic"), "y": ("wall", "wall"), "z": ("wall", "wall")}
    obc = OS.BC(x=bc["x"], y=bc["y"], z=bc["z"])
    cells, masks, t, _ = M.cut_links(V, F, shape)
    cfg = SolverConfig(nu=0.02, bc=bc, precision=precision)
    with Solver(SimGrid(shape), cfg) as s:
        s.set_mesh(V, F)
        gc, gm, gt, _ = s.cut_links()
        assert np.array_equal(gc, cells) and np.array_equal(gm, masks)    # the mesh part, unchanged
        if precision == "fp32":
            s.set_moments(*state)
            st = s.step(1)
            got = s.moments()
        else:
            w0, _ = codec.encode_state(state[0], state[1], neq_decompose(*state))
            s.codes = w0
            s.step(1)
            got = codec.unpack(s.codes)
    if precision == "fp32":
        r, m, sx, Fs, Ts = M.step_with_mesh(*state, cfg.tau, cells, t, bc=obc)
        for g, ref in zip(got, (r, m, sx)):
            assert np.linalg.norm(g - ref) / np.linalg.norm(ref) <= 1e-5
        np.testing.assert_allclose(st.force, Fs, rtol=1e-4, atol=1e-7)
    else:
        from oracle.moments import neq_recompose
        rho, mom, sn = codec.decode_state(w0)
        r, m, sx, _, _ = M.step_with_mesh(rho, mom, neq_recompose(rho, mom, sn), cfg.tau, cells, t, bc=obc)
        ref = codec.unpack(codec.encode_state(r, m, neq_decompose(r, m, sx))[0])
        assert np.abs(got.astype(np.int64) - ref.astype(np.int64)).max() <= 1
