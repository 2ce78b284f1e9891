"""Parity of the CUDA path (libhlbm.so on cuda:0) with the reference and the oracle.

Tolerances (stated per the north star):
  * fp32: per-moment relative L2 error ||m_gpu - m_ref|| / ||m_ref|| <= 1e-5 for each of the
    reference's moments rho, rho u, rho S (MomentSet fields, moments.py:136-172).
  * q16: code difference against the oracle's own quantized path (decode -> float64 step ->
    encode, oracle/step.py:fluid_step_q16) <= 1 LSB after one step; <= 8 LSB after 50 steps.
  * boundary lists / link masks: bit-exact.
"""

from pathlib import Path

import numpy as np
import pytest

from oracle import codec
from oracle import step as OS
from oracle.moments import neq_decompose, neq_recompose
from paper_2602_05295_b200 import QuantSpec, SimGrid, Solver, SolverConfig
from paper_2602_05295_b200.geometry import sphere_mask

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"
FP32_TOL = 1e-5


def moment_errors(got, ref, sel=None):
    out = []
    for g, r in zip(got, ref):
        if sel is not None:
            g, r = g[..., sel], r[..., sel]
        out.append(float(np.linalg.norm(g - r) / np.linalg.norm(r)))
    return out   # [rho, mom, stress]


def run_gpu(state, cfg, steps, mask=None, reference_kernel=False):
    shape = state[0].shape
    with Solver(SimGrid(shape, mask), cfg) as s:
        s.set_moments(*state)
        if reference_kernel:
            s.step_reference(steps)
        else:
            s.step(steps)
        return s.moments()


def test_golden_step16_matches_reference():
    z = np.load(G / "step16.npz")
    cfg = SolverConfig(nu=(float(z["tau"]) - 0.5) / 3)
    got = run_gpu((z["rho"], z["mom"], z["stress"]), cfg, 1)
    err = moment_errors(got, (z["rho1"], z["mom1"], z["stress1"]))
    assert max(err) <= FP32_TOL, err


def test_golden_tgv32_matches_reference():
    z = np.load(G / "tgv32.npz")
    cfg = SolverConfig(nu=(float(z["tau"]) - 0.5) / 3)
    got = run_gpu((z["rho0"], z["mom0"], z["stress0"]), cfg, int(z["steps"]))
    err = moment_errors(got, (z["rho"], z["mom"], z["stress"]))
    assert max(err) <= FP32_TOL, err


def test_tgv64_200_steps_config1():
    """BASELINE config 1: TGV 64^3, fp32, periodic, 200 steps vs the oracle."""
    state = OS.taylor_green(64)
    cfg = SolverConfig(nu=0.01)
    got = run_gpu(state, cfg, 200)
    ref = OS.run(*state, cfg.tau, 200)
    err = moment_errors(got, ref)
    print("TGV64x200 per-moment rel errors (rho, mom, stress):", err)
    assert max(err) <= FP32_TOL, err


@pytest.mark.parametrize("shape,steps", [((16, 16, 16), 1), ((20, 30, 68), 3), ((7, 40, 132), 2)])
@pytest.mark.parametrize("kernel", ["interior", "pull"])
def test_random_states(shape, steps, kernel):
    state = OS.random_state(shape, seed=1, drho=0.05, umax=0.08, sneq=0.005)
    cfg = SolverConfig(nu=0.02)
    got = run_gpu(state, cfg, steps, reference_kernel=(kernel == "pull"))
    ref = OS.run(*state, cfg.tau, steps)
    err = moment_errors(got, ref)
    assert max(err) <= FP32_TOL, err


def test_body_force():
    state = OS.random_state((12, 16, 24), seed=2, drho=0.05, umax=0.05, sneq=0.005)
    F = (2e-5, -1e-5, 3e-5)
    cfg = SolverConfig(nu=0.02, force=F)
    got = run_gpu(state, cfg, 3)
    ref = OS.run(*state, cfg.tau, 3, force=np.array(F))
    err = moment_errors(got, ref)
    assert max(err) <= FP32_TOL, err


def _channel_state(shape, mask, u0):
    rho = np.ones(shape)
    u = np.zeros((3,) + shape)
    u[0] = u0
    u[:, mask.astype(bool)] = 0
    mom = rho * u
    return rho, mom, neq_recompose(rho, mom, np.zeros((6,) + shape))


@pytest.mark.parametrize("bcname", ["channel", "closed", "walls_yz"])
def test_solids_and_domain_bcs(bcname):
    shape = (40, 24, 28)
    mask = sphere_mask(shape, (14, 11.5, 13.5), 5)
    if bcname == "channel":
        bc = {"x": ("inflow", "outflow"), "y": ("periodic", "periodic"), "z": ("wall", "wall")}
    elif bcname == "closed":
        bc = {"x": ("wall", "wall"), "y": ("wall", "wall"), "z": ("wall", "wall")}
    else:
        bc = {"x": ("periodic", "periodic"), "y": ("wall", "wall"), "z": ("wall", "wall")}
    cfg = SolverConfig(nu=0.02, bc=bc, u_in=(0.05, 0, 0))
    obc = OS.BC(x=bc["x"], y=bc["y"], z=bc["z"], u_in=(0.05, 0, 0))
    cells, masks = OS.boundary_lists(mask, obc)
    state = _channel_state(shape, mask, 0.05 if bcname == "channel" else 0.02)
    with Solver(SimGrid(shape, mask), cfg) as s:
        gc, gm = s.boundary()
        assert np.array_equal(gc, cells)          # bit-exact lists and link masks
        assert np.array_equal(gm, masks)
        s.set_moments(*state)
        st = s.step(5)
        got = s.moments()
    ref = state
    for _ in range(5):
        ref = OS.fluid_step(*ref, cfg.tau, obc, None, mask)
    fl = ~mask.astype(bool)
    err = moment_errors(got, ref, fl)
    assert max(err) <= FP32_TOL, err
    assert st.mass == pytest.approx(ref[0][fl].sum(), rel=1e-7)
    np.testing.assert_allclose(st.momentum, ref[1][:, fl].sum(axis=1), atol=1e-6 * fl.sum())
    # solid cells hold the rest state
    assert np.all(got[0][~fl] == 1.0) and np.all(got[1][:, ~fl] == 0.0)


def test_stats_match_oracle_sums():
    state = OS.random_state((16, 20, 24), seed=5, drho=0.05, umax=0.08, sneq=0.005)
    cfg = SolverConfig(nu=0.02)
    with Solver(SimGrid((16, 20, 24)), cfg) as s:
        s.set_moments(*state)
        st = s.step(2)
    ref = OS.run(*state, cfg.tau, 2)
    assert st.mass == pytest.approx(ref[0].sum(), rel=1e-7)
    np.testing.assert_allclose(st.momentum, ref[1].sum(axis=(1, 2, 3)), atol=1e-4)
    assert st.max_u == pytest.approx(np.sqrt(((ref[1] / ref[0]) ** 2).sum(0)).max(), rel=1e-5)
    assert st.n_fluid == 16 * 20 * 24


def test_divergence_raises_floating_point_error():
    shape = (8, 8, 8)
    rho = np.ones(shape)
    mom = np.zeros((3,) + shape)
    mom[0] = 0.95
    st = neq_recompose(rho, mom, np.zeros((6,) + shape))
    with Solver(SimGrid(shape), SolverConfig(nu=0.02)) as s:
        s.set_moments(rho, mom, st)
        with pytest.raises(FloatingPointError):
            s.step(1)


@pytest.mark.parametrize("precision", ["fp32", "q16"])
def test_divergence_report_names_step_and_node(precision):
    """the divergence report carries the step and the node -- here one fast spot in a
    fluid at rest; the locator scan runs only after a step reported divergence."""
    shape = (12, 8, 16)
    rho = np.ones(shape)
    mom = np.zeros((3,) + shape)
    blk = (slice(6, 9), slice(2, 5), slice(9, 12))     # a 3^3 block centred on (7, 3, 10): rho 0.8,
    rho[blk] = 0.8                                     # j = (0.6, 0.6, 0), |u| = 1.06 -- inside the
    mom[0][blk] = 0.6                                  # 16-bit ranges, so both precisions store it
    mom[1][blk] = 0.6
    st = neq_recompose(rho, mom, np.zeros((6,) + shape))
    with Solver(SimGrid(shape), SolverConfig(nu=0.02, precision=precision)) as s:
        s.set_moments(rho, mom, st)
        with pytest.raises(FloatingPointError) as e:
            s.step(1)
        msg = str(e.value)
    print(msg)
    assert "at step" in msg and "node (" in msg
    x, y, z = (int(v) for v in msg.split("node (")[1].split(")")[0].split(","))
    assert abs(x - 7) <= 1 and abs(y - 3) <= 1 and abs(z - 10) <= 1


def test_moment_set_accessor():
    state = OS.random_state((8, 8, 8), seed=6, drho=0.05, umax=0.05, sneq=0.005)
    with Solver(SimGrid((8, 8, 8)), SolverConfig(nu=0.02)) as s:
        s.set_moments(*state)
        ms = s.moment_set(3, 4, 5)
        np.testing.assert_allclose(ms.rho, state[0][3, 4, 5], rtol=1e-6)
        np.testing.assert_allclose(ms.velocity, state[1][:, 3, 4, 5] / state[0][3, 4, 5], atol=1e-7)
        with pytest.raises(ValueError):
            s.set_moments(-state[0], state[1], state[2])      # rho <= 0 (moments.py:147)


# ------------------------------------------------------------------ 16-bit path

def _q16_case(shape, seed, quant, steps, dither=False, tau=0.56):
    state = OS.random_state(shape, seed=seed, drho=0.05, umax=0.05, sneq=0.005)
    w0, _ = codec.encode_state(state[0], state[1], neq_decompose(*state),
                               np.array(quant.mmin), np.array(quant.mmax), np.array(quant.bits))
    cfg = SolverConfig(nu=(tau - 0.5) / 3, precision="q16", quant=quant, seed=7)
    with Solver(SimGrid(shape), cfg) as s:
        s.codes = w0
        for _ in range(steps):
            s.step(1)
        got = s.codes
    ref = w0
    for k in range(steps):
        ref, _ = OS.fluid_step_q16(ref, cfg.tau, k, mmin=np.array(quant.mmin), mmax=np.array(quant.mmax),
                                   bits=np.array(quant.bits), dither=dither, seed=7)
    return np.abs(codec.unpack(got).astype(np.int64) - codec.unpack(ref).astype(np.int64))


@pytest.mark.parametrize("dither", [False, True])
def test_q16_one_step_within_1_lsb(dither):
    d = _q16_case((16, 24, 32), 2, QuantSpec(dither=dither), 1, dither)
    assert d.max() <= 1
    assert np.mean(d > 0) < 0.01


@pytest.mark.parametrize("preset", ["16/15", "14/13", "12/11"])
def test_q16_bit_presets_one_step(preset):
    d = _q16_case((12, 16, 32), 3, QuantSpec.preset(preset), 1)
    assert d.max() <= 1


def test_q16_fifty_steps_within_8_lsb():
    d = _q16_case((12, 20, 64), 4, QuantSpec(), 50)
    print("q16 50 steps: max LSB", d.max(), "mean", d.mean())
    assert d.max() <= 8


def test_q16_saturation_counts():
    shape = (12, 16, 32)
    q = QuantSpec(mmin=(0.995,) + QuantSpec().mmin[1:], mmax=(1.005,) + QuantSpec().mmax[1:])
    state = OS.random_state(shape, seed=8, drho=0.004, umax=0.05, sneq=0.002)
    w0, _ = codec.encode_state(state[0], state[1], neq_decompose(*state), np.array(q.mmin), np.array(q.mmax))
    cfg = SolverConfig(nu=0.02, precision="q16", quant=q)
    with Solver(SimGrid(shape), cfg) as s:
        s.codes = w0
        st = s.step(1)
    rho, mom, sneq = codec.decode_state(w0, np.array(q.mmin), np.array(q.mmax))
    r, m, sn = OS.fluid_step(rho, mom, neq_recompose(rho, mom, sneq), cfg.tau)
    lo, hi = q.mmin[0], q.mmax[0]
    clear = np.count_nonzero((r < lo - 1e-6) | (r > hi + 1e-6))
    loose = np.count_nonzero((r < lo + 1e-6) | (r > hi - 1e-6))
    assert clear > 0
    assert clear <= st.saturation[0] <= loose
    assert np.all(st.saturation[1:] == 0)


@pytest.mark.parametrize("bcname", ["channel", "closed"])
def test_percell_step_matches_oracle_and_split(bcname):
    """The per-cell gather step (one kernel, solid links inline, same storage cut) against the
    oracle (fp32 tolerance) and against the split scheme (interior kernel + compacted boundary
    kernel): the two schemes compute the same step."""
    shape = (40, 24, 28)
    mask = sphere_mask(shape, (14, 11.5, 13.5), 5)
    if bcname == "channel":
        bc = {"x": ("inflow", "outflow"), "y": ("periodic", "periodic"), "z": ("wall", "wall")}
    else:
        bc = {"x": ("wall", "wall"), "y": ("wall", "wall"), "z": ("wall", "wall")}
    cfg = SolverConfig(nu=0.02, bc=bc, u_in=(0.05, 0, 0))
    obc = OS.BC(x=bc["x"], y=bc["y"], z=bc["z"], u_in=(0.05, 0, 0))
    state = _channel_state(shape, mask, 0.05)
    res = {}
    for scheme in ("fused", "split"):
        with Solver(SimGrid(shape, mask), cfg) as s:
            s.set_moments(*state)
            st = s.step_percell(5) if scheme == "fused" else s.step(5)
            res[scheme] = (s.moments(), st)
    ref = state
    for _ in range(5):
        ref = OS.fluid_step(*ref, cfg.tau, obc, None, mask)
    fl = ~mask.astype(bool)
    assert max(moment_errors(res["fused"][0], ref, fl)) <= FP32_TOL
    assert max(moment_errors(res["fused"][0], res["split"][0], fl)) <= FP32_TOL
    assert np.all(res["fused"][0][0][~fl] == 1.0) and np.all(res["fused"][0][1][:, ~fl] == 0.0)
    assert res["fused"][1].mass == pytest.approx(res["split"][1].mass, rel=1e-7)


def test_percell_q16_matches_split_within_1_lsb():
    shape = (32, 20, 24)
    mask = sphere_mask(shape, (12, 9.5, 11.5), 4)
    bc = {"x": ("inflow", "outflow"), "y": ("periodic", "periodic"), "z": ("periodic", "periodic")}
    cfg = SolverConfig(nu=0.02, bc=bc, u_in=(0.05, 0, 0), precision="q16", quant=QuantSpec())
    state = _channel_state(shape, mask, 0.05)
    words = {}
    for scheme in ("fused", "split"):
        with Solver(SimGrid(shape, mask), cfg) as s:
            s.set_moments(*state)
            if scheme == "fused":
                s.step_percell(1)
            else:
                s.step(1)
            words[scheme] = s.codes
    d = np.abs(codec.unpack(words["fused"]).astype(np.int64) - codec.unpack(words["split"]).astype(np.int64))
    assert d.max() <= 1


# ------------------------------------------------------------------------------------ D3Q19
def test_d3q19_matches_reference_golden():
    """D3Q19 (per-cell fused kernel) against the reference's own D3Q19 composition."""
    z = np.load(G / "d3q19.npz")
    cfg = SolverConfig(nu=(float(z["tau"]) - 0.5) / 3, lattice="D3Q19")
    for steps, key in ((1, "1"), (3, "3")):
        got = run_gpu((z["rho"], z["mom"], z["stress"]), cfg, steps)
        err = moment_errors(got, (z["rho" + key], z["mom" + key], z["stress" + key]))
        assert max(err) <= FP32_TOL, (steps, err)


@pytest.mark.parametrize("bcname", ["channel", "closed"])
def test_d3q19_solids_and_bcs(bcname):
    from oracle import lattice as OL
    shape = (24, 20, 28)
    mask = sphere_mask(shape, (10, 9.5, 13.5), 4)
    if bcname == "channel":
        bc = {"x": ("inflow", "outflow"), "y": ("periodic", "periodic"), "z": ("wall", "wall")}
    else:
        bc = {"x": ("wall", "wall"), "y": ("wall", "wall"), "z": ("wall", "wall")}
    cfg = SolverConfig(nu=0.02, bc=bc, u_in=(0.05, 0, 0), lattice="D3Q19")
    obc = OS.BC(x=bc["x"], y=bc["y"], z=bc["z"], u_in=(0.05, 0, 0))
    cells, masks = OS.boundary_lists(mask, obc, OL.D3Q19)
    state = _channel_state(shape, mask, 0.05)
    with Solver(SimGrid(shape, mask), cfg) as s:
        gc, gm = s.boundary()
        assert np.array_equal(gc, cells) and np.array_equal(gm, masks)   # 19-link masks, bit-exact
        s.set_moments(*state)
        st = s.step(4)
        got = s.moments()
    ref = OS.run(*state, cfg.tau, 4, obc, None, mask, OL.D3Q19)
    fl = ~mask.astype(bool)
    assert max(moment_errors(got, ref, fl)) <= FP32_TOL
    assert st.mass == pytest.approx(ref[0][fl].sum(), rel=1e-7)


def test_d3q19_q16_within_1_lsb():
    from oracle import lattice as OL
    shape = (12, 16, 20)
    state = OS.random_state(shape, seed=4, drho=0.05, umax=0.05, sneq=0.005)
    cfg = SolverConfig(nu=0.02, precision="q16", quant=QuantSpec(), lattice="D3Q19")
    words0, _ = codec.encode_state(state[0], state[1], neq_decompose(*state))
    with Solver(SimGrid(shape), cfg) as s:
        s.codes = words0
        s.step(1)
        words = s.codes
    ref, _ = OS.fluid_step_q16(words0, cfg.tau, 0, lat=OL.D3Q19)
    d = np.abs(codec.unpack(words).astype(np.int64) - codec.unpack(ref).astype(np.int64))
    assert d.max() <= 1


@pytest.mark.parametrize("precision", ["fp32", "q16"])
@pytest.mark.parametrize("bcname", ["periodic", "channel", "sphere"])
def test_d3q19_interior_kernel_matches_per_cell(precision, bcname):
    """D3Q19 steps run the interior kernel with two-chain streaming (216 w = prod(4,1,1) +
    prod(2,-1,-1)) plus the compacted 19-link kernels for solids; they match the per-cell D3Q19
    kernel (step_percell) and the oracle: fp32 per-moment relative error <= 1e-5, q16 codes within
    1 LSB."""
    from oracle import lattice as OL
    shape = (20, 33, 68)   # ragged tiles in y and z
    bc = None if bcname == "periodic" else {"x": ("inflow", "outflow"), "y": ("periodic", "periodic"),
                                            "z": ("wall", "wall") if bcname == "sphere" else ("periodic", "periodic")}
    mask = sphere_mask(shape, (9, 16.5, 33.5), 5) if bcname == "sphere" else None
    kw = {} if bc is None else {"bc": bc, "u_in": (0.05, 0, 0)}
    cfg = SolverConfig(nu=0.02, lattice="D3Q19", precision=precision, **kw)
    state = OS.random_state(shape, seed=6, drho=0.05, umax=0.05, sneq=0.005)
    if mask is not None:
        state = _channel_state(shape, mask, 0.05)
    res = {}
    for kind in ("interior", "per_cell"):
        with Solver(SimGrid(shape, mask), cfg) as s:
            if precision == "q16":
                s.codes = codec.encode_state(state[0], state[1], neq_decompose(*state))[0]
            else:
                s.set_moments(*state)
            s.step(2) if kind == "interior" else s.step_percell(2)
            res[kind] = s.codes if precision == "q16" else s.moments()
    if precision == "q16":
        d = np.abs(codec.unpack(res["interior"]).astype(np.int64) - codec.unpack(res["per_cell"]).astype(np.int64))
        assert d.max() <= 1
    else:
        fl = None if mask is None else ~mask.astype(bool)
        assert max(moment_errors(res["interior"], res["per_cell"], fl)) <= FP32_TOL
        if bc is None:
            ref = OS.run(*state, cfg.tau, 2, OS.BC(), None, None, OL.D3Q19)
            assert max(moment_errors(res["interior"], ref)) <= FP32_TOL


@pytest.mark.parametrize("shape", [(1, 1, 4), (3, 1, 8), (2, 3, 4), (1, 30, 8), (3, 2, 124), (2, 15, 68)])
@pytest.mark.parametrize("kernel", ["split", "fused"])
def test_tiny_and_ragged_grids(shape, kernel):
    """Degenerate and ragged periodic grids (single-cell rows/planes, partial tiles): both
    ghost rows / columns of a one-cell axis carry the periodic image."""
    state = OS.random_state(shape, seed=1, drho=0.05, umax=0.05, sneq=0.005)
    cfg = SolverConfig(nu=0.02)
    with Solver(SimGrid(shape), cfg) as s:
        s.set_moments(*state)
        s.step(2) if kernel == "split" else s.step_percell(2)
        got = s.moments()
    ref = OS.run(*state, cfg.tau, 2)
    err = moment_errors(got, ref)
    assert max(err) <= FP32_TOL, err


def component_errors(got, ref, sel=None):
    """Per component plane: relative L2 against the plane's own norm, against its moment's norm,
    and max |err| / (max - min) of the reference plane."""
    names = ["rho", "mx", "my", "mz", "Sxx", "Sxy", "Sxz", "Syy", "Syz", "Szz"]
    gp = [got[0]] + list(got[1]) + list(got[2])
    rp = [ref[0]] + list(ref[1]) + list(ref[2])
    mnorm = [np.linalg.norm(ref[0])] + [np.linalg.norm(ref[1])] * 3 + [np.linalg.norm(ref[2])] * 6
    out = {}
    for n, g, r, mn in zip(names, gp, rp, mnorm):
        if sel is not None:
            g, r = g[sel], r[sel]
        e = g - r
        out[n] = (float(np.linalg.norm(e) / np.linalg.norm(r)), float(np.linalg.norm(e) / mn),
                  float(np.abs(e).max() / (r.max() - r.min())))
    return out


@pytest.mark.parametrize("case", ["tgv64_200", "random_20"])
def test_per_component_errors(case):
    """Per-component-plane view of the fp32 error beside the per-moment metric.  Bound: every
    component's L2 error relative to its MOMENT's norm <= 1e-5 (the north star's per-moment
    reading) and max-abs error <= 1e-5 of the component's range.  The plane-relative number is
    reported, not bounded: a plane whose norm is ~1e-2 of its tensor's (rho S_zz of a TGV with
    u_z = 0 is pure non-equilibrium) carries the tensor's fp32 rounding at 1e2x magnification --
    the same figure the fp32 NumPy restatement of the reference formula reaches."""
    if case == "tgv64_200":
        state, steps, nu = OS.taylor_green(64), 200, 0.01
    else:
        state, steps, nu = OS.random_state((24, 28, 32), seed=9, drho=0.05, umax=0.06, sneq=0.004), 20, 0.02
    cfg = SolverConfig(nu=nu)
    got = run_gpu(state, cfg, steps)
    ref = OS.run(*state, cfg.tau, steps)
    ce = component_errors(got, ref)
    for n, (pl, mo, mx) in ce.items():
        print(f"{case} {n:4s} plane-rel {pl:.2e}  moment-rel {mo:.2e}  maxabs/range {mx:.2e}")
    assert max(v[1] for v in ce.values()) <= FP32_TOL
    assert max(v[2] for v in ce.values()) <= FP32_TOL


@pytest.mark.parametrize("quant", ["14/13", "12/11", "custom16"])
def test_d3q19_interior_non_default_codecs(quant):
    """D3Q19 with a bit preset or custom 16-bit ranges runs the two-chain interior kernel (codec
    modes 0 / 1) -- it matches the per-cell D3Q19 kernel and the oracle's quantized step within 1 LSB."""
    from oracle import lattice as OL
    q = (QuantSpec(mmin=(0.9,) + QuantSpec().mmin[1:], mmax=(1.2,) + QuantSpec().mmax[1:]) if quant == "custom16"
         else QuantSpec.preset(quant))
    shape = (12, 20, 36)
    state = OS.random_state(shape, seed=5, drho=0.04, umax=0.05, sneq=0.004)
    mn, mx, bits = np.array(q.mmin), np.array(q.mmax), np.array(q.bits)
    w0, _ = codec.encode_state(state[0], state[1], neq_decompose(*state), mn, mx, bits)
    cfg = SolverConfig(nu=0.02, precision="q16", quant=q, lattice="D3Q19")
    res = {}
    for kind in ("interior", "per_cell"):
        with Solver(SimGrid(shape), cfg) as s:
            s.codes = w0
            s.step(1) if kind == "interior" else s.step_percell(1)
            res[kind] = s.codes
    ref, _ = OS.fluid_step_q16(w0, cfg.tau, 0, mmin=mn, mmax=mx, bits=bits, lat=OL.D3Q19)
    for kind, w in res.items():
        d = np.abs(codec.unpack(w).astype(np.int64) - codec.unpack(ref).astype(np.int64))
        assert d.max() <= 1, (kind, d.max())


@pytest.mark.parametrize("shape", [(6, 1, 64), (6, 2, 64), (8, 16, 64), (6, 31, 72), (10, 47, 40)])
@pytest.mark.parametrize("dither", [False, True])
def test_q16_no_stats_path_matches_stats_path_and_oracle(shape, dither):
    """The no-statistics interior kernels (step_async: the bench's hot path) skip the arithmetic
    of rows past the first row beyond ny in the last y tile; ny values around the
    15-row tile cover 1, 2, 16 and 31 rows.  Bitwise equal to the statistics path over 3 steps,
    1 LSB of the oracle after one."""
    quant = QuantSpec(dither=dither)
    state = OS.random_state(shape, seed=5, drho=0.05, umax=0.05, sneq=0.005)
    w0, _ = codec.encode_state(state[0], state[1], neq_decompose(*state))
    cfg = SolverConfig(nu=0.02, precision="q16", quant=quant, seed=7)
    out = {}
    for path in ("stats", "async"):
        with Solver(SimGrid(shape), cfg) as s:
            s.codes = w0
            for k in range(3):
                s.step(1) if path == "stats" else s.step_async(1)
                if k == 0:
                    out[path + "1"] = s.codes
            out[path] = s.codes
    assert np.array_equal(out["stats"], out["async"])
    ref, _ = OS.fluid_step_q16(w0, cfg.tau, 0, dither=dither, seed=7)
    d = np.abs(codec.unpack(out["async1"]).astype(np.int64) - codec.unpack(ref).astype(np.int64))
    assert d.max() <= 1
