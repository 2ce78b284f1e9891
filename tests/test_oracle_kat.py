"""Known-answer and invariant tests of the oracle (SPEC.md examples and acceptance criteria)."""

import numpy as np
import pytest

from oracle import codec
from oracle import collision as OC
from oracle import lattice as OL
from oracle import moments as OM
from oracle import step as OS


def test_rest_state_reconstructs_weights():
    # rho=1, u=0, S=0 -> f_i = w_i
    f = OM.reconstruct_distributions(np.ones(1), np.zeros((3, 1)), np.zeros((6, 1)))
    np.testing.assert_allclose(f[:, 0], OL.W, rtol=0, atol=1e-16)


def test_round_trip_1e12():
    # reconstruct -> extract identity < 1e-12 over random valid sets
    rng = np.random.default_rng(5)
    n = 1000
    rho = rng.uniform(0.8, 1.5, n)
    u = rng.uniform(-1, 1, (3, n))
    u *= 0.4 * rng.uniform(0, 1, n) / np.maximum(np.linalg.norm(u, axis=0), 1e-12)
    mom = rho * u
    st = OM.neq_recompose(rho, mom, rng.uniform(-0.1, 0.1, (6, n)))
    r, m, s = OM.moments_from_distributions(OM.reconstruct_distributions(rho, mom, st))
    assert np.abs(r - rho).max() < 1e-12
    assert np.abs(m - mom).max() < 1e-12
    assert np.abs(s - st).max() < 1e-12


def test_collision_tau1_fixed_point():
    # tau=1, F=0 -> S_ab = u_a u_b (incl. diagonal in 3D); rho conserved
    rng = np.random.default_rng(1)
    rho = rng.uniform(0.9, 1.1, 50)
    mom = rho * rng.uniform(-0.1, 0.1, (3, 50))
    st = OM.neq_recompose(rho, mom, rng.uniform(-0.01, 0.01, (6, 50)))
    r, m, s = OC.collide_moments(rho, mom, st, None, 1.0)
    assert np.array_equal(r, rho)
    np.testing.assert_allclose(s, OM.outer_voigt(m) / r, atol=1e-15)


def test_uniform_rest_is_fixed_point():
    shape = (8, 8, 8)
    r, m, s = OS.fluid_step(np.ones(shape), np.zeros((3,) + shape), np.zeros((6,) + shape), 0.6)
    assert np.abs(r - 1).max() < 1e-15 and np.abs(m).max() < 1e-15 and np.abs(s).max() < 1e-15


def test_uniform_flow_invariant():
    shape = (8, 8, 8)
    u = np.array([0.05, -0.02, 0.03])
    rho = np.ones(shape)
    mom = np.broadcast_to(u[:, None, None, None], (3,) + shape).copy()
    st = OM.neq_recompose(rho, mom, np.zeros((6,) + shape))
    r, m, s = OS.run(rho, mom, st, 0.6, 3)
    np.testing.assert_allclose(m, mom, atol=1e-15)
    np.testing.assert_allclose(r, rho, atol=1e-15)


def test_mass_momentum_conservation_periodic():
    # SPEC.md:493-494 (drift < 1e-10 relative)
    r, m, s = OS.random_state((12, 12, 12), seed=3, drho=0.05, umax=0.05, sneq=0.005)
    M0, P0 = r.sum(), m.sum(axis=(1, 2, 3))
    r, m, s = OS.run(r, m, s, 0.56, 20)
    assert abs(r.sum() - M0) / M0 < 1e-12
    np.testing.assert_allclose(m.sum(axis=(1, 2, 3)), P0, atol=1e-11)


def test_bounce_back_conserves_mass_in_closed_box():
    shape = (10, 8, 8)
    bc = OS.BC(x=("wall", "wall"), y=("wall", "wall"), z=("wall", "wall"))
    mask = np.zeros(shape, dtype=np.uint8)
    mask[4:6, 3:5, 3:5] = 1
    r, m, s = OS.random_state(shape, seed=4, drho=0.05, umax=0.05, sneq=0.005)
    fl = ~mask.astype(bool)
    M0 = r[fl].sum()
    for _ in range(5):
        r, m, s = OS.fluid_step(r, m, s, 0.6, bc, None, mask)
    assert abs(r[fl].sum() - M0) < 1e-11


# ------------------------------------------------------------------ codec

def test_quantize_known_answers():
    assert codec.quantize(1.0, 0.8, 1.5, 16)[0] == 18724
    assert codec.quantize(0.8, 0.8, 1.5, 16)[0] == 0
    assert codec.quantize(1.5, 0.8, 1.5, 16)[0] == 65535


def test_pack_layout():
    codes = np.array([0xFFFF, 0x0000] * 5, dtype=np.uint32).reshape(10, 1)
    w = codec.pack(codes)
    assert w.shape == (5, 1) and np.all(w == 0x0000FFFF)
    rng = np.random.default_rng(0)
    c = rng.integers(0, 65536, (10, 100)).astype(np.uint32)
    assert np.array_equal(codec.unpack(codec.pack(c)), c)


def test_round_trip_error_bound():
    rng = np.random.default_rng(2)
    for k in range(10):
        lo, hi = codec.DEFAULT_MIN[k], codec.DEFAULT_MAX[k]
        m = rng.uniform(lo, hi, 10000)
        q, _ = codec.quantize(m, lo, hi, 16)
        err = np.abs(codec.dequantize(q, lo, hi, 16) - m)
        assert err.max() <= (hi - lo) / (2 * 65535) * (1 + 1e-12)


def test_words_per_node_is_half_of_fp32():
    # 5 u32 words vs 10 float32 per node
    assert codec.NWORDS * 4 * 2 == codec.NCOMP * 4


def test_dither_unbiased():
    # 1e6 samples, mean error within 3 sigma of 0
    cells = np.arange(1_000_000, dtype=np.int64)
    noise = codec.dither_noise(cells, 3, 11)
    lo, hi = 0.8, 1.5
    m = 1.0 + 1e-6
    q, _ = codec.quantize(np.full(cells.size, m), lo, hi, 16, noise[0])
    err = codec.dequantize(q, lo, hi, 16) - m
    step = (hi - lo) / 65535
    sigma = step / np.sqrt(12)
    assert abs(err.mean()) < 3 * sigma / np.sqrt(cells.size)
    assert np.all(noise >= -0.5) and np.all(noise < 0.5)
    # every component's noise is zero-mean uniform (std 1/sqrt(12)) and the components of a cell
    # are uncorrelated (words 1..4 are multiply-xorshift bijections of the cell hash)
    n = noise.reshape(10, -1)
    assert np.all(np.abs(n.mean(axis=1)) < 4 / np.sqrt(12 * n.shape[1]))
    assert np.allclose(n.std(axis=1), 1 / np.sqrt(12), rtol=2e-3)
    c = np.corrcoef(n)
    assert np.abs(c - np.eye(10)).max() < 5e-3
    # and neighbouring cells / steps are uncorrelated
    assert abs(np.corrcoef(n[0, :-1], n[0, 1:])[0, 1]) < 5e-3
    assert abs(np.corrcoef(n[0], codec.dither_noise(cells, 4, 11)[0])[0, 1]) < 5e-3


def test_saturation_counts_exact():
    m = np.array([0.79, 0.8, 1.0, 1.5, 1.51, 2.0])
    q, sat = codec.quantize(m, 0.8, 1.5, 16)
    assert sat.tolist() == [True, False, False, False, True, True]
    assert q.tolist()[0] == 0 and q.tolist()[-1] == 65535


def test_q16_step_runs_and_is_finite():
    r, m, s = OS.random_state((8, 8, 8), seed=1, drho=0.05, umax=0.05, sneq=0.005)
    w, _ = codec.encode_state(r, m, OM.neq_decompose(r, m, s))
    w2, sat = OS.fluid_step_q16(w, 0.6, 0, dither=True, seed=3)
    assert w2.shape == (5, 8, 8, 8) and sat.sum() == 0


# ------------------------------------------------------------------ mask -> lists

def brute_force_lists(mask, bc):
    nx, ny, nz = mask.shape
    cells, masks = [], []
    def solid(x, y, z):
        for ax, (v, n, kinds) in enumerate(((z, nz, bc.z), (y, ny, bc.y))):
            pass
        # z padded last -> checked first
        if z < 0 or z >= nz:
            if bc.z[0 if z < 0 else 1] == "wall":
                return True
            z %= nz
        if y < 0 or y >= ny:
            if bc.y[0 if y < 0 else 1] == "wall":
                return True
            y %= ny
        if x < 0 or x >= nx:
            k = bc.x[0 if x < 0 else 1]
            if k == "wall":
                return True
            if k in ("inflow", "outflow"):
                return False
            x %= nx
        return bool(mask[x, y, z])
    for x in range(nx):
        for y in range(ny):
            for z in range(nz):
                if mask[x, y, z]:
                    continue
                lm = 0
                for i in range(1, 27):
                    c = OL.C[i]
                    if solid(x - c[0], y - c[1], z - c[2]):
                        lm |= 1 << i
                if lm:
                    cells.append((x * ny + y) * nz + z)
                    masks.append(lm)
    return np.array(cells, dtype=np.int64), np.array(masks, dtype=np.uint32)


@pytest.mark.parametrize("bc", [OS.BC(),
                                OS.BC(x=("inflow", "outflow"), z=("wall", "wall")),
                                OS.BC(x=("wall", "wall"), y=("wall", "periodic")[:1] * 2)])
def test_boundary_lists_match_brute_force(bc):
    from paper_2602_05295_b200.geometry import sphere_mask
    mask = sphere_mask((9, 8, 8), (4, 3.5, 4), 2.5)
    mask[0, 0, 0] = 1   # a solid cell on the domain corner exercises the wrap rules
    cells, masks = OS.boundary_lists(mask, bc)
    c2, m2 = brute_force_lists(mask, bc)
    assert np.array_equal(cells, c2)
    assert np.array_equal(masks, m2)
