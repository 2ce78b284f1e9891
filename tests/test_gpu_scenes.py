"""Obstacle-crop parity at the full BASELINE scene sizes (configs 3 and 4), where the float64 oracle
cannot step the whole grid: the GPU runs the full scene, a window containing the obstacle surface
(plus a halo of one cell per compared step) is read back, and the oracle steps that window with
the same restated rules (collision.py:137-194, moments.py:25-90, bounce-back SPEC.md:501, codec
SPEC.md:345-361).  Each oracle step consumes one halo layer, so after `steps` steps the inner
window is exact without any boundary assumption.

  * config 3: channel past a sphere, 512x256x256, centre (128,128,128), R = 32, u_in = 0.1,
    nu = 1e-4, inflow / outflow in x, periodic y / z;
  * config 4: procedural vehicle 1000x400x400, 16-bit + dither, u_in = 0.1, nu = 1e-5, inflow /
    outflow in x, periodic y, walls in z (ground and ceiling).
Tolerances: fp32 per-moment relative L2 <= 1e-5 (fluid cells of the window), 16-bit codes within
2 LSB after 2 steps (1 LSB per step, as for the 512^3 box crop).
"""

import numpy as np
import pytest

from oracle import codec
from oracle import lattice as OL
from oracle import step as OS
from oracle.moments import neq_decompose, neq_recompose
from paper_2602_05295_b200 import QuantSpec, SimGrid, Solver, SolverConfig
from paper_2602_05295_b200.geometry import sphere_mask, vehicle_mask

pytestmark = pytest.mark.gpu

WARM, STEPS, C = 12, 2, 24     # GPU steps before the window is read, compared steps, window edge


def crop_step(state, solid, tau):
    """One oracle step of a window whose outer layer is the halo: returns the state of the window
    shrunk by one cell per side (solid sources inside the window take half-way bounce-back)."""
    padded = np.concatenate([state[0][None], state[1], state[2]])
    nx, ny, nz = (d - 2 for d in solid.shape)
    link = np.zeros((27, nx, ny, nz), dtype=bool)
    for i in range(1, 27):
        cx, cy, cz = OL.D3Q27.C[i]
        link[i] = solid[1 - cx:1 - cx + nx, 1 - cy:1 - cy + ny, 1 - cz:1 - cz + nz]
    inner = solid[1:-1, 1:-1, 1:-1]
    link[:, inner] = False
    r, m, s = OS.step_padded(padded, tau, None, link)
    r[inner] = 1.0
    m[:, inner] = 0.0
    s[:, inner] = 0.0
    return (r, m, s), solid[1:-1, 1:-1, 1:-1]


def scene(name):
    if name == "config3":
        dims = (512, 256, 256)
        mask = sphere_mask(dims, (128, 128, 128), 32)
        bc = {"x": ("inflow", "outflow"), "y": ("periodic", "periodic"), "z": ("periodic", "periodic")}
        return dims, mask, bc, 1e-4, (84, 116, 104)      # window at the upstream pole, off-axis in z
    dims = (1000, 400, 400)
    mask = vehicle_mask(dims, seed=0)
    bc = {"x": ("inflow", "outflow"), "y": ("periodic", "periodic"), "z": ("wall", "wall")}
    # window on the nose surface: first solid cell along the centre line
    yc, zc = dims[1] // 2, int(np.argmax(mask[:, dims[1] // 2, :].any(axis=0)) + 30)
    xs = int(np.argmax(mask[:, yc, zc]))
    return dims, mask, bc, 1e-5, (xs - C // 2, yc - C // 2, zc - C // 2)


@pytest.mark.parametrize("precision", ["fp32", "q16"])
@pytest.mark.parametrize("name", ["config3", "config4"])
def test_obstacle_crop_parity(name, precision):
    dims, mask, bc, nu, (x0, y0, z0) = scene(name)
    h = STEPS
    win = (slice(x0 - h, x0 + C + h), slice(y0 - h, y0 + C + h), slice(z0 - h, z0 + C + h))
    solid = mask[win].astype(bool)
    assert solid.any() and not solid.all(), "the window must contain the obstacle surface"
    dither = name == "config4" and precision == "q16"
    cfg = SolverConfig(nu=nu, precision=precision, bc=bc, u_in=(0.1, 0.0, 0.0), seed=5,
                       quant=QuantSpec(dither=dither))
    with Solver(SimGrid(dims, mask), cfg) as s:
        s.init_modes(np.array([[0, 0, 0, 0.1, 0.0, 0.0, np.pi / 2]]))   # uniform u_in everywhere
        s.step(WARM)
        init = s.moments_box(x0 - h, C + 2 * h, y0 - h, C + 2 * h, z0 - h, C + 2 * h)
        step0 = s.steps
        s.step(STEPS)
        got = s.moments_box(x0, C, y0, C, z0, C)
    fl = ~solid[h:-h, h:-h, h:-h]
    if precision == "fp32":
        ref, sol = init, solid
        for _ in range(STEPS):
            ref, sol = crop_step(ref, sol, cfg.tau)
        err = [float(np.linalg.norm((g - r)[..., fl]) / np.linalg.norm(r[..., fl])) for g, r in zip(got, ref)]
        print(f"{name} fp32 crop per-moment rel err (rho, mom, stress): {err}")
        assert max(err) <= 1e-5, err
        assert np.all(got[0][~fl] == 1.0)
        return
    words = codec.encode_state(init[0], init[1], neq_decompose(*init))[0]
    sol = solid
    for k in range(STEPS):
        rho, mom, sn = codec.decode_state(words)
        (r, m, st), sol = crop_step((rho, mom, neq_recompose(rho, mom, sn)), sol, cfg.tau)
        noise = None
        if dither:
            o = x0 - h + k + 1, y0 - h + k + 1, z0 - h + k + 1
            n = r.shape
            idx = (((np.arange(n[0]) + o[0])[:, None, None] * dims[1] + (np.arange(n[1]) + o[1])[None, :, None])
                   * dims[2] + (np.arange(n[2]) + o[2])[None, None, :])
            noise = codec.dither_noise(idx, step0 + k, cfg.seed)
        words = codec.encode_state(r, m, neq_decompose(r, m, st), noise=noise)[0]
    got_codes = codec.unpack(codec.encode_state(got[0], got[1], neq_decompose(*got))[0])
    d = np.abs(got_codes.astype(np.int64) - codec.unpack(words).astype(np.int64))
    print(f"{name} q16 crop: max LSB {d.max()}, share != {np.mean(d > 0):.2e}")
    assert d.max() <= 2
