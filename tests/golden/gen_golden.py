"""Generate the golden fixtures in tests/golden/ by running the REFERENCE package.

Run here (not on the GPU box, where /root/reference does not exist):
    python tests/golden/gen_golden.py
It imports momentlbm from /root/reference/pkg/src (or baseline/_ref) and records
outputs of the reference's own functions:
  lattice.npz        make_lattice("D3Q27") tables (lattice.py:172-211)
  moments.npz        reconstruct_distributions / moments_from_distributions /
                     neq_decompose on random moment sets (moments.py:25-102)
  collision.npz      collide_moments with and without a body force (collision.py:137-194)
  step16.npz         one periodic step of a random 16^3 state composed from the reference
                     functions + np.roll pull streaming (SURVEY.md §8c golden vector 1)
  tgv32.npz          Taylor-Green 32^3 after 10 steps, same composition
  d3q19.npz          make_lattice("D3Q19") tables and 1 / 3 periodic steps of a random
                     12x14x16 state with the D3Q19 lattice, same composition
`--extra` (SURVEY.md §8c's remaining golden vectors; same composition, codec and lists
written out here from SPEC, independent of oracle/):
  q16_step16.npz     16-bit codes of a random 16^3 state (SPEC.md:345-353 quantizer, default
                     QuantSpec, no dither) and of its state after one reference step
  sphere32.npz       sphere mask in a periodic 32^3 box -> sorted boundary list + link masks
                     (bit i: x - c_i solid, reference direction order) + solid list
  tgv64.npz          Taylor-Green 64^3 (nu = 0.01): kinetic energy and mass after every step to
                     200, and the planes x = 0 and x = 21 of the state after 1, 10 and 200 steps
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
for cand in ("/root/reference/pkg/src", str(ROOT / "baseline" / "_ref")):
    if Path(cand, "momentlbm").exists():
        sys.path.insert(0, cand)
        break

import momentlbm.collision as RC  # noqa: E402
import momentlbm.lattice as RL  # noqa: E402
import momentlbm.moments as RM  # noqa: E402

LAT = RL.make_lattice("D3Q27")
LAT19 = RL.make_lattice("D3Q19")


def ref_step(rho, mom, stress, tau, force=None, lat=LAT):
    """Alg. 2 from the reference's own functions."""
    r, m, s = RC.collide_moments(rho, mom, stress, force, tau, 3)
    f = RM.reconstruct_distributions(r, m, s, lat)
    fs = np.stack([np.roll(f[i], shift=tuple(lat.velocities[i]), axis=(0, 1, 2)) for i in range(lat.q)])
    return RM.moments_from_distributions(fs, lat)


def write_d3q19():
    h = LAT19.hermite
    tau = 0.5 + 3 * 0.02
    rho, mom, st = random_state((12, 14, 16), 3, 0.05, 0.08, 0.005)
    s1 = ref_step(rho, mom, st, tau, lat=LAT19)
    s3 = ref_step(*ref_step(*s1, tau, lat=LAT19), tau, lat=LAT19)
    np.savez_compressed(HERE / "d3q19.npz", velocities=LAT19.velocities, weights=LAT19.weights,
                        opposite=LAT19.opposite, h2c=h.h2_contract, h3=h.h3, tau=tau, rho=rho, mom=mom,
                        stress=st, rho1=s1[0], mom1=s1[1], stress1=s1[2], rho3=s3[0], mom3=s3[1],
                        stress3=s3[2])


def random_state(shape, seed, drho, umax, sneq):
    rng = np.random.default_rng(seed)
    rho = 1.0 + rng.uniform(-drho, drho, shape)
    mom = rho * rng.uniform(-umax, umax, (3,) + tuple(shape))
    n = rng.uniform(-sneq, sneq, (6,) + tuple(shape))
    return rho, mom, RM.neq_recompose(rho, mom, n)


def taylor_green(n, u0=0.05):
    k = 2 * np.pi / n
    x = np.arange(n)[:, None, None]
    y = np.arange(n)[None, :, None]
    z = np.arange(n)[None, None, :]
    ux = u0 * np.sin(k * x) * np.cos(k * y) * np.cos(k * z)
    uy = -u0 * np.cos(k * x) * np.sin(k * y) * np.cos(k * z)
    uz = np.zeros_like(ux + uy)
    rho = 1.0 + 3.0 * (u0 ** 2 / 16.0) * (np.cos(2 * k * x) + np.cos(2 * k * y)) * (np.cos(2 * k * z) + 2.0)
    rho = np.broadcast_to(rho, (n, n, n)).astype(np.float64)
    mom = np.stack([rho * ux, rho * uy, rho * uz])
    return rho, mom, RM.neq_recompose(rho, mom, np.zeros((6, n, n, n)))


def main():
    h = LAT.hermite
    np.savez_compressed(HERE / "lattice.npz", velocities=LAT.velocities, weights=LAT.weights,
                        opposite=LAT.opposite, h2=h.h2, h2c=h.h2_contract, h3=h.h3)

    rho, mom, st = random_state((64,), 0, 0.3, 0.4, 0.1)
    f = RM.reconstruct_distributions(rho, mom, st, LAT)
    rng = np.random.default_rng(1)
    fr = LAT.weights[:, None] * (1.0 + rng.uniform(-0.2, 0.2, (27, 64)))
    r2, m2, s2 = RM.moments_from_distributions(fr, LAT)
    np.savez_compressed(HERE / "moments.npz", rho=rho, mom=mom, stress=st, f=f, f_rand=fr,
                        rho_of_f=r2, mom_of_f=m2, stress_of_f=s2,
                        sneq=RM.neq_decompose(rho, mom, st))

    F = np.array([1e-4, -2e-4, 3e-5])
    c0 = RC.collide_moments(rho, mom, st, None, 0.53, 3)
    c1 = RC.collide_moments(rho, mom, st, F, 0.8, 3)
    np.savez_compressed(HERE / "collision.npz", rho=rho, mom=mom, stress=st, force=F,
                        tau0=0.53, rho0=c0[0], mom0=c0[1], stress0=c0[2],
                        tau1=0.8, rho1=c1[0], mom1=c1[1], stress1=c1[2])

    tau = 0.5 + 3 * 0.02
    rho, mom, st = random_state((16, 16, 16), 0, 0.1, 0.1, 0.01)
    out = ref_step(rho, mom, st, tau)
    np.savez_compressed(HERE / "step16.npz", tau=tau, rho=rho, mom=mom, stress=st,
                        rho1=out[0], mom1=out[1], stress1=out[2])

    tau = 0.5 + 3 * 0.01
    r, m, s = taylor_green(32)
    init = (r, m, s)
    for _ in range(10):
        r, m, s = ref_step(r, m, s, tau)
    np.savez_compressed(HERE / "tgv32.npz", tau=tau, steps=10, rho0=init[0], mom0=init[1],
                        stress0=init[2], rho=r, mom=m, stress=s)
    write_d3q19()
    print("golden fixtures written to", HERE)


QMIN = np.array([0.8, -0.6, -0.6, -0.6, -0.1, -0.1, -0.1, -0.1, -0.1, -0.1])
QMAX = np.array([1.5, 0.6, 0.6, 0.6, 0.1, 0.1, 0.1, 0.1, 0.1, 0.1])


def quantize16(rho, mom, stress):
    """q = floor((clamp(m) - min) / (max - min) * (2^16 - 1) + 1/2), m = (rho,
    rho u, sneq)."""
    m = np.concatenate([rho[None], mom, RM.neq_decompose(rho, mom, stress)])
    lo, hi = QMIN.reshape(-1, 1, 1, 1), QMAX.reshape(-1, 1, 1, 1)
    x = (np.clip(m, lo, hi) - lo) / (hi - lo)
    return np.clip(np.floor(x * 65535.0 + 0.5), 0, 65535).astype(np.uint16)


def dequantize16(q):
    lo, hi = QMIN.reshape(-1, 1, 1, 1), QMAX.reshape(-1, 1, 1, 1)
    m = lo + q.astype(np.float64) * (hi - lo) / 65535.0
    rho, mom = m[0], m[1:4]
    return rho, mom, RM.neq_recompose(rho, mom, m[4:])


def write_extra():
    tau = 0.5 + 3 * 0.02
    rho, mom, st = random_state((16, 16, 16), 5, 0.08, 0.08, 0.008)
    q0 = quantize16(rho, mom, st)
    q1 = quantize16(*ref_step(*dequantize16(q0), tau))
    np.savez_compressed(HERE / "q16_step16.npz", tau=tau, codes0=q0, codes1=q1)

    n = 32
    g = np.indices((n, n, n)).astype(np.float64)
    c = np.array([15.5, 16.2, 14.8]).reshape(3, 1, 1, 1)
    mask = (((g - c) ** 2).sum(0) <= 7.3 ** 2).astype(np.uint8)
    links = np.zeros((n, n, n), dtype=np.uint32)
    for i, ci in enumerate(LAT.velocities):
        if i:   # source x - c_i solid (periodic): np.roll(a, c)[x] = a[x - c]
            links |= (np.roll(mask, shift=tuple(ci), axis=(0, 1, 2)).astype(np.uint32) << np.uint32(i))
    fluid = mask == 0
    bsel = fluid & (links != 0)
    cells = np.flatnonzero(bsel.ravel()).astype(np.int64)
    np.savez_compressed(HERE / "sphere32.npz", mask=mask, boundary_cells=cells,
                        link_masks=links.ravel()[cells], solid_cells=np.flatnonzero(mask.ravel()).astype(np.int64))

    tau = 0.5 + 3 * 0.01
    r, m, s_ = taylor_green(64)
    ke, mass, planes = [], [], {}
    for k in range(1, 201):
        r, m, s_ = ref_step(r, m, s_, tau)
        ke.append(0.5 * float((m ** 2 / r).sum()))
        mass.append(float(r.sum()))
        if k in (1, 10, 200):
            sn = RM.neq_decompose(r, m, s_)
            planes[k] = np.concatenate([r[None], m, sn])[:, [0, 21]]
    np.savez_compressed(HERE / "tgv64.npz", tau=tau, ke=np.array(ke), mass=np.array(mass),
                        planes1=planes[1], planes10=planes[10], planes200=planes[200])


if __name__ == "__main__":
    if sys.argv[1:] == ["--d3q19"]:
        write_d3q19()
    elif sys.argv[1:] == ["--extra"]:
        write_extra()
    else:
        main()
