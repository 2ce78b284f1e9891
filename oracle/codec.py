"""ORACLE (test infrastructure only) -- the 16-bit moment codec, float64/uint.

No reference code exists for the codec (the ``quantization`` module is absent
from ``/root/reference/pkg``); this restates the SPEC contract:
  * QuantSpec default ranges rho [0.8,1.5], rho*u [-0.6,0.6], sneq [-0.1,0.1]
    -- SPEC.md:333,374; PAPER.md:695-699,728-738
  * quantize: m' = (clamp(m)-min)/(max-min); q = floor(m'(2^b-1) + 1/2 + noise),
    clamped to [0, 2^b-1]; saturation counted when m was clamped -- SPEC.md:345-353
  * dequantize: m = min + q (max-min)/(2^b-1) -- SPEC.md:354-357
  * pack: two 16-bit slots per little-endian u32, component order
    (rho, rho u_xyz, sneq xx,xy,xz,yy,yz,zz) -- SPEC.md:358-361
  * dither: zero-mean uniform noise in [-1/2, 1/2) LSB from a counter-based
    hash keyed by (node, component, step) -- SPEC.md:376,385

The dither hash below is the build's definition (SPEC only asks for a
counter-based generator); the CUDA codec reproduces it bit-for-bit.
"""

from __future__ import annotations

import numpy as np

NCOMP = 10
NWORDS = 5
DEFAULT_MIN = np.array([0.8, -0.6, -0.6, -0.6, -0.1, -0.1, -0.1, -0.1, -0.1, -0.1])
DEFAULT_MAX = np.array([1.5, 0.6, 0.6, 0.6, 0.1, 0.1, 0.1, 0.1, 0.1, 0.1])

# Fig. 11 presets b_rho_u / b_S
PRESETS = {"16/16": (16, 16), "16/15": (16, 15), "15/14": (15, 14),
           "14/13": (14, 13), "13/12": (13, 12), "12/11": (12, 11)}


def bits_for_preset(name: str) -> np.ndarray:
    b_ru, b_s = PRESETS[name]
    return np.array([b_ru] * 4 + [b_s] * 6, dtype=np.int64)


def _u32(x):
    return np.asarray(x, dtype=np.uint64) & np.uint64(0xFFFFFFFF)


def mix32(x):
    """lowbias32 integer hash (uint32 -> uint32), vectorised."""
    x = _u32(x)
    x ^= x >> np.uint64(16)
    x = (x * np.uint64(0x7FEB352D)) & np.uint64(0xFFFFFFFF)
    x ^= x >> np.uint64(15)
    x = (x * np.uint64(0x846CA68B)) & np.uint64(0xFFFFFFFF)
    x ^= x >> np.uint64(16)
    return x


def step_key(step: int, seed: int) -> int:
    return int(mix32(np.uint64((int(step) * 0x9E3779B9 + int(seed) * 0x85EBCA6B + 0x2545F491)
                               & 0xFFFFFFFF)))


DITHER_MULT = (0x9E3779B1, 0x85EBCA77, 0xC2B2AE3D, 0x27D4EB2F)   # odd multipliers, words 1..4


def dither_words(h0):
    """The 5 noise words of a cell from its hash h0: word 0 = h0, word k = m ^ (m >> 16) with
    m = h0 * M_k mod 2^32 (a bijection of h0 for every k, so each word is uniform when h0 is)."""
    h0 = _u32(h0)
    out = [h0]
    for mk in DITHER_MULT:
        m = (h0 * np.uint64(mk)) & np.uint64(0xFFFFFFFF)
        out.append(m ^ (m >> np.uint64(16)))
    return out


def dither_noise(cell_index, step: int, seed: int) -> np.ndarray:
    """Noise in LSB units, shape (10, ...) for global linear cell indices.

    h0 = mix32(cell + key(step, seed)); the 5 words come from ``dither_words(h0)``;
    component 2k takes the low 16 bits of word k, 2k+1 the high 16 bits;
    noise = bits/65536 - 1/2 (exact in float32 and float64)."""
    cell = np.asarray(cell_index, dtype=np.uint64)
    h0 = mix32(cell + np.uint64(step_key(step, seed)))
    out = []
    for hk in dither_words(h0):
        lo = (hk & np.uint64(0xFFFF)).astype(np.float64)
        hi = (hk >> np.uint64(16)).astype(np.float64)
        out.append(lo / 65536.0 - 0.5)
        out.append(hi / 65536.0 - 0.5)
    return np.stack(out, axis=0)


def quantize(m, mmin, mmax, bits, noise=None):
    """Return (codes uint32, saturated bool) for one component array."""
    m = np.asarray(m, dtype=np.float64)
    if np.any(~np.isfinite(m)):
        raise ValueError("non-finite moment value (solver divergence)")
    levels = float((1 << int(bits)) - 1)
    sat = (m < mmin) | (m > mmax)
    mc = np.clip(m, mmin, mmax)
    t = (mc - mmin) / (mmax - mmin) * levels + 0.5
    if noise is not None:
        t = t + noise
    q = np.clip(np.floor(t), 0.0, levels)
    return q.astype(np.uint32), sat


def dequantize(q, mmin, mmax, bits):
    levels = float((1 << int(bits)) - 1)
    return mmin + np.asarray(q, dtype=np.float64) * ((mmax - mmin) / levels)


def pack(codes):
    """codes (10, ...) -> words (5, ...): word k = code[2k] | code[2k+1] << 16."""
    codes = np.asarray(codes, dtype=np.uint32)
    return (codes[0::2] & np.uint32(0xFFFF)) | ((codes[1::2] & np.uint32(0xFFFF)) << np.uint32(16))


def unpack(words):
    words = np.asarray(words, dtype=np.uint32)
    out = np.empty((NCOMP,) + words.shape[1:], dtype=np.uint32)
    out[0::2] = words & np.uint32(0xFFFF)
    out[1::2] = words >> np.uint32(16)
    return out


def encode_state(rho, mom, sneq, mmin=DEFAULT_MIN, mmax=DEFAULT_MAX, bits=None,
                 noise=None):
    """(rho, mom(3), sneq(6)) -> (words(5,...), saturation counts(10))."""
    if bits is None:
        bits = np.full(NCOMP, 16, dtype=np.int64)
    comps = [rho, mom[0], mom[1], mom[2]] + [sneq[k] for k in range(6)]
    codes, sats = [], []
    for k, m in enumerate(comps):
        q, s = quantize(m, mmin[k], mmax[k], bits[k], None if noise is None else noise[k])
        codes.append(q)
        sats.append(int(np.count_nonzero(s)))
    return pack(np.stack(codes)), np.array(sats, dtype=np.int64)


def decode_state(words, mmin=DEFAULT_MIN, mmax=DEFAULT_MAX, bits=None):
    if bits is None:
        bits = np.full(NCOMP, 16, dtype=np.int64)
    codes = unpack(words)
    vals = np.stack([dequantize(codes[k], mmin[k], mmax[k], bits[k]) for k in range(NCOMP)])
    return vals[0], vals[1:4], vals[4:10]
