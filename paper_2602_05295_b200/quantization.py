"""Quantization configuration of the 16-bit moment codec (host-side description only).

The codec itself runs in registers inside the CUDA step kernels (csrc/hlbm_interior.cu,
csrc/hlbm_cells.cu).  This module carries the configuration the reference SPEC defines for
its absent ``quantization`` module:

  * QuantSpec default ranges rho [0.8,1.5], rho*u [-0.6,0.6], sneq [-0.1,0.1]
    
  * bit-allocation presets b_rho_u / b_S of Fig. 11
  * dither switch
"""

from __future__ import annotations

from dataclasses import dataclass, field

DEFAULT_MIN = (0.8, -0.6, -0.6, -0.6, -0.1, -0.1, -0.1, -0.1, -0.1, -0.1)
DEFAULT_MAX = (1.5, 0.6, 0.6, 0.6, 0.1, 0.1, 0.1, 0.1, 0.1, 0.1)
COMPONENTS = ("rho", "rho_ux", "rho_uy", "rho_uz",
              "sneq_xx", "sneq_xy", "sneq_xz", "sneq_yy", "sneq_yz", "sneq_zz")
PRESETS = {"16/16": (16, 16), "16/15": (16, 15), "15/14": (15, 14),
           "14/13": (14, 13), "13/12": (13, 12), "12/11": (12, 11)}


@dataclass
class QuantSpec:
    mmin: tuple = DEFAULT_MIN
    mmax: tuple = DEFAULT_MAX
    bits: tuple = (16,) * 10
    dither: bool = False

    def __post_init__(self):
        if len(self.mmin) != 10 or len(self.mmax) != 10 or len(self.bits) != 10:
            raise ValueError("QuantSpec needs 10 components")
        for lo, hi in zip(self.mmin, self.mmax):
            if not lo < hi:
                raise ValueError("quantization range needs min < max")
        for b in self.bits:
            if not 2 <= int(b) <= 16:
                raise ValueError("bits per component must lie in [2, 16] (16-bit slots)")

    @classmethod
    def preset(cls, name: str, dither: bool = False) -> "QuantSpec":
        b_ru, b_s = PRESETS[name]
        return cls(bits=(b_ru,) * 4 + (b_s,) * 6, dither=dither)

    @property
    def words_per_node(self) -> int:
        """Two 16-bit slots per u32: 5 words per 3-D node."""
        return 5

    def step(self, k: int) -> float:
        return (self.mmax[k] - self.mmin[k]) / ((1 << int(self.bits[k])) - 1)
