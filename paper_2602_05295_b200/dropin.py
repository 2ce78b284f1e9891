"""Install the B200 solver into the reference package's namespace as ``momentlbm.solver`` (and the
obstacle-geometry module ``momentlbm.geometry``).

The reference package (/root/reference/pkg, installed unmodified into baseline/_ref) lists
``momentlbm.solver`` in its layout (pkg/src/momentlbm/__init__.py:1-9) but does not ship it.
``install()`` imports the reference ``momentlbm`` (from sys.path, else from ``baseline/_ref``) and
appends ``overlay/momentlbm`` to its ``__path__``, so ``import momentlbm.solver`` finds the B200
module next to the reference's own ``lattice`` / ``moments`` / ``collision``.  A maintainer of the
reference would instead copy ``overlay/momentlbm/solver.py`` into ``pkg/src/momentlbm/``
(INTEGRATION.md §1).
"""

from __future__ import annotations

import importlib
import sys
from pathlib import Path

OVERLAY = Path(__file__).resolve().parent / "overlay" / "momentlbm"
REF_INSTALL = Path(__file__).resolve().parents[1] / "baseline" / "_ref"


def install():
    """Make ``momentlbm.solver`` importable; returns the reference ``momentlbm`` package."""
    try:
        pkg = importlib.import_module("momentlbm")
    except ImportError:
        if not (REF_INSTALL / "momentlbm").exists():
            raise ImportError("the reference package momentlbm is not importable (install it into "
                              "baseline/_ref, DESIGN.md §8)")
        sys.path.insert(0, str(REF_INSTALL))
        pkg = importlib.import_module("momentlbm")
    if str(OVERLAY) not in list(pkg.__path__):
        pkg.__path__.append(str(OVERLAY))
    return pkg
