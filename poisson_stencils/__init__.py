"""``poisson_stencils`` — the reference package's import path, served by the B200 engine.

The reference's callers import submodules by name (``from poisson_stencils.simulator
import run``, ``poisson_stencils.scheme``, ``.quadrature``, ``.interpolation``,
``.stability``, ``.benchmarks``: pkg/tests/test_simulator.py:6-18,
pkg/tests/test_acceptance.py:15-26, pkg/src/poisson_stencils/benchmarks.py:8-9).  With
this directory on ``sys.path`` (the repo root, or ``pip install -e .``) those imports bind
to :mod:`paper_1904_04048_b200` unchanged: every submodule name below is the SAME module
object as its ``paper_1904_04048_b200`` counterpart, so ``first_step`` / ``two_step`` /
``run`` execute in libps.so's sm_100a kernels (there is no CPU fallback).

Not provided: ``poisson_stencils.cli`` (the reference's argparse front-end,
pkg/src/poisson_stencils/cli.py) — out of scope for the accelerated path.
"""

import importlib as _importlib
import sys as _sys

import paper_1904_04048_b200 as _impl
from paper_1904_04048_b200 import *  # noqa: F401,F403
from paper_1904_04048_b200 import __all__, __version__  # noqa: F401

SUBMODULES = ("interpolation", "quadrature", "scheme", "stability", "simulator", "benchmarks")

for _name in SUBMODULES:
    _module = _importlib.import_module(f"paper_1904_04048_b200.{_name}")
    _sys.modules[f"{__name__}.{_name}"] = _module
    globals()[_name] = _module
del _name, _module
