"""pytest plugin: make ``import fftlattice`` resolve to the B200 drop-in.

Loaded with ``-p ref_shim`` by tools/run_reference_tests.py before the
reference's own tests are collected.  ``fftlattice`` and its submodules
(american, binomial, bsm, fft, model) are aliased to ``paper_2303_02317_b200``
and its same-named modules; ``fftlattice.cli`` -- the reference's command-line
driver, out of this repo's scope -- is the reference's own cli.py loaded from
baseline/_ref as a submodule of the alias, so its relative imports bind to the
drop-in's pricers (the reference CLI driving the GPU path).  Nothing of the
reference's pricing code is imported.
"""
from __future__ import annotations

import importlib
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2303_02317_b200 as _dropin  # noqa: E402

sys.modules["fftlattice"] = _dropin
for _name in ("american", "binomial", "bsm", "fft", "model"):
    sys.modules[f"fftlattice.{_name}"] = importlib.import_module(f"paper_2303_02317_b200.{_name}")

_cli_path = os.path.join(ROOT, "baseline", "_ref", "fftlattice", "cli.py")
if os.path.exists(_cli_path):
    _spec = importlib.util.spec_from_file_location("fftlattice.cli", _cli_path)
    _cli = importlib.util.module_from_spec(_spec)
    _cli.__package__ = "fftlattice"
    sys.modules["fftlattice.cli"] = _cli
    _spec.loader.exec_module(_cli)
    _dropin.cli = _cli
