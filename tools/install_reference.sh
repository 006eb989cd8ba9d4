#!/bin/sh
# Install the UNMODIFIED reference package into baseline/_ref (git-ignored,
# shipped to the GPU box by gpurun) for bench.py's reference arm.  The build
# writes into its source tree, so it installs from a copy under /tmp; numpy and
# numba are already in the image (--no-deps).
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/fftlattice_ref_src baseline/_ref
cp -r /root/reference/pkg /tmp/fftlattice_ref_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target baseline/_ref /tmp/fftlattice_ref_src
# the reference's own test suite, run against the drop-in by
# tools/run_reference_tests.py (the tests are data here, never product code)
cp -r /root/reference/pkg/tests baseline/_ref/tests
