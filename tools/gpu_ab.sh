#!/bin/bash
# A/B of prebuilt library variants on the headline batch (and the 1024 batch), then
# the GPU parity suite with the variant named in $PARITY (if any) installed.
set -u
mkdir -p gpurun_out
libs=$(ls tools/bin/lib_*.so)
timeout 300 python tools/ab_time.py $libs 2>&1 | tee gpurun_out/ab256.txt
AB_N=1024 timeout 300 python tools/ab_time.py $libs 2>&1 | tee gpurun_out/ab1024.txt
if [ -n "${PARITY:-}" ]; then
  cp tools/bin/lib_$PARITY.so paper_2303_02317_b200/libfftlattice_b200.so
  timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 | tee gpurun_out/parity_$PARITY.txt
fi
