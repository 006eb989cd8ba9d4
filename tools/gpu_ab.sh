#!/bin/bash
# A/B of prebuilt library variants (tools/bin/lib_*.so): headline batch, 1024
# puts, C2, C3, C4 and a 16384-option C5 subset; then the GPU parity suite with
# the variant named in $PARITY (if any) installed.
set -u
mkdir -p gpurun_out
libs=$(ls tools/bin/lib_*.so)
: > gpurun_out/ab_all.txt
for spec in "6 256" "6 1024" "2 256" "3 256" "4 64" ${AB_EXTRA:-"5 16384"}; do
  set -- $spec
  echo "== cfg $1 n $2" | tee -a gpurun_out/ab_all.txt
  AB_CFG=$1 AB_N=$2 timeout 300 python tools/ab_time.py $libs 2>&1 | tee -a gpurun_out/ab_all.txt
done
if [ -n "${PARITY:-}" ]; then
  cp tools/bin/lib_$PARITY.so paper_2303_02317_b200/libfftlattice_b200.so
  timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 | tee gpurun_out/parity_$PARITY.txt
fi
