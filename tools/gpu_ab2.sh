#!/bin/bash
# A/B of prebuilt library variants (tools/bin/lib_*.so) on the workloads listed
# in $AB_SPECS ("cfg n" pairs separated by ';'), see tools/ab_time.py.
set -u
mkdir -p gpurun_out
libs=$(ls tools/bin/lib_*.so)
: > gpurun_out/ab2.txt
IFS=';' read -ra specs <<< "${AB_SPECS:-6 256;4 64}"
for spec in "${specs[@]}"; do
  set -- $spec
  echo "== cfg $1 n $2" | tee -a gpurun_out/ab2.txt
  AB_CFG=$1 AB_N=$2 timeout 300 python tools/ab_time.py $libs 2>&1 | tee -a gpurun_out/ab2.txt
done
