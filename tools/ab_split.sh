#!/bin/bash
# A/B of the mixed-batch dispatch: one american_fast_kernel (FL_SPLIT_KINDS=0) vs the
# put and call kernels back to back (FL_SPLIT_KINDS=1), C5 subsets and the full C5.
mkdir -p gpurun_out
: > gpurun_out/ab_split.txt
for n in ${AB_SIZES:-4096 16384 65536}; do
  for s in 0 1; do
    echo "== C5 n $n split $s" | tee -a gpurun_out/ab_split.txt
    FL_SPLIT_KINDS=$s AB_CFG=5 AB_N=$n timeout 600 python tools/ab_time.py ${1:-tools/bin/lib_split.so} 2>&1 | tee -a gpurun_out/ab_split.txt
  done
done
