#!/bin/bash
# ncu --set full of one put_fast_kernel launch (after the same command ran plain).
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra"
timeout 300 $CMD > gpurun_out/plain_full.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:put_fast -s 1 -c 1 \
  -o gpurun_out/put16_full $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_full.log
