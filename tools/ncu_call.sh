#!/bin/bash
# ncu --set full of the C2 call kernel (bench line first runs plain).
mkdir -p gpurun_out
CMD="python bench.py --workload c2 --steps 1 --warmup 3 --no-cpu-baseline --no-extra"
timeout 300 $CMD > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:call_fast_kernel -s 1 -c 1 \
  -o gpurun_out/c2_full_${TAG:-x} $CMD > gpurun_out/ncu_c2_${TAG:-x}.log 2>&1
echo "ncu c2 rc=$?"
