#!/bin/bash
# One ncu --set full capture of the headline kernel (after bench.py exited 0
# without ncu in the same call), report into gpurun_out/.
mkdir -p gpurun_out
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > /dev/null 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:put_fast_kernel -s 1 -c 1 \
  -o gpurun_out/put16_full_r03 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/ncu_full_r03.log 2>&1
echo "ncu rc=$?"
