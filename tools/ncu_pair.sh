#!/bin/bash
# ncu --set full of the headline kernel (256 options) and of a single option,
# with the in-tree library (each command first runs plain and exits 0).
mkdir -p gpurun_out
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:put_fast_kernel -s 1 -c 1 \
  -o gpurun_out/put16_full_${TAG:-x} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/ncu_full_${TAG:-x}.log 2>&1
echo "ncu256 rc=$?"
AB_N=1 timeout 300 python tools/ab_time.py paper_2303_02317_b200/libfftlattice_b200.so > /dev/null 2>&1 || exit 1
AB_N=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:put_fast_kernel -s 3 -c 1 \
  -o gpurun_out/put1_full_${TAG:-x} python tools/ab_time.py paper_2303_02317_b200/libfftlattice_b200.so > gpurun_out/ncu_full1_${TAG:-x}.log 2>&1
echo "ncu1 rc=$?"
