#!/bin/bash
# Final round profile: ncu --set full of the headline kernel (after the same
# bench line exited 0 without ncu), then the in-place chain time split of a
# clock build (tools/bin/clk.so) at 256 / 148 / 1024 puts and C2.
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra"
timeout 300 $CMD > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:put_fast_kernel -s 1 -c 1 \
  -o gpurun_out/put16_full_final $CMD > gpurun_out/ncu_full_final.log 2>&1
echo "ncu rc=$?"
cp tools/bin/clk.so paper_2303_02317_b200/libfftlattice_b200.so
for spec in "256 6" "148 6" "1024 6" "256 2"; do timeout 120 python tools/strip_clock.py $spec; done > gpurun_out/chain_split_final.txt 2>&1
cat gpurun_out/chain_split_final.txt
