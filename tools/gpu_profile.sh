#!/bin/bash
# Round profile: default bench line, then (after the same command ran plain) the
# ncu launch list and one --set full capture of the headline put kernel.
set -u
mkdir -p gpurun_out
timeout 300 python bench.py > gpurun_out/bench_prof.json 2> gpurun_out/bench_prof.err; echo "bench rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
CMD2="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra"
timeout 300 $CMD2 > gpurun_out/plain_full.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:put_fast -s 1 -c 1 \
  -o gpurun_out/put16_full $CMD2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
