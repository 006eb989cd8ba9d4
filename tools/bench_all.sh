#!/bin/bash
# Every BASELINE.json config through bench.py (one JSON line each) and the
# ncu launch list of each (kernel shares), into gpurun_out/.
mkdir -p gpurun_out
for w in put16 c1 c2 c3 c4 c5; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  echo "$w rc=$? $(python -c "import json;d=json.load(open('gpurun_out/bench_$w.json'));print(round(d['ms_per_step'],3),'ms',round(d['roofline']['frac'],4),d.get('cpu_baseline',{}).get('value'))" 2>&1)"
done
for w in put16 c1 c2 c3 c4 c5; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$w.csv \
    python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --no-extra > /dev/null 2>&1
  echo "ncu $w rc=$?"
done
