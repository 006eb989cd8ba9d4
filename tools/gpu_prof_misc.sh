set -u
mkdir -p gpurun_out
timeout 200 python tools/prof_put.py 6 256 > gpurun_out/prof256.txt 2>&1
timeout 200 python tools/prof_put.py 6 1 > gpurun_out/prof1.txt 2>&1
for w in c5 c4 c2 c3; do timeout 300 python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/bench_$w.json 2>gpurun_out/bench_$w.err; done
