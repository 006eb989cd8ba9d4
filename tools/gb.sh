set -x
timeout 600 python bench.py --steps 5 --warmup 3 2>&1 | tail -5
timeout 300 python bench.py --steps 3 --warmup 3 --workload c3 --no-cpu-baseline 2>&1 | tail -3
timeout 300 python bench.py --steps 3 --warmup 3 --workload c2 --no-cpu-baseline 2>&1 | tail -3
timeout 300 python bench.py --steps 3 --warmup 3 --workload c1 --no-cpu-baseline 2>&1 | tail -3
