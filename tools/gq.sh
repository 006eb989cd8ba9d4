set -x
timeout 600 python -m pytest tests -m gpu -q --timeout 500 2>&1 | tail -15
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -3
