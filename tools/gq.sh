set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 600 python -m pytest tests -m gpu -q --timeout 500   2>&1 | tail -30
