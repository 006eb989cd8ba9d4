#!/bin/bash
# End-of-round check on one GPU box: GPU parity suite, smoke(), the randomised
# large-T parity sweep, the NCCL path of bench.py forced at world size 1, and
# both bench arms.  Outputs under gpurun_out/fc_*.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/fc_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/fc_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/fc_smoke.log
timeout 1500 python tools/stress_parity.py ${STRESS_SEED0:-1} ${STRESS_SEEDS:-6} ${STRESS_N:-128} > gpurun_out/fc_stress.log 2>&1; echo "stress rc=$?"
tail -12 gpurun_out/fc_stress.log
FL_BENCH_FORCE_DIST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fc_nccl.json 2> gpurun_out/fc_nccl.err
echo "nccl-forced bench rc=$?"; tail -c 600 gpurun_out/fc_nccl.json; tail -3 gpurun_out/fc_nccl.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fc_ref.json 2> gpurun_out/fc_ref.err; echo "ref rc=$?"
timeout 900 python bench.py > gpurun_out/fc_bench.json 2> gpurun_out/fc_bench.err; echo "bench rc=$?"
python - <<'P'
import json
for f in ("gpurun_out/fc_ref.json", "gpurun_out/fc_bench.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d.get("value"), d.get("ms_per_step"), (d.get("e2e") or {}).get("value"), (d.get("roofline") or {}).get("frac"),
              d.get("parity_vs_cpu") or d.get("parity"), (d.get("clocks") or {}))
    except Exception as e:
        print(f, "unreadable", e)
P
