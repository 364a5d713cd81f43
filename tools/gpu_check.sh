#!/bin/bash
# One GPU-box pass: GPU tests, bench lines for each config, launch list of the headline config.
# usage: tools/gpu_check.sh TAG [pytest-args...]
set -u
TAG=${1:-run}; shift || true
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q "$@" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for c in 4 2 3 1 5; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_launch.log 2>&1
echo done
