#!/bin/bash
# Round-2 closing evidence: bench lines of every config (+ the sharded world-1 step), launch list and
# ncu --set full of cfg4's hot kernels (the FEM kernels are unchanged since r02f).
O=gpurun_out/${1:-r02z}; mkdir -p $O
for c in 4 1 2 3 5; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29541 bench.py --sharded --config 5 --steps 5 --warmup 3 > $O/bench_sharded1.json 2> $O/bench_sharded1.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file $O/launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_launch.log 2>&1
python tools/radix_one.py 4 -1 > $O/plain_one.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_rpass|k_rfold|k_rup" -c 5 -o $O/prof_cfg4 python tools/radix_one.py 4 -1 > $O/ncu_cfg4.log 2>&1
python tools/big_column_probe.py > $O/long_columns.txt 2>&1
echo done
