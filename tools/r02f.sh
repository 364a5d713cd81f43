#!/bin/bash
# Final round-2 evidence: bench lines of every config (incl. the sharded world-1 step), ncu of cfg4 and cfg5 hot kernels.
O=gpurun_out/r02f; mkdir -p $O
for c in 4 1 2 3 5; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29541 bench.py --sharded --config 5 --steps 5 --warmup 3 > $O/bench_sharded1.json 2> $O/bench_sharded1.err
python tools/radix_one.py 4 -1 > $O/plain4.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_rpass|k_rfold|k_rup" -c 5 -o $O/prof_cfg4 python tools/radix_one.py 4 -1 > $O/ncu4.log 2>&1
python tools/radix_one.py 5 -1 > $O/plain5.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_tile_fold|k_colcount" -c 3 -o $O/prof_cfg5 python tools/radix_one.py 5 -1 > $O/ncu5.log 2>&1
echo done
