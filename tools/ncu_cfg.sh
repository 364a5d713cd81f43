#!/bin/bash
# ncu --set full of the hot kernels of BASELINE configs (one GPU).
# usage: tools/ncu_cfg.sh TAG "cfg:regex:count" ...
TAG=$1; shift
O=gpurun_out/$TAG; mkdir -p $O
for spec in "$@"; do
  IFS=: read cfg rx cnt <<< "$spec"
  python tools/radix_one.py $cfg -1 > $O/plain_cfg$cfg.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$rx" -c $cnt \
      -o $O/prof_cfg$cfg python tools/radix_one.py $cfg -1 > $O/ncu_cfg$cfg.log 2>&1
  echo "cfg$cfg rc=$?" >> $O/status.txt
done
