#!/bin/bash
# Copy the closing evidence of a tools/r02g.sh run (gpurun_out/TAG) into profiles/ (tracked).
# usage: tools/refresh_profiles.sh TAG
T=gpurun_out/${1:-r02z}; P=profiles
for c in 1 2 3 4 5; do cp $T/bench_cfg$c.json $P/r02_bench_cfg$c.json; done
cp $T/bench_sharded1.json $P/r02_bench_sharded1.json
cp $T/launches_cfg4.csv $P/r02_launches_cfg4.csv
python tools/launch_summary.py $T/launches_cfg4.csv heavy_dup_10000000_P100000000 $P/r02_launches_cfg4.md
{ echo "# ncu --set full --clock-control none, BASELINE cfg4, closing round-2 build (tools/r02g.sh; report $T/prof_cfg4.ncu-rep)"; python tools/ncu_sum.py $T/prof_cfg4.ncu-rep; } > $P/r02_ncu_cfg4.txt
{ python tools/ncu_lines.py $T/prof_cfg4.ncu-rep k_rpass_tma 25; python tools/ncu_lines.py $T/prof_cfg4.ncu-rep k_rfold 25; } > $P/r02_ncu_cfg4_lines.txt
cp $T/long_columns.txt $P/r02_long_columns.txt
python tools/traffic_json.py heavy_dup_10000000_P100000000 $T/prof_cfg4.ncu-rep
