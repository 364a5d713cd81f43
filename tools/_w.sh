O=gpurun_out/w25; mkdir -p $O
bash tools/abn.sh w25 4 b200
timeout 600 python tools/radix_check.py > $O/check.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
python bench.py --steps 10 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
