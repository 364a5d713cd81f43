O=gpurun_out/w15; mkdir -p $O
for v in b3; do echo "== $v" >> $O/hh.txt; timeout 600 python tools/heavy_hitter_probe.py paper_1406_1066_b200/lib/libsa_$v.so >> $O/hh.txt 2>&1; done
cp paper_1406_1066_b200/lib/libsa_b3.so paper_1406_1066_b200/lib/libsa_b200.so
timeout 600 python tools/radix_check.py > $O/check.txt 2>&1
timeout 600 python tools/big_column_probe.py > $O/long_columns.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "single_key or long_columns or sweep or fuzz or big_and_small or nan" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
