O=gpurun_out/w12; mkdir -p $O
cp paper_1406_1066_b200/lib/libsa_b1.so paper_1406_1066_b200/lib/libsa_b200.so
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "single_key or long_columns or sweep" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 600 python tools/big_column_probe.py > $O/long_columns.txt 2>&1
timeout 600 python tools/radix_check.py > $O/check.txt 2>&1
