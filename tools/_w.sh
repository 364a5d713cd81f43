O=gpurun_out/w23; mkdir -p $O
bash tools/abn.sh w23 4 u0 u1
cp paper_1406_1066_b200/lib/libsa_u1.so paper_1406_1066_b200/lib/libsa_b200.so
timeout 600 python tools/radix_check.py > $O/check.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "error or fuzz or three_pass or unaligned" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
