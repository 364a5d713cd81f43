O=gpurun_out/w9; mkdir -p $O
bash tools/abn.sh w9 4 k0 k1
cp paper_1406_1066_b200/lib/libsa_k1.so paper_1406_1066_b200/lib/libsa_b200.so
python tools/radix_check.py > $O/check.txt 2>&1
