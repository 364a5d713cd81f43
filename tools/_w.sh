O=gpurun_out/w22; mkdir -p $O
bash tools/abn.sh w22 4 r0 r1
cp paper_1406_1066_b200/lib/libsa_r1.so paper_1406_1066_b200/lib/libsa_b200.so
timeout 600 python tools/radix_check.py > $O/check.txt 2>&1
