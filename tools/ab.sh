# A/B: per-kernel times of libsa_base.so (saved reference build) vs the current build
O=gpurun_out/${1:-ab}; C=${2:-4}; mkdir -p $O
for i in 1 2; do
python tools/kernel_times.py paper_1406_1066_b200/lib/libsa_base.so $C >> $O/kt.txt 2>&1
python tools/kernel_times.py paper_1406_1066_b200/lib/libsa_b200.so $C >> $O/kt.txt 2>&1
done
if [ -n "$3" ]; then timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log; fi
