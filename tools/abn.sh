# A/B/n: per-kernel times of several libsa_<name>.so builds. usage: tools/abn.sh TAG CFG name1 name2 ...
O=gpurun_out/$1; C=$2; shift; shift; mkdir -p $O
for i in 1 2; do for n in "$@"; do
python tools/kernel_times.py paper_1406_1066_b200/lib/libsa_$n.so $C >> $O/kt.txt 2>&1
done; done
