#!/bin/bash
# Dev: build libsa_<NAME>.so with extra -D flags for sa_radix.cu only (other objects cached in /tmp/obj).
# usage: tools/build_variant.sh NAME [-DFLAG=1 ...]
NAME=$1; shift
C=paper_1406_1066_b200/csrc; O=/tmp/obj; mkdir -p $O
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC"
for f in sa_kernels sa_tile sa_prune sa_shard sa_capi; do
  if [ ! -f $O/$f.o ] || [ $C/$f.cu -nt $O/$f.o ] || [ $C/sa_internal.cuh -nt $O/$f.o ]; then nvcc $FL -c $C/$f.cu -o $O/$f.o & fi
done
nvcc $FL "$@" -c $C/sa_radix.cu -o $O/sa_radix_$NAME.o &
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o paper_1406_1066_b200/lib/libsa_$NAME.so $O/sa_kernels.o $O/sa_tile.o $O/sa_prune.o $O/sa_shard.o $O/sa_capi.o $O/sa_radix_$NAME.o
ls -la paper_1406_1066_b200/lib/libsa_$NAME.so
