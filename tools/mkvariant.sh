#!/bin/bash
# usage: mkvariant.sh name "extra flags"
name=$1; extra=$2
d=/tmp/var_$name; mkdir -p $d
C=paper_1901_00155_b200/csrc
for f in prep_kernels search_kernels tc_kernels probe_kernels engine; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -I include -I $C $extra -c $C/$f.cu -o $d/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -o paper_1901_00155_b200/_lib/var_$name.so $d/*.o -ldl -lpthread
echo built $name
