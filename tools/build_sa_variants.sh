#!/bin/bash
# A/B variants of libsssd.so differing only in sa_build.cu compile flags:
#   tools/build_sa_variants.sh name1 "-DFOO=1" name2 "-DFOO=2" ...
# -> paper_2411_05894_b200/libsssd_<name>.so (run with SSSD_LIB=...)
set -e
cd "$(dirname "$0")/.."
python -m paper_2411_05894_b200.buildlib > /dev/null
cd build/sssd
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr $flags -I ../../include -I ../../paper_2411_05894_b200/csrc -Xptxas -v \
    -c ../../paper_2411_05894_b200/csrc/sa_build.cu -o sa_build_$name.o 2>&1 | grep -A2 "rs_scatter_w" | grep "stack\|Used" | tr '\n' ' '
  echo " <- $name ($flags)"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../paper_2411_05894_b200/libsssd_$name.so \
    $(ls *.cu.o | grep -v '^sa_build.cu.o$') sa_build_$name.o -lcudart
done
