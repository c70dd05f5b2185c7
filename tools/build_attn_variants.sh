#!/bin/bash
# A/B variants of libsssd.so differing only in attention.cu compile flags:
#   tools/build_attn_variants.sh name1 "-DFOO=1" ... -> paper_2411_05894_b200/libsssd_<name>.so
set -e
cd "$(dirname "$0")/.."
python -m paper_2411_05894_b200.buildlib > /dev/null
cd build/sssd
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr $flags -I ../../include -I ../../paper_2411_05894_b200/csrc \
    -c ../../paper_2411_05894_b200/csrc/attention.cu -o attention_$name.o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../paper_2411_05894_b200/libsssd_$name.so \
    $(ls *.cu.o | grep -v '^attention.cu.o$') attention_$name.o -lcudart -lcuda
done
