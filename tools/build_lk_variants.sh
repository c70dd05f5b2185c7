#!/bin/bash
# A/B variants of libsssd.so differing only in propose.cu compile flags:
#   tools/build_lk_variants.sh name1 "-DFOO=1" name2 "-DFOO=2" ...
# -> paper_2411_05894_b200/libsssd_<name>.so (run with SSSD_LIB=...)
set -e
cd "$(dirname "$0")/.."
python -m paper_2411_05894_b200.buildlib > /dev/null
cd build/sssd
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr $flags -I ../../include -I ../../paper_2411_05894_b200/csrc -Xptxas -v \
    -c ../../paper_2411_05894_b200/csrc/propose.cu -o propose_$name.o 2>&1 | grep -A2 "ds_lookup_warp_kernel" | grep "stack\|Used" | tr '\n' ' '
  echo " <- $name ($flags)"
  # api.cu sees the same flags (it exports the probe switch of measurement builds)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr $flags -I ../../include -I ../../paper_2411_05894_b200/csrc \
    -c ../../paper_2411_05894_b200/csrc/api.cu -o api_lk_$name.o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../paper_2411_05894_b200/libsssd_$name.so \
    $(ls *.cu.o | grep -v '^propose.cu.o$' | grep -v '^api.cu.o$') propose_$name.o api_lk_$name.o -lcudart
done
