#!/bin/bash
# A/B variants of libsssd.so differing only in fusion_ls.cu (+ api.cu) compile flags:
#   tools/build_ls_variants.sh name1 "-DFOO=1 -DBAR=2" name2 "-DFOO=2" ...
# -> paper_2411_05894_b200/libsssd_<name>.so (run with SSSD_LIB=...)
set -e
cd "$(dirname "$0")/.."
python -m paper_2411_05894_b200.buildlib > /dev/null
cd build/sssd
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr $flags -I ../../include -I ../../paper_2411_05894_b200/csrc -Xptxas -v \
    -c ../../paper_2411_05894_b200/csrc/fusion_ls.cu -o fusion_ls_$name.o 2>&1 | grep -A2 "draft_ls_kernel" | grep "stack\|Used" | tr '\n' ' '
  echo " <- $name ($flags)"
  # api.cu launches the kernel: it sees the same flags (launch shape macros)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr $flags -I ../../include -I ../../paper_2411_05894_b200/csrc \
    -c ../../paper_2411_05894_b200/csrc/api.cu -o api_$name.o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../paper_2411_05894_b200/libsssd_$name.so \
    $(ls *.cu.o | grep -v '^fusion_ls.cu.o$' | grep -v '^api.cu.o$') fusion_ls_$name.o api_$name.o -lcudart
done
