#!/bin/bash
# A/B variants of libsssd.so differing only in fusion_cta.cu (+ api.cu) compile flags:
#   tools/build_cta_variants.sh name1 "-DSSSD_CTA_WARPS=4" ... -> paper_2411_05894_b200/libsssd_<name>.so
set -e
cd "$(dirname "$0")/.."
python -m paper_2411_05894_b200.buildlib > /dev/null
cd build/sssd
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  for f in fusion_cta api; do
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      --expt-relaxed-constexpr $flags -I ../../include -I ../../paper_2411_05894_b200/csrc \
      -c ../../paper_2411_05894_b200/csrc/$f.cu -o ${f}_$name.o
  done
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../paper_2411_05894_b200/libsssd_$name.so \
    $(ls *.cu.o | grep -v '^fusion_cta.cu.o$' | grep -v '^api.cu.o$') fusion_cta_$name.o api_$name.o -lcudart -lcuda
  echo "built $name ($flags)"
done
