#!/bin/bash
# Link A/B variants of libsssd.so that differ only in the fusion kernel's
# __launch_bounds__ min-blocks (SSSD_DRAFT_MINB): paper_2411_05894_b200/libsssd_minbN.so
set -e
cd "$(dirname "$0")/.."
python -m paper_2411_05894_b200.buildlib > /dev/null
cd build/sssd
for m in "$@"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -DSSSD_DRAFT_MINB=$m -I ../../include -I ../../paper_2411_05894_b200/csrc -Xptxas -v \
    -c ../../paper_2411_05894_b200/csrc/fusion.cu -o fusion_$m.o 2>&1 | grep -A2 "draft_kernel" | grep "stack\|Used" | tr '\n' ' '
  echo " <- minb $m"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../paper_2411_05894_b200/libsssd_minb$m.so \
    $(ls *.cu.o | grep -v '^fusion.cu.o$') fusion_$m.o -lcudart
done
