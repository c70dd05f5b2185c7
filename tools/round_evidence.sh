#!/bin/bash
# Regenerate the round's GPU evidence in one box call (run from the repo root on
# the GPU box; outputs under gpurun_out/, summarised into profiles/ afterwards
# with tools/ncu_summary.py):
#   gpu tests, the default bench line, the ncu launch list of the bench
#   command, one full-set capture of the propose kernels and of tree attention.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/ -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
tail -1 gpurun_out/bench.log > gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-extra --no-cpu-baseline \
  > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"ds_lookup|input_scan|propose_setup|lpt_scatter|draft_ls_kernel" -c 5 \
  -o gpurun_out/propose_full python tools/profile_propose.py 256 1 > gpurun_out/propose_full.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tree_attn -c 2 \
  -o gpurun_out/attn_full python tools/profile_attn.py > gpurun_out/attn_full.log 2>&1
ls -la gpurun_out | tail -12
