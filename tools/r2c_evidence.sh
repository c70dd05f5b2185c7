#!/bin/bash
# Round-2 final-session evidence: full GPU tests + the default bench line, the
# bench command's ncu launch list, full-set captures of the cfg2 propose kernels
# and of the B = 64 latency path.  Outputs under gpurun_out/ (summarised into
# profiles/ with tools/ncu_summary.py afterwards).
set -u
mkdir -p gpurun_out
SKIP_BENCH=${SKIP_BENCH:-0} bash tools/r2_check.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/r2c_launches.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline \
  > gpurun_out/r2c_launches_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"ds_lookup|input_scan|propose_setup|lpt_scatter|draft_ls_kernel" -c 5 \
  -o gpurun_out/r2c_propose_full -f python tools/profile_propose.py 256 1 > gpurun_out/r2c_propose_full.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"ds_lookup_kernel|input_scan|draft_cta_kernel" -s 6 -c 3 \
  -o gpurun_out/r2c_b64_full -f python tools/profile_propose.py 1 4 > gpurun_out/r2c_b64_full.log 2>&1
ls -la gpurun_out | tail -12
