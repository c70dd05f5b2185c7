#!/bin/bash
# Round-2 evidence refresh (after the CTA fusion, k-gram index and 4-gram SA
# round): the bench command's ncu launch list, full-set captures of the cfg2
# propose kernels (16,384 requests), of the B = 64 latency path (CTA fusion,
# small-batch lookup), of one 100M suffix-array build and of the k-gram index
# build.  Outputs under gpurun_out/ (summarised into profiles/ afterwards).
set -u
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline \
  > gpurun_out/r2_launches_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"ds_lookup|input_scan|propose_setup|lpt_scatter|draft_ls_kernel" -c 5 \
  -o gpurun_out/r2_propose_full -f python tools/profile_propose.py 256 1 > gpurun_out/r2_propose_full.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"ds_lookup_kernel|input_scan|draft_cta_kernel" -s 6 -c 3 \
  -o gpurun_out/r2_b64_full -f python tools/profile_propose.py 1 4 > gpurun_out/r2_b64_full.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"rs_scatter|rs_upsweep|sa_round_rank|sa_round_keys|sa_mgram_keys|kix_" -c 12 \
  -o gpurun_out/r2_sa_full -f python tools/sa_build_bench.py 1e8 > gpurun_out/r2_sa_full.log 2>&1
ls -la gpurun_out | tail -12
