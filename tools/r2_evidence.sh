#!/bin/bash
# Round-2 GPU evidence in one box call (outputs under gpurun_out/; summarised
# into profiles/ with tools/ncu_summary.py / tools/ncu_sum.py afterwards):
# the bench command's ncu launch list, a full-set capture of the propose
# kernels (cfg2, 16,384 requests), tensor-pipe metrics of tree attention
# (cfg3 / cfg4), and a full-set capture of one 100M suffix-array build.
set -u
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline \
  > gpurun_out/r2_launches_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"ds_lookup|input_scan|propose_setup|lpt_scatter|draft_ls_kernel" -c 5 \
  -o gpurun_out/r2_propose_full -f python tools/profile_propose.py 256 1 > gpurun_out/r2_propose_full.log 2>&1
timeout 600 ncu --clock-control none -k regex:tree_attn_kernel -c 4 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed \
  --csv python tools/bench_attn.py > gpurun_out/r2_attn_metrics.csv 2> gpurun_out/r2_attn_metrics.err
timeout 900 ncu --set full --clock-control none -k regex:"rs_scatter|rs_upsweep|sa_round_rank|sa_round_keys" -c 8 \
  -o gpurun_out/r2_sa_full -f python tools/sa_build_bench.py 1e8 > gpurun_out/r2_sa_full.log 2>&1
ls -la gpurun_out | tail -12
