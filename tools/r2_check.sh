#!/bin/bash
# Round-2 GPU check: full gpu test suite (incl. the reference's own suite,
# tests/refsuite) and the default bench line; logs under gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests/ -m gpu -q -p no:cacheprovider ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
tail -15 gpurun_out/pytest_gpu.log
if [ "${SKIP_BENCH:-0}" != "1" ]; then
  timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
  tail -1 gpurun_out/bench.log > gpurun_out/bench.json
  head -c 3000 gpurun_out/bench.json
fi
