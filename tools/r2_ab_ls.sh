#!/bin/bash
# A/B of fusion-kernel build variants (tools/build_ls_variants.sh) on the cfg2
# workload: tools/ab_draft.py per variant; optional correctness tests first.
set -u
mkdir -p gpurun_out
if [ -n "${AB_TESTS:-}" ]; then
  timeout 900 python -m pytest $AB_TESTS -q -x -p no:cacheprovider > gpurun_out/pytest_ab.log 2>&1; tail -3 gpurun_out/pytest_ab.log
fi
bash tools/ab_ls.sh ${AB_VARIANTS} 2>&1 | tee gpurun_out/ab_ls.log
