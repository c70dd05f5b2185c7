#!/bin/bash
# tools/ab_draft.py for each libsssd_<name>.so variant given
cd "$(dirname "$0")/.."
for n in "$@"; do
  SSSD_LIB=$PWD/paper_2411_05894_b200/libsssd_$n.so timeout 300 python tools/ab_draft.py 2>&1 | tail -1 | cut -c1-140
done
