#!/bin/bash
# tools/ab_draft.py under each environment assignment given, e.g. SSSD_LKW_PAD=16000
cd "$(dirname "$0")/.."
for a in "$@"; do
  echo "$a $(env $a timeout 300 python tools/ab_draft.py 2>&1 | tail -1 | cut -c1-100)"
done
