#!/bin/bash
# tree-attention timing (cfg3 / cfg4 and the s_q sweep) under each environment assignment given
cd "$(dirname "$0")/.."
for a in "$@"; do
  echo "$a $(env $a python tools/bench_attn.py | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["cfg3"]["ms"],4), round(d["cfg4"]["ms"],4))') | $(env $a python tools/bench_attn_sq.py | tr '\n' ' ')"
done
