"""Run bench.py's cfg1 decode block alone (spec vs autoregressive, B=8)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

print(json.dumps(bench.bench_decode_cfg1(), default=str))
