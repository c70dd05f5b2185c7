import os, sys, json
sys.path.insert(0, os.getcwd())
import bench
print(json.dumps({k: v for k, v in bench.bench_decode_b64(True).get("llama3_8b", {}).items() if "tokens" in k or "step" in k}))
