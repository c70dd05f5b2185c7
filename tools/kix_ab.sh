set -x
python tools/ab_draft.py 2>&1 | tail -1
SSSD_NO_KIX=1 python tools/ab_draft.py 2>&1 | tail -1
python tools/latency_ab.py
SSSD_NO_KIX=1 python tools/latency_ab.py
timeout 900 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
