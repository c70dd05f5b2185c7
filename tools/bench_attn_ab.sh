# tree-attention timing at cfg3 / cfg4 (tools/bench_attn.py), optionally for A/B builds:
#   bash tools/bench_attn_ab.sh [libsssd_variant.so ...]
for lib in "${@:-paper_2411_05894_b200/libsssd.so}"; do
  echo "$lib $(SSSD_LIB=$PWD/$lib python tools/bench_attn.py)"
done
