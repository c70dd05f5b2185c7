set -u
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --kernel-name kns=sssd --print-limit 20 python tools/sanitize_r2.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/san_$tool.log
done
