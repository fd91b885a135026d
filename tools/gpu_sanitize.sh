# compute-sanitizer over every kernel family (tools/sanitize.py), logs into gpurun_out/
set -x
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --print-limit 50 python tools/sanitize.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.txt
done
timeout 900 $CS --tool memcheck --print-limit 50 python tools/sanitize.py --large > gpurun_out/sanitize_memcheck_large.txt 2>&1
echo "memcheck large rc=$?"; tail -3 gpurun_out/sanitize_memcheck_large.txt
