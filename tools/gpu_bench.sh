# one GPU pass: selected tests ($1, a pytest -k expression), then bench.py (default workload)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
if [ -n "$1" ]; then timeout 900 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider -k "$1" > gpurun_out/gputest_sel.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_sel.log; fi
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -5 gpurun_out/bench.err
