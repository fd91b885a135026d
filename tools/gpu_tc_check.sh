# tensor-core kernel change check: parity tests on the tc paths, timed configs, then the bench and a split sweep
timeout 1200 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider -k "tensor_core or timed or config3 or sharded or smoke or c4 or 2p16 or in_graph" > gpurun_out/gputest_tc.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_tc.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/bench.err
for S in 32 37 64; do CLB_TC_SPLITS=$S timeout 300 python bench.py --quick --no-cpu-baseline --steps 10 > gpurun_out/bench_S$S.json 2>/dev/null; echo "S=$S rc=$?"; done
