# ncu evidence for round 2: launch list of the default bench command (cold-cache, serialised per-launch times),
# one --set full capture of the pair tcgen05 kernel at n = 2^20 (fp16) inside the bench, and of the
# real-plan FFT kernels at n = 2^24 (cADMM FFT engine)
ls -d /usr/include/eigen3 /usr/local/include/eigen3 > gpurun_out/eigen_probe.txt 2>&1; echo "eigen probe rc=$?" >> gpurun_out/eigen_probe.txt; nproc >> gpurun_out/eigen_probe.txt
set -x
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2.csv \
  python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_bench.log 2>&1; echo "launch list rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_tc_dense -s 2 -c 1 \
  -o gpurun_out/prof_tc_pair python bench.py --steps 2 --warmup 3 --quick --no-cpu-baseline > gpurun_out/ncu_tc.log 2>&1; echo "tc full rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_rows_r2c|k_cols|k_mid" -s 20 -c 5 \
  -o gpurun_out/prof_fft_real python tools/fft_probe.py cadmm 24 > gpurun_out/ncu_fft.log 2>&1; echo "fft full rc=$?"
ls -la gpurun_out
