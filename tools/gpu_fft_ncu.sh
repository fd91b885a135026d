# ncu --set full of the FFT engine's kernels: C3 ISTA (n = 2^20, real FINE plan) and cADMM n = 2^24 (three-level
# real plan)
set -x
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_rows_r2c|k_cols|k_mid" -s 40 -c 5 \
  -o gpurun_out/prof_fft24 python tools/fft_probe.py cadmm 24 > gpurun_out/ncu_fft24.log 2>&1; echo "fft24 rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_rows_r2c|k_cols" -s 30 -c 5 \
  -o gpurun_out/prof_fft20 python tools/fft_probe.py ista 20 > gpurun_out/ncu_fft20.log 2>&1; echo "fft20 rc=$?"
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -s 200 -c 60 --csv \
  --log-file gpurun_out/launches_fft20.csv python tools/fft_probe.py ista 20 > /dev/null 2>&1; echo "list rc=$?"
