# ncu --set full of the FFT engine's kernels (C3 ISTA n = 2^20, cADMM n = 2^24), summarised to CSV on the box
# (the reports themselves stay there: gpurun_out/ is capped at 64 MiB)
set -x
NCU=/usr/local/cuda/bin/ncu
mkdir -p /tmp/ncu
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_rows_r2c|k_cols|k_mid" -s 40 -c 5 \
  -o /tmp/ncu/prof_fft24 python tools/fft_probe.py cadmm 24 > gpurun_out/ncu_fft24.log 2>&1; echo "fft24 rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_rows_r2c|k_cols" -s 30 -c 5 \
  -o /tmp/ncu/prof_fft20 python tools/fft_probe.py ista 20 > gpurun_out/ncu_fft20.log 2>&1; echo "fft20 rc=$?"
for r in prof_fft24 prof_fft20; do $NCU -i /tmp/ncu/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null; done
ls -la gpurun_out
