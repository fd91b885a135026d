# ncu --set full of the FFT engine's passes at 2^24 (cADMM), report brought back for source-level reading here
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_rows_r2c|k_cols|k_mid" -s 20 -c 4 \
  -o gpurun_out/prof_fft24_new python tools/fft_probe.py cadmm 24 > gpurun_out/ncu_fft24_new.log 2>&1; echo "rc=$?"
