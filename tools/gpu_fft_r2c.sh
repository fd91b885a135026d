# FFT engine: parity tests (incl. real vs complex plans), then step times: real vs complex plans and
# three-level vs two-level (N1 = 2048, 8-column tiles)
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_timed_configs.py -m gpu -x -q -s -p no:cacheprovider -k "fft or deblur or smoke or padded or small" > gpurun_out/gputest_fft.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/gputest_fft.log
for mode in 0 1; do
  CLB_FFT_C2C=$mode timeout 300 python tools/fft_probe.py cadmm 20 22 23 24 2>&1 | sed "s/^/c2c=$mode /"
  CLB_FFT_C2C=$mode timeout 300 python tools/fft_probe.py ista 22 24 2>&1 | sed "s/^/c2c=$mode /"
done | tee gpurun_out/fft_r2c_probe.log
CLB_FFT_TWO_LEVEL=1 timeout 300 python tools/fft_probe.py cadmm 22 23 24 2>&1 | sed "s/^/two_level /" | tee -a gpurun_out/fft_r2c_probe.log
