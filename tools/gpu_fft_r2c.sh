# FFT engine: real plans vs complex plans (parity tests, then step times)
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_timed_configs.py -m gpu -x -q -s -p no:cacheprovider -k "fft or deblur or smoke or padded or small" > gpurun_out/gputest_fft.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/gputest_fft.log
for mode in 0 1; do
  CLB_FFT_C2C=$mode timeout 300 python tools/fft_probe.py cadmm 20 22 23 24 2>&1 | sed "s/^/c2c=$mode /"
  CLB_FFT_C2C=$mode timeout 300 python tools/fft_probe.py ista 22 24 2>&1 | sed "s/^/c2c=$mode /"
done | tee gpurun_out/fft_r2c_probe.log
