timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -s -p no:cacheprovider -k "fft4 or fft_engine" > gpurun_out/gputest_fft.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_fft.log
python tools/fft_probe.py cadmm 20 22 23 24 > gpurun_out/fft_probe.log 2>&1
CLB_FFT_TWO_LEVEL=1 python tools/fft_probe.py cadmm 22 23 24 >> gpurun_out/fft_probe.log 2>&1
python tools/fft_probe.py ista 20 22 24 >> gpurun_out/fft_probe.log 2>&1
cat gpurun_out/fft_probe.log
