# FFT engine at L2-resident sizes: FINE launches (half the work per CTA) vs the default tiles; parity subset
set -x
for f in 0 1; do
  CLB_FFT_FINE=$f timeout 300 python tools/fft_probe.py ista 20 21 2>&1 | sed "s/^/fine=$f /"
  CLB_FFT_FINE=$f timeout 300 python tools/fft_probe.py cadmm 20 21 2>&1 | sed "s/^/fine=$f /"
done | tee gpurun_out/fft_fine.log
for c in 1; do CLB_FFT_C2C=$c timeout 300 python tools/fft_probe.py ista 18 19 20 2>&1 | sed "s/^/c2c=$c /"; done | tee -a gpurun_out/fft_fine.log
CLB_FFT_C2C=0 timeout 300 python tools/fft_probe.py ista 18 19 2>&1 | sed "s/^/real /" | tee -a gpurun_out/fft_fine.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "fft" 2>&1 | tail -3
