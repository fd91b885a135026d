# FFT engine plan comparison at large n: three-level (default) vs two-level (N1 = 2048, 8-column tiles)
set -x
for tl in "" 1; do
  CLB_FFT_TWO_LEVEL=$tl timeout 300 python tools/fft_probe.py cadmm 22 23 24 2>&1 | sed "s/^/two_level=$tl /"
  CLB_FFT_TWO_LEVEL=$tl timeout 300 python tools/fft_probe.py ista 24 2>&1 | sed "s/^/two_level=$tl /"
done | tee gpurun_out/fft_plans.log
CLB_FFT_TWO_LEVEL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "three_level or real_plan" 2>&1 | tail -3
