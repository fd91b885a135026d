timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "fft4 or fft_engine" 2>&1 | tail -2
python tools/fft_probe.py cadmm 20 22 24 2>&1; python tools/fft_probe.py ista 20 24 2>&1
