# A/B on one box for an FFT-engine change: bitwise hashes and step times of the in-tree library (B) against
# _exp/oldlib/libcirclasso_b200.so (A), then the FFT parity tests on B
set -x
rm -rf /tmp/A && mkdir -p /tmp/A && cp -r paper_1707_02244_b200 tools /tmp/A/
cp _exp/oldlib/libcirclasso_b200.so /tmp/A/paper_1707_02244_b200/_lib/libcirclasso_b200.so
(cd /tmp/A && python tools/fft_hash.py) > gpurun_out/hash_A.txt 2>&1
python tools/fft_hash.py > gpurun_out/hash_B.txt 2>&1
diff gpurun_out/hash_A.txt gpurun_out/hash_B.txt && echo "BITWISE IDENTICAL"
for r in 1 2; do
  (cd /tmp/A && python tools/fft_probe.py cadmm 22 24 && python tools/fft_probe.py ista 20 24) 2>&1 | sed 's/^/A /'
  (python tools/fft_probe.py cadmm 22 24 && python tools/fft_probe.py ista 20 24) 2>&1 | sed 's/^/B /'
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "fft" 2>&1 | tail -2
