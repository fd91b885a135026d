# cta_group::2 pair kernel vs single-CTA kernel: correctness (sampled fp64 sums) and timing;
# tc_probe_mmaonly: the MMA pipe alone (no tile production after the first fill, no drain)
set -x
cd tools/microbench
for lg in 18 20; do
  for pair in 1 0; do
    CLB_TC_PAIR=$pair timeout 120 ./tc_probe $lg 10; echo "rc=$? pair=$pair lg=$lg"
    CLB_TC_PAIR=$pair timeout 120 ./tc_probe_mmaonly $lg 10 | grep time; echo "mmaonly rc=$? pair=$pair lg=$lg"
  done
done 2>&1 | tee ../../gpurun_out/tc_pair.log
