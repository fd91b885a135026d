# A/B on one box: the in-tree library (B) against _exp/oldlib/libcirclasso_b200.so (A), the bench line (ISTA + cADMM
# phase times) twice each
set -x
rm -rf /tmp/A && mkdir -p /tmp/A && cp -r paper_1707_02244_b200 bench.py oracle tools MEASURED_PEAKS.json profiles /tmp/A/ 2>/dev/null
cp _exp/oldlib/libcirclasso_b200.so /tmp/A/paper_1707_02244_b200/_lib/libcirclasso_b200.so
for round in 1 2; do
  (cd /tmp/A && timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | python tools/ab_summary.py A)
  timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | python tools/ab_summary.py B
done
