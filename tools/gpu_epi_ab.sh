# split-sum variants of the contiguous epilogues (CLB_EPI_SUM=0/1/2): bench phase times (ISTA) and the cADMM line
for r in 1 2; do for v in 0 1 2; do
  CLB_EPI_SUM=$v timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('sumv=$v', 'ista', round(d['value'],2), 'phases', [round(x,4) for x in d['roofline']['phase_ms']], 'admm', round((d.get('admm') or {}).get('value',0),2), (d.get('admm') or {}).get('phase_ms'))"
done; done
