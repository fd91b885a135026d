"""Prints one bench line's rate and phase times (tools/gpu_ab.sh): python tools/ab_summary.py TAG < bench.json"""
import json
import sys

d = json.loads(sys.stdin.read().strip().splitlines()[-1])
adm = d.get("admm") or {}
print(sys.argv[1], round(d["value"], 2), [round(x, 4) for x in d["roofline"]["phase_ms"]],
      round(adm.get("value", 0.0), 2), [round(x, 4) for x in adm.get("phase_ms", [])])
