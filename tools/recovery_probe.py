"""Time-to-recovery probe: iterations and seconds until MSE(x, x*) <= target
(paper protocol target 1e-4) through the public API.

    python tools/recovery_probe.py [n_log2] [engine fft|direct] [kind ista|cadmm] [max_iter]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_02244_b200 as cl

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 20
engine = sys.argv[2] if len(sys.argv) > 2 else "fft"
kind = sys.argv[3] if len(sys.argv) > 3 else "ista"
max_iter = int(sys.argv[4]) if len(sys.argv) > 4 else 5000
n = 1 << lg
p = cl.make_problem(n, n // 4, max(1, n // 256), 1)
for target in (1e-4, 1e-5, 1e-6):
    cfg = cl.SolverConfig(max_iter=max_iter, check_every=10, target_mse=target, use_fft=(engine == "fft"))
    run = cl.ista_run if kind == "ista" else cl.cadmm_run
    t0 = time.perf_counter()
    rep = run(p.measurements, p.op, cfg, truth=p.signal.values)
    wall = time.perf_counter() - t0
    print(f"{kind} n=2^{lg} {engine}: target {target:g} reached={rep.reached_target} iterations={rep.iterations} "
          f"final_mse={rep.final_metric:.3e} setup={rep.setup_seconds:.3f}s total={rep.total_seconds:.3f}s wall={wall:.3f}s",
          flush=True)
