"""BASELINE config 5 on one GPU: compressed-domain deblurring of a 4096x4096 star field
(gen_star_field(4096, 4096, 0.1, 1), 1-D blur L=5, m=n/2, alpha=1e-2) through
run_deblur_experiment (deblur.hpp:141-156).  FFT engine for the full recovery, the direct engine
for a timed pair of iterations.  Prints one JSON object."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_02244_b200 as cl

W = H = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 300
direct_iters = int(sys.argv[3]) if len(sys.argv) > 3 else 2
out = {"workload": f"BASELINE config 5: deblur {W}x{H} star field (density 0.1, seed 1), L=5, m=n/2, alpha=1e-2, cADMM"}
t0 = time.perf_counter()
img = cl.gen_star_field(W, H, 0.1, 1)
out["gen_s"] = time.perf_counter() - t0
for eng, it in (("fft", iters), ("direct", direct_iters)):
    if it <= 0:
        continue
    cfg = cl.SolverConfig(alpha=1e-2, max_iter=it, check_every=it, use_fft=(eng == "fft"))
    t0 = time.perf_counter()
    res = cl.run_deblur_experiment(img, 5, W * H // 2, cfg, 1)
    wall = time.perf_counter() - t0
    rep = res.report
    run_s = rep.total_seconds - rep.setup_seconds
    out[eng] = {"iterations": rep.iterations, "wall_s": wall, "setup_s": rep.setup_seconds, "solve_s": run_s,
                "iters_per_s": rep.iterations / run_s if run_s > 0 else None, "mse_vs_truth": res.mse_vs_truth,
                "normalized_mse": res.normalized_mse, "error_map_mean": res.error_map_mean}
    print(json.dumps({eng: out[eng]}), file=sys.stderr, flush=True)
print(json.dumps(out))
