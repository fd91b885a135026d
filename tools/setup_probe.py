"""Where does an ista_run/cadmm_run call spend its host time?  (e2e diagnostics)"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_02244_b200 as cl

n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
p = cl.make_problem(n, n // 4, n // 256, 1)
cl.ista_run(p.measurements, p.op, cl.SolverConfig(max_iter=2, check_every=2))  # warm the context
for kind in ("ista", "cadmm"):
    setup = cl.ista_setup if kind == "ista" else cl.cadmm_setup
    for rep in range(2):
        t0 = time.perf_counter()
        st = setup(p.op, p.measurements, cl.SolverConfig(max_iter=20, check_every=20))
        t1 = time.perf_counter()
        r = cl.api._run(st, None, st.cfg)
        t2 = time.perf_counter()
        del st
        t3 = time.perf_counter()
        print(f"{kind}: setup call {t1-t0:.3f}s (report setup {r.setup_seconds:.3f}s)  run call {t2-t1:.3f}s "
              f"(report total {r.total_seconds:.3f}s)  destroy {t3-t2:.3f}s", flush=True)
pr = cProfile.Profile()
pr.enable()
cl.ista_run(p.measurements, p.op, cl.SolverConfig(max_iter=20, check_every=20))
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
