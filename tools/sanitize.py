"""Small solves on every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck):
    compute-sanitizer --tool memcheck python tools/sanitize.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_02244_b200 as cl

for n, m, k in ((1000, 300, 10), (4096, 1024, 64), (1 << 14, 1 << 12, 64), (1 << 17, 1 << 15, 512)):
    p = cl.make_problem(n, m, k, 2)
    for fft in (False, True):
        if fft and (n & (n - 1)):
            continue
        for run in (cl.ista_run, cl.cadmm_run):
            rep = run(p.measurements, p.op, cl.SolverConfig(max_iter=4, check_every=2, use_fft=fft),
                      truth=p.signal.values)
            print(f"n={n} {run.__name__} fft={fft}: {rep.iterations} iterations, metric {rep.final_metric:.3e}",
                  flush=True)
