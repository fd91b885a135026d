import sys, time
sys.path.insert(0, "/root/repo")
import paper_1707_02244_b200 as cl
p = cl.make_problem(1 << 20, 1 << 18, 1 << 12, 1)
for rep in range(3):
    t0 = time.perf_counter()
    st = cl.ista_setup(p.op, p.measurements, cl.SolverConfig(use_fft=True, max_iter=20, check_every=20))
    t1 = time.perf_counter()
    r = cl.api._run(st, None, st.cfg)
    t2 = time.perf_counter()
    del st
    t3 = time.perf_counter()
    print(f"fft ista: setup {t1-t0:.4f}s (report {r.setup_seconds:.4f}) run {t2-t1:.4f}s (report total {r.total_seconds:.4f}) destroy {t3-t2:.4f}s")
