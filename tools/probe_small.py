"""Small-config timing (graph replay): BASELINE configs 1 and 2, both engines."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_02244_b200 as cl
p = cl.make_problem(4096, 1024, 64, 1)
for kind, iters in (("ista", 1000), ("cadmm", 200)):
    for fft in (False, True):
        st = (cl.ista_setup if kind == "ista" else cl.cadmm_setup)(p.op, p.measurements, cl.SolverConfig(use_fft=fft))
        st.step(10); st.synchronize()
        st.step(iters); st.synchronize()
        ms = st.last_step_ms()
        cfg = cl.SolverConfig(max_iter=iters, check_every=iters, use_fft=fft)
        t0 = time.perf_counter()
        rep = (cl.ista_run if kind == "ista" else cl.cadmm_run)(p.measurements, p.op, cfg)
        e2e = time.perf_counter() - t0
        print(f"{kind} n=4096 fft={fft}: {iters} iters in {ms:.2f} ms device ({iters/ms*1e3:.0f} it/s); "
              f"ista_run/cadmm_run e2e {e2e*1e3:.1f} ms", flush=True)
