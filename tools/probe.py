"""Quick per-phase timing probe (not the bench): python tools/probe.py"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1707_02244_b200 as cl

def probe(kind, n, m, k, iters=3):
    t0 = time.time()
    p = cl.make_problem(n, m, k, 1)
    t1 = time.time()
    st = (cl.ista_setup if kind == "ista" else cl.cadmm_setup)(p.op, p.measurements)
    t2 = time.time()
    st.profile(True)
    st.step(1); st.synchronize()
    st.step(iters); st.synchronize()
    ms = st.last_step_ms() / iters
    st.step_checked()
    ph = st.phase_ms()
    flops = 4.0 * m * n if kind == "ista" else 6.0 * n * n
    print(f"{kind} n={n} m={m}: gen {t1-t0:.2f}s setup {t2-t1:.2f}s  {ms:.3f} ms/iter  {flops/ms/1e9:.2f} TFLOP/s  phases(ms)={['%.3f'%v for v in ph]}", flush=True)

if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "ista20":
        probe("ista", 1 << 20, 1 << 18, 1 << 12, 3)
        sys.exit(0)
    print("ffma peak TF/s", cl.ffma_peak_tflops(0))
    probe("ista", 4096, 1024, 64, 20)
    probe("cadmm", 4096, 1024, 64, 20)
    probe("ista", 1 << 20, 1 << 18, 1 << 12, 3)
    probe("cadmm", 1 << 18, 1 << 16, 1 << 10, 3)
