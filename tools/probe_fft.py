"""FFT-engine timing probe: python tools/probe_fft.py"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_02244_b200 as cl
for kind, n, m, k in (("ista", 4096, 1024, 64), ("cadmm", 4096, 1024, 64), ("ista", 1 << 20, 1 << 18, 1 << 12),
                      ("cadmm", 1 << 20, 1 << 18, 1 << 12), ("cadmm", 1 << 24, 1 << 22, 1 << 16), ("ista", 1 << 24, 1 << 22, 1 << 16)):
    p = cl.make_problem(n, m, k, 1)
    st = (cl.ista_setup if kind == "ista" else cl.cadmm_setup)(p.op, p.measurements, cl.SolverConfig(use_fft=True))
    st.profile(True)
    st.step(3); st.synchronize()
    it = 50
    st.step(it); st.synchronize()
    ms = st.last_step_ms() / it
    st.step_checked()
    print(f"fft {kind} n={n}: {ms:.4f} ms/iter = {1e3/ms:.1f} it/s  phases {['%.3f'%v for v in st.phase_ms()]}", flush=True)
