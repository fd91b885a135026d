import os, sys
sys.path.insert(0, os.getcwd())
import paper_1707_02244_b200 as cl
for lg in (22, 24):
    n = 1 << lg
    p = cl.make_problem(n, n // 4, n // 256, 1)
    st = cl.cadmm_setup(p.op, p.measurements, cl.SolverConfig(use_fft=True))
    st.profile(2)
    st.step(5); st.synchronize()
    print(lg, [round(x, 4) for x in st.phase_ms()], flush=True)
    del st
