"""Runs `iters` solver iterations at a given size (profiling driver)."""
import sys, os, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_02244_b200 as cl
ap = argparse.ArgumentParser()
ap.add_argument("--kind", default="ista"); ap.add_argument("--n", type=int, default=1 << 20)
ap.add_argument("--m", type=int, default=1 << 18); ap.add_argument("--k", type=int, default=1 << 12)
ap.add_argument("--iters", type=int, default=1); ap.add_argument("--fft", action="store_true")
a = ap.parse_args()
p = cl.make_problem(a.n, a.m, a.k, 1)
st = (cl.ista_setup if a.kind == "ista" else cl.cadmm_setup)(p.op, p.measurements, cl.SolverConfig(use_fft=a.fft))
st.step(a.iters); st.synchronize()
print("done", st.last_step_ms())
