import sys, os
sys.path.insert(0, "/root/repo")
import paper_1707_02244_b200 as cl
p = cl.make_problem(4096, 1024, 64, 1)
st = cl.ista_setup(p.op, p.measurements)
st.step(200); st.synchronize()
print("ms", st.last_step_ms())
