#!/usr/bin/env python3
"""Where the e2e time goes: ista_run at BASELINE config 3 (20 iterations, the bench's e2e call) with
CLB_TRACE=1 stage timings from the library on stderr, plus the Python-side wall clock."""
import os
import sys
import time

os.environ.setdefault("CLB_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_02244_b200 as cl  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "ista"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
p = cl.make_problem(1 << 20, 1 << 18, 1 << 12, 1)
run = cl.ista_run if kind == "ista" else cl.cadmm_run
for rep in range(4):
    print(f"---- call {rep}", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    r = run(p.measurements, p.op, cl.SolverConfig(max_iter=iters, check_every=iters))
    dt = time.perf_counter() - t0
    print(f"call {rep}: {dt * 1e3:.1f} ms wall, {iters / dt:.1f} it/s, setup {r.setup_seconds * 1e3:.1f} ms, "
          f"total {r.total_seconds * 1e3:.1f} ms", file=sys.stderr, flush=True)

# per-step device time of a fresh state: single synced steps, then back-to-back runs
import ctypes as C  # noqa: E402
from paper_1707_02244_b200._native import lib  # noqa: E402
os.environ["CLB_TRACE"] = "0"
st = (cl.ista_setup if kind == "ista" else cl.cadmm_setup)(p.op, p.measurements)
ms = C.c_double()
seq = []
for i in range(12):
    st.step(1)
    st.synchronize()
    lib.cl_solver_last_step_ms(st.handle, C.byref(ms))
    seq.append(round(ms.value, 3))
print("single synced steps (ms):", seq, file=sys.stderr)
for k in (5, 20, 50):
    st.step(k)
    st.synchronize()
    lib.cl_solver_last_step_ms(st.handle, C.byref(ms))
    print(f"{k} back-to-back steps: {ms.value / k:.3f} ms/step", file=sys.stderr)
    time.sleep(1.0)
    st.step(k)
    st.synchronize()
    lib.cl_solver_last_step_ms(st.handle, C.byref(ms))
    print(f"{k} back-to-back steps after 1 s idle: {ms.value / k:.3f} ms/step", file=sys.stderr)
