#!/usr/bin/env python3
"""sha256 of the FFT engine's iterate after 5 steps at several sizes: a bitwise A/B check between two builds of
the library (a change that only reorders loads must leave every bit unchanged)."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1707_02244_b200 as cl  # noqa: E402

for kind, lg in [("ista", 16), ("ista", 18), ("ista", 20), ("cadmm", 20), ("cadmm", 22), ("cadmm", 23), ("cadmm", 24),
                 ("ista", 24)]:
    n = 1 << lg
    p = cl.make_problem(n, n // 4, max(1, n // 256), 1)
    st = (cl.cadmm_setup if kind == "cadmm" else cl.ista_setup)(p.op, p.measurements, cl.SolverConfig(use_fft=True))
    st.step(5)
    st.synchronize()
    x = np.ascontiguousarray(st.get("z" if kind == "cadmm" else "x"))
    print(f"{kind} 2^{lg}: {hashlib.sha256(x.tobytes()).hexdigest()[:16]}", flush=True)
    del st
