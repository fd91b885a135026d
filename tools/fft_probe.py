#!/usr/bin/env python3
"""FFT-engine step time and algorithmic HBM rate at large n (cADMM: 3 products per iteration; ISTA: 2),
CUDA-graph replay, L2 flushed between steps.  CLB_FFT_TWO_LEVEL=1 selects the two-level plan."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1707_02244_b200 as cl  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "cadmm"
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for lg in [int(a) for a in sys.argv[2:]] or [20, 22, 23, 24]:
    n = 1 << lg
    p = cl.make_problem(n, n // 4, n // 256, 1)
    st = (cl.cadmm_setup if kind == "cadmm" else cl.ista_setup)(p.op, p.measurements, cl.SolverConfig(use_fft=True))
    st.step(3)
    st.synchronize()
    import ctypes as C
    from paper_1707_02244_b200._native import lib
    sp = C.c_void_p()
    lib.cl_solver_stream(st.handle, C.byref(sp))
    stream = torch.cuda.ExternalStream(sp.value)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    for a, b in ev:
        with torch.cuda.stream(stream):
            flush.zero_()
            a.record(stream)
        st.step(1)
        with torch.cuda.stream(stream):
            b.record(stream)
    st.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / len(ev)
    nprod = 3 if kind == "cadmm" else 2
    print(f"{kind} n=2^{lg} plan={'two' if os.environ.get('CLB_FFT_TWO_LEVEL') else 'default'}: {ms:.4f} ms/step, "
          f"{nprod * 48 * n / (ms * 1e-3) / 1e9:.0f} GB/s at 48 n bytes per product", flush=True)
    del st
