"""Small solves on every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck):
    compute-sanitizer --tool memcheck python tools/sanitize.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_02244_b200 as cl

for n, m, k in ((1000, 300, 10), (4096, 1024, 64), (1 << 14, 1 << 12, 64), (1 << 17, 1 << 15, 512)):
    p = cl.make_problem(n, m, k, 2)
    for fft in (False, True):
        if fft and (n & (n - 1)):
            continue
        for run in (cl.ista_run, cl.cadmm_run):
            rep = run(p.measurements, p.op, cl.SolverConfig(max_iter=4, check_every=2, use_fft=fft),
                      truth=p.signal.values)
            print(f"n={n} {run.__name__} fft={fft}: {rep.iterations} iterations, metric {rep.final_metric:.3e}",
                  flush=True)

# the tcgen05 dense-product kernel (k_tc_dense) in both operand formats: fp16 2-term split (n >= 2^18)
# and 3xTF32 (smaller n), on CTA pairs (cta_group::2) and single CTAs, unsharded and sharded (tile_lo > 0)
# through the phase API
import ctypes as C  # noqa: E402

from paper_1707_02244_b200._native import lib as L  # noqa: E402

for n in (1 << 16, 1 << 18):
    p = cl.make_problem(n, n // 4, n // 256, 3)
    for setup in (cl.ista_setup, cl.cadmm_setup):
        st = setup(p.op, p.measurements)
        st.step(2)
        st.synchronize()
        # shard 1 of 2 (tile_lo > 0, whole CTA pairs) and shard 1 of 3 (odd tile range: single CTAs)
        for world in (2, 3):
            sh = setup(p.op, p.measurements)
            assert L.cl_solver_shard(sh.handle, 1, world) == 0
            for ph in range(2 if setup is cl.ista_setup else 3):
                assert L.cl_solver_run_phase(sh.handle, ph) == 0
            sh.synchronize()
        print(f"tc n={n} {setup.__name__}: 2 steps + one shard-1-of-2 and one shard-1-of-3 step", flush=True)

# the dense ADMM baseline (Gram matrix, blocked Gauss-Jordan, fused mat-vec; n not a multiple of 64) and the
# library-owned sharded data plane (peer-copy transport, 2 ranks on one device)
p = cl.make_problem(200, 100, 10, 4)
rep = cl.admm_dense_run(p.measurements, p.op, cl.SolverConfig(max_iter=4, check_every=2), truth=p.signal.values)
print(f"dense admm n=200: {rep.iterations} iterations, metric {rep.final_metric:.3e}", flush=True)
p = cl.make_problem(1 << 16, 1 << 14, 256, 5)
for kind in ("ista", "cadmm"):
    for transport in ("copy", "peer"):
        g = cl.ShardedSolve(kind, p.op, p.measurements, cl.SolverConfig(max_iter=2, check_every=2), devices=[0, 0],
                            transport=transport)
        print(f"sharded {kind} 2 ranks ({transport}): {g.run(truth=p.signal.values).iterations} iterations",
              flush=True)

if "--large" in sys.argv:  # the three-level FFT plan (n >= 2^22): memcheck only (slow under racecheck)
    p = cl.make_problem(1 << 22, 1 << 20, 1 << 14, 6)
    for run in (cl.ista_run, cl.cadmm_run):
        rep = run(p.measurements, p.op, cl.SolverConfig(max_iter=2, check_every=2, use_fft=True))
        print(f"three-level fft n=2^22 {run.__name__}: {rep.iterations} iterations", flush=True)
