#!/usr/bin/env python3
"""Generates tests/golden/c3_recovery.npz -- the oracle's time-to-recovery runs at BASELINE config 3.

make_problem(2^20, 2^18, 2^12, seed=1), ista_run / cadmm_run (solvers.hpp:479-534, run_loop :426-472) with
SolverConfig(target_mse=1e-4, check_every=10) and the true signal, on the oracle's fp64 FFT engine
(oracle/circlasso_oracle.cpp; test infrastructure).  Stored per solver: the iteration count at which the
stop rule fired, whether the target was reached, the final MSE, the whole (iteration, MSE) trace, the
support of the final iterate (packed bitmap + sha256) and its values at 32768 seeded positions.

Run from the repo root: python tests/golden/make_recovery_fixture.py  (~20 minutes, single-threaded FFT).
"""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as orc  # noqa: E402

N, M, K, SEED = 1 << 20, 1 << 18, 1 << 12, 1
OUT = os.path.join(ROOT, "tests", "golden", "c3_recovery.npz")


def main():
    p = orc.make_problem(N, M, K, SEED)
    pos = np.sort(np.random.default_rng(20261018).choice(N, 32768, replace=False)).astype(np.int64)
    rec = {"y_sha256": np.frombuffer(hashlib.sha256(p.y.tobytes()).digest(), dtype=np.uint8), "sample_pos": pos}
    for kind in ("ista", "cadmm"):
        t0 = time.time()
        r = orc.run(kind, p.row, p.omega, p.y, truth=p.x_true, engine=orc.ENGINE_FFT, max_iter=20000,
                    target_mse=1e-4, check_every=10)
        bits = np.packbits(r.final_x != 0)
        rec.update({
            f"{kind}_iterations": np.int64(r.iterations), f"{kind}_reached": np.bool_(r.reached_target),
            f"{kind}_final_mse": np.float64(r.final_metric),
            f"{kind}_trace": np.array(r.trace, dtype=np.float64).reshape(-1, 2),
            f"{kind}_support_bits": bits,
            f"{kind}_support_sha256": np.frombuffer(hashlib.sha256(bits.tobytes()).digest(), dtype=np.uint8),
            f"{kind}_nnz": np.int64(np.count_nonzero(r.final_x)),
            f"{kind}_sample": r.final_x[pos], f"{kind}_norm": np.float64(np.linalg.norm(r.final_x)),
        })
        print(f"{kind}: {r.iterations} iterations, reached {r.reached_target}, final MSE {r.final_metric:.6e}, "
              f"nnz {np.count_nonzero(r.final_x)}, {time.time() - t0:.0f} s", flush=True)
    np.savez_compressed(OUT, **rec)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
