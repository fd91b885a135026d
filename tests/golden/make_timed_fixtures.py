#!/usr/bin/env python3
"""Generates tests/golden/c3_fixture.npz -- oracle states at the configuration the bench times.

BASELINE config 3: make_problem(2^20, 2^18, 2^12, seed=1), SolverConfig defaults (alpha = 1e-4,
tau = 0.9, literal pairing; cADMM rho = sigma = 0.1, tau1 = tau2 = 1).  The oracle
(oracle/circlasso_oracle.cpp, test infrastructure; its FFT engine agrees with the reference's
phase engine to <= 1e-12, tests/parallel_test.cpp:191-238) is stepped in fp64:

  ista_25, ista_200   x and r after 25 / 200 ISTA iterations (solvers.hpp:252-263)
  cadmm_5             z and x after 5 cADMM iterations (solvers.hpp:399-415)

For each state the fixture keeps, compactly (the full fp64 vectors are 8 MB each):
  * the support of the iterate as a packed bitmap plus its sha256 and size;
  * the l2 norms of the iterate and of the second vector;
  * the values at 32768 seeded sample positions (iterate) and 8192 (second vector);
  * the threshold margin of every entry: | |v_i| - g | with v the pre-threshold value of the
    last step (ISTA: v = x_{t-1} + tau delta_t, g = alpha; cADMM: v = x_t + nu_{t-1},
    g = alpha / sigma).  An fp32 solver can only disagree on the support where this margin is
    below its own rounding; SURVEY hard part 3.  Stored: the 256 smallest margins with their
    positions, and quantiles.

Run from the repo root: python tests/golden/make_timed_fixtures.py  (about 2 minutes).
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
OUT = os.path.join(ROOT, "tests", "golden", "c3_fixture.npz")
N_SAMPLE, M_SAMPLE, N_SMALLEST = 32768, 8192, 256


def sample_positions():
    rng = np.random.default_rng(20261017)
    return (np.sort(rng.choice(N, N_SAMPLE, replace=False)).astype(np.int64),
            np.sort(rng.choice(M, M_SAMPLE, replace=False)).astype(np.int64))


def support_record(prefix, x):
    bits = np.packbits(x != 0)
    return {f"{prefix}_support_bits": bits,
            f"{prefix}_support_sha256": np.frombuffer(hashlib.sha256(bits.tobytes()).digest(), dtype=np.uint8),
            f"{prefix}_nnz": np.int64(np.count_nonzero(x))}


def margin_record(prefix, v, g):
    marg = np.abs(np.abs(v) - g)
    order = np.argsort(marg, kind="stable")[:N_SMALLEST]
    return {f"{prefix}_margin_pos": order.astype(np.int64), f"{prefix}_margin_val": marg[order],
            f"{prefix}_margin_quantiles": np.quantile(marg, [0.0, 1e-6, 1e-5, 1e-4, 1e-3, 0.5]),
            f"{prefix}_threshold": np.float64(g)}


def main():
    t0 = time.time()
    p = orc.make_problem(N, M, K, SEED)
    ns, ms = sample_positions()
    rec = {"n": np.int64(N), "m": np.int64(M), "k": np.int64(K), "seed": np.int64(SEED),
           "sample_n": ns, "sample_m": ms,
           "y_sha256": np.frombuffer(hashlib.sha256(p.y.tobytes()).digest(), dtype=np.uint8)}

    ista = orc.Ista(p.row, p.omega, p.y)
    sc = ista.scalars()
    done = 0
    for target in (25, 200):
        ista.step(target - 1 - done, orc.ENGINE_FFT)
        x_prev = ista.get("x")
        ista.step(1, orc.ENGINE_FFT)
        done = target
        x, r, d = ista.get("x"), ista.get("r"), ista.get("delta")
        pre = f"ista_{target}"
        rec.update(support_record(pre, x))
        rec.update(margin_record(pre, x_prev + sc["tau"] * d, sc["threshold"]))
        rec[f"{pre}_x_norm"] = np.float64(np.linalg.norm(x))
        rec[f"{pre}_r_norm"] = np.float64(np.linalg.norm(r))
        rec[f"{pre}_x_sample"] = x[ns]
        rec[f"{pre}_r_sample"] = r[ms]
        print(f"{pre}: nnz {np.count_nonzero(x)}, |x| {np.linalg.norm(x):.6e}, min margin "
              f"{rec[pre + '_margin_val'][0]:.3e} ({time.time() - t0:.0f} s)", flush=True)

    cadmm = orc.Cadmm(p.row, p.omega, p.y)
    csc = cadmm.scalars()
    cadmm.step(4, orc.ENGINE_FFT)
    nu_prev = cadmm.get("nu")
    cadmm.step(1, orc.ENGINE_FFT)
    z, x = cadmm.get("z"), cadmm.get("x")
    pre = "cadmm_5"
    rec.update(support_record(pre, z))
    rec.update(margin_record(pre, x + nu_prev, csc["threshold"]))
    rec[f"{pre}_z_norm"] = np.float64(np.linalg.norm(z))
    rec[f"{pre}_x_norm"] = np.float64(np.linalg.norm(x))
    rec[f"{pre}_z_sample"] = z[ns]
    rec[f"{pre}_x_sample"] = x[ns]
    print(f"{pre}: nnz {np.count_nonzero(z)}, |z| {np.linalg.norm(z):.6e}, min margin "
          f"{rec[pre + '_margin_val'][0]:.3e} ({time.time() - t0:.0f} s)", flush=True)

    np.savez_compressed(OUT, **rec)
    print(f"wrote {OUT} ({os.path.getsize(OUT) / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
