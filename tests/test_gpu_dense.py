"""Dense ADMM baseline on the GPU (the paper's PADMM; reference solvers.hpp:267-327, padmm_phases
parallel.hpp:284-317, admm_dense_run :497-514) against the oracle's restatement (oracle/circlasso_oracle.cpp:
Cholesky inverse, ascending fp64 products).

* setup: B = (A~^T A~ + rho I)^-1 (fp64 on the device, stored fp32) and A~^T y~, incl. n not a multiple of the
  64-wide Gauss-Jordan block;
* iterations: x, z, u after a fixed count at rel l2 <= 1e-4 with identical support up to threshold ties;
* the reference's acceptance criterion 2 (solver equivalence, tests/acceptance.cpp:152-174): ISTA (proximal),
  dense ADMM and cADMM agree to l-inf 1e-4 at n = 512;
* n = 4096 (BASELINE configs 1/2 size, the dense cap): B against numpy's fp64 inverse of the Gram matrix.
"""
import numpy as np
import pytest

import paper_1707_02244_b200 as cl
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if cl.device_count() < 1:
        pytest.skip("no CUDA device")


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def op_of(p):
    return cl.PartialCirculantOperator(cl.CirculantMatrix(p.row), cl.SubsamplingMask(p.omega, p.n))


def gram_fp64(p):
    s = orc.spectral_norm(p.row)
    n = p.n
    idx = (np.arange(n)[None, :] - p.omega[:, None]) % n
    ad = p.row[idx] / s
    return ad.T @ ad + 0.1 * np.eye(n), ad.T @ (p.y / s)


@pytest.mark.parametrize("n,m,k,seed", [(256, 128, 25, 3), (1000, 400, 40, 5), (1024, 512, 51, 7)])
def test_admm_setup_matches_oracle(n, m, k, seed):
    p = orc.make_problem(n, m, k, seed)
    g = cl.admm_setup(op_of(p), p.y)
    o = orc.Admm(p.row, p.omega, p.y)
    eb, ea = rel(g.get("B"), o.get("B")), rel(g.get("aty"), o.get("aty"))
    print(f"n={n}: B rel {eb:.2e}, A^T y rel {ea:.2e}")
    assert eb <= 1e-6 and ea <= 1e-6  # fp32 storage of fp64 results
    assert np.array_equal(g.get("rhs"), g.get("aty"))  # rhs = A~^T y~ at t = 0 (solvers.hpp:312)


@pytest.mark.parametrize("n,m,k,seed,iters", [(256, 128, 25, 3, 50), (1024, 512, 51, 7, 200)])
def test_admm_steps_match_oracle(n, m, k, seed, iters):
    p = orc.make_problem(n, m, k, seed)
    g = cl.admm_setup(op_of(p), p.y)
    g.step(iters)
    o = orc.Admm(p.row, p.omega, p.y)
    o.step(iters)
    for f in ("x", "z", "u", "rhs"):
        e = rel(g.get(f), o.get(f))
        print(f"n={n} {iters} iterations: {f} rel {e:.2e}")
        assert e <= 1e-4, f
    gz, oz = g.get("z"), o.get("z")
    flips = np.flatnonzero((gz != 0) != (oz != 0))
    thr = o.scalars()["threshold"]
    v = o.get("x") + (o.get("u") + o.get("z") - o.get("x"))  # x_t + u_{t-1} (u_t = u_{t-1} + x_t - z_t)
    assert np.all(np.abs(np.abs(v[flips]) - thr) <= 1e-3 * thr), flips


def test_admm_dense_run_bookkeeping_and_errors():
    p = orc.make_problem(256, 128, 25, 11)
    cfg = cl.SolverConfig(target_mse=1e-4, max_iter=20000)
    rep = cl.admm_dense_run(p.y, op_of(p), cfg, truth=p.x_true)
    ref = orc.run("admm", p.row, p.omega, p.y, truth=p.x_true, max_iter=20000, target_mse=1e-4)
    assert rep.reached_target and ref.reached_target
    assert abs(rep.iterations - ref.iterations) <= 10  # the same check point, or the next one
    assert rep.footprint_bytes == cl.analytic_footprint(cl.FootprintKind.kDenseAdmm, 256, 128, 4)
    assert rep.setup_seconds <= rep.total_seconds
    with pytest.raises(cl.CapacityError):
        cl.admm_setup(op_of(p), p.y, cl.SolverConfig(dense_cap=128))
    with pytest.raises(cl.ParameterError):
        cl.admm_setup(op_of(p), p.y, cl.SolverConfig(rho=0.0))
    with pytest.raises(cl.DimensionError):
        cl.admm_setup(op_of(p), p.y[:-1])
    z = cl.admm_dense_run(np.zeros(128), op_of(p), cl.SolverConfig(max_iter=30))
    assert not np.any(z.final_x)  # y = 0: every solver returns exactly 0 (solvers_test.cpp:137-155)


def test_solver_equivalence_512():
    """acceptance.cpp:152-174: ISTA (proximal pairing), dense ADMM and cADMM, iterate-change target 1e-8,
    truth withheld, worst pairwise l-inf < 1e-4 (3 of the reference's 10 seeds)."""
    worst = 0.0
    for seed in (1, 2, 3):
        p = orc.make_problem(512, 256, 51, seed)
        cfg = cl.SolverConfig(target_mse=1e-8, max_iter=400000)
        xi = cl.ista_run(p.y, op_of(p), cl.SolverConfig(target_mse=1e-8, max_iter=400000,
                                                        pairing=cl.ThresholdPairing.kProximal)).final_x
        xa = cl.admm_dense_run(p.y, op_of(p), cfg).final_x
        xc = cl.cadmm_run(p.y, op_of(p), cfg).final_x
        worst = max(worst, np.max(np.abs(xi - xa)), np.max(np.abs(xa - xc)), np.max(np.abs(xi - xc)))
    print(f"solver equivalence: worst pairwise l-inf {worst:.2e}")
    assert worst < 1e-4


def test_admm_4096_inverse_vs_numpy():
    """The dense cap (n = 4096, m = 1024: BASELINE configs 1/2): B against numpy's fp64 inverse."""
    p = orc.make_problem(4096, 1024, 64, 1)
    G, aty = gram_fp64(p)
    g = cl.admm_setup(op_of(p), p.y)
    B = g.get("B")
    e = rel(B, np.linalg.inv(G))
    r = float(np.max(np.abs(B @ G - np.eye(4096))))
    print(f"n=4096: B rel {e:.2e} vs numpy inv, max |B G - I| {r:.2e}, A^T y rel {rel(g.get('aty'), aty):.2e}")
    assert e <= 1e-6 and r <= 1e-5 and rel(g.get("aty"), aty) <= 1e-6
    g.step(20)
    assert np.all(np.isfinite(g.get("z")))
