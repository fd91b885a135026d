"""Pins the CPU oracle (oracle/) against the reference's own known answers.

The reference cannot be built in this image (no Eigen), so these KATs -- every
one taken from the reference test suite or the C++ standard, see
tests/golden/kats.json -- are what make the oracle a trustworthy checker for
the GPU parity tests.  CPU only.
"""
import math

import numpy as np
import pytest

from oracle import oracle as orc


def dense_circulant(row):
    # tests/oracles.hpp:20-27 -- element (i, j) = row[(j - i) mod n]
    n = len(row)
    return np.array([[row[(j - i) % n] for j in range(n)] for i in range(n)])


def random_vector(n, seed):
    # tests/solvers_test.cpp:39-44 -- SeededRng(seed).normal() draws
    return orc.rng_draws(seed, "normal", n)


def test_mt19937_64_standard_kat(kats):
    k = kats["mt19937_64_10000th"]
    draws = orc.mt19937_64(k["seed"], k["index"])
    assert int(draws[-1]) == int(k["value"])


def test_rng_transforms():
    # sensing.hpp:61-63: uniform = (u64 >> 11) * 2^-53 over the raw engine
    raw = orc.mt19937_64(42, 4)
    u = orc.rng_draws(42, "uniform", 4)
    assert np.array_equal(u, (raw >> np.uint64(11)).astype(np.float64) * 2.0 ** -53)
    # tests/sensing_test.cpp:21-67: ranges, moments, bounded ints
    u = orc.rng_draws(42, "uniform", 20000)
    assert u.min() >= 0.0 and u.max() < 1.0 and abs(u.mean() - 0.5) < 0.01
    z = orc.rng_draws(43, "normal", 20000)
    assert abs(z.mean()) < 0.05 and abs(z.var() - 1.0) < 0.05
    b = orc.rng_draws(44, "below", 70000, bound=7)
    counts = np.bincount(b.astype(int), minlength=7)
    assert np.all(np.abs(counts - 10000) < 5 * math.sqrt(10000))
    assert orc.rng_draws(44, "below", 1, bound=1)[0] == 0
    with pytest.raises(orc.OracleError):
        orc.rng_draws(44, "below", 1, bound=0)


def test_entry_rule_and_shift_products(kats):
    k = kats["entry_rule_3x3"]
    row = np.array(k["row"], float)
    cols = np.stack([orc.circ_matvec(row, e) for e in np.eye(3)], axis=1)
    assert np.array_equal(cols, np.array(k["dense"], float))
    k = kats["shift_products"]
    assert np.array_equal(orc.circ_matvec(k["row"], k["x"]), k["Cx"])
    assert np.array_equal(orc.circ_matvec(k["row"], k["x"], transpose=True), k["CTx"])
    assert np.allclose(orc.circ_matvec(k["row"], k["x"], use_fft=True), k["Cx"], atol=1e-14)


def test_soft_threshold(kats):
    for v, g, want in kats["soft_threshold"]["cases"]:
        assert orc.soft_threshold(v, g)[0] == want


def test_mask_gram_inverse(kats):
    k = kats["mask_gram_inverse"]
    assert np.allclose(orc.mask_gram_inverse(k["omega"], k["n"], k["rho"]), k["d"], rtol=1e-15)
    with pytest.raises(orc.OracleError):
        orc.mask_gram_inverse(k["omega"], k["n"], 0.0)


def test_spectral_norm(kats):
    n = kats["spectral_norm_identity"]["n"]
    assert abs(orc.spectral_norm(np.eye(n)[0]) - 1.0) < 1e-12
    k = kats["spectral_norm_scaled_shift"]
    assert abs(orc.spectral_norm(k["row"]) - k["value"]) < 1e-12
    # tests/circulant_test.cpp:247-256 -- equals the largest singular value
    for n in (2, 8, 32, 128):
        row = random_vector(n, 800 + n)
        want = np.linalg.svd(dense_circulant(row), compute_uv=False)[0]
        assert abs(orc.spectral_norm(row) - want) <= 1e-10 * want


def test_gram_inverse(kats):
    k = kats["gram_singular"]
    with pytest.raises(orc.OracleError) as e:
        orc.regularized_gram_inverse(k["row"], k["rho"], k["sigma_singular"])
    assert e.value.code == orc.ESINGULAR
    orc.regularized_gram_inverse(k["row"], k["rho"], k["sigma_ok"])
    for bad in ((-0.1, 0.1), (0.1, -0.1), (0.0, 0.0)):
        with pytest.raises(orc.OracleError) as e:
            orc.regularized_gram_inverse(k["row"], *bad)
        assert e.value.code == orc.EPARAM
    # tests/circulant_test.cpp:163-179 -- matches dense inversion
    for n in (4, 16, 64, 256):
        row = random_vector(n, 500 + n)
        b = orc.regularized_gram_inverse(row, 0.1, 0.1)
        C = dense_circulant(row)
        want = np.linalg.inv(0.1 * C.T @ C + 0.1 * np.eye(n))
        got = dense_circulant(b)
        assert np.linalg.norm(got - want) / max(1.0, np.linalg.norm(want)) < 1e-8


def test_matvec_paths_vs_dense():
    # tests/circulant_test.cpp:59-74 (naive 1e-12, FFT 1e-10), incl. non-power-of-two n
    for n in (1, 2, 3, 5, 16, 64, 97, 256):
        row = random_vector(n, 40 + n)
        x = random_vector(n, 80 + n)
        D = dense_circulant(row)
        for tr, want in ((False, D @ x), (True, D.T @ x)):
            scale = max(1.0, np.linalg.norm(want))
            assert np.linalg.norm(orc.circ_matvec(row, x, transpose=tr) - want) / scale < 1e-12
            assert np.linalg.norm(orc.circ_matvec(row, x, transpose=tr, use_fft=True) - want) / scale < 1e-10


def test_dft_vs_direct_series():
    # tests/fft_test.cpp:47-57
    for n in (1, 2, 3, 8, 17, 64, 257):
        x = random_vector(n, 900 + n)
        jk = np.outer(np.arange(n), np.arange(n))
        want = (x[None, :] * np.exp(-2j * np.pi * jk / n)).sum(axis=1)
        got = orc.dft(x)
        assert np.max(np.abs(got - want)) / max(1.0, np.max(np.abs(want))) < 1e-10
        assert np.max(np.abs(orc.idft_real(got) - x)) < 1e-12 * max(1.0, np.max(np.abs(x)))
    with pytest.raises(orc.OracleError) as e:  # tests/fft_test.cpp:80-90
        orc.idft_real(np.array([0, 1j, 0, 0]))
    assert e.value.code == orc.ECONSIST


def test_compose_and_blur(kats):
    k = kats["blur_delta"]
    B = orc.blur_row(k["n"], k["L"])
    delta = np.zeros(k["n"])
    delta[0] = 1.0
    y = orc.circ_matvec(B, delta, use_fft=True)
    for i in range(k["n"]):
        assert abs(y[i] - (k["value"] if i in k["hit"] else 0.0)) < 1e-12
    # tests/circulant_test.cpp:231-245
    for n in (2, 8, 64, 128):
        c, b = random_vector(n, 600 + n), random_vector(n, 700 + n)
        want = dense_circulant(c) @ dense_circulant(b)
        got = dense_circulant(orc.circ_compose(c, b))
        assert np.linalg.norm(got - want) / max(1.0, np.linalg.norm(want)) < 1e-10


def test_generation_contracts(kats):
    k = kats["floor_k"]
    v, s = orc.gen_sparse_signal(k["n"], k["k"], k["seed"])
    assert len(s) == 409 and np.count_nonzero(v) == 409 and np.all(np.diff(s) > 0)
    k = kats["star_field"]
    px = orc.gen_star_field(k["width"], k["height"], k["density"], k["seed"])
    lit = px[px != 0]
    assert len(lit) == k["lit"] and lit.min() >= k["lo"] and lit.max() < k["hi"]
    # tests/sensing_test.cpp:69-81 -- bit reproducibility
    a, b = orc.make_problem(128, 64, 12, 9), orc.make_problem(128, 64, 12, 9)
    for f in ("row", "omega", "x_true", "support", "y"):
        assert np.array_equal(getattr(a, f), getattr(b, f))
    c = orc.make_problem(128, 64, 12, 10)
    assert not np.array_equal(a.row, c.row)
    # tests/sensing_test.cpp:141-175 -- mask contract, measure vs dense
    row, om = orc.gen_circulant_sensing(16, 16, 3)
    assert np.array_equal(om, np.arange(16))
    row, om = orc.gen_circulant_sensing(64, 24, 5)
    sv, _ = orc.gen_sparse_signal(64, 6, 5)
    want = dense_circulant(row)[om] @ sv
    assert np.linalg.norm(orc.measure(row, om, sv) - want) / max(1, np.linalg.norm(want)) < 1e-10
    for bad in ((8, 0), (8, 9)):
        with pytest.raises(orc.OracleError):
            orc.gen_circulant_sensing(*bad, 1)


def test_identity_operator_ista(kats):
    k = kats["identity_ista"]
    n = k["n"]
    y = k["y_scale"] * random_vector(n, k["y_seed"])
    row = np.eye(n)[0]
    rep = orc.run("ista", row, np.arange(n), y, alpha=k["alpha"], proximal=True, max_iter=k["max_iter"],
                  target_mse=k["target"])
    assert rep.reached_target
    want = np.sign(y) * np.maximum(np.abs(y) - k["alpha"], 0.0)
    assert np.max(np.abs(rep.final_x - want)) < k["tol"]


def test_zero_measurements(kats):
    k = kats["zero_measurement_stop"]
    p = orc.make_problem(k["n"], k["m"], k["k"], k["seed"])
    zero = np.zeros(k["m"])
    rep = orc.run("ista", p.row, p.omega, zero, target_mse=k["target"], check_every=k["check_every"])
    assert rep.iterations == k["check_every"] and rep.reached_target
    for kind in ("ista", "cadmm"):
        rep = orc.run(kind, p.row, p.omega, zero, max_iter=40)
        assert np.all(rep.final_x == 0.0)


def test_parameter_validation():
    p = orc.make_problem(32, 16, 3, 13)
    for kw in ({"tau": 1.5}, {"tau": -0.2}, {"alpha": 0.0}):
        with pytest.raises(orc.OracleError) as e:
            orc.Ista(p.row, p.omega, p.y, **kw)
        assert e.value.code == orc.EPARAM
    for kw in ({"alpha": 0.0}, {"rho": 0.0}, {"tau1": 1.7}, {"tau2": 0.0}):
        with pytest.raises(orc.OracleError) as e:
            orc.Cadmm(p.row, p.omega, p.y, **kw)
        assert e.value.code == orc.EPARAM
    bad = p.y.copy()
    bad[3] = np.nan
    for cls in (orc.Ista, orc.Cadmm):
        with pytest.raises(orc.OracleError) as e:
            cls(p.row, p.omega, bad)
        assert e.value.code == orc.EDIVERGE
    # tests/solvers_test.cpp:203-214 -- zero operator: singular unless y == 0
    z = np.zeros(16)
    orc.Cadmm(z, np.arange(16), np.zeros(16))
    with pytest.raises(orc.OracleError) as e:
        orc.Cadmm(z, np.arange(16), random_vector(16, 15))
    assert e.value.code == orc.ESINGULAR


def test_literal_equals_proximal_bitwise(kats):
    k = kats["literal_equals_proximal"]
    p = orc.make_problem(k["n"], k["m"], k["k"], k["seed"])
    a = orc.run("ista", p.row, p.omega, p.y, tau=k["tau"], alpha=k["alpha_literal"], max_iter=k["iters"])
    b = orc.run("ista", p.row, p.omega, p.y, tau=k["tau"], alpha=k["alpha_proximal"], proximal=True,
                max_iter=k["iters"])
    assert np.array_equal(a.final_x, b.final_x)


def test_phases_vs_fft_engine(kats):
    k = kats["phases_vs_fft"]
    p = orc.make_problem(k["n"], k["m"], k["k"], k["seed"])
    for cls, fields in ((orc.Ista, ("x", "r")), (orc.Cadmm, ("x", "z", "v"))):
        a, b = cls(p.row, p.omega, p.y), cls(p.row, p.omega, p.y)
        a.step(k["iters"], orc.ENGINE_PHASES, threads=2)
        b.step(k["iters"], orc.ENGINE_FFT)
        for f in fields:
            assert np.max(np.abs(a.get(f) - b.get(f))) < k["tol"]
        # bitwise across thread counts (tests/parallel_test.cpp:136-189)
        c = cls(p.row, p.omega, p.y)
        c.step(k["iters"], orc.ENGINE_PHASES, threads=7)
        for f in fields:
            assert np.array_equal(a.get(f), c.get(f))


def test_ista_objective_nonincreasing():
    # tests/solvers_test.cpp:303-323 (literal pairing solves the alpha/tau-weighted problem)
    p = orc.make_problem(256, 128, 25, 20)
    h = orc.Ista(p.row, p.omega, p.y)
    s = orc.spectral_norm(p.row)
    A = dense_circulant(p.row)[p.omega]
    w = 1e-4 / 0.9

    def obj(x):
        r = p.y / s - (A @ x) / s
        return r @ r + 2 * w * np.abs(x).sum()

    prev = obj(h.get("x"))
    for _ in range(400):
        h.step(1, orc.ENGINE_FFT)
        cur = obj(h.get("x"))
        assert cur <= prev + 1e-12
        prev = cur


def test_protocol_recovery_1024(kats):
    k = kats["protocol_recovery_1024"]
    p = orc.make_problem(k["n"], k["m"], k["k"], k["seed"])
    rep = orc.run("cadmm", p.row, p.omega, p.y, truth=p.x_true, engine=orc.ENGINE_FFT,
                  max_iter=k["cadmm_max_iter"], target_mse=k["target"])
    assert rep.reached_target and rep.final_metric <= k["target"]
    assert rep.trace[-1][1] == rep.final_metric
    assert all(a[0] < b[0] for a, b in zip(rep.trace, rep.trace[1:]))


def test_phase_sample_full_range_is_a_step():
    # bench.py's CPU baseline times phase_sample(); over the full ranges it is exactly one phase step
    p = orc.make_problem(512, 128, 8, 3)
    a, b = orc.Ista(p.row, p.omega, p.y), orc.Ista(p.row, p.omega, p.y)
    for _ in range(3):
        a.step(1, orc.ENGINE_PHASES, 2)
        tr, tg = b.phase_sample(128, 512, 2)
        assert tr >= 0 and tg >= 0
    assert np.array_equal(a.get("x"), b.get("x"))
    ca, cb = orc.Cadmm(p.row, p.omega, p.y), orc.Cadmm(p.row, p.omega, p.y)
    for _ in range(3):
        ca.step(1, orc.ENGINE_PHASES, 2)
        assert len(cb.phase_sample(512, 2)) == 3
    assert np.array_equal(ca.get("z"), cb.get("z"))
    with pytest.raises(orc.OracleError):
        b.phase_sample(129, 512)


def test_dense_admm_oracle_against_numpy():
    """The dense ADMM restatement (solvers.hpp:267-327): its Cholesky inverse and iterations against an
    independent numpy evaluation (np.linalg.inv of A~^T A~ + rho I); the validation order of admm_setup
    (:288-296: dense cap, then rho, then alpha)."""
    p = orc.make_problem(192, 96, 10, 4)
    o = orc.Admm(p.row, p.omega, p.y, alpha=2e-3, rho=0.3)
    s = orc.spectral_norm(p.row)
    idx = (np.arange(p.n)[None, :] - p.omega[:, None]) % p.n
    ad = p.row[idx] / s
    B = np.linalg.inv(ad.T @ ad + 0.3 * np.eye(p.n))
    aty = ad.T @ (p.y / s)
    assert np.max(np.abs(o.get("B") - B)) <= 1e-12 and np.max(np.abs(o.get("aty") - aty)) <= 1e-12
    x = z = u = np.zeros(p.n)
    rhs = aty.copy()
    thr = 2e-3 / 0.3
    for _ in range(25):
        x = B @ rhs
        z = orc.soft_threshold(x + u, thr)
        u = u + x - z
        rhs = aty + 0.3 * (z - u)
    o.step(25)
    assert np.max(np.abs(o.get("z") - z)) <= 1e-10 and np.max(np.abs(o.get("u") - u)) <= 1e-10
    assert o.scalars()["threshold"] == thr
    with pytest.raises(orc.OracleError) as e:
        orc.Admm(p.row, p.omega, p.y, dense_cap=100)
    assert e.value.code == orc.ECAPACITY and "exceeds the dense cap 100" in str(e.value)
    with pytest.raises(orc.OracleError) as e:
        orc.Admm(p.row, p.omega, p.y, rho=0.0)
    assert e.value.code == orc.EPARAM
    rep = orc.run("admm", p.row, p.omega, p.y, truth=p.x_true, max_iter=40, check_every=10)
    assert rep.iterations == 40 and [t for t, _ in rep.trace] == [10, 20, 30, 40]
