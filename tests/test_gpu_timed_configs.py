"""Parity at the configurations the bench times (BASELINE configs 3, 4 and 5), on the GPU through the C-ABI.

* C3 (ISTA n = 2^20, m = 2^18; the bench's `value`): 25 and 200 iterations against the committed oracle
  fixture (tests/golden/c3_fixture.npz, tests/golden/make_timed_fixtures.py), plus 25 iterations against the
  live oracle on the full vectors; cADMM at the same size (the bench's `admm` line) for 5 iterations.
* C4 (cADMM n = 2^24, m = 2^22, k = 2^16): 3 iterations of the direct engine against the oracle's FFT engine.
* C5 (4096 x 4096 star field, order-5 blur, m = n/2): the composed operator, then 3 cADMM (alpha = 1e-2) and
  3 ISTA iterations on it against the oracle.

North-star bar: identical support and relative l2 <= 1e-4.  Every support flip is reported together with the
oracle's threshold margin | |v| - g | at that entry (v the pre-threshold value of the last step); the test
fails on a flip whose margin exceeds FLIP_MARGIN * g, i.e. one not explained by fp32 rounding at the
threshold.  The minimum margin and the flip count are printed for the record (pytest -s).
"""
import concurrent.futures as cf
import os

import numpy as np
import pytest

import paper_1707_02244_b200 as cl
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIXTURE = os.path.join(ROOT, "tests", "golden", "c3_fixture.npz")
REL_TOL = 1e-4
FLIP_MARGIN = 1e-3  # a flip must sit within 1e-3 of the threshold (relative) in the fp64 oracle


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if cl.device_count() < 1:
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def fx():
    return dict(np.load(FIXTURE))


@pytest.fixture(scope="module")
def c3():
    return orc.make_problem(1 << 20, 1 << 18, 1 << 12, 1)


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def op_of(p):
    return cl.PartialCirculantOperator(cl.CirculantMatrix(p.row), cl.SubsamplingMask(p.omega, p.n))


def check_support(got, want_nonzero, margin, thr, what):
    """Flips between the GPU support and the oracle's; each must be explained by a sub-threshold margin."""
    flips = np.flatnonzero((got != 0) != want_nonzero)
    worst = float(np.max(margin[flips])) / thr if len(flips) else 0.0
    print(f"{what}: {len(flips)} support flips of {len(got)} entries; min oracle margin "
          f"{float(np.min(margin)):.3e} ({float(np.min(margin)) / thr:.2e} of g); largest margin at a flip "
          f"{worst:.2e} of g")
    assert worst <= FLIP_MARGIN, f"{what}: flips at {flips[:8]} with margins {margin[flips[:8]] / thr} of g"
    return len(flips)


def fixture_margins(fx, pre, n):
    """Margins of the fixture's 256 closest entries; everything else is at least the 256th margin."""
    marg = np.full(n, float(fx[f"{pre}_margin_val"][-1]))
    marg[fx[f"{pre}_margin_pos"]] = fx[f"{pre}_margin_val"]
    return marg


def check_against_fixture(fx, pre, it, second, second_name, second_sample):
    n = int(fx["n"])
    want_nz = np.unpackbits(fx[f"{pre}_support_bits"])[:n].astype(bool)
    thr = float(fx[f"{pre}_threshold"])
    flips = check_support(it, want_nz, fixture_margins(fx, pre, n), thr, pre)
    e_s = rel(it[fx["sample_n"]], fx[f"{pre}_{'z' if pre.startswith('cadmm') else 'x'}_sample"])
    norm_name = f"{pre}_{'z' if pre.startswith('cadmm') else 'x'}_norm"
    e_n = abs(np.linalg.norm(it) - float(fx[norm_name])) / float(fx[norm_name])
    idx = fx["sample_m"] if second_name == "r" else fx["sample_n"]
    e_2 = rel(second[idx], fx[second_sample])
    print(f"{pre}: rel l2 on {len(fx['sample_n'])} sampled entries {e_s:.2e}, norm {e_n:.2e}, "
          f"{second_name} sampled {e_2:.2e}")
    assert e_s <= REL_TOL and e_n <= REL_TOL and e_2 <= REL_TOL
    return flips


def test_fixture_pins_the_c3_problem(fx, c3):
    """The fixture belongs to this problem: make_problem is bit-exact, so y's sha256 matches."""
    import hashlib
    assert hashlib.sha256(c3.y.tobytes()).digest() == fx["y_sha256"].tobytes()


def test_c3_ista_25_and_200_iterations(fx, c3):
    g = cl.ista_setup(op_of(c3), c3.y)
    with cf.ThreadPoolExecutor(1) as pool:  # the live oracle (fp64 FFT engine, CPU) runs beside the GPU
        def oracle25():
            o = orc.Ista(c3.row, c3.omega, c3.y)
            o.step(25, orc.ENGINE_FFT)
            return o.get("x"), o.get("r")
        fut = pool.submit(oracle25)
        g.step(25)
        x25, r25 = g.get("x"), g.get("r")
        check_against_fixture(fx, "ista_25", x25, r25, "r", "ista_25_r_sample")
        g.step(175)
        x200, r200 = g.get("x"), g.get("r")
        check_against_fixture(fx, "ista_200", x200, r200, "r", "ista_200_r_sample")
        ox, orr = fut.result()
    e_x, e_r = rel(x25, ox), rel(r25, orr)
    print(f"ista_25 vs the live oracle (full vectors): x {e_x:.2e}, r {e_r:.2e}")
    assert e_x <= REL_TOL and e_r <= REL_TOL
    check_support(x25, ox != 0, fixture_margins(fx, "ista_25", len(ox)), float(fx["ista_25_threshold"]),
                  "ista_25 vs live oracle")


def test_c3_cadmm_5_iterations(fx, c3):
    g = cl.cadmm_setup(op_of(c3), c3.y)
    g.step(5)
    check_against_fixture(fx, "cadmm_5", g.get("z"), g.get("x"), "x", "cadmm_5_x_sample")


def margins_from_step(pre_vals, thr):
    return np.abs(np.abs(pre_vals) - thr)


def test_c4_cadmm_2p24_direct_engine_vs_oracle():
    """BASELINE config 4 at G = 1: cADMM n = 2^24, m = 2^22, k = 2^16, 3 iterations (the 512-tile x 2-split
    tensor-core plan) against the oracle's FFT engine (<= 1e-12 from the phase engine)."""
    p = orc.make_problem(1 << 24, 1 << 22, 1 << 16, 1)

    def oracle():
        o = orc.Cadmm(p.row, p.omega, p.y)
        o.step(2, orc.ENGINE_FFT)
        nu_prev = o.get("nu")
        o.step(1, orc.ENGINE_FFT)
        x = o.get("x")
        return o.get("z"), x, x + nu_prev, o.scalars()["threshold"]

    with cf.ThreadPoolExecutor(1) as pool:
        fut = pool.submit(oracle)
        g = cl.cadmm_setup(op_of(p), p.y)
        g.step(3)
        z, x = g.get("z"), g.get("x")
        oz, ox, v, thr = fut.result()
    print(f"C4 cADMM 3 iterations: rel l2 z {rel(z, oz):.2e}, x {rel(x, ox):.2e}")
    check_support(z, oz != 0, margins_from_step(v, thr), thr, "C4 z")
    assert rel(z, oz) <= REL_TOL and rel(x, ox) <= REL_TOL


def test_c5_deblur_4096x4096_cadmm_and_ista():
    """BASELINE config 5 on one GPU: gen_star_field(4096, 4096, 0.1, 1), order-5 blur, m = n/2, seed 1
    (run_deblur_experiment, deblur.hpp:141-156): the composed operator row against the oracle's fp64
    composition, then 3 cADMM iterations (alpha = 1e-2, cli:544) and 3 ISTA iterations on the composed A."""
    img = cl.gen_star_field(4096, 4096, 0.1, 1)
    n = img.size()
    B = cl.blur_matrix(n, 5)
    sensing = cl.gen_circulant_sensing(n, n // 2, 1)
    A = cl.compose_sensing(sensing.circulant(), B, sensing.mask())
    y = cl.measure(A, img.pixels)
    row = A.circulant().first_row()
    om = A.mask().omega()

    def oracle():
        ref_row = orc.circ_compose(sensing.circulant().first_row(), B.first_row())
        oc = orc.Cadmm(row, om, y, alpha=1e-2)
        oc.step(2, orc.ENGINE_FFT)
        nu_prev = oc.get("nu")
        oc.step(1, orc.ENGINE_FFT)
        cz, cv, cthr = oc.get("z"), oc.get("x") + nu_prev, oc.scalars()["threshold"]
        del oc
        oi = orc.Ista(row, om, y, alpha=1e-2)
        oi.step(2, orc.ENGINE_FFT)
        x_prev = oi.get("x")
        oi.step(1, orc.ENGINE_FFT)
        sc = oi.scalars()
        return ref_row, cz, cv, cthr, oi.get("x"), x_prev + sc["tau"] * oi.get("delta"), sc["threshold"]

    with cf.ThreadPoolExecutor(1) as pool:
        fut = pool.submit(oracle)
        gc = cl.cadmm_setup(A, y, cl.SolverConfig(alpha=1e-2))
        gc.step(3)
        z = gc.get("z")
        del gc
        gi = cl.ista_setup(A, y, cl.SolverConfig(alpha=1e-2))
        gi.step(3)
        xi = gi.get("x")
        ref_row, cz, cv, cthr, ix, iv, ithr = fut.result()
    assert rel(row, ref_row) <= 1e-12
    print(f"C5 cADMM 3 iterations: rel l2 z {rel(z, cz):.2e}; ISTA 3 iterations: rel l2 x {rel(xi, ix):.2e}")
    check_support(z, cz != 0, margins_from_step(cv, cthr), cthr, "C5 cADMM z")
    check_support(xi, ix != 0, margins_from_step(iv, ithr), ithr, "C5 ISTA x")
    assert rel(z, cz) <= REL_TOL and rel(xi, ix) <= REL_TOL


def test_concurrent_solvers_on_one_device_bitwise():
    """Two solvers on the fp16 tensor-core path (n = 2^18) with operand scales 10^6 apart, stepped
    interleaved on their own streams with no synchronization between them (graph replays), equal the solo
    runs bitwise: each product's scale hand-over goes through its own solver's scratch."""
    n, m = 1 << 18, 1 << 16
    pa, pb = orc.make_problem(n, m, n // 256, 21), orc.make_problem(n, m, n // 256, 22)
    ya, yb = pa.y, pb.y * 1e6
    for setup, field in ((cl.ista_setup, "x"), (cl.cadmm_setup, "z")):
        solo = []
        for p, y in ((pa, ya), (pb, yb)):
            s = setup(op_of(p), y)
            s.step(4)
            solo.append(s.get(field))
        a, b = setup(op_of(pa), ya), setup(op_of(pb), yb)
        for _ in range(4):
            a.step(1)
            b.step(1)
        assert np.array_equal(a.get(field), solo[0]) and np.array_equal(b.get(field), solo[1]), setup.__name__


@pytest.mark.parametrize("kind,n", [("ista", 1 << 18), ("cadmm", 1 << 16), ("ista", 4096)])
def test_in_graph_phase_timing(kind, n):
    """profile(2): event-record nodes inside the captured step graph stamp every phase of each replay (the
    bench's roofline reads its kernel time from them); results are unchanged by the extra nodes."""
    p = orc.make_problem(n, n // 4, max(8, n // 256), 3)
    setup = cl.ista_setup if kind == "ista" else cl.cadmm_setup
    field = "x" if kind == "ista" else "z"
    ref = setup(op_of(p), p.y)
    ref.step(4)
    g = setup(op_of(p), p.y)
    g.profile(2)
    for _ in range(4):  # back-to-back replays, no synchronization in between
        g.step(1)
    g.synchronize()
    ms = g.phase_ms()
    assert len(ms) == (4 if kind == "ista" else 6) and all(v >= 0.0 for v in ms) and sum(ms) > 0.0, ms
    hist = g.phase_history()
    if n >= 1 << 15:  # every replay stamped its own slot
        assert len(hist) == 4 and all(len(h) == len(ms) and sum(h) > 0.0 for h in hist), hist
        assert hist[-1] == ms
    if n >= 1 << 15:  # same kernels, extra graph nodes: bitwise
        assert np.array_equal(g.get(field), ref.get(field))
    else:  # profiled small solves run the multi-kernel step instead of the persistent launch
        assert rel(g.get(field), ref.get(field)) <= 1e-5


# ------------------------------------------------------------- time to recovery at C3 (the bench's line)
RECOVERY = os.path.join(ROOT, "tests", "golden", "c3_recovery.npz")


@pytest.mark.parametrize("kind,use_fft", [("ista", False), ("ista", True), ("cadmm", False), ("cadmm", True)])
def test_c3_time_to_recovery_matches_oracle(kind, use_fft, c3):
    """ista_run / cadmm_run(target_mse = 1e-4, check_every = 10, truth = x*) at BASELINE config 3 -- the bench's
    time-to-recovery line -- against the oracle's own run (tests/golden/c3_recovery.npz,
    tests/golden/make_recovery_fixture.py): the stop rule fires at the same check, the MSE trace agrees check by
    check, and the final iterate matches (support flips only at the threshold, sampled rel l2 <= 1e-4)."""
    import hashlib
    rf = dict(np.load(RECOVERY))
    assert hashlib.sha256(c3.y.tobytes()).digest() == rf["y_sha256"].tobytes()
    run = cl.ista_run if kind == "ista" else cl.cadmm_run
    rep = run(c3.y, op_of(c3), cl.SolverConfig(target_mse=1e-4, check_every=10, max_iter=20000, use_fft=use_fft),
              truth=c3.x_true)
    want_it = int(rf[f"{kind}_iterations"])
    trace = np.array([(t.iteration, t.value) for t in rep.mse_trace]) if rep.mse_trace else np.zeros((0, 2))
    wt = rf[f"{kind}_trace"]
    k = min(len(trace), len(wt))
    e_tr = float(np.max(np.abs(trace[:k, 1] - wt[:k, 1]) / wt[:k, 1]))
    x = np.asarray(rep.final_x)
    e_x = rel(x[rf["sample_pos"]], rf[f"{kind}_sample"])
    want_nz = np.unpackbits(rf[f"{kind}_support_bits"])[:len(x)].astype(bool)
    fl = np.flatnonzero((x != 0) != want_nz)
    flips = len(fl)
    # the GPU value at a flip (zero where the oracle's is not): soft-thresholding maps a pre-threshold value
    # within fp32 resolution of the threshold to (nearly) zero, so a flip must carry a tiny value
    worst = float(np.max(np.abs(x[fl]))) / float(np.max(np.abs(x))) if flips else 0.0
    print(f"C3 {kind} {'fft' if use_fft else 'direct'}: {rep.iterations} iterations (oracle {want_it}), final MSE "
          f"{rep.final_metric:.6e} (oracle {float(rf[f'{kind}_final_mse']):.6e}), MSE trace max rel diff {e_tr:.2e} "
          f"over {k} checks, final x sampled rel l2 {e_x:.2e}, {flips} support flips (largest |x| at a flip "
          f"{worst:.1e} of max|x|)")
    assert rep.reached_target == bool(rf[f"{kind}_reached"])
    assert rep.iterations == want_it
    assert np.array_equal(trace[:k, 0], wt[:k, 0]) and len(trace) == len(wt)
    assert e_tr <= 1e-3 and e_x <= REL_TOL  # MSE vs truth: a difference of nearly equal vectors
    assert flips <= 5e-5 * len(x) and worst <= 1e-5  # threshold-margin flips only
