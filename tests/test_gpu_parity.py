"""GPU parity: the sm_100a kernels (through the C-ABI) against the CPU oracle.

Tolerances (north star, BASELINE.json): after a fixed iteration count the
recovered iterate has the identical support and a relative l2 difference
<= 1e-4 from the reference solver (fp32 on device vs the oracle's fp64).
Single products are checked at relative l2 <= 5e-5 (fp32 sums of up to 2^16
terms)."""
import numpy as np
import pytest

import paper_1707_02244_b200 as cl
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

REL_TOL = 1e-4


def rel_l2(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


EDGE = 1e-5  # support flips allowed only for entries this small relative to max|x| (fp32 vs fp64 at the threshold)


def assert_parity(got, want, tol=REL_TOL, what=""):
    """Identical support and rel l2 <= tol.  An entry whose pre-threshold value sits within fp32 resolution
    of the threshold can land on either side (the reference's own support test needs a margin for the same
    reason, tests/solvers_test.cpp:395-405); such flips are tolerated only when the entry is below
    EDGE * max|x| in both solvers, and are reported."""
    flips = np.flatnonzero((got != 0) != (want != 0))
    scale = max(float(np.max(np.abs(want))), 1e-30)
    bad = [int(i) for i in flips if max(abs(got[i]), abs(want[i])) > EDGE * scale]
    if len(flips):
        print(f"{what}: {len(flips)} near-threshold support flips, max |x| among them "
              f"{max(max(abs(got[i]), abs(want[i])) for i in flips) / scale:.2e} of max|x|")
    assert not bad, f"{what}: support differs at {bad[:10]} (got {got[bad[:5]]}, want {want[bad[:5]]})"
    assert rel_l2(got, want) <= tol, f"{what}: rel l2 {rel_l2(got, want):.3e}"


def op_of(p):
    return cl.PartialCirculantOperator(cl.CirculantMatrix(p.row), cl.SubsamplingMask(p.omega, p.n))


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if cl.device_count() < 1:
        pytest.skip("no CUDA device")


# --------------------------------------------------------------- single products
@pytest.mark.parametrize("n", [1, 2, 3, 5, 16, 64, 97, 256, 1000, 4096, 10000, 1 << 16])
def test_circ_products(n):
    row = orc.rng_draws(40 + n, "normal", n)
    x = orc.rng_draws(80 + n, "normal", n)
    C = cl.CirculantMatrix(row)
    want = orc.circ_matvec(row, x, use_fft=n > 4096)
    assert rel_l2(cl.circ_matvec(C, x), want) <= 5e-5
    want_t = orc.circ_matvec(row, x, transpose=True, use_fft=n > 4096)
    assert rel_l2(cl.circ_transpose_matvec(C, x), want_t) <= 5e-5


@pytest.mark.parametrize("n,m,seed", [(8, 4, 1), (97, 48, 3), (128, 64, 5), (4096, 1024, 1), (4096, 4096, 2),
                                      (10007, 2500, 4), (1 << 16, 1 << 14, 6)])
def test_partial_products(n, m, seed):
    row, om = orc.gen_circulant_sensing(n, m, seed)
    A = cl.PartialCirculantOperator(cl.CirculantMatrix(row), cl.SubsamplingMask(om, n))
    x = orc.rng_draws(seed + 100, "normal", n)
    r = orc.rng_draws(seed + 200, "normal", m)
    full = orc.circ_matvec(row, x, use_fft=True)
    assert rel_l2(cl.partial_matvec(A, x), full[om]) <= 5e-5
    emb = np.zeros(n)
    emb[om] = r
    assert rel_l2(cl.partial_transpose_matvec(A, r), orc.circ_matvec(row, emb, transpose=True, use_fft=True)) <= 5e-5


def test_sparse_edge_masks():
    # rows only at chunk boundaries / first and last index, m = 1, m = n
    n = 5000
    row = orc.rng_draws(11, "normal", n)
    x = orc.rng_draws(12, "normal", n)
    full = orc.circ_matvec(row, x, use_fft=True)
    for om in (np.array([0]), np.array([n - 1]), np.array([0, 2047, 2048, 4095, 4096, n - 1]), np.arange(n)):
        A = cl.PartialCirculantOperator(cl.CirculantMatrix(row), cl.SubsamplingMask(om, n))
        assert rel_l2(cl.partial_matvec(A, x), full[om]) <= 5e-5
        r = orc.rng_draws(13, "normal", len(om))
        emb = np.zeros(n)
        emb[om] = r
        assert rel_l2(cl.partial_transpose_matvec(A, r), orc.circ_matvec(row, emb, transpose=True, use_fft=True)) <= 5e-5


# --------------------------------------------------------------- solver steps
@pytest.mark.parametrize("n,m,k,seed,iters", [(128, 64, 12, 5, 25), (97, 48, 9, 3, 40), (1000, 300, 30, 2, 50)])
def test_ista_steps_match_oracle(n, m, k, seed, iters):
    p = orc.make_problem(n, m, k, seed)
    g = cl.ista_setup(op_of(p), p.y)
    g.step(iters)
    o = orc.Ista(p.row, p.omega, p.y)
    o.step(iters, orc.ENGINE_PHASES)
    assert_parity(g.get("x"), o.get("x"), what="x")
    assert rel_l2(g.get("r"), o.get("r")) <= REL_TOL
    assert rel_l2(g.get("delta"), o.get("delta")) <= 1e-3  # delta of the last step: small, cancellation-prone
    assert g.t == iters


@pytest.mark.parametrize("n,m,k,seed,iters", [(128, 64, 12, 5, 25), (97, 48, 9, 3, 40), (1000, 500, 100, 2, 60)])
def test_cadmm_steps_match_oracle(n, m, k, seed, iters):
    p = orc.make_problem(n, m, k, seed)
    g = cl.cadmm_setup(op_of(p), p.y)
    g.step(iters)
    o = orc.Cadmm(p.row, p.omega, p.y)
    o.step(iters, orc.ENGINE_PHASES)
    assert_parity(g.get("z"), o.get("z"), what="z")
    for f in ("x", "v", "mu", "nu", "beta"):
        assert rel_l2(g.get(f), o.get(f)) <= REL_TOL, f


def test_config1_ista_4096(capsys):
    """BASELINE config 1: ISTA n=4096, m=1024, k=64, 1000 iterations, seeds 1..10."""
    worst = 0.0
    for seed in range(1, 11):
        p = orc.make_problem(4096, 1024, 64, seed)
        cfg = cl.SolverConfig(max_iter=1000, check_every=1000)
        rep = cl.ista_run(p.y, op_of(p), cfg)
        ref = orc.run("ista", p.row, p.omega, p.y, max_iter=1000, check_every=1000)
        assert rep.iterations == ref.iterations == 1000
        assert_parity(rep.final_x, ref.final_x, what=f"seed {seed}")
        worst = max(worst, rel_l2(rep.final_x, ref.final_x))
    print(f"config1 worst rel l2 {worst:.3e}")


def test_config2_cadmm_4096():
    """BASELINE config 2: cADMM (circulant Gram inverse) on the same problems, 200 iterations."""
    for seed in range(1, 6):
        p = orc.make_problem(4096, 1024, 64, seed)
        cfg = cl.SolverConfig(max_iter=200, check_every=200)
        rep = cl.cadmm_run(p.y, op_of(p), cfg)
        ref = orc.run("cadmm", p.row, p.omega, p.y, max_iter=200, check_every=200)
        assert_parity(rep.final_x, ref.final_x, what=f"seed {seed}")


# --------------------------------------------------------------- run-loop semantics (solvers_test.cpp)
def test_zero_measurements_and_stop(kats):
    k = kats["zero_measurement_stop"]
    p = cl.make_problem(k["n"], k["m"], k["k"], k["seed"])
    zero = np.zeros(k["m"])
    rep = cl.ista_run(zero, p.op, cl.SolverConfig(target_mse=k["target"]))
    assert rep.iterations == k["check_every"] and rep.reached_target
    for run in (cl.ista_run, cl.cadmm_run):
        assert np.all(run(zero, p.op, cl.SolverConfig(max_iter=40)).final_x == 0.0)


def test_identity_operator_fixed_point(kats):
    k = kats["identity_ista"]
    n = k["n"]
    y = k["y_scale"] * orc.rng_draws(k["y_seed"], "normal", n)
    I = cl.PartialCirculantOperator(cl.CirculantMatrix.Identity(n), cl.SubsamplingMask.Full(n))
    cfg = cl.SolverConfig(alpha=k["alpha"], pairing=cl.ThresholdPairing.kProximal, target_mse=k["target"],
                          max_iter=k["max_iter"])
    rep = cl.ista_run(y, I, cfg)
    assert rep.reached_target
    assert np.max(np.abs(rep.final_x - cl.soft_threshold(y, k["alpha"]))) < k["tol"]


def test_literal_equals_proximal_bitwise(kats):
    k = kats["literal_equals_proximal"]
    p = cl.make_problem(k["n"], k["m"], k["k"], k["seed"])
    a = cl.ista_run(p.measurements, p.op, cl.SolverConfig(tau=k["tau"], alpha=k["alpha_literal"], max_iter=k["iters"]))
    b = cl.ista_run(p.measurements, p.op, cl.SolverConfig(tau=k["tau"], alpha=k["alpha_proximal"],
                                                           pairing=cl.ThresholdPairing.kProximal, max_iter=k["iters"]))
    assert np.array_equal(a.final_x, b.final_x)


def test_report_bookkeeping_and_determinism():
    p = cl.make_problem(256, 128, 25, 17)
    cfg = cl.SolverConfig(target_mse=1e-4, max_iter=20000)
    rep = cl.cadmm_run(p.measurements, p.op, cfg, truth=p.signal.values)
    assert rep.reached_target and rep.metric == cl.StopMetric.kMseVsTruth and rep.final_metric <= 1e-4
    assert rep.footprint_bytes == cl.analytic_footprint(cl.FootprintKind.kCpadmm, 256, 128, 4)
    assert rep.mse_trace[-1].value == rep.final_metric
    assert all(a.iteration < b.iteration for a, b in zip(rep.mse_trace, rep.mse_trace[1:]))
    rep2 = cl.cadmm_run(p.measurements, p.op, cfg, truth=p.signal.values)
    assert np.array_equal(rep.final_x, rep2.final_x) and rep.iterations == rep2.iterations
    nt = cl.cadmm_run(p.measurements, p.op, cl.SolverConfig(target_mse=1e-8, max_iter=50))
    assert nt.metric == cl.StopMetric.kIterateChange


def test_protocol_recovery_1024():
    p = cl.make_problem(1024, 512, 102, 1)
    rep = cl.cadmm_run(p.measurements, p.op, cl.SolverConfig(target_mse=1e-4, max_iter=20000), truth=p.signal.values)
    assert rep.reached_target and cl.mse(rep.final_x, p.signal.values) <= 1e-4
    rep = cl.ista_run(p.measurements, p.op, cl.SolverConfig(target_mse=1e-4, max_iter=100000), truth=p.signal.values)
    assert rep.reached_target


def test_nonfinite_iterate_flag():
    # cADMM iterate z = eta(x + nu): an infinite dual propagates into z and must raise the flag
    # (run_loop's check_finite, solvers.hpp:190-197).  (ISTA cannot be poisoned this way: the
    # soft threshold maps NaN to 0, exactly as in the reference.)
    p = cl.make_problem(256, 128, 10, 3)
    st = cl.cadmm_setup(p.op, p.measurements)
    nu = np.zeros(256)
    nu[7] = np.inf
    st.set("nu", nu)
    _, nonfinite = st.step_checked()
    assert nonfinite
    st2 = cl.cadmm_setup(p.op, p.measurements)
    _, nonfinite = st2.step_checked()
    assert not nonfinite


# --------------------------------------------------------------- large-n properties (config 3 scale)
def test_config3_scale_ista_vs_fft_oracle():
    """n = 2^20, m = 2^18: 3 GPU iterations vs the oracle's FFT engine (<=1e-12 from the phases)."""
    n, m = 1 << 20, 1 << 18
    p = orc.make_problem(n, m, 1 << 12, 1)
    g = cl.ista_setup(op_of(p), p.y)
    g.step(3)
    o = orc.Ista(p.row, p.omega, p.y)
    o.step(3, orc.ENGINE_FFT)
    assert_parity(g.get("x"), o.get("x"), what="x")
    assert rel_l2(g.get("r"), o.get("r")) <= REL_TOL


def test_config3_scale_cadmm_vs_fft_oracle():
    """cADMM at n = 2^20 (the bench's `admm` line; tensor-core products with fp16 operands):
    3 GPU iterations vs the oracle's FFT engine."""
    n, m = 1 << 20, 1 << 18
    p = orc.make_problem(n, m, 1 << 12, 1)
    g = cl.cadmm_setup(op_of(p), p.y)
    g.step(3)
    o = orc.Cadmm(p.row, p.omega, p.y)
    o.step(3, orc.ENGINE_FFT)
    assert_parity(g.get("z"), o.get("z"), what="z")
    for f in ("x", "v"):
        assert rel_l2(g.get(f), o.get(f)) <= REL_TOL, f


def test_cpp_adapter_gpu():
    """Reference-style C++ code through include/circlasso_b200.hpp on the GPU."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1707_02244_b200", "_lib",
                       "adapter_test")
    out = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "PASS" in out.stdout, out.stdout + out.stderr
    eig = os.path.join(os.path.dirname(exe), "eigen_style_test")  # the adapter's Eigen branch (test double)
    out = subprocess.run([eig, "gpu"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "PASS" in out.stdout, out.stdout + out.stderr


# --------------------------------------------------------------- FFT engine (SolverConfig.use_fft=True)
@pytest.mark.parametrize("n,m,k,seed,iters", [(128, 64, 12, 5, 25), (4096, 1024, 64, 1, 200), (1 << 16, 1 << 14, 256, 2, 30)])
def test_fft_engine_ista_matches_oracle(n, m, k, seed, iters):
    p = orc.make_problem(n, m, k, seed)
    g = cl.ista_setup(op_of(p), p.y, cl.SolverConfig(use_fft=True))
    g.step(iters)
    o = orc.Ista(p.row, p.omega, p.y)
    o.step(iters, orc.ENGINE_FFT)
    assert_parity(g.get("x"), o.get("x"), what="x")
    assert rel_l2(g.get("r"), o.get("r")) <= REL_TOL


@pytest.mark.parametrize("n,m,k,seed,iters", [(128, 64, 12, 5, 25), (4096, 1024, 64, 1, 200), (1 << 16, 1 << 14, 256, 2, 30)])
def test_fft_engine_cadmm_matches_oracle(n, m, k, seed, iters):
    p = orc.make_problem(n, m, k, seed)
    g = cl.cadmm_setup(op_of(p), p.y, cl.SolverConfig(use_fft=True))
    g.step(iters)
    o = orc.Cadmm(p.row, p.omega, p.y)
    o.step(iters, orc.ENGINE_FFT)
    assert_parity(g.get("z"), o.get("z"), what="z")
    for f in ("x", "v", "mu", "nu"):
        assert rel_l2(g.get(f), o.get(f)) <= REL_TOL, f


def test_fft_engine_matches_direct_engine_c3():
    """Both engines on BASELINE config 3 (n = 2^20): same iterate after 5 iterations."""
    p = orc.make_problem(1 << 20, 1 << 18, 1 << 12, 1)
    a = cl.ista_setup(op_of(p), p.y, cl.SolverConfig(use_fft=True))
    b = cl.ista_setup(op_of(p), p.y)
    a.step(5)
    b.step(5)
    assert_parity(a.get("x"), b.get("x"), what="fft vs direct")


@pytest.mark.parametrize("kind,n,m,k,seed,iters", [("ista", 1000, 300, 10, 1, 60), ("cadmm", 1000, 500, 10, 2, 40),
                                                   ("ista", 10007, 2500, 40, 3, 30), ("cadmm", 10007, 5000, 40, 4, 20),
                                                   ("ista", 300007, 75000, 1000, 5, 5)])
def test_fft_engine_non_power_of_two_matches_oracle(kind, n, m, k, seed, iters):
    """use_fft=True (the reference's default engine) at any n: the circulant is embedded as a linear
    convolution in the next power of two >= 2n-1 (Stockham passes below 2^14, four-step above)."""
    p = orc.make_problem(n, m, k, seed)
    setup = cl.ista_setup if kind == "ista" else cl.cadmm_setup
    g = setup(op_of(p), p.y, cl.SolverConfig(use_fft=True))
    g.step(iters)
    o = (orc.Ista if kind == "ista" else orc.Cadmm)(p.row, p.omega, p.y)
    o.step(iters, orc.ENGINE_FFT)
    f = "x" if kind == "ista" else "z"
    assert_parity(g.get(f), o.get(f), what=f)
    for h in (("r",) if kind == "ista" else ("x", "v", "mu", "nu", "beta")):
        assert rel_l2(g.get(h), o.get(h)) <= REL_TOL, h


def test_fft_engine_protocol_recovery():
    p = cl.make_problem(4096, 2048, 409, 1)
    rep = cl.cadmm_run(p.measurements, p.op, cl.SolverConfig(target_mse=1e-4, max_iter=20000, use_fft=True),
                       truth=p.signal.values)
    assert rep.reached_target


# --------------------------------------------------------------- deblurring (deblur.hpp)
def test_deblur_order1_blur_equals_plain_recovery():
    """tests/image_deblur_test.cpp:261-280"""
    n = 256
    sensing = cl.gen_circulant_sensing(n, n, 9)
    img = cl.gen_star_field(16, 16, 0.12, 3)
    y = cl.measure(sensing, img.pixels)
    cfg = cl.SolverConfig(target_mse=1e-8, max_iter=30000)
    via = cl.deblur_recover(y, sensing.circulant(), cl.blur_matrix(n, 1), sensing.mask(), 16, 16, cfg, img)
    direct = cl.cadmm_run(y, sensing, cfg)
    assert np.array_equal(via.report.final_x, direct.final_x) and via.report.iterations == direct.iterations
    assert np.isfinite(via.mse_vs_truth)


def test_deblur_black_image_and_shape_contract():
    black = cl.GrayImage(8, 8, np.zeros(64))
    res = cl.run_deblur_experiment(black, 3, 32, cl.SolverConfig(max_iter=30), 4)
    assert np.all(res.recovered.pixels == 0) and res.mse_vs_truth == 0 and res.normalized_mse == 0
    sensing = cl.gen_circulant_sensing(64, 32, 2)
    with pytest.raises(cl.DimensionError):
        cl.deblur_recover(np.zeros(32), sensing.circulant(), cl.blur_matrix(64, 2), sensing.mask(), 7, 8)
    with pytest.raises(cl.ParameterError):
        cl.deblur_recover(np.zeros(32), sensing.circulant(), cl.blur_matrix(64, 2), sensing.mask(), 0, 8)


@pytest.mark.parametrize("use_fft", [False, True])
def test_deblur_acceptance_64x64(use_fft):
    """tests/acceptance.cpp:398-427: 64x64 star field, L=5, m=n/2 -> MSE <= 5e-2; control L=1, m=n -> <= 1e-6."""
    truth = cl.gen_star_field(64, 64, 0.1, 7)
    main = cl.run_deblur_experiment(truth, 5, 2048, cl.SolverConfig(alpha=1e-2, target_mse=1e-7, max_iter=50000,
                                                                     use_fft=use_fft), 7)
    control = cl.run_deblur_experiment(truth, 1, 4096, cl.SolverConfig(alpha=1e-6, target_mse=1e-8, max_iter=50000,
                                                                        use_fft=use_fft), 7)
    print(f"deblur 64x64 fft={use_fft}: MSE {main.mse_vs_truth:.3e} in {main.report.iterations} it; "
          f"control {control.mse_vs_truth:.3e} in {control.report.iterations} it")
    assert main.mse_vs_truth <= 5e-2 and control.mse_vs_truth <= 1e-6
    assert np.all((main.recovered.pixels >= 0) & (main.recovered.pixels <= 1))


def test_deblur_matches_oracle_iterates():
    truth = cl.gen_star_field(24, 24, 0.08, 11)
    n = truth.size()
    B = cl.blur_matrix(n, 3)
    sensing = cl.gen_circulant_sensing(n, 288, 11)
    A = cl.compose_sensing(sensing.circulant(), B, sensing.mask())
    y = cl.measure(A, truth.pixels)
    g = cl.cadmm_setup(A, y, cl.SolverConfig(alpha=1e-2))
    g.step(300)
    o = orc.Cadmm(A.circulant().first_row(), A.mask().omega(), y, alpha=1e-2)
    o.step(300, orc.ENGINE_PHASES)
    assert_parity(g.get("z"), o.get("z"), what="deblur z")


# --------------------------------------------------------------- virtual shards on one GPU
@pytest.mark.parametrize("kind", ["ista", "cadmm"])
@pytest.mark.parametrize("world", [2, 3])
def test_virtual_shards_bitwise(kind, world):
    """G solver shards on one device, all-gathered through torch copies between phases: the iterate must be
    bitwise identical to the unsharded solve (no reduction crosses shards)."""
    import torch
    from paper_1707_02244_b200 import dist as cdist
    n, m = (40000, 10000) if kind == "ista" else (40000, 20000)
    p = cl.make_problem(n, m, 100, 3)
    setup = cl.ista_setup if kind == "ista" else cl.cadmm_setup
    ref = setup(p.op, p.measurements)
    ref.step(4)
    shards = [cdist.CudaShard(setup(p.op, p.measurements), g, world) for g in range(world)]
    for _ in range(4):
        for ph in shards[0].phases():
            outs = []
            for sh in shards:
                sh.run_phase(ph)
                outs.append(sh.phase_output(ph))
            for sh in shards:
                sh.state.synchronize()
            for g, (full_g, a_g, b_g) in enumerate(outs):  # "all-gather": every shard copies every slice
                for h, (full_h, _, _) in enumerate(outs):
                    if h != g and b_g > a_g:
                        full_h[a_g:b_g].copy_(full_g[a_g:b_g])
            torch.cuda.synchronize()
    field = "x" if kind == "ista" else "v"
    for sh in shards:
        assert np.array_equal(sh.state.get(field), ref.get(field))
    if kind == "cadmm":
        z = np.zeros(n)
        for sh in shards:  # z is slice-local: assemble it
            full, a, b = sh.phase_output(1)
            lo, hi = a, b
            z[lo:hi] = sh.state.get("z")[lo:hi]
        assert np.array_equal(z, ref.get("z"))


def test_sharded_step_over_nccl_world1():
    """The production sharded path (CudaShard + TorchGather over NCCL on the solver stream), world size 1."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    from paper_1707_02244_b200 import dist as cdist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        p = cl.make_problem(1 << 16, 1 << 14, 100, 5)
        ref = cl.ista_setup(p.op, p.measurements)
        ref.step(3)
        st = cl.ista_setup(p.op, p.measurements)
        shard = cdist.CudaShard(st, 0, 1)
        cdist.sharded_step(shard, cdist.TorchGather(), 3)
        st.synchronize()
        assert np.array_equal(st.get("x"), ref.get("x"))
    finally:
        dist.destroy_process_group()


# ------------------------------------------------- setup transforms on the device
def _states(kind, p, host_setup, iters=20, use_fft=False):
    import os
    old = os.environ.get("CLB_HOST_SETUP")
    os.environ["CLB_HOST_SETUP"] = "1" if host_setup else "0"
    os.environ["CLB_FFT_STOCKHAM"] = "1"  # same FFT engine either way (the four-step one needs the device setup)
    try:
        setup = cl.ista_setup if kind == "ista" else cl.cadmm_setup
        g = setup(op_of(p), p.y, cl.SolverConfig(use_fft=use_fft))
        g.step(iters)
        return {f: g.get(f) for f in (("x", "r", "delta") if kind == "ista" else ("x", "z", "v", "mu", "nu", "beta"))}
    finally:
        del os.environ["CLB_FFT_STOCKHAM"]
        if old is None:
            del os.environ["CLB_HOST_SETUP"]
        else:
            os.environ["CLB_HOST_SETUP"] = old


@pytest.mark.parametrize("kind,use_fft", [("ista", False), ("cadmm", False), ("ista", True), ("cadmm", True)])
def test_device_setup_matches_host_setup(kind, use_fft):
    """Spectral norm, Gram inverse and operator rows computed by the device fp64 FFT (n >= 2^14, power of
    two) agree with the host fp64 transforms: the two setups differ only in fp64 rounding, far below fp32."""
    p = orc.make_problem(1 << 16, 1 << 14, 1 << 8, 4)
    dev = _states(kind, p, host_setup=False, use_fft=use_fft)
    host = _states(kind, p, host_setup=True, use_fft=use_fft)
    for f in dev:
        assert rel_l2(dev[f], host[f]) <= 1e-6, (f, rel_l2(dev[f], host[f]))


def test_cadmm_2p16_vs_fft_oracle():
    """cADMM at n = 2^16 (device setup path) against the oracle's FFT engine."""
    p = orc.make_problem(1 << 16, 1 << 14, 1 << 8, 6)
    g = cl.cadmm_setup(op_of(p), p.y)
    g.step(10)
    o = orc.Cadmm(p.row, p.omega, p.y)
    o.step(10, orc.ENGINE_FFT)
    assert_parity(g.get("z"), o.get("z"), what="z")
    for f in ("x", "v", "mu", "nu", "beta"):
        assert rel_l2(g.get(f), o.get(f)) <= REL_TOL, f


def test_device_gram_floor_raises():
    """regularized_gram_inverse's 1e-14 invertibility floor (circulant.hpp:309-316) on the device path:
    a constant first row has a zero spectrum off k = 0, so rho |c_k|^2 + sigma = sigma = 1e-15."""
    n = 1 << 14
    c = np.ones(n)
    op = cl.PartialCirculantOperator(cl.CirculantMatrix(c), cl.SubsamplingMask(np.arange(0, n, 2), n))
    with pytest.raises(cl.SingularityError):
        cl.cadmm_setup(op, np.zeros(n // 2), cl.SolverConfig(sigma=1e-15))


# ------------------------------------------------------- four-step FFT engine
@pytest.mark.parametrize("kind,lg", [("ista", 14), ("ista", 15), ("ista", 17), ("cadmm", 14), ("cadmm", 17)])
def test_fft4_engine_matches_oracle(kind, lg):
    """The four-step engine (n >= 2^14; N1 = N2 and N1 != N2 splits) against the oracle's FFT engine."""
    n = 1 << lg
    p = orc.make_problem(n, n // 4, n // 256, 3)
    setup = cl.ista_setup if kind == "ista" else cl.cadmm_setup
    g = setup(op_of(p), p.y, cl.SolverConfig(use_fft=True))
    g.step(20)
    o = (orc.Ista if kind == "ista" else orc.Cadmm)(p.row, p.omega, p.y)
    o.step(20, orc.ENGINE_FFT)
    f = "x" if kind == "ista" else "z"
    assert_parity(g.get(f), o.get(f), what=f)
    for h in (("r", "delta") if kind == "ista" else ("x", "v", "mu", "nu")):
        assert rel_l2(g.get(h), o.get(h)) <= (1e-3 if h == "delta" else REL_TOL), h


@pytest.mark.parametrize("kind,lg,iters", [("ista", 22, 3), ("cadmm", 23, 2)])
def test_fft4_three_level_matches_oracle(kind, lg, iters):
    """The three-level plan (n >= 2^22: 256 x A x B, the length-N2 rows themselves four-step) against the
    oracle's fp64 FFT engine."""
    n = 1 << lg
    p = orc.make_problem(n, n // 4, n // 256, 3)
    setup = cl.ista_setup if kind == "ista" else cl.cadmm_setup
    g = setup(op_of(p), p.y, cl.SolverConfig(use_fft=True))
    g.step(iters)
    o = (orc.Ista if kind == "ista" else orc.Cadmm)(p.row, p.omega, p.y)
    o.step(iters, orc.ENGINE_FFT)
    f = "x" if kind == "ista" else "z"
    assert_parity(g.get(f), o.get(f), what=f)
    for h in (("r",) if kind == "ista" else ("x", "v")):
        assert rel_l2(g.get(h), o.get(h)) <= REL_TOL, h


@pytest.mark.parametrize("kind,lg", [("ista", 14), ("cadmm", 15), ("ista", 18), ("cadmm", 20), ("ista", 22),
                                     ("cadmm", 23), ("ista", 24), ("cadmm", 24)])
def test_fft4_real_plan_matches_complex_plan(kind, lg):
    """Real plans (n / 2 complex points, the spectrum unpacked pairwise between the row FFTs; the default)
    against the complex plans (CLB_FFT_C2C=1: n complex points), two- and three-level, up to n = 2^24."""
    import os
    n = 1 << lg
    p = orc.make_problem(n, n // 4, n // 256, 2)
    setup = cl.ista_setup if kind == "ista" else cl.cadmm_setup
    got = {}
    for c2c in ("0", "1"):  # force the real / the complex plan
        os.environ["CLB_FFT_C2C"] = c2c
        try:
            g = setup(op_of(p), p.y, cl.SolverConfig(use_fft=True))
            g.step(4)
            got[c2c] = {f: g.get(f) for f in (("x", "r") if kind == "ista" else ("z", "x", "v"))}
            del g
        finally:
            del os.environ["CLB_FFT_C2C"]
    for f in got["0"]:
        assert rel_l2(got["0"][f], got["1"][f]) <= 1e-5, (f, rel_l2(got["0"][f], got["1"][f]))


@pytest.mark.parametrize("kind,lg", [("ista", 20), ("ista", 23), ("cadmm", 22), ("ista", 24)])
def test_fft4_engine_matches_stockham_engine(kind, lg):
    """Four-step engine vs the multi-pass Stockham engine (CLB_FFT_STOCKHAM=1) up to n = 2^24."""
    import os
    n = 1 << lg
    p = orc.make_problem(n, n // 4, n // 256, 1)
    setup = cl.ista_setup if kind == "ista" else cl.cadmm_setup
    got = {}
    for stock in ("0", "1"):
        os.environ["CLB_FFT_STOCKHAM"] = stock
        try:
            g = setup(op_of(p), p.y, cl.SolverConfig(use_fft=True))
            g.step(4)
            got[stock] = {f: g.get(f) for f in (("x", "r") if kind == "ista" else ("z", "x", "v"))}
            del g
        finally:
            del os.environ["CLB_FFT_STOCKHAM"]
    for f in got["0"]:
        assert rel_l2(got["0"][f], got["1"][f]) <= 1e-5, (f, rel_l2(got["0"][f], got["1"][f]))


# ------------------------------------------------- persistent small-n ISTA (one cooperative launch)
@pytest.mark.parametrize("n,m,k,seed,iters", [(4096, 1024, 64, 1, 300), (2048, 700, 40, 4, 120),
                                              (8192, 2048, 100, 5, 80), (4096, 4096, 64, 2, 50)])
def test_small_coop_ista_matches_oracle(n, m, k, seed, iters):
    """The single-launch small-n ISTA kernel (cooperative grid) against the oracle's phase engine."""
    p = orc.make_problem(n, m, k, seed)
    g = cl.ista_setup(op_of(p), p.y)
    g.step(iters)
    o = orc.Ista(p.row, p.omega, p.y)
    o.step(iters, orc.ENGINE_PHASES)
    assert g.t == iters
    assert_parity(g.get("x"), o.get("x"), what="x")
    assert rel_l2(g.get("r"), o.get("r")) <= REL_TOL
    assert rel_l2(g.get("delta"), o.get("delta")) <= 1e-3


def test_small_coop_ista_matches_multikernel():
    """Cooperative small-n kernel vs the multi-kernel path (CLB_NO_SMALL=1) on config 1, seed 3: same iterates."""
    import os
    p = orc.make_problem(4096, 1024, 64, 3)
    got = {}
    for off in ("0", "1"):
        os.environ["CLB_NO_SMALL"] = off
        try:
            g = cl.ista_setup(op_of(p), p.y)
            g.step(200)
            got[off] = g.get("x")
        finally:
            del os.environ["CLB_NO_SMALL"]
    assert rel_l2(got["0"], got["1"]) <= 1e-5


def test_device_measure_and_compose_match_host():
    """measure / compose_rows through the device fp64 FFT (power-of-two n >= 2^14) agree with the host
    fp64 DFT to the reference's own FFT tolerance (tests/fft_test.cpp:136-148: 1e-10)."""
    import os
    n = 1 << 16
    p = orc.make_problem(n, n // 4, 256, 9)
    blur = cl.blur_matrix(n, 5)
    out = {}
    for host in ("0", "1"):
        os.environ["CLB_HOST_SETUP"] = host
        try:
            A = op_of(p)
            out[host] = (cl.measure(A, p.x_true), cl.compose_sensing(A.circulant(), blur, A.mask()).circulant().first_row(),
                         cl.make_problem(n, n // 4, 256, 9).measurements)
        finally:
            del os.environ["CLB_HOST_SETUP"]
    for a, b in zip(out["0"], out["1"]):
        assert np.max(np.abs(a - b)) <= 1e-12 * max(1.0, np.max(np.abs(b)))
    assert np.max(np.abs(out["0"][0] - p.y)) <= 1e-12 * max(1.0, np.max(np.abs(p.y)))


# ------------------------------------------- large, ragged sizes (streamed kernels, 96x148 units)
@pytest.mark.parametrize("n,m,seed", [(131075, 32771, 7), (524309, 131073, 8), (1 << 19, 1 << 17, 9)])
def test_partial_products_large_ragged(n, m, seed):
    """Streamed-window kernels at n >= 2^17: n not a multiple of 4 (scalar staging path), ragged last
    tile, and the large unit target (n >= 2^19)."""
    row, om = orc.gen_circulant_sensing(n, m, seed)
    A = cl.PartialCirculantOperator(cl.CirculantMatrix(row), cl.SubsamplingMask(om, n))
    x = orc.rng_draws(seed + 100, "normal", n)
    r = orc.rng_draws(seed + 200, "normal", m)
    full = orc.circ_matvec(row, x, use_fft=True)
    assert rel_l2(cl.partial_matvec(A, x), full[om]) <= 5e-5
    emb = np.zeros(n)
    emb[om] = r
    assert rel_l2(cl.partial_transpose_matvec(A, r), orc.circ_matvec(row, emb, transpose=True, use_fft=True)) <= 5e-5


def test_sparse_edge_masks_large():
    """Rows only at the ends and at chunk boundaries, m = 1 and m = n, at a size the streamed kernels run."""
    n = 200003
    row = orc.rng_draws(21, "normal", n)
    x = orc.rng_draws(22, "normal", n)
    full = orc.circ_matvec(row, x, use_fft=True)
    for om in (np.array([0]), np.array([n - 1]), np.array([0, 1023, 1024, 2047, 2048, 131071, 131072, n - 1]),
               np.arange(n)):
        A = cl.PartialCirculantOperator(cl.CirculantMatrix(row), cl.SubsamplingMask(om, n))
        assert rel_l2(cl.partial_matvec(A, x), full[om]) <= 5e-5
        r = orc.rng_draws(23, "normal", len(om))
        emb = np.zeros(n)
        emb[om] = r
        assert rel_l2(cl.partial_transpose_matvec(A, r), orc.circ_matvec(row, emb, transpose=True, use_fft=True)) <= 5e-5


@pytest.mark.parametrize("n", [524291])
def test_circ_products_large_ragged(n):
    """Dense products at n >= 2^19 (large unit target), n odd."""
    row = orc.rng_draws(50, "normal", n)
    x = orc.rng_draws(51, "normal", n)
    C = cl.CirculantMatrix(row)
    assert rel_l2(cl.circ_matvec(C, x), orc.circ_matvec(row, x, use_fft=True)) <= 5e-5
    assert rel_l2(cl.circ_transpose_matvec(C, x), orc.circ_matvec(row, x, transpose=True, use_fft=True)) <= 5e-5


@pytest.mark.parametrize("kind", ["ista", "cadmm"])
def test_steps_large_ragged_vs_fft_oracle(kind):
    """Solver steps at n = 262147 (odd, streamed sparse kernels / dense kernel) vs the oracle's FFT engine."""
    n = 262147
    p = orc.make_problem(n, n // 4, 1000, 11)
    setup = cl.ista_setup if kind == "ista" else cl.cadmm_setup
    g = setup(op_of(p), p.y)
    g.step(3)
    o = (orc.Ista if kind == "ista" else orc.Cadmm)(p.row, p.omega, p.y)
    o.step(3, orc.ENGINE_FFT)
    f = "x" if kind == "ista" else "z"
    assert_parity(g.get(f), o.get(f), what=f)


@pytest.mark.parametrize("n,m,k,seed,iters", [(4096, 1024, 64, 1, 500), (1024, 300, 20, 2, 100), (8192, 2048, 80, 3, 60)])
def test_small_fft_engine_ista_matches_oracle(n, m, k, seed, iters):
    """One-CTA FFT-engine ISTA (all iterations in one launch) against the oracle's FFT engine."""
    p = orc.make_problem(n, m, k, seed)
    g = cl.ista_setup(op_of(p), p.y, cl.SolverConfig(use_fft=True))
    g.step(iters)
    o = orc.Ista(p.row, p.omega, p.y)
    o.step(iters, orc.ENGINE_FFT)
    assert g.t == iters
    assert_parity(g.get("x"), o.get("x"), what="x")
    assert rel_l2(g.get("r"), o.get("r")) <= REL_TOL
    assert rel_l2(g.get("delta"), o.get("delta")) <= 1e-3


@pytest.mark.parametrize("n,m,k,seed,iters", [(4096, 1024, 64, 2, 200), (2048, 1024, 40, 4, 80)])
def test_small_fft_engine_cadmm_matches_oracle(n, m, k, seed, iters):
    """One-CTA FFT-engine cADMM against the oracle's FFT engine."""
    p = orc.make_problem(n, m, k, seed)
    g = cl.cadmm_setup(op_of(p), p.y, cl.SolverConfig(use_fft=True))
    g.step(iters)
    o = orc.Cadmm(p.row, p.omega, p.y)
    o.step(iters, orc.ENGINE_FFT)
    assert_parity(g.get("z"), o.get("z"), what="z")
    for f in ("x", "v", "mu", "nu", "beta"):
        assert rel_l2(g.get(f), o.get(f)) <= REL_TOL, f


def test_bench_sweeps_the_protocol_problem():
    """The reference's `bench` sweep (io_cli_test.cpp:317-336) through the GPU solvers: pinned CSV, m = n/2,
    k = n/10, status ok at the protocol target."""
    import io
    from paper_1707_02244_b200 import io as cio
    out = io.StringIO()
    cio.bench([128, 4096], solvers=("cadmm", "ista", "admm"), seeds=1,
              cfg=cl.SolverConfig(target_mse=1e-4, max_iter=20000), out=out)
    lines = out.getvalue().splitlines()
    assert lines[0] == cio.kBenchCsvHeader and len(lines) == 7
    f = lines[1].split(",")
    assert f[:4] == ["cadmm", "128", "64", "12"] and f[11] == "ok"
    rows = [ln.split(",") for ln in lines[1:]]
    assert all(len(r) == 12 for r in rows)
    assert [r[11] for r in rows if r[0] == "admm"] == ["skipped", "skipped"]
    assert all(r[11] == "ok" and float(r[8]) <= 1e-4 for r in rows if r[0] != "admm")


def test_matvec_scheme_bench_accounts_fetches():
    """parallel_test.cpp:259-277 and io_cli_test.cpp:297-315 on the GPU: fetch accounting, both schemes compute
    the same product (fp32: to tolerance, the reference's loops agree exactly in fp64), pinned CSV rows."""
    import io
    from paper_1707_02244_b200 import io as cio
    n = 64
    c = cio.matvec_scheme_bench(n, "circulant", 3, 9)
    r = cio.matvec_scheme_bench(n, "reference", 3, 9)
    assert c.unique_fetches == 2 * n and c.vector_fetches == 2 * n
    assert r.unique_fetches == n * n + n and r.vector_fetches == 3 * n
    assert abs(c.checksum - r.checksum) <= 1e-4 * max(1.0, abs(r.checksum))
    assert c.min_seconds <= c.mean_seconds and r.min_seconds <= r.mean_seconds and c.repeats == 3
    big = cio.matvec_scheme_bench(cio.kDenseCap + 1, "circulant", 1)  # no cap on the circulant scheme
    assert big.unique_fetches == 2 * (cio.kDenseCap + 1)
    out = io.StringIO()
    cio.matvec_bench([64], repeats=2, out=out)
    lines = out.getvalue().splitlines()
    assert lines[0] == cio.kBenchCsvHeader and len(lines) == 3
    circ, ref = lines[1].split(","), lines[2].split(",")
    assert circ[0] == "matvec-circulant" and ref[0] == "matvec-reference" and circ[5] == "2"
    assert circ[9] == "1024" and ref[9] == "33280"


@pytest.mark.parametrize("n,m,k,seed,iters", [(4096, 1024, 64, 1, 200), (2048, 1024, 40, 2, 100), (8192, 2048, 80, 3, 40)])
def test_coop_cadmm_matches_oracle(n, m, k, seed, iters):
    """Persistent cooperative cADMM (all iterations in one launch, grid barriers between phases) against the
    oracle's phase engine."""
    p = orc.make_problem(n, m, k, seed)
    g = cl.cadmm_setup(op_of(p), p.y)
    g.step(iters)
    o = orc.Cadmm(p.row, p.omega, p.y)
    o.step(iters, orc.ENGINE_PHASES)
    assert g.t == iters
    assert_parity(g.get("z"), o.get("z"), what="z")
    for f in ("x", "v", "mu", "nu", "beta"):
        assert rel_l2(g.get(f), o.get(f)) <= REL_TOL, f


# ------------------------------------------------- tensor-core products (csrc/tc_dense.cu)
@pytest.mark.parametrize("kind,lg,iters,f16", [("ista", 18, 4, "0"), ("ista", 17, 4, "0"), ("cadmm", 16, 3, "0"),
                                               ("cadmm", 15, 3, "0"), ("ista", 18, 4, "1"), ("cadmm", 16, 3, "1")])
def test_tensor_core_products_match_ffma_kernels(kind, lg, iters, f16, monkeypatch):
    """k_tc_dense (3xTF32, or the fp16 2-term split with CLB_TC_F16=1; TMEM drained to fp32) against
    the FFMA kernels (CLB_NO_TC=1), which are themselves oracle-checked: same iterates to fp32
    accuracy after a few iterations."""
    monkeypatch.setenv("CLB_TC_F16", f16)
    n = 1 << lg
    p = orc.make_problem(n, n // 4, max(1, n // 256), 3)
    setup = cl.ista_setup if kind == "ista" else cl.cadmm_setup
    fields = ("x", "r", "delta") if kind == "ista" else ("z", "x", "v", "beta")
    got = {}
    for off in ("0", "1"):
        monkeypatch.setenv("CLB_NO_TC", off)
        g = setup(op_of(p), p.y)
        g.step(iters)
        got[off] = {f: g.get(f) for f in fields}
        del g
    for f in fields:
        tol = 1e-3 if f == "delta" else 2e-5
        assert rel_l2(got["0"][f], got["1"][f]) <= tol, (f, rel_l2(got["0"][f], got["1"][f]))


@pytest.mark.parametrize("kind,lg", [("ista", 18), ("cadmm", 17)])
def test_tensor_core_sharded_matches_unsharded(kind, lg):
    """Two shards of one solve on one GPU, slices exchanged locally after every phase (the
    all-gather's effect), against the unsharded solve: bitwise identical iterates, since the
    split-K decomposition depends on n only."""
    import torch
    from paper_1707_02244_b200.dist import CudaShard
    n = 1 << lg
    p = orc.make_problem(n, n // 4, max(1, n // 256), 5)
    setup = cl.ista_setup if kind == "ista" else cl.cadmm_setup
    iters = 3
    ref = setup(op_of(p), p.y)
    ref.step(iters)
    want = ref.get("x")
    states = [setup(op_of(p), p.y) for _ in range(2)]
    shards = [CudaShard(s, r, 2) for r, s in enumerate(states)]
    for _ in range(iters):
        for ph in shards[0].phases():
            outs = []
            for sh in shards:
                sh.run_phase(ph)
                sh.state.synchronize()
                outs.append(sh.phase_output(ph))
            (f0, b0, e0), (f1, b1, e1) = outs
            f1[b0:e0].copy_(f0[b0:e0])
            f0[b1:e1].copy_(f1[b1:e1])
            torch.cuda.synchronize()
    for s in states:
        s.synchronize()
    got = states[0].get("x")
    assert np.array_equal(got, want), rel_l2(got, want)


@pytest.mark.parametrize("f16", ["0", "1"])
@pytest.mark.parametrize("case", ["wide", "tiny", "huge", "sparse"])
def test_tensor_core_product_scaling(case, f16, monkeypatch):
    """k_tc_dense at n = 2^20 on inputs that stress the fp16 path's power-of-two scaling (and the
    3xTF32 path on the same data): 12 decades of dynamic range, uniformly tiny (1e-30) or huge
    (1e30) magnitudes, and a vector that is zero except for a few entries.  Same 5e-5 bar as every
    other product."""
    monkeypatch.setenv("CLB_TC_F16", f16)
    n = 1 << 20
    rng = np.random.default_rng(11)
    row = rng.standard_normal(n)
    x = rng.standard_normal(n)
    if case == "wide":
        x *= 10.0 ** rng.uniform(-6, 6, n)
    elif case == "tiny":
        x *= 1e-30
        row *= 1e-5
    elif case == "huge":
        x *= 1e30
    else:
        x[:] = 0.0
        x[rng.choice(n, 7, replace=False)] = rng.standard_normal(7)
    C = cl.CirculantMatrix(row)
    want = orc.circ_matvec(row, x, use_fft=True)
    assert rel_l2(cl.circ_matvec(C, x), want) <= 5e-5
    want_t = orc.circ_matvec(row, x, transpose=True, use_fft=True)
    assert rel_l2(cl.circ_transpose_matvec(C, x), want_t) <= 5e-5


@pytest.mark.parametrize("lg", [20, 24])
def test_tensor_core_product_error_bound(lg):
    """The fp16-split tcgen05 product's error budget, pinned in a test at the bench size (2^20) and at C4/C5's
    2^24: at sampled outputs, |got - exact| / sum_j |c_{j-i} u_j| <= 2e-8 (fp32 FFMA-level; measured 2.2e-9 to
    4.6e-9, tools/microbench/tc_probe.cu), the exact sum in fp64 over all n terms."""
    n = 1 << lg
    rng = np.random.default_rng(5)
    row = rng.standard_normal(n).astype(np.float32).astype(np.float64)  # exactly representable: the
    u = rng.standard_normal(n).astype(np.float32).astype(np.float64)    # bound measures the product alone
    got = cl.circ_matvec(cl.CirculantMatrix(row), u)
    worst = 0.0
    for i in rng.choice(n, 24, replace=False):
        terms = row[(np.arange(n) - i) % n] * u  # C u: out[i] = sum_j c[(j - i) mod n] u[j] (circulant.hpp:6-8)
        worst = max(worst, abs(got[i] - terms.sum()) / np.abs(terms).sum())
    print(f"tcgen05 product n=2^{lg}: max |err| / sum|terms| = {worst:.2e} over 24 sampled outputs")
    assert worst <= 2e-8


@pytest.mark.parametrize("kind,lg", [("cadmm", 18), ("cadmm", 22), ("ista", 20), ("ista", 22)])
def test_fft_unchecked_and_checked_steps_bitwise(kind, lg):
    """The FFT engine's unchecked iterations (16-byte cADMM duals, batched consumer loads) and its checked ones
    (the scalar metric-producing epilogues) advance the state identically, bit for bit."""
    n = 1 << lg
    p = cl.make_problem(n, n // 4, n // 256, 11)
    setup = cl.cadmm_setup if kind == "cadmm" else cl.ista_setup
    fields = ("x", "z", "nu", "mu", "v", "beta") if kind == "cadmm" else ("x", "r", "delta")
    a = setup(p.op, p.measurements, cl.SolverConfig(use_fft=True))
    b = setup(p.op, p.measurements, cl.SolverConfig(use_fft=True))
    a.step(6)
    for _ in range(6):
        b.step_checked()
    a.synchronize()
    b.synchronize()
    for f in fields:
        assert np.array_equal(a.get(f), b.get(f)), f
