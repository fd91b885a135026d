"""The library-owned sharded solve on one GPU: the data plane of 2/4/8 ranks with the exchange
inside the library (cl_group_*, peer-copy transport: every rank on device 0), and the NCCL paths at world
size 1 (cl_group_* over ncclCommInitAll, cl_comm_* + cl_solver_attach_comm).  Every sharding must give the
unsharded iterate bitwise: each output is computed by the same arithmetic on whichever rank owns it."""
import os

import numpy as np
import pytest

import paper_1707_02244_b200 as cl
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if cl.device_count() < 1:
        pytest.skip("no CUDA device")


def op_of(p):
    return cl.PartialCirculantOperator(cl.CirculantMatrix(p.row), cl.SubsamplingMask(p.omega, p.n))


CASES = [("ista", 1 << 18), ("ista", 1 << 16), ("cadmm", 1 << 16), ("cadmm", 1 << 15)]


@pytest.mark.parametrize("kind,n", CASES)
@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("transport", ["copy", "peer"])
def test_group_transport_bitwise(kind, n, world, transport):
    """World 2/4/8 on one GPU through the library's data plane: peer copies after each phase ("copy"), or the
    exchange fused into the producing epilogue kernels as stores into every rank's copy ("peer"); the iterate
    and every state vector equal the unsharded solve's, bitwise."""
    p = orc.make_problem(n, n // 4, n // 256, 5)
    setup = cl.ista_setup if kind == "ista" else cl.cadmm_setup
    solo = setup(op_of(p), p.y)
    solo.step(4)
    g = cl.ShardedSolve(kind, op_of(p), p.y, devices=[0] * world, transport=transport)
    g.step(4)
    fields = ("x", "r", "delta") if kind == "ista" else ("x", "z", "nu", "mu", "v", "beta")
    for f in fields:
        assert np.array_equal(g.get(f), solo.get(f)), f
    assert g.info() == {"world": world, "t": 4, "transport": cl.ShardedSolve.TRANSPORTS[transport]}


@pytest.mark.parametrize("kind", ["ista", "cadmm"])
def test_group_run_loop_matches_unsharded(kind):
    """run() through the group: same check cadence, the metrics summed over ranks, the same iterate."""
    p = orc.make_problem(1 << 16, 1 << 14, 256, 9)
    cfg = cl.SolverConfig(max_iter=40, check_every=10, target_mse=1e-30)
    run = cl.ista_run if kind == "ista" else cl.cadmm_run
    ref = run(p.y, op_of(p), cfg, truth=p.x_true)
    for world, transport in ((4, "copy"), (3, "peer"), (1, "nccl")):
        rep = cl.ShardedSolve(kind, op_of(p), p.y, cfg, devices=[0] * world, transport=transport).run(truth=p.x_true)
        assert rep.iterations == ref.iterations == 40
        assert np.array_equal(rep.final_x, ref.final_x)
        assert [t.iteration for t in rep.mse_trace] == [10, 20, 30, 40]
        assert all(abs(a.value - b.value) <= 1e-12 * max(1.0, abs(b.value))
                   for a, b in zip(rep.mse_trace, ref.mse_trace))
        assert all(t.elapsed_seconds >= 0 for t in rep.mse_trace)


@pytest.mark.parametrize("kind", ["ista", "cadmm"])
def test_native_comm_world1_attach(kind):
    """cl_comm_unique_id + cl_comm_init_rank (world 1) + cl_solver_attach_comm: the NCCL-backed sharded step
    and run loop of the one-process-per-GPU mode."""
    from paper_1707_02244_b200.dist import NativeComm
    p = orc.make_problem(1 << 18, 1 << 16, 1024, 3)
    setup = cl.ista_setup if kind == "ista" else cl.cadmm_setup
    solo = setup(op_of(p), p.y)
    solo.step(3)
    comm = NativeComm(NativeComm.unique_id(), 1, 0, 0)
    st = setup(op_of(p), p.y)
    comm.attach(st)
    st.step(3)
    f = "x" if kind == "ista" else "z"
    assert np.array_equal(st.get(f), solo.get(f))


def test_group_rejects_bad_arguments():
    p = orc.make_problem(4096, 1024, 64, 1)
    with pytest.raises(cl.ParameterError):
        cl.ShardedSolve("ista", op_of(p), p.y, devices=[0, 0], transport="copy",
                        cfg=cl.SolverConfig(use_fft=True))
    with pytest.raises(cl.DimensionError):
        cl.ShardedSolve("ista", op_of(p), p.y[:-1], devices=[0])


def test_cpp_adapter_sharded_config4():
    """BASELINE config 4 (cADMM n = 2^24, m = 2^22) sharded through the C-ABI from C++ in one process
    (circlasso_b200::ShardedSolve over cl_group_*): NCCL world 1 and a 2-rank peer-copy split, each bitwise
    equal to the unsharded solve (tests/cpp/adapter_test.cpp, mode c4)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1707_02244_b200", "_lib",
                       "adapter_test")
    out = subprocess.run([exe, "c4"], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0 and "PASS" in out.stdout and out.stdout.count("bitwise equal") == 2, \
        out.stdout + out.stderr


@pytest.mark.parametrize("kind,n,world", [("ista", 1 << 18, 2), ("cadmm", 1 << 16, 2), ("ista", 1 << 16, 3)])
def test_ipc_peer_transport_processes(kind, n, world, tmp_path):
    """One process per rank (all on device 0) over the CUDA IPC peer-store transport (cl_solver_peer_export /
    _attach; no NCCL): the run loop's iterations, trace and final iterate equal the unsharded solve's, and the
    exchanged vectors are complete on every rank, bitwise."""
    import subprocess
    import sys
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "helpers", "ipc_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, kind, str(n), str(r), str(world), str(tmp_path)],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(world)]
    outs = [pr.communicate(timeout=300)[0] for pr in procs]
    assert all(pr.returncode == 0 for pr in procs), outs
    p = orc.make_problem(n, n // 4, n // 256, 5)
    cfg = cl.SolverConfig(max_iter=12, check_every=4, target_mse=1e-30)
    run = cl.ista_run if kind == "ista" else cl.cadmm_run
    ref = run(p.y, op_of(p), cfg, truth=p.x_true)
    setup = cl.ista_setup if kind == "ista" else cl.cadmm_setup
    solo = setup(op_of(p), p.y, cfg)
    solo.step(12)
    for r in range(world):
        got = dict(np.load(tmp_path / f"out_{r}.npz"))
        assert int(got["iterations"]) == ref.iterations == 12
        assert np.array_equal(got["final_x"], ref.final_x)
        assert np.allclose(got["trace"][:, 1], [t.value for t in ref.mse_trace], rtol=1e-12, atol=0)
        for f in (("x", "r") if kind == "ista" else ("x", "beta", "v")):
            assert np.array_equal(got[f], solo.get(f)), (r, f)
