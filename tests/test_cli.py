"""The reference's command-line front end over the B200 engine (tools/cli/circlasso_b200_cli.cpp mirrors
/root/reference/proj/tools/circlasso_cli.cpp): subcommands, files, CSV schema and exit codes.  CPU tests
cover generation and usage errors; the -m gpu tests run recover / bench / matvec-bench / deblur."""
import csv
import os
import subprocess

import numpy as np
import pytest

import paper_1707_02244_b200 as cl
from paper_1707_02244_b200 import io as clio
from oracle import oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1707_02244_b200", "_lib", "circlasso_b200_cli")
HEADER = "algorithm,n,m,k,seed,iterations,setup_s,total_s,final_mse,footprint_bytes,iters_per_s,status"


def run(*args, timeout=600):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=timeout)


def test_gen_writes_the_reference_files_bit_exact(tmp_path):
    """cli:186-199: defaults k = n/10, m = n/2; the three CIRCVEC1/CIRCOPR1 files hold make_problem's vectors."""
    out = run("gen", "--n", 1000, "--seed", 4, "--out", tmp_path / "p")
    assert out.returncode == 0 and "gen: n=1000 m=500 k=100 seed=4" in out.stdout
    p = orc.make_problem(1000, 500, 100, 4)
    A = clio.read_operator(str(tmp_path / "p.operator.bin"))
    assert np.array_equal(clio.read_vector(str(tmp_path / "p.signal.bin")), p.x_true)
    assert np.array_equal(clio.read_vector(str(tmp_path / "p.measurements.bin")), p.y)
    assert np.array_equal(A.circulant().first_row(), p.row) and np.array_equal(A.mask().omega(), p.omega)


def test_usage_errors_exit_1(tmp_path):
    assert run().returncode == 1
    assert run("--help").returncode == 0
    assert run("bogus").returncode == 1
    assert run("recover").returncode == 1  # --problem required
    assert run("gen", "--n", 16).returncode == 1  # --out required
    assert run("gen", "--n", "abc", "--out", tmp_path / "x").returncode == 1
    bad = run("recover", "--problem", tmp_path / "missing")
    assert bad.returncode == 1 and "cannot open" in bad.stderr
    run("gen", "--n", 64, "--out", tmp_path / "q")
    e = run("recover", "--problem", tmp_path / "q", "--engine", "opencl")
    assert e.returncode == 1 and "--engine" in e.stderr
    e = run("recover", "--problem", tmp_path / "q", "--pairing", "odd")
    assert e.returncode == 1 and "--pairing" in e.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("solver,engine", [("ista", "cuda"), ("cadmm", "cuda"), ("cadmm", "cuda-fft"),
                                           ("ista", "fft"), ("admm", "cuda"), ("ista", "phases"),
                                           ("cadmm", "phases"), ("admm", "phases")])
def test_recover_matches_the_library_and_writes_csv(tmp_path, solver, engine):
    if cl.device_count() < 1:
        pytest.skip("no CUDA device")
    run("gen", "--n", 512, "--seed", 2, "--out", tmp_path / "p")
    out = run("recover", "--problem", tmp_path / "p", "--solver", solver, "--engine", engine, "--max-iter", 300,
              "--target-mse", 1e-4, "--out", tmp_path / "r.csv", "--out-x", tmp_path / "x.bin")
    assert out.stdout.startswith(f"{solver}: n=512 m=256 iterations=")
    assert "final mse vs truth" in out.stdout and "footprint_bytes=" in out.stdout
    rows = list(csv.reader(open(tmp_path / "r.csv")))
    assert ",".join(rows[0]) == HEADER and rows[1][0] == solver and rows[1][3] == "51"
    p = orc.make_problem(512, 256, 51, 2)
    cfg = cl.SolverConfig(max_iter=300, target_mse=1e-4, use_fft=engine in ("cuda-fft", "fft"))
    run_fn = {"ista": cl.ista_run, "cadmm": cl.cadmm_run, "admm": cl.admm_dense_run}[solver]
    ref = run_fn(p.y, cl.PartialCirculantOperator(cl.CirculantMatrix(p.row), cl.SubsamplingMask(p.omega, 512)),
                 cfg, truth=p.x_true)
    assert np.array_equal(clio.read_vector(str(tmp_path / "x.bin")), ref.final_x)
    assert out.returncode == (0 if ref.reached_target else 2)
    assert rows[1][-1] == ("ok" if ref.reached_target else "max_iter")


@pytest.mark.gpu
def test_bench_matvec_bench_and_deblur(tmp_path):
    if cl.device_count() < 1:
        pytest.skip("no CUDA device")
    b = run("bench", "--n", 1024, "--n", 8192, "--seeds", 1, "--out", tmp_path / "b.csv")
    assert b.returncode == 0, b.stderr
    rows = list(csv.DictReader(open(tmp_path / "b.csv")))
    assert [(r["algorithm"], r["n"]) for r in rows] == [("ista", "1024"), ("admm", "1024"), ("cadmm", "1024"),
                                                      ("ista", "8192"), ("admm", "8192"), ("cadmm", "8192")]
    assert rows[4]["status"] == "skipped" and all(r["status"] == "ok" for r in rows if r["algorithm"] != "admm"
                                                  or r["n"] == "1024")
    mv = run("matvec-bench", "--n", 4096, "--n", 8192, "--repeats", 3, "--out", tmp_path / "m.csv")
    assert mv.returncode == 0, mv.stderr
    mrows = list(csv.DictReader(open(tmp_path / "m.csv")))
    assert [r["algorithm"] for r in mrows] == ["matvec-circulant", "matvec-reference"] * 2
    assert mrows[3]["status"] == "skipped" and mrows[0]["footprint_bytes"] == str(2 * 4096 * 8)
    d = run("deblur", "--star-field", "64x64", "--max-iter", 20000, "--out", tmp_path / "d")
    assert d.returncode == 0, d.stdout + d.stderr
    for suffix in ("truth", "blurred", "recovered", "errmap"):
        img = cl.read_pgm(str(tmp_path / f"d.{suffix}.pgm"))
        assert (img.width, img.height) == (64, 64)
    st = list(csv.DictReader(open(tmp_path / "d.stats.csv")))[0]
    assert (st["width"], st["n"], st["m"], st["L"]) == ("64", "4096", "2048", "5")
    assert float(st["mse"]) <= 5e-2  # acceptance criterion 8 (tests/acceptance.cpp:398-427)
