"""CPU-only checks of the product library: it loads, exports the whole C-ABI,
and its host-side parts (generation, fp64 setup transforms, validation) agree
with the oracle.  No kernel is launched here."""
import os
import re

import numpy as np
import pytest

import paper_1707_02244_b200 as cl
from paper_1707_02244_b200 import _native
from oracle import oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            src = open(os.path.join(ROOT, "include", fn)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            names |= set(re.findall(r"\b(cl_[a-z0-9_]+)\s*\(", src))
    return names


def test_library_exports_every_declared_symbol():
    names = declared_symbols()
    assert len(names) > 30
    missing = [n for n in sorted(names) if not hasattr(_native.lib, n)]
    assert not missing, missing
    assert set(_native.EXPORTED) == names
    assert _native.lib.cl_abi_version() == 3


def test_nvtx_ranges_name_the_reference_phases():
    """The tracing ranges carry the reference's KernelPhase names (parallel.hpp:179-307)."""
    blob = open(_native.lib._name, "rb").read()
    for name in (b"cpista residual computation", b"cpista thresholded gradient", b"cpadmm primal variables update",
                 b"cpadmm signal recovery", b"cpadmm thresholded variables update", b"cl_solver_run",
                 b"cl_group_step"):
        assert name + b"\0" in blob, name
    assert b"nvtxRangePushA" in blob or b"libnvToolsExt" in blob or b"NVTX_INJECTION" in blob


def test_config_defaults_match_reference():
    cfg = cl.SolverConfig()
    c = cfg._c()
    assert (c.alpha, c.tau, c.rho, c.sigma, c.tau1, c.tau2) == (1e-4, 0.0, 0.1, 0.1, 1.0, 1.0)
    assert c.max_iter == 100000 and np.isnan(c.target_mse) and c.check_every == 10 and c.pairing == 0
    assert c.engine == 0 and cl.SolverConfig(use_fft=True)._c().engine == 1


@pytest.mark.parametrize("n,m,k,seed", [(128, 64, 12, 9), (97, 48, 9, 3), (4096, 1024, 64, 1), (1 << 14, 1 << 12, 64, 7)])
def test_make_problem_bit_exact_with_oracle(n, m, k, seed):
    a = cl.make_problem(n, m, k, seed)
    b = orc.make_problem(n, m, k, seed)
    assert np.array_equal(a.op.circulant().first_row(), b.row)
    assert np.array_equal(a.op.mask().omega(), b.omega)
    assert np.array_equal(a.signal.values, b.x_true)
    assert np.array_equal(a.signal.support, b.support)
    # y is DFT-evaluated in fp64 by both (different FFTs): tolerance, as the reference's own tests
    assert np.max(np.abs(a.measurements - b.y)) <= 1e-12 * max(1.0, np.max(np.abs(b.y)))


def test_star_field_and_blur_bit_exact():
    assert np.array_equal(cl.gen_star_field(64, 64, 0.1, 21).pixels, orc.gen_star_field(64, 64, 0.1, 21))
    img = cl.make_image(2, 2, [-1.0, 0.5, 2.0, 1.0])
    assert np.array_equal(img.pixels, [0.0, 0.5, 1.0, 1.0])
    with pytest.raises(cl.ParameterError):
        cl.make_image(0, 2, [])
    assert np.array_equal(cl.blur_matrix(16, 5).first_row(), orc.blur_row(16, 5))
    with pytest.raises(cl.ParameterError):
        cl.blur_matrix(8, 9)
    with pytest.raises(cl.ParameterError):
        cl.gen_star_field(8, 8, 1.5, 1)


@pytest.mark.parametrize("n", [2, 8, 17, 97, 256, 4096])
def test_setup_transforms_match_oracle(n):
    row = orc.rng_draws(800 + n, "normal", n)
    C = cl.CirculantMatrix(row)
    assert abs(cl.spectral_norm(C) - orc.spectral_norm(row)) <= 1e-12 * orc.spectral_norm(row)
    b = cl.regularized_gram_inverse(C, 0.1, 0.1).first_row()
    assert np.max(np.abs(b - orc.regularized_gram_inverse(row, 0.1, 0.1))) < 1e-10
    row2 = orc.rng_draws(900 + n, "normal", n)
    comp = cl.compose_sensing(C, cl.CirculantMatrix(row2), cl.SubsamplingMask.Full(n))
    assert np.max(np.abs(comp.circulant().first_row() - orc.circ_compose(row, row2))) < 1e-10


def test_setup_errors_mirror_reference(kats):
    k = kats["gram_singular"]
    with pytest.raises(cl.SingularityError):
        cl.regularized_gram_inverse(cl.CirculantMatrix(k["row"]), k["rho"], k["sigma_singular"])
    with pytest.raises(cl.ParameterError):
        cl.regularized_gram_inverse(cl.CirculantMatrix(k["row"]), 0.0, 0.0)
    k = kats["mask_gram_inverse"]
    d = cl.mask_gram_inverse(cl.SubsamplingMask(k["omega"], k["n"]), k["rho"]).diag()
    assert np.allclose(d, k["d"], rtol=1e-15)
    with pytest.raises(cl.ParameterError):
        cl.SubsamplingMask([4, 1], 8)
    with pytest.raises(cl.ParameterError):
        cl.SubsamplingMask([1, 8], 8)


def test_solver_validation_before_device():
    """ista_setup / cadmm_setup raise exactly where the reference does, before any device work."""
    p = cl.make_problem(32, 16, 3, 13)
    for kw in ({"tau": 1.5}, {"tau": -0.2}, {"alpha": 0.0}):
        with pytest.raises(cl.ParameterError):
            cl.ista_setup(p.op, p.measurements, cl.SolverConfig(**kw))
    for kw in ({"alpha": 0.0}, {"rho": 0.0}, {"sigma": 0.0}, {"tau1": 1.7}, {"tau2": 0.0}):
        with pytest.raises(cl.ParameterError):
            cl.cadmm_setup(p.op, p.measurements, cl.SolverConfig(**kw))
    with pytest.raises(cl.DimensionError):
        cl.ista_setup(p.op, np.zeros(15))
    bad = p.measurements.copy()
    bad[3] = np.nan
    with pytest.raises(cl.DivergenceError):
        cl.ista_setup(p.op, bad)
    Z = cl.PartialCirculantOperator(cl.CirculantMatrix(np.zeros(16)), cl.SubsamplingMask.Full(16))
    with pytest.raises(cl.SingularityError):
        cl.cadmm_setup(Z, orc.rng_draws(15, "normal", 16))


def test_analytic_footprint():
    n18 = 1 << 18
    assert cl.analytic_footprint(cl.FootprintKind.kCpista, n18, n18 // 2, 4) == 4 * n18 * 4
    assert cl.analytic_footprint(cl.FootprintKind.kCpadmm, 1 << 20, 1 << 19, 4) == 40 * 1024 * 1024
    assert cl.analytic_footprint(cl.FootprintKind.kDenseAdmm, 256, 128, 8) == (256 * 256 + 4 * 256 + 128) * 8


def test_cpp_adapter_cpu_parts():
    """The reference-style C++ drop-in (include/circlasso_b200.hpp) links and behaves on the host."""
    import subprocess
    exe = os.path.join(ROOT, "paper_1707_02244_b200", "_lib", "adapter_test")
    assert os.path.exists(exe), "build the package first (make -C paper_1707_02244_b200)"
    out = subprocess.run([exe, "cpu"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and "PASS" in out.stdout, out.stdout + out.stderr


def test_cpp_adapter_eigen_branch_cpu_parts():
    """Reference-style Eigen code (Vector<double>::Zero, comma initializer, <double> templates) against the
    adapter's __has_include(<Eigen/Dense>) branch, built with the Eigen test double of tests/cpp/eigen_stub."""
    import subprocess
    exe = os.path.join(ROOT, "paper_1707_02244_b200", "_lib", "eigen_style_test")
    out = subprocess.run([exe, "cpu"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and "PASS" in out.stdout, out.stdout + out.stderr


# ---------------------------------------------------------------- artifact formats (io.hpp)
def test_vector_files_roundtrip_bit_for_bit(tmp_path):
    """io_cli_test.cpp:81-95"""
    from paper_1707_02244_b200 import io as cio
    v = np.array([0.0, -0.0, 5e-324, np.finfo(float).max, -1e-300, 3.141592653589793, np.nan, -np.inf])
    path = tmp_path / "vector.bin"
    cio.write_vector(v, path)
    assert path.read_bytes() == b"CIRCVEC1" + (8).to_bytes(8, "little") + v.astype("<f8").tobytes()
    back = cio.read_vector(path)
    assert back.tobytes() == v.tobytes()
    cio.write_vector(np.zeros(0), path)
    assert len(cio.read_vector(path)) == 0


def test_operator_files_roundtrip_exactly(tmp_path):
    """io_cli_test.cpp:97-107 (and the byte layout io.hpp:99-112)"""
    from paper_1707_02244_b200 import io as cio
    A = cl.gen_circulant_sensing(64, 24, 99)
    path = tmp_path / "operator.bin"
    cio.write_operator(A, path)
    raw = path.read_bytes()
    assert raw[:8] == b"CIRCOPR1" and int.from_bytes(raw[8:16], "little") == 64
    assert int.from_bytes(raw[16:24], "little") == 24 and len(raw) == 24 + 64 * 8 + 24 * 8
    back = cio.read_operator(path)
    assert back.n() == 64 and back.m() == 24
    assert np.array_equal(back.circulant().first_row(), A.circulant().first_row())
    assert np.array_equal(back.mask().omega(), A.mask().omega())


def test_binary_readers_reject_malformed_files(tmp_path):
    """io_cli_test.cpp:109-152"""
    from paper_1707_02244_b200 import io as cio
    path = tmp_path / "malformed.bin"
    with pytest.raises(cl.FormatError, match="cannot open"):
        cio.read_vector(tmp_path / "missing.bin")
    path.write_bytes(b"CIRCVEX1\x02\x00\x00\x00\x00\x00\x00\x00")
    with pytest.raises(cl.FormatError, match="bad magic"):
        cio.read_vector(path)
    with pytest.raises(cl.FormatError, match="bad magic"):
        cio.read_operator(path)
    path.write_bytes(b"CIRC")
    with pytest.raises(cl.FormatError):
        cio.read_vector(path)
    path.write_bytes(b"CIRCVEC1" + (10).to_bytes(8, "little") + np.full(3, 1.5).tobytes())
    with pytest.raises(cl.FormatError, match="truncated"):
        cio.read_vector(path)
    path.write_bytes(b"CIRCOPR1" + (4).to_bytes(8, "little") + (5).to_bytes(8, "little"))
    with pytest.raises(cl.FormatError, match="m exceeds n"):
        cio.read_operator(path)


def test_bench_rows_compute_throughput_defensively():
    """io_cli_test.cpp:154-167"""
    from paper_1707_02244_b200 import io as cio
    row = cio.BenchRow(iterations=1000, setup_seconds=0.5, total_seconds=2.5)
    assert row.iterations_per_second() == pytest.approx(500.0)
    row.iterations = 0
    assert row.iterations_per_second() == 0.0
    row.iterations, row.total_seconds = 10, row.setup_seconds
    assert row.iterations_per_second() == 0.0


def test_bench_csv_schema_is_pinned():
    """io_cli_test.cpp:169-206"""
    import io
    from paper_1707_02244_b200 import io as cio
    assert cio.kBenchCsvHeader == ("algorithm,n,m,k,seed,iterations,setup_s,total_s,final_mse,"
                                   "footprint_bytes,iters_per_s,status")
    row = cio.BenchRow("cadmm", 1024, 512, 102, 7, 1180, 0.25, 1.5, 9.41674e-05, 40960)
    out = io.StringIO()
    cio.write_bench_header(out)
    cio.write_bench_row(out, row)
    header, line = out.getvalue().splitlines()
    assert header == cio.kBenchCsvHeader
    f = line.split(",")
    assert len(f) == 12 and f[0] == "cadmm" and f[1] == "1024" and f[4] == "7" and f[5] == "1180"
    assert float(f[8]) == row.final_mse and f[9] == "40960" and f[11] == "ok"
    assert float(f[10]) == pytest.approx(1180.0 / 1.25)
    assert f[6] == "0.25" and f[7] == "1.5"  # ostream setprecision(9) general format


def test_matvec_scheme_bench_validation_before_device():
    """parallel_test.cpp:279-289: argument and capacity errors are raised before any device work."""
    from paper_1707_02244_b200 import io as cio
    with pytest.raises(cl.ParameterError):
        cio.matvec_scheme_bench(0, "circulant", 1)
    with pytest.raises(cl.ParameterError):
        cio.matvec_scheme_bench(8, "circulant", 0)
    with pytest.raises(cl.CapacityError):
        cio.matvec_scheme_bench(cio.kDenseCap + 1, "reference", 1)


def test_dense_admm_validation_before_any_device_work():
    """admm_setup's checks (solvers.hpp:288-296): size, then the dense cap, then rho/alpha -- all raised on
    the host before the library touches a device, so they hold on a CPU-only machine too."""
    p = cl.make_problem(256, 128, 25, 11)
    with pytest.raises(cl.CapacityError, match="exceeds the dense cap 128"):
        cl.admm_setup(p.op, p.measurements, cl.SolverConfig(dense_cap=128))
    with pytest.raises(cl.DimensionError):
        cl.admm_setup(p.op, p.measurements[:-1], cl.SolverConfig(dense_cap=128))
    with pytest.raises(cl.ParameterError, match="rho"):
        cl.admm_setup(p.op, p.measurements, cl.SolverConfig(rho=0.0))
    with pytest.raises(cl.ParameterError, match="alpha"):
        cl.admm_dense_run(p.measurements, p.op, cl.SolverConfig(alpha=-1.0))
    assert cl.analytic_footprint(cl.FootprintKind.kDenseAdmm, 256, 128, 4) == (256 * 256 + 4 * 256 + 128) * 4


# ---- PGM images (image.hpp:56-153), the reference's own cases (tests/image_deblur_test.cpp:62-140) ----
def test_pgm_roundtrip_and_quantization(tmp_path):
    rng = np.random.default_rng(77)
    img = cl.make_image(9, 5, rng.uniform(size=45))
    path = tmp_path / "roundtrip.pgm"
    cl.write_pgm(img, path)
    back = cl.read_pgm(path)
    assert (back.width, back.height, len(back.pixels)) == (9, 5, 45)
    assert np.max(np.abs(back.pixels - img.pixels)) <= 0.5 / 255.0 + 1e-12
    raw = cl.GrayImage(3, 1, np.array([-3.0, 0.5, 1.7]))  # deliberately unclamped
    cl.write_pgm(raw, tmp_path / "q.pgm")
    q = cl.read_pgm(tmp_path / "q.pgm")
    assert q.pixels[0] == 0.0 and q.pixels[1] == 128.0 / 255.0 and q.pixels[2] == 1.0  # lround(127.5) = 128
    assert open(tmp_path / "q.pgm", "rb").read() == b"P5\n3 1\n255\n\x00\x80\xff"


def test_pgm_header_comments_and_errors(tmp_path):
    p = tmp_path / "h.pgm"
    p.write_bytes(b"P5\n# a comment line\n 3 2 # trailing comment\n255\n" + bytes([0, 0x40, 0x80, 0xC0, 0xFF, 0x20]))
    img = cl.read_pgm(p)
    assert (img.width, img.height) == (3, 2) and img.pixels[0] == 0.0 and img.pixels[4] == 1.0
    with pytest.raises(cl.FormatError, match="cannot open"):
        cl.read_pgm(tmp_path / "missing.pgm")
    for content, needle in ((b"P2\n2 2\n255\n0 0 0 0\n", "'P2'"), (b"P5\nabc 2\n255\n", "'abc'"),
                            (b"P5\n2 2\n65535\n", "65535"), (b"P5\n2 2\n0\n", "maxval"),
                            (b"P5\n4 4\n255\nabcde", "truncated")):
        p.write_bytes(content)
        with pytest.raises(cl.FormatError, match=needle):
            cl.read_pgm(p)
    with pytest.raises(cl.ParameterError):
        cl.write_pgm(cl.GrayImage(0, 0, np.zeros(0)), tmp_path / "e.pgm")


def test_makefile_builds_every_engine_source():
    """The library's Makefile compiles and links exactly the sources under csrc/ and tracks every header (a
    stale list once linked a deleted kernel's object from an old build tree)."""
    mk = open(os.path.join(ROOT, "paper_1707_02244_b200", "Makefile")).read()
    src = set(re.search(r"^SRC := (.*)$", mk, re.M).group(1).split())
    hdr = set(re.search(r"^HDR := (.*)$", mk, re.M).group(1).split())
    csrc = os.path.join(ROOT, "paper_1707_02244_b200", "csrc")
    files = os.listdir(csrc)
    assert src == {f"csrc/{f}" for f in files if f.endswith((".cu", ".cpp"))}
    assert {f"csrc/{f}" for f in files if f.endswith((".cuh", ".hpp"))} <= hdr
    assert "$(OUT): $(OBJ)" in mk
