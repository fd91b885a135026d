"""Artifact formats of the reference (io.hpp) and its protocol bench sweep (cli:263-333).

CIRCVEC1 vectors and CIRCOPR1 operators are read and written by the library
(csrc/io.cpp) byte for byte as the reference does, with its FormatError
messages; the bench CSV rows use its pinned schema and ostream formatting, so
tables from this engine and from the reference concatenate.
"""
from __future__ import annotations

import ctypes as C
import math
import sys
from dataclasses import dataclass
from typing import Iterable, Optional, TextIO

import numpy as np

from ._native import cl_bench_row, lib
from .api import (CirculantMatrix, FormatError, PartialCirculantOperator, SolverConfig, SubsamplingMask, _check, _f64,
                  _pd, _pi, cadmm_run, ista_run, make_problem)

_d = C.POINTER(C.c_double)
_i64 = C.POINTER(C.c_int64)


def _path(p) -> bytes:
    return str(p).encode()


def write_vector(v, path) -> None:
    """io.hpp:80-87"""
    v = _f64(v)
    _check(lib.cl_write_vector(_path(path), _pd(v), len(v)))


def read_vector(path) -> np.ndarray:
    """io.hpp:89-97"""
    n = C.c_int64(0)
    _check(lib.cl_read_vector(_path(path), None, 0, C.byref(n)))
    out = np.zeros(n.value)
    _check(lib.cl_read_vector(_path(path), _pd(out), n.value, C.byref(n)))
    return out


def write_operator(A: PartialCirculantOperator, path) -> None:
    """io.hpp:99-112"""
    row = _f64(A.circulant().first_row())
    om = np.ascontiguousarray(A.mask().omega(), dtype=np.int64)
    _check(lib.cl_write_operator(_path(path), A.n(), A.m(), _pd(row), _pi(om)))


def read_operator(path) -> PartialCirculantOperator:
    """io.hpp:114-131"""
    n, m = C.c_int64(0), C.c_int64(0)
    _check(lib.cl_read_operator(_path(path), None, 0, None, 0, C.byref(n), C.byref(m)))
    row = np.zeros(n.value)
    om = np.zeros(m.value, dtype=np.int64)
    _check(lib.cl_read_operator(_path(path), _pd(row), n.value, _pi(om), m.value, C.byref(n), C.byref(m)))
    return PartialCirculantOperator(CirculantMatrix(row), SubsamplingMask(om, n.value))


kBenchCsvHeader = ("algorithm,n,m,k,seed,iterations,setup_s,total_s,final_mse,"
                   "footprint_bytes,iters_per_s,status")


@dataclass
class BenchRow:
    """io.hpp:133-153"""
    algorithm: str = ""
    n: int = 0
    m: int = 0
    k: int = 0
    seed: int = 0
    iterations: int = 0
    setup_seconds: float = 0.0
    total_seconds: float = 0.0
    final_mse: float = 0.0
    footprint_bytes: int = 0
    status: str = "ok"

    def _c(self) -> cl_bench_row:
        r = cl_bench_row()
        r.algorithm, r.n, r.m, r.k, r.seed = self.algorithm.encode(), self.n, self.m, self.k, self.seed
        r.iterations, r.setup_seconds, r.total_seconds = self.iterations, self.setup_seconds, self.total_seconds
        r.final_mse, r.footprint_bytes, r.status = self.final_mse, self.footprint_bytes, self.status.encode()
        return r

    def iterations_per_second(self) -> float:
        r = self._c()
        return lib.cl_bench_iters_per_second(C.byref(r))


def _text(fn, *args) -> str:
    n = C.c_int64(0)
    _check(fn(*args, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(fn(*args, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def write_bench_header(out: TextIO) -> None:
    """io.hpp:157-159"""
    out.write(_text(lib.cl_bench_csv_header) + "\n")


def write_bench_row(out: TextIO, row: BenchRow) -> None:
    """io.hpp:161-168"""
    r = row._c()
    out.write(_text(lib.cl_bench_csv_row, C.byref(r)) + "\n")


def bench(sizes: Iterable[int], solvers: Iterable[str] = ("ista", "cadmm"), seeds: int = 1,
          cfg: Optional[SolverConfig] = None, out: Optional[TextIO] = None, device: int = 0) -> None:
    """The reference's `bench` sweep (cli:263-333): for each n, m = n/2, k = n/10, seeds 1..seeds, each
    solver run on make_problem with the truth as the stopping metric, one pinned-CSV row per run.
    `admm` (dense ADMM, out of scope here: SURVEY 8f row 4) is written as status "skipped"."""
    cfg = cfg or SolverConfig()
    out = out or sys.stdout
    write_bench_header(out)
    for n in sizes:
        m, k = n // 2, n // 10
        for seed in range(1, seeds + 1):
            p = make_problem(n, m, k, seed)
            for solver in solvers:
                row = BenchRow(algorithm=solver, n=n, m=m, k=k, seed=seed)
                if solver == "admm":
                    row.status = "skipped"
                    write_bench_row(out, row)
                    continue
                if solver not in ("ista", "cadmm"):
                    raise ValueError("--solver must be ista, admm, or cadmm")
                try:
                    run = ista_run if solver == "ista" else cadmm_run
                    rep = run(p.measurements, p.op, cfg, truth=p.signal.values, device=device)
                    row.iterations, row.setup_seconds, row.total_seconds = (rep.iterations, rep.setup_seconds,
                                                                            rep.total_seconds)
                    row.final_mse, row.footprint_bytes = rep.final_metric, rep.footprint_bytes
                    row.status = "ok" if rep.reached_target or math.isnan(cfg.target_mse) else "max_iter"
                except FormatError:
                    raise
                except Exception as e:  # DivergenceError -> "diverged", others -> "error" (cli:313-320)
                    row.status = "diverged" if type(e).__name__ == "DivergenceError" else "error"
                write_bench_row(out, row)


# ---- matvec scheme benchmark (parallel.hpp:318-406, cli:334-372; the paper's Fig. 5) ----
kDenseCap = 4096  # circulant.hpp:31


@dataclass
class SchemeTiming:
    """parallel.hpp:329-338"""
    scheme: str = "circulant"
    n: int = 0
    repeats: int = 0
    min_seconds: float = 0.0
    mean_seconds: float = 0.0
    unique_fetches: int = 0
    vector_fetches: int = 0
    checksum: float = 0.0


def matvec_scheme_bench(n: int, scheme: str = "circulant", repeats: int = 1, seed: int = 1,
                        dense_cap: int = kDenseCap, device: int = 0) -> SchemeTiming:
    """`repeats` device-timed products of the seeded circulant: "circulant" = the direct engine,
    "reference" = a dense row-major copy through a plain GEMV (fp32 on the GPU)."""
    if scheme not in ("circulant", "reference"):
        raise ValueError("scheme must be 'circulant' or 'reference'")
    mn, me, ck = C.c_double(0), C.c_double(0), C.c_double(0)
    uf, vf = C.c_uint64(0), C.c_uint64(0)
    _check(lib.cl_matvec_scheme_bench(device, n, 0 if scheme == "circulant" else 1, repeats, seed, dense_cap,
                                      C.byref(mn), C.byref(me), C.byref(uf), C.byref(vf), C.byref(ck)))
    return SchemeTiming(scheme, n, repeats, mn.value, me.value, uf.value, vf.value, ck.value)


def matvec_bench(sizes: Iterable[int], repeats: int = 5, seed: int = 1, out: Optional[TextIO] = None,
                 dense_cap: int = kDenseCap, device: int = 0) -> None:
    """cli:334-372: one pinned-CSV row per (n, scheme); the dense scheme above the cap is "skipped"."""
    out = out or sys.stdout
    write_bench_header(out)
    for n in sizes:
        for scheme in ("circulant", "reference"):
            row = BenchRow(algorithm=f"matvec-{scheme}", n=n, m=n, k=0, seed=seed)
            if scheme == "reference" and n > dense_cap:
                row.status = "skipped"
                write_bench_row(out, row)
                continue
            t = matvec_scheme_bench(n, scheme, repeats, seed, dense_cap, device)
            row.iterations, row.setup_seconds, row.total_seconds = repeats, 0.0, t.mean_seconds * repeats
            row.final_mse, row.footprint_bytes = 0.0, t.unique_fetches * 8
            write_bench_row(out, row)
