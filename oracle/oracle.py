"""ctypes wrapper over oracle/_build/liborc.so — TEST INFRASTRUCTURE ONLY.

The CPU restatement of the reference circlasso solver (see the header of
oracle/circlasso_oracle.cpp for what it restates and how it is pinned).
Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg; the product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liborc.so")

OK, EDIM, EPARAM, ESINGULAR, EDIVERGE, ECAPACITY, EFORMAT, ECONSIST, EPHASE = range(9)
ENGINE_PHASES, ENGINE_FFT = 0, 1


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build() -> str:
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
        os.path.join(_HERE, "circlasso_oracle.cpp")
    ):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _decl(_lib)
    return _lib


_d = C.POINTER(C.c_double)
_i64 = C.POINTER(C.c_int64)
_u64 = C.POINTER(C.c_uint64)


def _decl(L):
    L.orc_last_error.restype = C.c_char_p
    L.orc_splitmix64.restype = C.c_uint64
    L.orc_splitmix64.argtypes = [C.c_uint64]
    L.orc_derive_seed.restype = C.c_uint64
    L.orc_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
    L.orc_mt19937_64.argtypes = [C.c_uint64, C.c_int64, _u64]
    L.orc_rng_draws.argtypes = [C.c_uint64, C.c_int, C.c_uint64, C.c_int64, _d]
    L.orc_gen_sparse_signal.argtypes = [C.c_int64, C.c_int64, C.c_uint64, _d, _i64]
    L.orc_gen_circulant_sensing.argtypes = [C.c_int64, C.c_int64, C.c_uint64, _d, _i64]
    L.orc_measure.argtypes = [C.c_int64, C.c_int64, _d, _i64, _d, _d]
    L.orc_make_problem.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_uint64, _d, _i64, _d, _i64, _d]
    L.orc_gen_star_field.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_uint64, _d]
    L.orc_blur_row.argtypes = [C.c_int64, C.c_int64, _d]
    L.orc_dft.argtypes = [C.c_int64, _d, _d, _d]
    L.orc_idft.argtypes = [C.c_int64, _d, _d, _d, _d]
    L.orc_idft_real.argtypes = [C.c_int64, _d, _d, C.c_double, _d]
    L.orc_spectral_norm.argtypes = [C.c_int64, _d, _d]
    L.orc_regularized_gram_inverse.argtypes = [C.c_int64, _d, C.c_double, C.c_double, _d]
    L.orc_mask_gram_inverse.argtypes = [C.c_int64, C.c_int64, _i64, C.c_double, _d]
    L.orc_circ_compose.argtypes = [C.c_int64, _d, _d, _d]
    L.orc_circ_matvec.argtypes = [C.c_int64, _d, _d, C.c_int, C.c_int, _d]
    L.orc_soft_threshold.restype = C.c_double
    L.orc_soft_threshold.argtypes = [C.c_double, C.c_double]
    L.orc_ista_setup.restype = C.c_void_p
    L.orc_ista_setup.argtypes = [C.c_int64, C.c_int64, _d, _i64, _d, C.c_double, C.c_double, C.c_int,
                                 C.POINTER(C.c_int)]
    L.orc_ista_step.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int]
    L.orc_ista_get.argtypes = [C.c_void_p, C.c_int, _d]
    L.orc_ista_phase_sample.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int, _d]
    L.orc_cadmm_phase_sample.argtypes = [C.c_void_p, C.c_int64, C.c_int, _d]
    L.orc_ista_scalars.argtypes = [C.c_void_p, _d, _d, _d]
    L.orc_ista_free.argtypes = [C.c_void_p]
    L.orc_cadmm_setup.restype = C.c_void_p
    L.orc_cadmm_setup.argtypes = [C.c_int64, C.c_int64, _d, _i64, _d, C.c_double, C.c_double, C.c_double,
                                  C.c_double, C.c_double, C.POINTER(C.c_int)]
    L.orc_cadmm_step.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int]
    L.orc_cadmm_get.argtypes = [C.c_void_p, C.c_int, _d]
    L.orc_cadmm_scalars.argtypes = [C.c_void_p, _d, _d]
    L.orc_cadmm_free.argtypes = [C.c_void_p]
    L.orc_admm_setup.restype = C.c_void_p
    L.orc_admm_setup.argtypes = [C.c_int64, C.c_int64, _d, _i64, _d, C.c_double, C.c_double, C.c_int64, C.c_int,
                                 C.POINTER(C.c_int)]
    L.orc_admm_step.argtypes = [C.c_void_p, C.c_int64, C.c_int]
    L.orc_admm_get.argtypes = [C.c_void_p, C.c_int, _d]
    L.orc_admm_scalars.argtypes = [C.c_void_p, _d, _d]
    L.orc_admm_free.argtypes = [C.c_void_p]
    L.orc_run_loop.argtypes = [C.c_void_p, C.c_int, _d, C.c_int64, C.c_double, C.c_int64, C.c_int, C.c_int,
                               _i64, C.POINTER(C.c_int), _d, _i64, _d, C.c_int64, _i64]


def _check(rc: int):
    if rc != OK:
        raise OracleError(rc, lib().orc_last_error().decode())


def _pd(a):
    return a.ctypes.data_as(_d)


def _pi(a):
    return a.ctypes.data_as(_i64)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


# ---------------------------------------------------------------- generation
def mt19937_64(seed: int, count: int) -> np.ndarray:
    out = np.zeros(count, dtype=np.uint64)
    lib().orc_mt19937_64(seed, count, out.ctypes.data_as(_u64))
    return out


def rng_draws(seed: int, kind: str, count: int, bound: int = 0) -> np.ndarray:
    k = {"uniform": 0, "normal": 1, "below": 2}[kind]
    out = np.zeros(count)
    _check(lib().orc_rng_draws(seed, k, bound, count, _pd(out)))
    return out


def gen_sparse_signal(n: int, k: int, seed: int):
    v = np.zeros(max(n, 0))
    s = np.zeros(max(k, 0), dtype=np.int64)
    _check(lib().orc_gen_sparse_signal(n, k, seed, _pd(v), _pi(s)))
    return v, s


def gen_circulant_sensing(n: int, m: int, seed: int):
    row = np.zeros(n)
    om = np.zeros(max(m, 0), dtype=np.int64)
    _check(lib().orc_gen_circulant_sensing(n, m, seed, _pd(row), _pi(om)))
    return row, om


def measure(row, omega, x):
    row, omega, x = f64(row), i64(omega), f64(x)
    y = np.zeros(len(omega))
    _check(lib().orc_measure(len(row), len(omega), _pd(row), _pi(omega), _pd(x), _pd(y)))
    return y


@dataclass
class Problem:
    n: int
    m: int
    k: int
    seed: int
    row: np.ndarray
    omega: np.ndarray
    x_true: np.ndarray
    support: np.ndarray
    y: np.ndarray


def make_problem(n: int, m: int, k: int, seed: int) -> Problem:
    row = np.zeros(n)
    om = np.zeros(m, dtype=np.int64)
    xt = np.zeros(n)
    sup = np.zeros(k, dtype=np.int64)
    y = np.zeros(m)
    _check(lib().orc_make_problem(n, m, k, seed, _pd(row), _pi(om), _pd(xt), _pi(sup), _pd(y)))
    return Problem(n, m, k, seed, row, om, xt, sup, y)


def gen_star_field(width: int, height: int, density: float, seed: int) -> np.ndarray:
    px = np.zeros(width * height)
    _check(lib().orc_gen_star_field(width, height, density, seed, _pd(px)))
    return px


def blur_row(n: int, L: int) -> np.ndarray:
    row = np.zeros(n)
    _check(lib().orc_blur_row(n, L, _pd(row)))
    return row


# ---------------------------------------------------------------- operators
def dft(x):
    x = f64(x)
    re, im = np.zeros(len(x)), np.zeros(len(x))
    _check(lib().orc_dft(len(x), _pd(x), _pd(re), _pd(im)))
    return re + 1j * im


def idft_real(f, rel_tol=1e-10):
    re, im = f64(np.real(f)), f64(np.imag(f))
    out = np.zeros(len(re))
    _check(lib().orc_idft_real(len(re), _pd(re), _pd(im), rel_tol, _pd(out)))
    return out


def spectral_norm(c) -> float:
    c = f64(c)
    out = np.zeros(1)
    _check(lib().orc_spectral_norm(len(c), _pd(c), _pd(out)))
    return float(out[0])


def regularized_gram_inverse(c, rho, sigma):
    c = f64(c)
    b = np.zeros(len(c))
    _check(lib().orc_regularized_gram_inverse(len(c), _pd(c), rho, sigma, _pd(b)))
    return b


def mask_gram_inverse(omega, n, rho):
    omega = i64(omega)
    d = np.zeros(n)
    _check(lib().orc_mask_gram_inverse(n, len(omega), _pi(omega), rho, _pd(d)))
    return d


def circ_compose(c, b):
    c, b = f64(c), f64(b)
    out = np.zeros(len(c))
    _check(lib().orc_circ_compose(len(c), _pd(c), _pd(b), _pd(out)))
    return out


def circ_matvec(c, x, transpose=False, use_fft=False):
    c, x = f64(c), f64(x)
    y = np.zeros(len(c))
    _check(lib().orc_circ_matvec(len(c), _pd(c), _pd(x), int(transpose), int(use_fft), _pd(y)))
    return y


def soft_threshold(v, g):
    return np.array([lib().orc_soft_threshold(float(a), float(g)) for a in np.atleast_1d(v)])


# ---------------------------------------------------------------- solvers
class _Handle:
    _kind = -1

    def __del__(self):
        if getattr(self, "_h", None):
            self._free(self._h)
            self._h = None


class Ista(_Handle):
    """ista_setup + ista_step (reference solvers.hpp:222-263)."""

    _kind = 0

    def __init__(self, row, omega, y, alpha=1e-4, tau=0.0, proximal=False):
        row, omega, y = f64(row), i64(omega), f64(y)
        if len(y) != len(omega):
            raise OracleError(EDIM, "ista_setup: dimension mismatch")
        st = C.c_int(0)
        self._free = lib().orc_ista_free
        self._h = lib().orc_ista_setup(len(row), len(omega), _pd(row), _pi(omega), _pd(y), alpha, tau,
                                       int(proximal), C.byref(st))
        _check(st.value)
        self.n, self.m = len(row), len(omega)

    def step(self, iters=1, engine=ENGINE_PHASES, threads=None):
        _check(lib().orc_ista_step(self._h, iters, engine, threads or os.cpu_count() or 1))

    def phase_sample(self, rows, outs, threads=None):
        """Times the phase engine on rows [0, rows) / outputs [0, outs) -> (t_residual, t_gradient) s."""
        t = np.zeros(2)
        _check(lib().orc_ista_phase_sample(self._h, rows, outs, threads or os.cpu_count() or 1, _pd(t)))
        return float(t[0]), float(t[1])

    def get(self, name):
        which = {"x": 0, "r": 1, "delta": 2, "c": 3, "y": 4}[name]
        out = np.zeros(self.m if name in ("r", "y") else self.n)
        _check(lib().orc_ista_get(self._h, which, _pd(out)))
        return out

    def scalars(self):
        a, b, c = np.zeros(1), np.zeros(1), np.zeros(1)
        lib().orc_ista_scalars(self._h, _pd(a), _pd(b), _pd(c))
        return {"tau": a[0], "threshold": b[0], "s": c[0]}


class Cadmm(_Handle):
    """cadmm_setup + cadmm_step (reference solvers.hpp:359-415)."""

    _kind = 1
    FIELDS = ("x", "z", "nu", "mu", "v", "beta", "c", "b", "d", "pty")

    def __init__(self, row, omega, y, alpha=1e-4, rho=0.1, sigma=0.1, tau1=1.0, tau2=1.0):
        row, omega, y = f64(row), i64(omega), f64(y)
        if len(y) != len(omega):
            raise OracleError(EDIM, "cadmm_setup: dimension mismatch")
        st = C.c_int(0)
        self._free = lib().orc_cadmm_free
        self._h = lib().orc_cadmm_setup(len(row), len(omega), _pd(row), _pi(omega), _pd(y), alpha, rho, sigma,
                                        tau1, tau2, C.byref(st))
        _check(st.value)
        self.n, self.m = len(row), len(omega)

    def step(self, iters=1, engine=ENGINE_PHASES, threads=None):
        _check(lib().orc_cadmm_step(self._h, iters, engine, threads or os.cpu_count() or 1))

    def phase_sample(self, outs, threads=None):
        """Times the three phases on outputs [0, outs) -> (t_primal, t_recovery, t_duals) s."""
        t = np.zeros(3)
        _check(lib().orc_cadmm_phase_sample(self._h, outs, threads or os.cpu_count() or 1, _pd(t)))
        return float(t[0]), float(t[1]), float(t[2])

    def get(self, name):
        out = np.zeros(self.n)
        _check(lib().orc_cadmm_get(self._h, self.FIELDS.index(name), _pd(out)))
        return out

    def scalars(self):
        a, b = np.zeros(1), np.zeros(1)
        lib().orc_cadmm_scalars(self._h, _pd(a), _pd(b))
        return {"threshold": a[0], "s": b[0]}


class Admm(_Handle):
    """admm_setup + admm_step (reference solvers.hpp:267-327): the dense baseline with the explicit
    n x n inverse B = (A~^T A~ + rho I)^-1 (Cholesky), phases parallel.hpp:284-317."""

    _kind = 2
    FIELDS = ("x", "z", "u", "rhs", "aty", "B")
    DENSE_CAP = 4096  # circulant.hpp:31 kDenseCap

    def __init__(self, row, omega, y, alpha=1e-4, rho=0.1, dense_cap=DENSE_CAP, threads=None):
        row, omega, y = f64(row), i64(omega), f64(y)
        if len(y) != len(omega):
            raise OracleError(EDIM, "admm_setup: dimension mismatch")
        st = C.c_int(0)
        self._free = lib().orc_admm_free
        self._h = lib().orc_admm_setup(len(row), len(omega), _pd(row), _pi(omega), _pd(y), alpha, rho, dense_cap,
                                       threads or os.cpu_count() or 1, C.byref(st))
        _check(st.value)
        self.n, self.m = len(row), len(omega)

    def step(self, iters=1, engine=ENGINE_PHASES, threads=None):
        _check(lib().orc_admm_step(self._h, iters, threads or os.cpu_count() or 1))

    def get(self, name):
        out = np.zeros(self.n * self.n if name == "B" else self.n)
        _check(lib().orc_admm_get(self._h, self.FIELDS.index(name), _pd(out)))
        return out.reshape(self.n, self.n) if name == "B" else out

    def scalars(self):
        a, b = np.zeros(1), np.zeros(1)
        lib().orc_admm_scalars(self._h, _pd(a), _pd(b))
        return {"threshold": a[0], "s": b[0]}


@dataclass
class Report:
    final_x: np.ndarray
    iterations: int
    reached_target: bool
    final_metric: float
    trace: list = field(default_factory=list)


def run(kind: str, row, omega, y, truth=None, engine=ENGINE_PHASES, threads=None, max_iter=100000,
        target_mse=float("nan"), check_every=10, **params) -> Report:
    """ista_run / cadmm_run (reference solvers.hpp:479-534) incl. run_loop :426-472."""
    h = {"ista": Ista, "cadmm": Cadmm, "admm": Admm}[kind](row, omega, y, **params)
    cap = max_iter // max(check_every, 1) + 2
    tit = np.zeros(cap, dtype=np.int64)
    tval = np.zeros(cap)
    it, tl = C.c_int64(0), C.c_int64(0)
    reached = C.c_int(0)
    fm = np.zeros(1)
    tr = f64(truth) if truth is not None else None
    _check(lib().orc_run_loop(h._h, h._kind, _pd(tr) if tr is not None else None, max_iter, target_mse,
                              check_every, engine, threads or os.cpu_count() or 1, C.byref(it), C.byref(reached),
                              _pd(fm), _pi(tit), _pd(tval), cap, C.byref(tl)))
    fx = h.get("x" if kind == "ista" else "z")
    n_tr = min(tl.value, cap)
    return Report(fx, it.value, bool(reached.value), float(fm[0]),
                  [(int(tit[i]), float(tval[i])) for i in range(n_tr)])
