"""Python mirror of the reference circlasso solver API over the C-ABI.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/circlasso/): ``ista_run``/``cadmm_run``
(solvers.hpp:479-534), ``ista_setup``/``ista_step`` and the cADMM pair
(:222-263, :359-415), ``SolverConfig`` (:112-125), ``RecoveryReport``
(:139-150), ``make_problem`` & co. (sensing.hpp), the operator types and
setup transforms (circulant.hpp), and the typed exceptions (errors.hpp).
Every solver call runs the sm_100a kernels of libcirclasso_b200.so; there is
no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from ._native import cl_config, cl_report, lib

# --------------------------------------------------------------------------- errors


class Error(RuntimeError):
    """errors.hpp:13-16"""


class DimensionError(Error):
    pass


class ParameterError(Error):
    pass


class SingularityError(Error):
    pass


class DivergenceError(Error):
    pass


class CapacityError(Error):
    pass


class FormatError(Error):
    pass


class ConsistencyError(Error):
    pass


class PhaseError(Error):
    def __init__(self, what: str, global_id: int = -1):
        super().__init__(what)
        self.global_id = global_id


class CudaError(Error):
    """Device/runtime failure (no reference counterpart: the reference has no device)."""


class CommError(Error):
    """Collective failure in a sharded solve."""


_ERRORS = {1: DimensionError, 2: ParameterError, 3: SingularityError, 4: DivergenceError, 5: CapacityError,
           6: FormatError, 7: ConsistencyError, 8: PhaseError, 9: CudaError, 10: CommError}


def _check(rc: int):
    if rc != 0:
        msg = lib.cl_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, Error)(msg)


_d = C.POINTER(C.c_double)
_i64 = C.POINTER(C.c_int64)


def _f64(a, name="array"):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a


def _pd(a):
    return a.ctypes.data_as(_d) if a is not None else None


def _pi(a):
    return a.ctypes.data_as(_i64)


def _idx(a):
    return np.ascontiguousarray(a, dtype=np.int64)


# --------------------------------------------------------------------------- config / report


class ThresholdPairing(enum.IntEnum):
    """solvers.hpp:83"""
    kLiteral = 0
    kProximal = 1


class StopMetric(enum.IntEnum):
    """solvers.hpp:130"""
    kMseVsTruth = 0
    kIterateChange = 1


@dataclass
class SolverConfig:
    """solvers.hpp:112-125.

    ``use_fft`` selects the product engine.  The reference defaults to its
    FFT engine; here the default is the direct shift-indexed sm_100a kernels
    (the paper's scheme and the north-star path, the reference's
    ``use_fft=false`` arithmetic); ``use_fft=True`` runs the on-device FFT
    engine (any n: non-power-of-two n is embedded as a linear convolution in the
    next power of two >= 2n-1).  ``dense_cap`` bounds the dense ADMM baseline
    (admm_setup / admm_dense_run: CapacityError above it)."""
    alpha: float = 1e-4
    tau: float = 0.0
    rho: float = 0.1
    sigma: float = 0.1
    tau1: float = 1.0
    tau2: float = 1.0
    max_iter: int = 100000
    target_mse: float = float("nan")
    check_every: int = 10
    pairing: ThresholdPairing = ThresholdPairing.kLiteral
    use_fft: bool = False
    dense_cap: int = 4096

    def _c(self) -> cl_config:
        c = cl_config()
        lib.cl_config_default(C.byref(c))
        c.alpha, c.tau, c.rho, c.sigma = self.alpha, self.tau, self.rho, self.sigma
        c.tau1, c.tau2 = self.tau1, self.tau2
        c.max_iter, c.target_mse = int(self.max_iter), float(self.target_mse)
        c.check_every, c.pairing = int(self.check_every), int(self.pairing)
        c.engine = 1 if self.use_fft else 0
        c.dense_cap = int(self.dense_cap)
        return c


@dataclass
class TracePoint:
    iteration: int
    value: float
    elapsed_seconds: float = float("nan")


@dataclass
class RecoveryReport:
    """solvers.hpp:139-150"""
    final_x: np.ndarray
    iterations: int = 0
    mse_trace: List[TracePoint] = field(default_factory=list)
    setup_seconds: float = 0.0
    total_seconds: float = 0.0
    footprint_bytes: int = 0
    metric: StopMetric = StopMetric.kIterateChange
    reached_target: bool = False
    final_metric: float = float("nan")


class FootprintKind(enum.IntEnum):
    kCpista = 0
    kCpadmm = 1
    kDenseIsta = 2
    kDenseAdmm = 3


def analytic_footprint(kind: FootprintKind, n: int, m: int, scalar_width: int) -> int:
    """solvers.hpp:90-106"""
    if kind == FootprintKind.kCpista:
        return 4 * n * scalar_width
    if kind == FootprintKind.kCpadmm:
        return 10 * n * scalar_width
    if kind == FootprintKind.kDenseIsta:
        return (2 * m * n + 2 * n + 2 * m) * scalar_width
    if kind == FootprintKind.kDenseAdmm:
        return (n * n + 4 * n + m) * scalar_width
    raise ParameterError("analytic_footprint: unknown solver kind")


# --------------------------------------------------------------------------- operators


class CirculantMatrix:
    """circulant.hpp:36-105 (first row only; A(i,j) = first_row[(j-i) mod n])."""

    def __init__(self, first_row):
        self._row = _f64(first_row)

    @staticmethod
    def Identity(n: int) -> "CirculantMatrix":
        r = np.zeros(n)
        if n > 0:
            r[0] = 1.0
        return CirculantMatrix(r)

    def first_row(self) -> np.ndarray:
        return self._row

    def n(self) -> int:
        return len(self._row)

    def stored_scalars(self) -> int:
        return self.n()


class SubsamplingMask:
    """circulant.hpp:130-184"""

    def __init__(self, omega, n: int):
        self._omega = _idx(omega)
        self._n = int(n)
        if n < 0:
            raise ParameterError("SubsamplingMask: negative dimension")
        if len(self._omega) and (np.any(np.diff(self._omega) <= 0) or self._omega[0] < 0 or self._omega[-1] >= n):
            raise ParameterError("SubsamplingMask: indices must be strictly increasing and within [0, n)")

    @staticmethod
    def Full(n: int) -> "SubsamplingMask":
        return SubsamplingMask(np.arange(n), n)

    def m(self) -> int:
        return len(self._omega)

    def n(self) -> int:
        return self._n

    def omega(self) -> np.ndarray:
        return self._omega

    def apply(self, x):
        x = _f64(x)
        if len(x) != self._n:
            raise DimensionError(f"SubsamplingMask::apply: dimension mismatch, {len(x)} vs {self._n}")
        return x[self._omega]

    def embed(self, y):
        y = _f64(y)
        if len(y) != self.m():
            raise DimensionError(f"SubsamplingMask::embed: dimension mismatch, {len(y)} vs {self.m()}")
        out = np.zeros(self._n)
        out[self._omega] = y
        return out


class PartialCirculantOperator:
    """circulant.hpp:188-212 (A = P C)."""

    def __init__(self, circulant: CirculantMatrix, mask: SubsamplingMask):
        if circulant.n() != mask.n():
            raise DimensionError(
                f"PartialCirculantOperator: dimension mismatch, {circulant.n()} vs {mask.n()}")
        self._c, self._mask = circulant, mask

    def n(self) -> int:
        return self._c.n()

    def m(self) -> int:
        return self._mask.m()

    def circulant(self) -> CirculantMatrix:
        return self._c

    def mask(self) -> SubsamplingMask:
        return self._mask


class DiagonalOperator:
    def __init__(self, diag):
        self._d = _f64(diag)

    def diag(self):
        return self._d

    def apply(self, x):
        x = _f64(x)
        if len(x) != len(self._d):
            raise DimensionError("DiagonalOperator::apply: dimension mismatch")
        return self._d * x


# --------------------------------------------------------------------------- generation


@dataclass
class SparseSignal:
    values: np.ndarray
    support: np.ndarray

    def n(self):
        return len(self.values)

    def k(self):
        return len(self.support)


@dataclass
class SensingProblem:
    signal: SparseSignal
    op: PartialCirculantOperator
    measurements: np.ndarray
    seed: int = 0

    def n(self):
        return self.op.n()

    def m(self):
        return self.op.m()

    def k(self):
        return self.signal.k()


def gen_sparse_signal(n: int, k: int, seed: int) -> SparseSignal:
    """sensing.hpp:129-145"""
    v = np.zeros(max(n, 0))
    s = np.zeros(max(k, 0), dtype=np.int64)
    _check(lib.cl_gen_sparse_signal(n, k, seed, _pd(v), _pi(s)))
    return SparseSignal(v, s)


def gen_circulant_sensing(n: int, m: int, seed: int) -> PartialCirculantOperator:
    """sensing.hpp:149-168"""
    row = np.zeros(max(n, 0))
    om = np.zeros(max(m, 0), dtype=np.int64)
    _check(lib.cl_gen_circulant_sensing(n, m, seed, _pd(row), _pi(om)))
    return PartialCirculantOperator(CirculantMatrix(row), SubsamplingMask(om, n))


def measure(A: PartialCirculantOperator, x) -> np.ndarray:
    """sensing.hpp:171-182 (fp64, DFT-evaluated like the reference)."""
    if isinstance(x, SparseSignal):
        x = x.values
    x = _f64(x)
    if len(x) != A.n():
        raise DimensionError(f"measure: dimension mismatch, {len(x)} vs {A.n()}")
    y = np.zeros(A.m())
    _check(lib.cl_measure(A.n(), A.m(), _pd(A.circulant().first_row()), _pi(A.mask().omega()), _pd(x), _pd(y)))
    return y


def make_problem(n: int, m: int, k: int, seed: int) -> SensingProblem:
    """sensing.hpp:198-207"""
    row = np.zeros(n)
    om = np.zeros(m, dtype=np.int64)
    xt = np.zeros(n)
    sup = np.zeros(k, dtype=np.int64)
    y = np.zeros(m)
    _check(lib.cl_make_problem(n, m, k, seed, _pd(row), _pi(om), _pd(xt), _pi(sup), _pd(y)))
    op = PartialCirculantOperator(CirculantMatrix(row), SubsamplingMask(om, n))
    return SensingProblem(SparseSignal(xt, sup), op, y, seed)


@dataclass
class GrayImage:
    """image.hpp:24-38 (row-major pixels in [0, 1])."""
    width: int
    height: int
    pixels: np.ndarray

    def size(self) -> int:
        return self.width * self.height

    def at(self, row: int, col: int) -> float:
        return float(self.pixels[row * self.width + col])


def make_image(width: int, height: int, values) -> GrayImage:
    """image.hpp:41-54: clamp into [0, 1]."""
    if width < 1 or height < 1:
        raise ParameterError("make_image: dimensions must be positive")
    values = _f64(values)
    if len(values) != width * height:
        raise DimensionError(f"make_image: dimension mismatch, {len(values)} vs {width * height}")
    return GrayImage(width, height, np.clip(values, 0.0, 1.0))


def write_pgm(img: GrayImage, path: str):
    """image.hpp:137-153: binary P5, maxval 255, intensities clamped to [0, 1] and rounded."""
    if img.width < 1 or img.height < 1:
        raise ParameterError("write_pgm: empty image")
    px = _f64(img.pixels)
    if len(px) != img.size():
        raise DimensionError(f"write_pgm: dimension mismatch, {len(px)} vs {img.size()}")
    _check(lib.cl_write_pgm(str(path).encode(), img.width, img.height, _pd(px)))


def read_pgm(path: str) -> GrayImage:
    """image.hpp:95-135: binary P5 with maxval 1..255 -> intensities in [0, 1]."""
    w, h = C.c_int64(), C.c_int64()
    _check(lib.cl_read_pgm(str(path).encode(), None, 0, C.byref(w), C.byref(h)))
    px = np.zeros(w.value * h.value)
    _check(lib.cl_read_pgm(str(path).encode(), _pd(px), len(px), C.byref(w), C.byref(h)))
    return GrayImage(w.value, h.value, px)


def gen_star_field(width: int, height: int, density: float, seed: int) -> GrayImage:
    """deblur.hpp:69-86: floor(density n) stars at uniform positions, intensities U[0.3, 1)."""
    px = np.zeros(max(width * height, 0))
    _check(lib.cl_gen_star_field(width, height, density, seed, _pd(px)))
    return GrayImage(width, height, px)


def blur_matrix(n: int, L: int) -> CirculantMatrix:
    """deblur.hpp:26-36"""
    row = np.zeros(max(n, 0))
    _check(lib.cl_blur_row(n, L, _pd(row)))
    return CirculantMatrix(row)


def compose_sensing(C_: CirculantMatrix, B: CirculantMatrix, mask: SubsamplingMask) -> PartialCirculantOperator:
    """deblur.hpp:53-64"""
    if C_.n() != B.n():
        raise DimensionError(f"compose_sensing: dimension mismatch, {C_.n()} vs {B.n()}")
    if mask.n() != C_.n():
        raise DimensionError(f"compose_sensing: dimension mismatch, {mask.n()} vs {C_.n()}")
    out = np.zeros(C_.n())
    _check(lib.cl_compose_rows(C_.n(), _pd(C_.first_row()), _pd(B.first_row()), _pd(out)))
    return PartialCirculantOperator(CirculantMatrix(out), mask)


# --------------------------------------------------------------------------- setup transforms


def spectral_norm(C_: CirculantMatrix) -> float:
    """circulant.hpp:347-351"""
    out = np.zeros(1)
    _check(lib.cl_spectral_norm(C_.n(), _pd(C_.first_row()), _pd(out)))
    return float(out[0])


def regularized_gram_inverse(C_: CirculantMatrix, rho: float, sigma: float) -> CirculantMatrix:
    """circulant.hpp:297-320"""
    b = np.zeros(C_.n())
    _check(lib.cl_regularized_gram_inverse(C_.n(), _pd(C_.first_row()), rho, sigma, _pd(b)))
    return CirculantMatrix(b)


def mask_gram_inverse(P: SubsamplingMask, rho: float) -> DiagonalOperator:
    """circulant.hpp:324-333"""
    d = np.zeros(P.n())
    _check(lib.cl_mask_gram_inverse(P.n(), P.m(), _pi(P.omega()), rho, _pd(d)))
    return DiagonalOperator(d)


def soft_threshold(x, gamma: float) -> np.ndarray:
    """solvers.hpp:47-53 (host helper; strict inequality, NaN -> 0)."""
    if gamma < 0:
        raise ParameterError("soft_threshold: gamma must be nonnegative")
    x = _f64(x)
    out = np.zeros_like(x)
    out[x > gamma] = x[x > gamma] - gamma
    out[x < -gamma] = x[x < -gamma] + gamma
    return out


def mse(a, b) -> float:
    """solvers.hpp:56-61"""
    a, b = _f64(a), _f64(b)
    if len(a) != len(b):
        raise DimensionError(f"mse: dimension mismatch, {len(a)} vs {len(b)}")
    return float(np.sum((a - b) ** 2) / len(a)) if len(a) else 0.0


# --------------------------------------------------------------------------- device products


def circ_matvec(M: CirculantMatrix, x, device: int = 0) -> np.ndarray:
    """C x on the GPU (circulant.hpp:216-244; fp32 direct kernel)."""
    x = _f64(x)
    if len(x) != M.n():
        raise DimensionError(f"circ_matvec: dimension mismatch, {len(x)} vs {M.n()}")
    out = np.zeros(M.n())
    _check(lib.cl_circ_matvec(device, M.n(), _pd(M.first_row()), _pd(x), 0, _pd(out)))
    return out


def circ_transpose_matvec(M: CirculantMatrix, x, device: int = 0) -> np.ndarray:
    """C^T x on the GPU (circulant.hpp:248-274)."""
    x = _f64(x)
    if len(x) != M.n():
        raise DimensionError(f"circ_transpose_matvec: dimension mismatch, {len(x)} vs {M.n()}")
    out = np.zeros(M.n())
    _check(lib.cl_circ_matvec(device, M.n(), _pd(M.first_row()), _pd(x), 1, _pd(out)))
    return out


def partial_matvec(A: PartialCirculantOperator, x, device: int = 0) -> np.ndarray:
    """A x = P C x on the GPU, rows generated on the fly (circulant.hpp:277-282)."""
    x = _f64(x)
    if len(x) != A.n():
        raise DimensionError(f"partial_matvec: dimension mismatch, {len(x)} vs {A.n()}")
    out = np.zeros(A.m())
    _check(lib.cl_partial_matvec(device, A.n(), A.m(), _pd(A.circulant().first_row()), _pi(A.mask().omega()),
                                 _pd(x), _pd(out)))
    return out


def partial_transpose_matvec(A: PartialCirculantOperator, y, device: int = 0) -> np.ndarray:
    """A^T y = C^T P^T y on the GPU (circulant.hpp:286-291)."""
    y = _f64(y)
    if len(y) != A.m():
        raise DimensionError(f"partial_transpose_matvec: dimension mismatch, {len(y)} vs {A.m()}")
    out = np.zeros(A.n())
    _check(lib.cl_partial_transpose_matvec(device, A.n(), A.m(), _pd(A.circulant().first_row()),
                                           _pi(A.mask().omega()), _pd(y), _pd(out)))
    return out


# --------------------------------------------------------------------------- solver states


class _DeviceState:
    """Owns a cl_solver handle (IstaState / CadmmState analogue, on device)."""

    KIND = -1
    FIELDS: tuple = ()

    def __init__(self, A: PartialCirculantOperator, y, cfg: SolverConfig, device: int = 0):
        y = _f64(y)
        if len(y) != A.m():
            raise DimensionError(f"{self._name}: dimension mismatch, {len(y)} vs {A.m()}")
        self.cfg = cfg
        self._n, self._m = A.n(), A.m()
        h = C.c_void_p()
        c = cfg._c()
        _check(lib.cl_solver_create(self.KIND, A.n(), A.m(), _pd(A.circulant().first_row()), _pi(A.mask().omega()),
                                    _pd(y), C.byref(c), device, C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.cl_solver_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def step(self, iters: int = 1):
        _check(lib.cl_solver_step(self._h, int(iters)))

    def step_checked(self):
        v = C.c_double(0)
        nf = C.c_int(0)
        _check(lib.cl_solver_step_checked(self._h, C.byref(v), C.byref(nf)))
        return v.value, bool(nf.value)

    def synchronize(self):
        _check(lib.cl_solver_synchronize(self._h))

    def get(self, name: str) -> np.ndarray:
        size = self._m if name in ("r", "y") else self._n
        out = np.zeros(size)
        _check(lib.cl_solver_get(self._h, name.encode(), _pd(out)))
        return out

    def set(self, name: str, values):
        values = _f64(values)
        size = self._m if name in ("r", "y") else self._n
        if len(values) != size:  # the C side reads exactly `size` doubles
            raise DimensionError(f"set('{name}'): expected {size} values, got {len(values)}")
        _check(lib.cl_solver_set(self._h, name.encode(), _pd(values)))

    def set_truth(self, truth):
        t = _f64(truth) if truth is not None else None
        if t is not None and len(t) != self._n:
            raise DimensionError("truth: dimension mismatch")
        _check(lib.cl_solver_set_truth(self._h, _pd(t)))

    def info(self):
        n, m, t = C.c_int64(), C.c_int64(), C.c_int64()
        s, thr = C.c_double(), C.c_double()
        _check(lib.cl_solver_info(self._h, C.byref(n), C.byref(m), C.byref(t), C.byref(s), C.byref(thr)))
        return {"n": n.value, "m": m.value, "t": t.value, "scale": s.value, "threshold": thr.value}

    @property
    def t(self) -> int:
        return self.info()["t"]

    def last_step_ms(self) -> float:
        v = C.c_double()
        _check(lib.cl_solver_last_step_ms(self._h, C.byref(v)))
        return v.value

    def profile(self, enable=True):
        """Per-phase CUDA events: False/0 off, True/1 eager launches, 2 = event nodes inside the captured
        step graph (times the graph-replayed step itself)."""
        _check(lib.cl_solver_profile(self._h, int(enable)))

    def phase_history(self, max_steps=256):
        """profile(2): per-phase times (ms) of each of the last graph replays, oldest first (list of lists)."""
        steps, nph = C.c_int64(0), C.c_int(0)
        _check(lib.cl_solver_phase_history(self._h, None, 0, C.byref(steps), C.byref(nph)))
        k = min(int(steps.value), max_steps)
        arr = (C.c_double * max(1, k * max(nph.value, 1)))()
        _check(lib.cl_solver_phase_history(self._h, arr, k, C.byref(steps), C.byref(nph)))
        return [[arr[i * nph.value + j] for j in range(nph.value)] for i in range(int(steps.value))]

    def phase_ms(self):
        arr = (C.c_double * 8)()
        cnt = C.c_int(8)
        _check(lib.cl_solver_phase_ms(self._h, arr, C.byref(cnt)))
        return [arr[i] for i in range(cnt.value)]

    def __getattr__(self, name):
        if name in type(self).FIELDS:
            return self.get(name)
        raise AttributeError(name)


class IstaState(_DeviceState):
    """solvers.hpp:208-220 + ista_setup :222-249 (state resident on the GPU)."""
    KIND = 0
    FIELDS = ("x", "r", "delta", "c", "y")
    _name = "ista_setup"


class CadmmState(_DeviceState):
    """solvers.hpp:337-357 + cadmm_setup :359-395 (state resident on the GPU)."""
    KIND = 1
    FIELDS = ("x", "z", "nu", "mu", "v", "beta", "c", "b", "d", "pty")
    _name = "cadmm_setup"


class AdmmState(_DeviceState):
    """solvers.hpp:267-283 + admm_setup :285-314: the dense baseline; B = (A~^T A~ + rho I)^-1 is built in
    fp64 on the GPU (Gram matrix + blocked Gauss-Jordan) and iterated in fp32."""
    KIND = 2
    FIELDS = ("x", "z", "u", "rhs", "aty", "B")
    _name = "admm_setup"

    def get(self, name: str) -> np.ndarray:
        if name != "B":
            return super().get(name)
        out = np.zeros(self._n * self._n)
        _check(lib.cl_solver_get(self._h, b"B", _pd(out)))
        return out.reshape(self._n, self._n)


def ista_setup(A: PartialCirculantOperator, y, cfg: SolverConfig = None, device: int = 0) -> IstaState:
    return IstaState(A, y, cfg or SolverConfig(), device)


def ista_step(state: IstaState, use_fft: bool = True):
    state.step(1)


def cadmm_setup(A: PartialCirculantOperator, y, cfg: SolverConfig = None, device: int = 0) -> CadmmState:
    return CadmmState(A, y, cfg or SolverConfig(), device)


def cadmm_step(state: CadmmState, use_fft: bool = True):
    state.step(1)


def admm_setup(A: PartialCirculantOperator, y, cfg: SolverConfig = None, device: int = 0) -> AdmmState:
    """solvers.hpp:285-314 (DimensionError, then CapacityError for n > cfg.dense_cap, before anything is built)."""
    return AdmmState(A, y, cfg or SolverConfig(), device)


def admm_step(state: AdmmState):
    """solvers.hpp:318-327"""
    state.step(1)


def _report(call, n: int, cfg: SolverConfig) -> RecoveryReport:
    rep = cl_report()
    cap = (int(cfg.max_iter) // max(int(cfg.check_every), 1)) + 2 if cfg.max_iter >= 0 else 0
    cap = min(cap, 1 << 22)
    tit = np.zeros(max(cap, 1), dtype=np.int64)
    tval = np.zeros(max(cap, 1))
    tsec = np.zeros(max(cap, 1))
    fx = np.zeros(n)
    _check(call(C.byref(rep), _pd(fx), _pi(tit), _pd(tval), _pd(tsec), cap))
    trace = [TracePoint(int(tit[i]), float(tval[i]), float(tsec[i])) for i in range(min(rep.trace_len, cap))]
    return RecoveryReport(final_x=fx, iterations=rep.iterations, mse_trace=trace, setup_seconds=rep.setup_seconds,
                          total_seconds=rep.total_seconds, footprint_bytes=rep.footprint_bytes,
                          metric=StopMetric(rep.metric), reached_target=bool(rep.reached_target),
                          final_metric=rep.final_metric)


def _run(state: _DeviceState, truth, cfg: SolverConfig) -> RecoveryReport:
    if truth is not None:
        state.set_truth(truth)
    return _report(lambda *a: lib.cl_solver_run(state.handle, *a), state._n, cfg)


def ista_run(y, A: PartialCirculantOperator, cfg: SolverConfig = None, truth=None, device: int = 0,
             comm=None) -> RecoveryReport:
    """solvers.hpp:479-495.  ``comm`` (dist.NativeComm): this process's rank of a sharded solve; every rank
    makes the same call and gets the same report."""
    cfg = cfg or SolverConfig()
    st = ista_setup(A, y, cfg, device)
    if comm is not None:
        comm.attach(st)
    return _run(st, truth, cfg)


def cadmm_run(y, A: PartialCirculantOperator, cfg: SolverConfig = None, truth=None, device: int = 0,
              comm=None) -> RecoveryReport:
    """solvers.hpp:518-534 (``comm`` as for ista_run)"""
    cfg = cfg or SolverConfig()
    st = cadmm_setup(A, y, cfg, device)
    if comm is not None:
        comm.attach(st)
    return _run(st, truth, cfg)


def admm_dense_run(y, A: PartialCirculantOperator, cfg: SolverConfig = None, truth=None,
                   device: int = 0) -> RecoveryReport:
    """solvers.hpp:497-514: dense ADMM; the O(n^3) inversion is timed into setup_seconds."""
    cfg = cfg or SolverConfig()
    st = admm_setup(A, y, cfg, device)
    return _run(st, truth, cfg)


class ShardedSolve:
    """A sharded ISTA / cADMM solve driven from one process (cl_group_*): rank r on devices[r],
    the slice exchange after every phase inside the library -- NCCL (``transport="nccl"``: ncclCommInitAll,
    one grouped set of in-place broadcasts per phase), peer copies (``"copy"``: devices may repeat, e.g.
    [0, 0, 0, 0] runs the 4-rank data plane on one GPU), or peer stores fused into the kernels that produce
    each slice (``"peer"``: no separate exchange; NVLink stores across GPUs, at most 8 ranks).  Same iterate
    as the unsharded solve, bitwise."""

    TRANSPORTS = {"nccl": 0, "copy": 1, "peer": 2}

    def __init__(self, kind: str, A: PartialCirculantOperator, y, cfg: SolverConfig = None, devices=(0,),
                 transport: str = "nccl"):
        cfg = cfg or SolverConfig()
        y = _f64(y)
        if len(y) != A.m():
            raise DimensionError(f"{kind}_setup: dimension mismatch, {len(y)} vs {A.m()}")
        self.kind = {"ista": 0, "cadmm": 1}[kind]
        self.cfg = cfg
        self._n, self._m = A.n(), A.m()
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        c = cfg._c()
        _check(lib.cl_group_create(self.kind, A.n(), A.m(), _pd(A.circulant().first_row()), _pi(A.mask().omega()),
                                   _pd(y), C.byref(c), devs, len(devices), self.TRANSPORTS[transport],
                                   C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.cl_group_destroy(h)
            self._h = None

    def step(self, iters: int = 1):
        _check(lib.cl_group_step(self._h, int(iters)))

    def synchronize(self):
        _check(lib.cl_group_synchronize(self._h))

    def get(self, name: str) -> np.ndarray:
        out = np.zeros(self._m if name in ("r", "y") else self._n)
        _check(lib.cl_group_get(self._h, name.encode(), _pd(out)))
        return out

    def info(self):
        w, t, tr = C.c_int(), C.c_int64(), C.c_int()
        _check(lib.cl_group_info(self._h, C.byref(w), C.byref(t), C.byref(tr)))
        return {"world": w.value, "t": t.value, "transport": tr.value}

    def run(self, truth=None) -> RecoveryReport:
        if truth is not None:
            t = _f64(truth)
            if len(t) != self._n:
                raise DimensionError("truth: dimension mismatch")
            _check(lib.cl_group_set_truth(self._h, _pd(t)))
        return _report(lambda *a: lib.cl_group_run(self._h, *a), self._n, self.cfg)


def device_count() -> int:
    c = C.c_int(0)
    rc = lib.cl_device_count(C.byref(c))
    return c.value if rc == 0 else 0


def ffma_peak_tflops(device: int = 0) -> float:
    v = C.c_double()
    _check(lib.cl_ffma_peak(device, C.byref(v)))
    return v.value


# --------------------------------------------------------------------------- deblurring (deblur.hpp)


@dataclass
class DeblurResult:
    """deblur.hpp:93-101"""
    recovered: GrayImage
    report: RecoveryReport
    error_map: Optional[np.ndarray] = None
    mse_vs_truth: float = float("nan")
    error_map_mean: float = float("nan")
    normalized_mse: float = float("nan")


def deblur_recover(y, C_: CirculantMatrix, B: CirculantMatrix, mask: SubsamplingMask, width: int, height: int,
                   cfg: SolverConfig = None, truth: Optional[GrayImage] = None, device: int = 0) -> DeblurResult:
    """deblur.hpp:107-136: cadmm_run on A = P C B (iterate-change stopping; truth only for statistics)."""
    cfg = cfg or SolverConfig()
    if width < 1 or height < 1:
        raise ParameterError("deblur_recover: dimensions must be positive")
    A = compose_sensing(C_, B, mask)
    if A.n() != width * height:
        raise DimensionError(f"deblur_recover: dimension mismatch, {A.n()} vs {width * height}")
    y = _f64(y)
    if len(y) != A.m():
        raise DimensionError(f"deblur_recover: dimension mismatch, {len(y)} vs {A.m()}")
    if truth is not None and len(truth.pixels) != A.n():
        raise DimensionError("deblur_recover: truth dimension mismatch")
    rep = cadmm_run(y, A, cfg, None, device)
    res = DeblurResult(recovered=make_image(width, height, rep.final_x), report=rep)
    if truth is not None:
        res.mse_vs_truth = mse(rep.final_x, truth.pixels)
        mean = float(np.mean(truth.pixels))
        scale = mean if mean > 0 else 1.0
        res.error_map = np.abs(rep.final_x - truth.pixels) / scale
        res.error_map_mean = float(np.mean(res.error_map))
        res.normalized_mse = res.mse_vs_truth / (scale * scale)
    return res


def run_deblur_experiment(image: GrayImage, L: int, m: int, cfg: SolverConfig = None, seed: int = 1,
                          device: int = 0) -> DeblurResult:
    """deblur.hpp:141-156: blur (order L), sense (seeded circulant, m of n rows), recover with cADMM."""
    n = image.size()
    if len(image.pixels) != n:
        raise DimensionError("run_deblur_experiment: dimension mismatch")
    B = blur_matrix(n, L)
    sensing = gen_circulant_sensing(n, m, seed)
    A = compose_sensing(sensing.circulant(), B, sensing.mask())
    y = measure(A, image.pixels)
    return deblur_recover(y, sensing.circulant(), B, sensing.mask(), image.width, image.height, cfg, image, device)
