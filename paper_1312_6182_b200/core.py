"""Domain types of the GP-SPCA engine, mirroring reference core.py.

Conventions are the reference's (core.py:1-7): A is p x n with the n
columns as variables; sphere iterates x live in R^p, loadings z in R^n.
The one structural difference is `DataMatrix`: its storage is a
device-resident, column-major, zero-padded copy managed by
libgpspca_b200 (fp32 inputs stay fp32 on the device; every reduction is
fp64), and its column norms / finiteness flag come from one device pass.
"""

from dataclasses import dataclass, field

import numpy as np

from . import _native

PENALTIES = ("l1", "l0")
MODES = ("single_unit", "block")
INITS = ("max_norm_column", "random_orthonormal", "user_supplied")
DEFLATIONS = ("orthogonal_projection",)

ALGEBRAIC_TOL = 1e-12  # core.py:21
STIEFEL_TOL = 1e-10    # core.py:22


def _storage_dtype(arr, dtype):
    if dtype is not None:
        dt = np.dtype(dtype)
        if dt not in (np.float32, np.float64):
            raise ValueError("storage dtype must be float32 or float64")
        return dt
    return np.dtype(np.float32) if arr.dtype == np.float32 else np.dtype(np.float64)


class DataMatrix:
    """Dense p x n matrix, device-resident (reference core.py:25-61).

    `DataMatrix(values)` copies the input to the GPU once; the object is
    immutable, so the cached column norms (core.py:243) stay valid.  Storage
    dtype follows the input (float32 stays float32, anything else becomes
    float64) unless `dtype=` overrides it.  `.values` downloads a float64
    column-major host copy on first access.
    """

    __slots__ = ("_handle", "_ctx", "p", "n", "dtype", "_values", "_norms", "_nonfinite", "_owner", "__weakref__")

    def __init__(self, values, dtype=None, device=None):
        if isinstance(values, DataMatrix):
            values = values.values
        arr = np.asarray(values)
        if arr.ndim != 2:
            raise ValueError(f"expected a 2-d matrix, got ndim={arr.ndim}")
        p, n = arr.shape
        if p < 1 or n < 1:
            raise ValueError(f"matrix must be at least 1x1, got {p}x{n}")
        dt = _storage_dtype(arr, dtype)
        code = _native.F32 if dt == np.float32 else _native.F64
        ctx = _native.context(device)
        object.__setattr__(self, "_ctx", ctx)
        object.__setattr__(self, "_handle", None)
        object.__setattr__(self, "_owner", None)
        object.__setattr__(self, "_values", None)
        object.__setattr__(self, "_norms", None)
        object.__setattr__(self, "p", int(p))
        object.__setattr__(self, "n", int(n))
        object.__setattr__(self, "dtype", dt)
        h = _native.C.c_void_p()
        if arr.dtype == dt and arr.flags.f_contiguous:
            rc = _native.lib().gps_matrix_create(ctx.handle, arr.ctypes.data, p, n, p, code, _native.C.byref(h))
        else:
            src = np.ascontiguousarray(arr, dtype=dt)
            rc = _native.lib().gps_matrix_create_rowmajor(ctx.handle, src.ctypes.data, p, n, code,
                                                          _native.C.byref(h))
        _native.check(rc, "DataMatrix upload")
        object.__setattr__(self, "_handle", h)
        norms, bad = self._column_pass()
        if bad:
            raise ValueError("matrix entries must be finite")
        object.__setattr__(self, "_norms", norms)
        object.__setattr__(self, "_nonfinite", False)

    @classmethod
    def from_device(cls, ptr, p, n, ld=None, dtype=np.float32, device=None, owner=None):
        """A device-resident column-major p x n buffer (e.g. a torch CUDA
        tensor's data_ptr).  With `owner` given and ld == roundup(p, 32) the
        buffer is adopted WITHOUT a copy (owner is kept alive); otherwise it is
        copied into engine storage.  Finiteness is checked either way."""
        dt = np.dtype(dtype)
        code = _native.F32 if dt == np.float32 else _native.F64
        ctx = _native.context(device)
        h = _native.C.c_void_p()
        ld = int(ld or p)
        if owner is not None and ld == -(-int(p) // 32) * 32:
            _native.check(_native.lib().gps_matrix_wrap_device(ctx.handle, _native.C.c_void_p(ptr), int(p), int(n),
                                                               ld, code, _native.C.byref(h)))
        else:
            owner = None
            _native.check(_native.lib().gps_matrix_create_device(ctx.handle, _native.C.c_void_p(ptr), int(p),
                                                                 int(n), ld, code, _native.C.byref(h)))
        self = cls._wrap(ctx, h)
        object.__setattr__(self, "_owner", owner)
        if self._nonfinite:
            raise ValueError("matrix entries must be finite")
        return self

    @classmethod
    def _wrap(cls, ctx, handle):
        """Adopt a gps_matrix handle produced by the library (e.g. deflate)."""
        self = object.__new__(cls)
        p, n, ld = _native.C.c_int64(), _native.C.c_int64(), _native.C.c_int64()
        code = _native.C.c_int()
        _native.check(_native.lib().gps_matrix_info(handle, _native.C.byref(p), _native.C.byref(n),
                                                    _native.C.byref(ld), _native.C.byref(code)))
        for name, value in (("_ctx", ctx), ("_handle", handle), ("_values", None), ("_owner", None), ("p", p.value),
                            ("n", n.value), ("dtype", np.dtype(np.float32 if code.value == _native.F32
                                                               else np.float64))):
            object.__setattr__(self, name, value)
        norms, bad = self._column_pass()
        object.__setattr__(self, "_norms", norms)
        object.__setattr__(self, "_nonfinite", bool(bad))
        return self

    def _column_pass(self):
        norms = np.empty(self.n)
        bad = _native.C.c_int(0)
        _native.check(_native.lib().gps_column_norms(self._handle, _native.dptr(norms), _native.C.byref(bad)))
        norms.flags.writeable = False
        return norms, bad.value

    def __setattr__(self, name, value):
        raise AttributeError("DataMatrix is immutable")

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and _native._lib is not None:
            _native.lib().gps_matrix_destroy(h)

    @property
    def handle(self):
        return self._handle

    @property
    def context(self):
        return self._ctx

    @property
    def shape(self):
        return (self.p, self.n)

    @property
    def norms(self):
        """fp64 column norms computed on the device at construction."""
        return self._norms

    @property
    def values(self):
        """float64 F-ordered host copy (downloaded lazily, read-only)."""
        if self._values is None:
            host = np.empty((self.p, self.n), dtype=self.dtype, order="F")
            _native.check(_native.lib().gps_matrix_download(self._handle, host.ctypes.data))
            host = np.asarray(host, dtype=np.float64, order="F")
            host.flags.writeable = False
            object.__setattr__(self, "_values", host)
        return self._values

    def column(self, i):
        """Column a_i as a float64 vector (core.py:52-54)."""
        i = int(i)
        if not -self.n <= i < self.n:
            raise IndexError(i)
        out = np.empty(self.p)
        _native.check(_native.lib().gps_matrix_column(self._handle, i % self.n, _native.dptr(out)))
        return out

    def __repr__(self):
        return f"DataMatrix(p={self.p}, n={self.n}, dtype={self.dtype.name}, device={self._ctx.device})"


def as_data_matrix(A):
    """Coerce an array-like (or pass through a DataMatrix), core.py:64-68."""
    return A if isinstance(A, DataMatrix) else DataMatrix(A)


class SparseLoadings:
    """n x m loadings with unit-or-zero columns and an explicit pattern
    (reference core.py:71-110)."""

    __slots__ = ("values", "pattern", "m")

    def __init__(self, values):
        arr = np.array(values, dtype=np.float64, copy=True)
        if arr.ndim == 1:
            arr = arr.reshape(-1, 1)
        if arr.ndim != 2:
            raise ValueError("loadings must be a vector or a 2-d matrix")
        col_norms = np.linalg.norm(arr, axis=0)
        off = (col_norms > 0) & (np.abs(col_norms - 1.0) > ALGEBRAIC_TOL)
        if off.any():
            raise ValueError(f"columns {np.flatnonzero(off).tolist()} are neither zero nor unit norm")
        pattern = tuple(np.flatnonzero(arr[:, j]) for j in range(arr.shape[1]))
        arr.flags.writeable = False
        object.__setattr__(self, "values", arr)
        object.__setattr__(self, "pattern", pattern)
        object.__setattr__(self, "m", arr.shape[1])

    def __setattr__(self, name, value):
        raise AttributeError("SparseLoadings is immutable")

    @property
    def n(self):
        return self.values.shape[0]

    def nnz_per_component(self):
        return [int(ix.size) for ix in self.pattern]

    def __repr__(self):
        return f"SparseLoadings(n={self.n}, m={self.m}, nnz={self.nnz_per_component()})"


class StiefelPoint:
    """p x m matrix with orthonormal columns (reference core.py:113-140)."""

    __slots__ = ("values",)

    def __init__(self, values, tol=STIEFEL_TOL):
        arr = np.array(values, dtype=np.float64, copy=True)
        if arr.ndim == 1:
            arr = arr.reshape(-1, 1)
        p, m = arr.shape
        if m > p:
            raise ValueError(f"need m <= p, got p={p}, m={m}")
        err = np.linalg.norm(arr.T @ arr - np.eye(m))
        if err > tol:
            raise ValueError(f"columns not orthonormal: ||X'X - I||_F = {err:.3e}")
        arr.flags.writeable = False
        object.__setattr__(self, "values", arr)

    def __setattr__(self, name, value):
        raise AttributeError("StiefelPoint is immutable")

    @property
    def p(self):
        return self.values.shape[0]

    @property
    def m(self):
        return self.values.shape[1]


def _broadcast_m(value, m, name):
    v = np.atleast_1d(np.asarray(value, dtype=np.float64))
    if v.size == 1:
        v = np.full(m, v[0])
    if v.shape != (m,):
        raise ValueError(f"{name} must be a scalar or length-{m} vector")
    return v


@dataclass(frozen=True)
class SolverConfig:
    """One solve's settings (reference core.py:152-209); gamma / mu are
    stored as read-only length-m fp64 vectors."""

    penalty: str = "l1"
    mode: str = "single_unit"
    m: int = 1
    gamma: object = 0.0
    mu: object = 1.0
    tol: float = 1e-6
    max_iter: int = 1000
    init: str = "max_norm_column"
    deflation: str = "orthogonal_projection"
    seed: int = 0
    x0: object = None
    restarts: int = 1
    refine: bool = False

    def __post_init__(self):
        for value, allowed, name in ((self.penalty, PENALTIES, "penalty"), (self.mode, MODES, "mode"),
                                     (self.init, INITS, "init"), (self.deflation, DEFLATIONS, "deflation")):
            if value not in allowed:
                raise ValueError(f"{name} must be one of {allowed}")
        if self.m < 1:
            raise ValueError("m must be >= 1")
        if self.restarts < 1:
            raise ValueError("restarts must be >= 1")
        if not self.tol > 0:
            raise ValueError("tol must be > 0")
        if self.max_iter < 1:
            raise ValueError("max_iter must be >= 1")
        gamma = _broadcast_m(self.gamma, self.m, "gamma")
        if (gamma < 0).any():
            raise ValueError("gamma entries must be >= 0")
        mu = _broadcast_m(self.mu, self.m, "mu")
        if (mu <= 0).any():
            raise ValueError("mu entries must be > 0")
        gamma.flags.writeable = False
        mu.flags.writeable = False
        object.__setattr__(self, "gamma", gamma)
        object.__setattr__(self, "mu", mu)
        if self.init == "user_supplied" and self.x0 is None:
            raise ValueError("init='user_supplied' requires x0")


@dataclass(frozen=True)
class RunReport:
    """Per-solve diagnostics (reference core.py:212-226) plus device
    records the reference keeps implicitly:

    - `kernel_launches`: device kernels the solve launched;
    - `near_threshold`: per component, the column indices whose (mu-scaled)
      correlation in the final sweep lies within 1e-6 gamma of the
      threshold -- ||c| - gamma| <= 1e-6 gamma (l1), |c^2 - gamma| <=
      1e-6 gamma (l0) -- the entries whose support membership is decided by
      rounding (north_star: logged, not counted as a support mismatch);
      `near_threshold_total` counts them (the device keeps the first 8192);
    - `stiefel_errors` (block solves): ||X_k'X_k - I||_F of every iterate,
      k = 0 .. iterations -- the feasibility the reference asserts by
      building a StiefelPoint from each polar output (block.py:149,
      core.py:113-129).
    """

    objective_history: list = field(default_factory=list)
    iterations: int = 0
    wall_time: float = 0.0
    nnz_per_component: list = field(default_factory=list)
    converged: bool = False
    component_histories: list = None
    kernel_launches: int = 0
    near_threshold: list = None
    near_threshold_total: int = 0
    stiefel_errors: list = None


BAND_COMPONENTS = 64  # entries are col * 64 + component (csrc/common.cuh BandLog)


def decode_band(entries, m, offset=0):
    """Per-component sorted column indices of a device near-threshold list."""
    e = np.asarray(entries, dtype=np.int64)
    cols, comp = e // BAND_COMPONENTS + offset, e % BAND_COMPONENTS
    return [np.unique(cols[comp == j]) for j in range(m)]


def positive_part(t):
    """max(0, t) elementwise (core.py:229-231)."""
    return np.maximum(t, 0.0)


def column_norms(A):
    """Euclidean norm of every column (core.py:243-246), from the device pass."""
    return np.array(as_data_matrix(A).norms)


def center_columns(A):
    """Subtract each column's mean; a new fp64 DataMatrix (core.py:234-240),
    formed on the device (column means by a 1/p-weighted A'1 sweep, then a
    rank-1 copy kernel)."""
    return center_columns_with_means(A)[0]


def center_columns_with_means(A):
    """center_columns plus the fp64 column means it subtracted."""
    A = as_data_matrix(A)
    h = _native.C.c_void_p()
    means = np.empty(A.n)
    _native.check(_native.lib().gps_matrix_center(A.handle, _native.dptr(means), _native.C.byref(h)))
    return DataMatrix._wrap(A.context, h), means


def gram_quadratic(A, z):
    """z'(A'A)z evaluated as ||Az||^2 without forming the Gram matrix
    (core.py:249-256); Az by the device column accumulation."""
    A = as_data_matrix(A)
    z = np.asarray(z, dtype=np.float64)
    if z.shape != (A.n,):
        raise ValueError(f"z must have length n={A.n}, got shape {z.shape}")
    v = np.empty(A.p)
    _native.check(_native.lib().gps_gram_apply(A.handle, _native.dptr(np.ascontiguousarray(z)), _native.dptr(v)))
    return float(v @ v)
