"""ctypes wrapper of the CPU oracle (ldpc_oracle.c).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg -- never by the product
package.  It is the checker the CUDA path is compared against, and the CPU
baseline it is timed beside.

The arithmetic lives in ldpc_oracle.c (a restatement of the reference's
serial.py / tables.py, file:line cited there).  The prior is restated twice:
priors_awgn() is the reference's own numpy expression (serial.py:39-50), the
only way to get numpy's last-ulp values on the machine at hand; npexp.c
restates the exp numpy runs on AVX512_SKX hosts (SVML exp8_ha) in C, the
checker for the device prior kernel (priors_awgn_svml / npexp below).
"""

from __future__ import annotations

import ctypes
import os
import pathlib
import subprocess

import numpy as np

_HERE = pathlib.Path(__file__).resolve().parent
_LIB_PATH = _HERE / "build" / "liboracle.so"
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_f64p = ctypes.POINTER(ctypes.c_double)

_ERRORS = {
    -1: "matrix dimensions must be positive",
    -2: "entry outside the matrix",
    -3: "duplicate entry",
    -4: "row has no entries",
    -5: "column has no entries",
    -6: "out of memory",
}


def build(force: bool = False) -> pathlib.Path:
    """Compile the oracle (gcc, -ffp-contract=off) into oracle/build/."""
    srcs = [_HERE / "ldpc_oracle.c", _HERE / "npexp.c"]
    if force or not _LIB_PATH.exists() or any(_LIB_PATH.stat().st_mtime < s.stat().st_mtime for s in srcs):
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        L.oracle_tables_create.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, _i32p, _i32p,
                                           ctypes.POINTER(ctypes.c_void_p)]
        L.oracle_tables_create.restype = ctypes.c_int
        L.oracle_tables_destroy.argtypes = [ctypes.c_void_p]
        L.oracle_tables_export.argtypes = [ctypes.c_void_p, ctypes.c_int] + [_i64p] * 6
        L.oracle_tables_var_groups.argtypes = [ctypes.c_void_p, _i64p, _i64p]
        L.oracle_values_to_check.argtypes = [ctypes.c_void_p, _f64p, _f64p, _f64p]
        L.oracle_values_to_variable.argtypes = [ctypes.c_void_p, _f64p, _f64p]
        L.oracle_estimate.argtypes = [ctypes.c_void_p, _f64p, _f64p, _u8p]
        L.oracle_syndrome.argtypes = [ctypes.c_void_p, _u8p, _u8p]
        L.oracle_decode.argtypes = [ctypes.c_void_p, _f64p, ctypes.c_int32, ctypes.c_int32, _u8p, _u8p, _i32p,
                                    _u8p]
        L.oracle_decode.restype = ctypes.c_int
        L.oracle_decode_batch.argtypes = [ctypes.c_void_p, _f64p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_int32, _u8p, _u8p, _i32p, _u8p]
        L.oracle_decode_batch.restype = ctypes.c_int
        L.oracle_npexp_array.argtypes = [_f64p, ctypes.c_long, _f64p]
        L.oracle_npexp_array.restype = None
        L.oracle_priors_awgn.argtypes = [_f64p, ctypes.c_long, ctypes.c_double, _f64p]
        L.oracle_priors_awgn.restype = None
        _lib = L
    return _lib


def _ptr(a: np.ndarray, typ):
    return a.ctypes.data_as(typ)


def priors_awgn(y, sigma2: float) -> np.ndarray:
    """serial.py:39-50, the identical numpy expression."""
    if sigma2 <= 0:
        raise ValueError("sigma2 must be positive")
    y = np.asarray(y, dtype=np.float64)
    with np.errstate(over="ignore"):
        return 1.0 / (1.0 + np.exp(-2.0 * y / sigma2))


def npexp(x) -> np.ndarray:
    """npexp.c: numpy's AVX512_SKX float64 exp (SVML exp8_ha), restated in C."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    lib().oracle_npexp_array(_ptr(x, _f64p), x.size, _ptr(out, _f64p))
    return out


def priors_awgn_svml(y, sigma2: float) -> np.ndarray:
    """serial.py:49-50 evaluated with npexp (one rounding per operation)."""
    if sigma2 <= 0:
        raise ValueError("sigma2 must be positive")
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.empty_like(y)
    lib().oracle_priors_awgn(_ptr(y, _f64p), y.size, float(sigma2), _ptr(out, _f64p))
    return out


class OracleTables:
    """Both table orientations of one code (tables.py:95-116), built in C."""

    def __init__(self, n: int, m: int, ones):
        arr = np.asarray(ones, dtype=np.int64).reshape(-1, 2)
        rows = np.ascontiguousarray(arr[:, 0], dtype=np.int32)
        cols = np.ascontiguousarray(arr[:, 1], dtype=np.int32)
        h = ctypes.c_void_p()
        rc = lib().oracle_tables_create(int(n), int(m), len(rows), _ptr(rows, _i32p), _ptr(cols, _i32p),
                                        ctypes.byref(h))
        if rc != 0:
            raise ValueError(_ERRORS.get(rc, f"oracle error {rc}"))
        self._h = h
        self.n, self.m, self.total_edges = int(n), int(m), len(rows)

    @classmethod
    def from_matrix(cls, H) -> "OracleTables":
        return cls(H.n, H.m, H.ones)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib().oracle_tables_destroy(h)
            self._h = None

    def export(self, orientation: str) -> dict:
        E = self.total_edges
        out = {k: np.empty(E, dtype=np.int64) for k in "evctsu"}
        lib().oracle_tables_export(self._h, 0 if orientation == "variable" else 1,
                                   *[_ptr(out[k], _i64p) for k in "evctsu"])
        return out

    def var_groups(self):
        gs = np.empty(self.n, dtype=np.int64)
        gz = np.empty(self.n, dtype=np.int64)
        lib().oracle_tables_var_groups(self._h, _ptr(gs, _i64p), _ptr(gz, _i64p))
        return gs, gz

    # -- phases (serial.py:63-147), canonical edge order -------------------
    def values_to_check(self, p, r):
        p = np.ascontiguousarray(p, dtype=np.float64)
        r = np.ascontiguousarray(r, dtype=np.float64)
        q = np.empty(self.total_edges)
        lib().oracle_values_to_check(self._h, _ptr(p, _f64p), _ptr(r, _f64p), _ptr(q, _f64p))
        return q

    def values_to_variable(self, q):
        q = np.ascontiguousarray(q, dtype=np.float64)
        r = np.empty(self.total_edges)
        lib().oracle_values_to_variable(self._h, _ptr(q, _f64p), _ptr(r, _f64p))
        return r

    def estimate(self, p, r):
        p = np.ascontiguousarray(p, dtype=np.float64)
        r = np.ascontiguousarray(r, dtype=np.float64)
        c = np.empty(self.n, dtype=np.uint8)
        lib().oracle_estimate(self._h, _ptr(p, _f64p), _ptr(r, _f64p), _ptr(c, _u8p))
        return c

    def syndrome(self, chat):
        chat = np.ascontiguousarray(chat, dtype=np.uint8)
        if chat.shape[-1] != self.n:
            raise ValueError(f"estimate length {chat.shape[-1]} does not match n={self.n}")
        z = np.empty(self.m, dtype=np.uint8)
        lib().oracle_syndrome(self._h, _ptr(chat, _u8p), _ptr(z, _u8p))
        return z

    # -- decode (serial.py:150-178) ---------------------------------------
    def decode_priors(self, p, max_iterations: int, fixed_iterations: bool = False):
        """One frame from priors; returns (estimate, success, iterations, syndrome)."""
        if max_iterations < 0:
            raise ValueError("max_iterations must be non-negative")
        p = np.ascontiguousarray(p, dtype=np.float64)
        if p.shape != (self.n,):
            raise ValueError(f"expected {self.n} observations, got {p.shape}")
        est = np.empty(self.n, dtype=np.uint8)
        z = np.empty(self.m, dtype=np.uint8)
        ok = ctypes.c_uint8()
        it = ctypes.c_int32()
        rc = lib().oracle_decode(self._h, _ptr(p, _f64p), int(max_iterations), int(bool(fixed_iterations)),
                                 _ptr(est, _u8p), ctypes.byref(ok), ctypes.byref(it), _ptr(z, _u8p))
        if rc:
            raise RuntimeError(f"oracle decode failed ({rc})")
        return est, bool(ok.value), int(it.value), z

    def decode_awgn(self, y, sigma2: float, max_iterations: int, fixed_iterations: bool = False):
        return self.decode_priors(priors_awgn(y, sigma2), max_iterations, fixed_iterations)

    def decode_batch(self, P, max_iterations: int, fixed_iterations: bool = False, n_threads: int | None = None):
        """Frames [B, n] of priors decoded on host threads (the CPU baseline)."""
        P = np.ascontiguousarray(P, dtype=np.float64)
        B = P.shape[0]
        if P.shape != (B, self.n):
            raise ValueError("priors must be [B, n]")
        est = np.empty((B, self.n), dtype=np.uint8)
        z = np.empty((B, self.m), dtype=np.uint8)
        ok = np.empty(B, dtype=np.uint8)
        it = np.empty(B, dtype=np.int32)
        nt = int(n_threads or os.cpu_count() or 1)
        rc = lib().oracle_decode_batch(self._h, _ptr(P, _f64p), B, int(max_iterations), int(bool(fixed_iterations)),
                                       nt, _ptr(est, _u8p), _ptr(ok, _u8p), _ptr(it, _i32p), _ptr(z, _u8p))
        if rc:
            raise RuntimeError(f"oracle batch decode failed ({rc})")
        return est, ok.astype(bool), it, z
