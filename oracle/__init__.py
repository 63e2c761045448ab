"""CPU oracle for WQ formation of IGA Galerkin matrices (arXiv:1605.01238).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  It wraps ``oracle/wq_oracle.c`` (binary128 weights, long-double
coefficients and row sums, direct nested sums -- see the header of that file
for the paper passage behind every step).  It shares no code with the CUDA
path in ``paper_1605_01238_b200/``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "wq_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

MASS, STIFFNESS = 0, 1
ORC_OK, ORC_EINVAL, ORC_EKNOTS, ORC_ESINGULAR, ORC_EGEOMETRY = 0, 1, 2, 3, 4
FAMILIES = ((0, 0), (1, 0), (0, 1), (1, 1))  # (a, b) = (test, trial) derivative order


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (binary128 via libquadmath, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared", "-o", _LIB, _SRC,
               "-lquadmath", "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = C.CDLL(_LIB)
            P = C.c_void_p
            i64p = C.POINTER(C.c_int64)
            dp = C.POINTER(C.c_double)
            lib.orc_create.restype = P
            lib.orc_create.argtypes = [C.c_int, C.c_int, i64p, C.POINTER(dp), dp]
            lib.orc_destroy.argtypes = [P]
            lib.orc_status.argtypes = [P]
            lib.orc_message.argtypes = [P]
            lib.orc_message.restype = C.c_char_p
            lib.orc_info.argtypes = [P, C.c_int, C.c_int]
            lib.orc_info.restype = C.c_int64
            lib.orc_export_dir.argtypes = [P, C.c_int] + [C.c_void_p] * 9
            lib.orc_coef_box.argtypes = [P, i64p, i64p, C.c_void_p, C.c_void_p]
            lib.orc_row_nnz.argtypes = [P, C.c_int64]
            lib.orc_row_nnz.restype = C.c_int64
            lib.orc_rows.argtypes = [P, C.c_int, C.c_int64] + [C.c_void_p] * 6
            lib.orc_pattern.argtypes = [P, C.c_void_p, C.c_void_p]
            lib.orc_pattern_rows.argtypes = [P, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
            lib.orc_set_coefficients.argtypes = [P, C.c_void_p, C.c_void_p]
            lib.orc_sgq_dense.argtypes = [P, C.c_int, C.c_void_p]
            lib.orc_check_knots.argtypes = [C.c_int, C.c_int64, dp]
            lib.orc_num_points.argtypes = [C.c_int, C.c_int64]
            lib.orc_num_points.restype = C.c_int64
            lib.orc_points.argtypes = [C.c_int, C.c_int64, dp, dp]
            lib.orc_basis_all.argtypes = [C.c_int, C.c_int64, dp, C.c_double, dp, dp]
            lib.orc_gauss.argtypes = [C.c_int, dp, dp]
            _lib = lib
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _vp(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"oracle status {status}: {msg}")
        self.status = status


# ---- stand-alone univariate helpers (pins) --------------------------------
def check_knots(p, knots) -> int:
    k = np.ascontiguousarray(knots, dtype=np.float64)
    return _load().orc_check_knots(p, k.size, _dp(k))


def points(p, knots) -> np.ndarray:
    """Global point grid of Remark 1, reading R1."""
    lib = _load()
    k = np.ascontiguousarray(knots, dtype=np.float64)
    out = np.empty(lib.orc_num_points(p, k.size))
    st = lib.orc_points(p, k.size, _dp(k), _dp(out))
    if st:
        raise OracleError(st, "invalid knots")
    return out


def basis_all(p, knots, x):
    """All B-splines of degree p and their derivatives at x (binary128, rounded)."""
    k = np.ascontiguousarray(knots, dtype=np.float64)
    n = k.size - p - 1
    v, dv = np.empty(n), np.empty(n)
    _load().orc_basis_all(p, k.size, _dp(k), float(x), _dp(v), _dp(dv))
    return v, dv


def gauss(n):
    t, w = np.empty(n), np.empty(n)
    _load().orc_gauss(n, _dp(t), _dp(w))
    return t, w


# ---- full context ------------------------------------------------------------
class Oracle:
    """One WQ problem: d knot vectors of degree p plus an optional control net."""

    def __init__(self, p: int, knots, ctrl=None, kappa=None, gamma=None):
        self._lib = _load()
        self.p = int(p)
        self.knots = [np.ascontiguousarray(k, dtype=np.float64) for k in knots]
        self.d = len(self.knots)
        nk = (C.c_int64 * self.d)(*[k.size for k in self.knots])
        arr = (C.POINTER(C.c_double) * self.d)(*[_dp(k) for k in self.knots])
        self._ctrl = None if ctrl is None else np.ascontiguousarray(ctrl, dtype=np.float64).reshape(-1, self.d)
        self._h = self._lib.orc_create(self.d, self.p, nk, arr,
                                       None if self._ctrl is None else _dp(self._ctrl))
        st = self._lib.orc_status(self._h)
        if st:
            msg = self._lib.orc_message(self._h).decode()
            self._lib.orc_destroy(self._h)
            self._h = None
            raise OracleError(st, msg)
        self._kappa = None if kappa is None else np.ascontiguousarray(kappa, dtype=np.float64).reshape(-1)
        self._gamma = None if gamma is None else np.ascontiguousarray(gamma, dtype=np.float64).reshape(-1)
        if self._kappa is not None or self._gamma is not None:
            self._lib.orc_set_coefficients(self._h, _vp(self._kappa), _vp(self._gamma))
        self.n = [int(self._lib.orc_info(self._h, l, 0)) for l in range(self.d)]
        self.nq = [int(self._lib.orc_info(self._h, l, 1)) for l in range(self.d)]
        self.maxq = [int(self._lib.orc_info(self._h, l, 2)) for l in range(self.d)]
        self.ndof = int(np.prod(self.n))

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.orc_destroy(self._h)
            self._h = None

    def direction(self, l: int) -> dict:
        n, nq, mq, p = self.n[l], self.nq[l], self.maxq[l], self.p
        out = dict(points=np.empty(nq), qlo=np.empty(n, np.int64), qlen=np.empty(n, np.int64),
                   jlo=np.empty(n, np.int64), jlen=np.empty(n, np.int64),
                   w=np.empty((n, 4, mq)), Bv=np.empty((nq, n)), Bd=np.empty((nq, n)),
                   I4=np.empty((n, 2 * p + 1, 4)))
        self._lib.orc_export_dir(self._h, l, *[_vp(out[k]) for k in
                                               ("points", "qlo", "qlen", "jlo", "jlen", "w", "Bv", "Bd", "I4")])
        return out

    def coef_box(self, qb, qe):
        """c and C (row-major d x d) on the grid box [qb, qe) -> (npts, 1+d*d), det."""
        qb = np.asarray(list(qb) + [0] * (3 - self.d), np.int64)
        qe = np.asarray(list(qe) + [1] * (3 - self.d), np.int64)
        npts = int(np.prod((qe - qb)[: self.d]))
        out = np.empty((npts, 1 + self.d * self.d))
        det = np.empty(npts)
        st = self._lib.orc_coef_box(self._h, qb.ctypes.data_as(C.POINTER(C.c_int64)),
                                    qe.ctypes.data_as(C.POINTER(C.c_int64)), _vp(out), _vp(det))
        return out, det, st

    def row_nnz(self, rows) -> np.ndarray:
        return np.array([self._lib.orc_row_nnz(self._h, int(r)) for r in rows], np.int64)

    def rows(self, matrix: int, rows):
        """Direct-sum WQ values of the given global rows.

        Returns (ptr, col, val, kappa, scale): CSR of the selected rows in the
        order given, kappa_i and scale_i = max_j sum_q |term_ijq| per row."""
        if self._ctrl is None:
            raise OracleError(1, "no control net")
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        nnz = self.row_nnz(rows)
        ptr = np.zeros(rows.size + 1, np.int64)
        np.cumsum(nnz, out=ptr[1:])
        col = np.empty(int(ptr[-1]), np.int32)
        val = np.empty(int(ptr[-1]))
        kappa = np.empty(rows.size)
        scale = np.empty(rows.size)
        st = self._lib.orc_rows(self._h, int(matrix), rows.size, _vp(rows), _vp(ptr), _vp(col), _vp(val),
                                _vp(kappa), _vp(scale))
        if st:
            raise OracleError(st, "row evaluation failed (geometry?)")
        return ptr, col, val, kappa, scale

    def pattern(self):
        """Full CSR pattern (row_ptr int64, col int32) by definition."""
        rp = np.empty(self.ndof + 1, np.int64)
        self._lib.orc_pattern(self._h, _vp(rp), None)
        col = np.empty(int(rp[-1]), np.int32)
        self._lib.orc_pattern(self._h, _vp(rp), _vp(col))
        return rp, col

    def pattern_rows(self, r_lo: int, r_hi: int):
        """Pattern of rows [r_lo, r_hi) (global row_ptr offsets, columns), by definition."""
        rp = np.empty(r_hi - r_lo + 1, np.int64)
        self._lib.orc_pattern_rows(self._h, int(r_lo), int(r_hi), _vp(rp), None)
        col = np.empty(int(rp[-1] - rp[0]), np.int32)
        self._lib.orc_pattern_rows(self._h, int(r_lo), int(r_hi), _vp(rp), _vp(col))
        return rp, col

    def sgq_dense(self, matrix: int) -> np.ndarray:
        """Element-loop Gauss (p+1 pts/dir/elem) dense matrix; self-check only."""
        A = np.empty((self.ndof, self.ndof))
        st = self._lib.orc_sgq_dense(self._h, int(matrix), _vp(A))
        if st:
            raise OracleError(st, "sgq failed")
        return A

    def dense(self, matrix: int) -> np.ndarray:
        ptr, col, val, _, _ = self.rows(matrix, np.arange(self.ndof))
        A = np.zeros((self.ndof, self.ndof))
        for r in range(self.ndof):
            A[r, col[ptr[r]:ptr[r + 1]]] = val[ptr[r]:ptr[r + 1]]
        return A
