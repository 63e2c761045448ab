"""paper_1605_01238_b200 -- B200-native weighted-quadrature (WQ) formation of
isogeometric Galerkin mass/stiffness matrices (arXiv:1605.01238).

Thin ctypes binding of ``libwq.so`` (C-ABI in ``include/wq.h``).  Functions
carry the C names; this module only marshals arguments.  Every step of the
path runs in the CUDA kernels of ``csrc/``; there is no CPU fallback: if the
library is missing or no CUDA device is present, calls raise.

PyTorch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WQ_LIB_DEBUG_PATH") or os.path.join(_HERE, "libwq.so")  # override: debug builds (tools/)

WQ_OK, WQ_EINVAL, WQ_EKNOTS, WQ_ESINGULAR, WQ_EGEOMETRY, WQ_ENOMEM, WQ_ECUDA, WQ_ERANGE = range(8)
WQ_MASS, WQ_STIFFNESS = 0, 1
WQ_KERNEL_AUTO, WQ_KERNEL_DIRECT, WQ_KERNEL_TILE, WQ_KERNEL_WS, WQ_KERNEL_LINE, WQ_KERNEL_ZLINE = 0, 1, 2, 3, 4, 5
WQ_LAYOUT_AUTO, WQ_LAYOUT_STANDARD = 0, 1
WQ_MAX_DEGREE = 10

EXPORTED = ("wq_plan_create", "wq_plan_destroy", "wq_plan_info", "wq_build_rules", "wq_build_coef",
            "wq_pattern", "wq_assemble", "wq_assemble_ex", "wq_check", "wq_form_host", "wq_export_rules",
            "wq_export_coef", "wq_status_string", "wq_last_error", "wq_version", "wq_launch_count")


class WQError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: status {status} ({detail})")
        self.status = status
        self.detail = detail


class _Desc(C.Structure):
    _fields_ = [("d", C.c_int), ("p", C.c_int), ("n_knots", C.POINTER(C.c_int64)),
                ("knots", C.POINTER(C.POINTER(C.c_double))), ("slab_begin", C.c_int64), ("slab_end", C.c_int64),
                ("need_mass", C.c_int), ("need_stiffness", C.c_int), ("device", C.c_int), ("coef_layout", C.c_int)]


class _Info(C.Structure):
    _fields_ = [("n_dof_total", C.c_int64), ("nnz_total", C.c_int64), ("row_begin", C.c_int64),
                ("n_rows_local", C.c_int64), ("nnz_local", C.c_int64), ("n_dof", C.c_int64 * 3),
                ("n_qp", C.c_int64 * 3), ("max_q", C.c_int32 * 3), ("coef_points", C.c_int64),
                ("workspace_bytes", C.c_int64)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libwq.so; raises (loudly) if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libwq.so not found at {path}: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    vp = C.c_void_p
    lib.wq_plan_create.argtypes = [C.POINTER(_Desc), C.POINTER(vp)]
    lib.wq_plan_destroy.argtypes = [vp]
    lib.wq_plan_info.argtypes = [vp, C.POINTER(_Info)]
    lib.wq_build_rules.argtypes = [vp, vp]
    lib.wq_build_coef.argtypes = [vp, vp, vp]
    lib.wq_pattern.argtypes = [vp, C.c_int64, vp, vp, vp]
    lib.wq_assemble.argtypes = [vp, C.c_int, vp, vp, vp]
    lib.wq_assemble_ex.argtypes = [vp, C.c_int, C.c_int, vp, vp, vp]
    lib.wq_check.argtypes = [vp, vp]
    lib.wq_form_host.argtypes = [vp, C.c_int, vp, C.c_int64, vp, vp, vp, vp]
    lib.wq_export_rules.argtypes = [vp, C.c_int, vp, vp, vp, vp, vp, vp]
    lib.wq_export_coef.argtypes = [vp, vp, C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
    lib.wq_status_string.argtypes = [C.c_int]
    lib.wq_status_string.restype = C.c_char_p
    lib.wq_last_error.restype = C.c_char_p
    lib.wq_version.restype = C.c_char_p
    lib.wq_launch_count.restype = C.c_uint64
    for name in EXPORTED:
        if not name.startswith(("wq_status", "wq_last", "wq_version", "wq_launch_count")):
            getattr(lib, name).restype = C.c_int
    _lib = lib
    return lib


def _chk(st: int, where: str):
    if st != WQ_OK:
        lib = load_library()
        raise WQError(st, where, f"{lib.wq_status_string(st).decode()}; {lib.wq_last_error().decode()}")


def _ptr(t):
    """Device/host pointer of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


# ---------------------------------------------------------------- C names
def wq_plan_create(p, knots, slab=(0, -1), need_mass=True, need_stiffness=True, device=0, coef_layout=0):
    lib = load_library()
    ks = [np.ascontiguousarray(k, dtype=np.float64) for k in knots]
    d = len(ks)
    nk = (C.c_int64 * d)(*[k.size for k in ks])
    arr = (C.POINTER(C.c_double) * d)(*[k.ctypes.data_as(C.POINTER(C.c_double)) for k in ks])
    desc = _Desc(d, int(p), nk, arr, int(slab[0]), int(slab[1]), int(bool(need_mass)), int(bool(need_stiffness)),
                 int(device), int(coef_layout))
    h = C.c_void_p()
    _chk(lib.wq_plan_create(C.byref(desc), C.byref(h)), "wq_plan_create")
    return h.value


def wq_plan_destroy(plan):
    _chk(load_library().wq_plan_destroy(plan), "wq_plan_destroy")


def wq_plan_info(plan) -> dict:
    info = _Info()
    _chk(load_library().wq_plan_info(plan, C.byref(info)), "wq_plan_info")
    return dict(n_dof_total=info.n_dof_total, nnz_total=info.nnz_total, row_begin=info.row_begin,
                n_rows_local=info.n_rows_local, nnz_local=info.nnz_local, n_dof=list(info.n_dof),
                n_qp=list(info.n_qp), max_q=list(info.max_q), coef_points=info.coef_points,
                workspace_bytes=info.workspace_bytes)


def wq_build_rules(plan, stream=None):
    _chk(load_library().wq_build_rules(plan, _stream(stream)), "wq_build_rules")


def wq_build_coef(plan, d_ctrl, stream=None):
    _chk(load_library().wq_build_coef(plan, _ptr(d_ctrl), _stream(stream)), "wq_build_coef")


def wq_pattern(plan, nnz_base, d_row_ptr, d_col=None, stream=None):
    _chk(load_library().wq_pattern(plan, int(nnz_base), _ptr(d_row_ptr), _ptr(d_col), _stream(stream)), "wq_pattern")


def wq_assemble(plan, matrix, d_val, d_col=None, stream=None, kernel=WQ_KERNEL_AUTO):
    _chk(load_library().wq_assemble_ex(plan, int(matrix), int(kernel), _ptr(d_val), _ptr(d_col), _stream(stream)),
         "wq_assemble")


def wq_check(plan, stream=None):
    _chk(load_library().wq_check(plan, _stream(stream)), "wq_check")


def wq_form_host(plan, matrix, h_ctrl, nnz_base, h_row_ptr, h_col, h_val, stream=None):
    _chk(load_library().wq_form_host(plan, int(matrix), _ptr(h_ctrl), int(nnz_base), _ptr(h_row_ptr), _ptr(h_col),
                                     _ptr(h_val), _stream(stream)), "wq_form_host")


def wq_export_rules(plan, dir: int, p: int) -> dict:
    info = wq_plan_info(plan)
    n, nq, mq = info["n_dof"][dir], info["n_qp"][dir], info["max_q"][dir]
    out = dict(points=np.empty(nq), qlo=np.empty(n, np.int32), qlen=np.empty(n, np.int32),
               w=np.empty((n, 4, mq)), basis=np.empty((nq, 3, p + 1)), span=np.empty(nq, np.int32))
    _chk(load_library().wq_export_rules(plan, dir, *[_ptr(out[k]) for k in ("points", "qlo", "qlen", "w", "basis",
                                                                              "span")]), "wq_export_rules")
    return out


def wq_export_coef(plan):
    lib = load_library()
    nv, nc, qb = C.c_int64(), C.c_int32(), C.c_int64()
    _chk(lib.wq_export_coef(plan, None, C.byref(nv), C.byref(nc), C.byref(qb)), "wq_export_coef")
    out = np.empty(nv.value)
    _chk(lib.wq_export_coef(plan, _ptr(out), C.byref(nv), C.byref(nc), C.byref(qb)), "wq_export_coef")
    return out.reshape(nc.value, -1), qb.value


def wq_version() -> str:
    return load_library().wq_version().decode()


def wq_launch_count() -> int:
    return int(load_library().wq_launch_count())


# ---------------------------------------------------------------- convenience
class Plan:
    """RAII wrapper: one plan (one GPU, one slab) + torch-allocated buffers."""

    def __init__(self, p, knots, slab=(0, -1), need_mass=True, need_stiffness=True, device=0, coef_layout=0):
        self.p = int(p)
        self.d = len(knots)
        self.device = device
        self.h = wq_plan_create(p, knots, slab, need_mass, need_stiffness, device, coef_layout)
        self.info = wq_plan_info(self.h)

    def close(self):
        if getattr(self, "h", None):
            wq_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def alloc_csr(self, with_col=True):
        import torch
        dev = torch.device("cuda", self.device)
        rp = torch.empty(self.info["n_rows_local"] + 1, dtype=torch.int64, device=dev)
        col = torch.empty(self.info["nnz_local"], dtype=torch.int32, device=dev) if with_col else None
        val = torch.empty(self.info["nnz_local"], dtype=torch.float64, device=dev)
        return rp, col, val

    def setup(self, d_ctrl, stream=None):
        wq_build_rules(self.h, stream)
        wq_build_coef(self.h, d_ctrl, stream)

    def form(self, matrix, d_ctrl, nnz_base=0, out=None, stream=None, kernel=WQ_KERNEL_AUTO, check=True):
        """Whole hot path on device: rules, coefficients, pattern, values."""
        rp, col, val = out if out is not None else self.alloc_csr()
        self.setup(d_ctrl, stream)
        wq_pattern(self.h, nnz_base, rp, None, stream)
        wq_assemble(self.h, matrix, val, col, stream, kernel)
        if check:
            wq_check(self.h, stream)
        return rp, col, val
