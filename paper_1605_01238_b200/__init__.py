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
WQ_KERNEL_AUTO, WQ_KERNEL_DIRECT, WQ_KERNEL_TILE, WQ_KERNEL_ZLINE, WQ_KERNEL_ZHP, WQ_KERNEL_SF2 = 0, 1, 2, 3, 4, 5
WQ_BPTS_INTERIOR, WQ_BPTS_ENDPOINTS = 0, 1
WQ_MAX_DEGREE = 10
KERNEL_NAMES = {0: "none", 1: "direct", 2: "tile", 3: "zline", 4: "zhp", 5: "sf2"}

EXPORTED = ("wq_plan_create", "wq_plan_destroy", "wq_plan_info", "wq_build_rules", "wq_build_coef",
            "wq_pattern", "wq_assemble", "wq_assemble_ex", "wq_assemble_sgq", "wq_check", "wq_form_host",
            "wq_export_rules", "wq_export_coef", "wq_status_string", "wq_last_error", "wq_version",
            "wq_launch_count")


class WQError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: status {status} ({detail})")
        self.status = status
        self.detail = detail


class _Desc(C.Structure):
    _fields_ = [("d", C.c_int), ("p", C.c_int), ("n_knots", C.POINTER(C.c_int64)),
                ("knots", C.POINTER(C.POINTER(C.c_double))), ("ctrl", C.c_void_p), ("kappa", C.c_void_p),
                ("gamma", C.c_void_p), ("slab_begin", C.c_int64), ("slab_end", C.c_int64),
                ("need_mass", C.c_int), ("need_stiffness", C.c_int), ("bpts", C.c_int), ("device", C.c_int)]


class _Info(C.Structure):
    _fields_ = [("n_dof_total", C.c_int64), ("nnz_total", C.c_int64), ("row_begin", C.c_int64),
                ("n_rows_local", C.c_int64), ("nnz_local", C.c_int64), ("n_dof", C.c_int64 * 3),
                ("n_qp", C.c_int64 * 3), ("max_q", C.c_int32 * 3), ("coef_points", C.c_int64),
                ("workspace_bytes", C.c_int64), ("kernel", C.c_int32 * 2), ("uniform_rules", C.c_int32)]


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
    lib.wq_build_coef.argtypes = [vp, vp, vp, vp, vp]
    lib.wq_pattern.argtypes = [vp, C.c_int64, vp, vp, vp]
    lib.wq_assemble.argtypes = [vp, C.c_int, vp, vp, vp]
    lib.wq_assemble_ex.argtypes = [vp, C.c_int, C.c_int, vp, vp, vp]
    lib.wq_assemble_sgq.argtypes = [vp, C.c_int, vp, vp, vp, vp, vp, vp]
    lib.wq_check.argtypes = [vp, vp]
    lib.wq_form_host.argtypes = [vp, C.c_int, vp, vp, vp, C.c_int64, vp, vp, vp, vp]
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


_DT = {"f64": ("float64", "torch.float64"), "i64": ("int64", "torch.int64"), "i32": ("int32", "torch.int32")}


def _ptr(t, kind=None, n=None, where="argument", device=None, host=False):
    """Pointer of a torch tensor or numpy array (None -> NULL), after checking what the C side
    assumes: dtype `kind` ("f64" / "i64" / "i32"), contiguity, at least `n` elements, and the
    memory space (device tensors on the plan's device, or host memory when host=True)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        if not host:
            raise WQError(WQ_EINVAL, where, "numpy array passed where a device buffer is required")
        if kind and str(t.dtype) != _DT[kind][0]:
            raise WQError(WQ_EINVAL, where, f"dtype {t.dtype}, expected {_DT[kind][0]}")
        if not t.flags["C_CONTIGUOUS"]:
            raise WQError(WQ_EINVAL, where, "array is not contiguous")
        if n is not None and t.size < n:
            raise WQError(WQ_EINVAL, where, f"{t.size} elements, need {n}")
        return t.ctypes.data
    if kind and str(t.dtype) != _DT[kind][1]:
        raise WQError(WQ_EINVAL, where, f"dtype {t.dtype}, expected {_DT[kind][1]}")
    if not t.is_contiguous():
        raise WQError(WQ_EINVAL, where, "tensor is not contiguous")
    if n is not None and t.numel() < n:
        raise WQError(WQ_EINVAL, where, f"{t.numel()} elements, need {n}")
    if host:
        if t.is_cuda:
            raise WQError(WQ_EINVAL, where, "device tensor passed where host memory is required")
    else:
        if not t.is_cuda:
            raise WQError(WQ_EINVAL, where, "host tensor passed where a device buffer is required")
        if device is not None and t.device.index != device:
            raise WQError(WQ_EINVAL, where, f"tensor on cuda:{t.device.index}, plan on cuda:{device}")
    return t.data_ptr()


def _host_f64(a, n, where):
    """Host FP64 copy (contiguous numpy) of an optional net with n values."""
    if a is None:
        return None
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    if a.size != n:
        raise WQError(WQ_EINVAL, where, f"{a.size} values, need {n}")
    return a


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


# ---------------------------------------------------------------- C names
def wq_plan_create(p, knots, ctrl=None, kappa=None, gamma=None, slab=(0, -1), need_mass=True, need_stiffness=True,
                   device=0, bpts=WQ_BPTS_INTERIOR):
    lib = load_library()
    ks = [np.ascontiguousarray(k, dtype=np.float64) for k in knots]
    d = len(ks)
    ndof = int(np.prod([k.size - p - 1 for k in ks])) if ks else 0
    hc = _host_f64(ctrl, ndof * d, "wq_plan_create(ctrl)")
    hk = _host_f64(kappa, ndof, "wq_plan_create(kappa)")
    hg = _host_f64(gamma, ndof, "wq_plan_create(gamma)")
    nk = (C.c_int64 * d)(*[k.size for k in ks])
    arr = (C.POINTER(C.c_double) * d)(*[k.ctypes.data_as(C.POINTER(C.c_double)) for k in ks])
    vp = lambda a: None if a is None else a.ctypes.data
    desc = _Desc(d, int(p), nk, arr, vp(hc), vp(hk), vp(hg), int(slab[0]), int(slab[1]), int(bool(need_mass)),
                 int(bool(need_stiffness)), int(bpts), int(device))
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
                workspace_bytes=info.workspace_bytes, kernel=list(info.kernel), uniform_rules=info.uniform_rules)


def wq_build_rules(plan, stream=None):
    _chk(load_library().wq_build_rules(plan, _stream(stream)), "wq_build_rules")


def wq_build_coef(plan, d_ctrl, d_kappa=None, d_gamma=None, stream=None):
    info = wq_plan_info(plan)
    n, d = info["n_dof_total"], sum(1 for x in info["n_qp"] if x > 1) or 1
    _chk(load_library().wq_build_coef(plan, _ptr(d_ctrl, "f64", None, "wq_build_coef(ctrl)"),
                                      _ptr(d_kappa, "f64", n, "wq_build_coef(kappa)"),
                                      _ptr(d_gamma, "f64", n, "wq_build_coef(gamma)"), _stream(stream)),
         "wq_build_coef")


def wq_pattern(plan, nnz_base, d_row_ptr, d_col=None, stream=None):
    info = wq_plan_info(plan)
    _chk(load_library().wq_pattern(plan, int(nnz_base), _ptr(d_row_ptr, "i64", info["n_rows_local"] + 1, "row_ptr"),
                                   _ptr(d_col, "i32", info["nnz_local"], "col"), _stream(stream)), "wq_pattern")


def wq_assemble(plan, matrix, d_val, d_col=None, stream=None, kernel=WQ_KERNEL_AUTO):
    info = wq_plan_info(plan)
    _chk(load_library().wq_assemble_ex(plan, int(matrix), int(kernel), _ptr(d_val, "f64", info["nnz_local"], "val"),
                                       _ptr(d_col, "i32", info["nnz_local"], "col"), _stream(stream)),
         "wq_assemble")


def wq_assemble_sgq(plan, matrix, d_ctrl, d_val, d_col=None, d_kappa=None, d_gamma=None, stream=None):
    info = wq_plan_info(plan)
    n = info["n_dof_total"]
    _chk(load_library().wq_assemble_sgq(plan, int(matrix), _ptr(d_ctrl, "f64", None, "ctrl"),
                                        _ptr(d_kappa, "f64", n, "kappa"), _ptr(d_gamma, "f64", n, "gamma"),
                                        _ptr(d_val, "f64", info["nnz_local"], "val"),
                                        _ptr(d_col, "i32", info["nnz_local"], "col"), _stream(stream)),
         "wq_assemble_sgq")


def wq_check(plan, stream=None):
    _chk(load_library().wq_check(plan, _stream(stream)), "wq_check")


def wq_form_host(plan, matrix, h_ctrl, nnz_base, h_row_ptr, h_col, h_val, stream=None, h_kappa=None, h_gamma=None):
    info = wq_plan_info(plan)
    n, nnz, rows = info["n_dof_total"], info["nnz_local"], info["n_rows_local"]
    _chk(load_library().wq_form_host(plan, int(matrix), _ptr(h_ctrl, "f64", None, "h_ctrl", host=True),
                                     _ptr(h_kappa, "f64", n, "h_kappa", host=True),
                                     _ptr(h_gamma, "f64", n, "h_gamma", host=True), int(nnz_base),
                                     _ptr(h_row_ptr, "i64", rows + 1, "h_row_ptr", host=True),
                                     _ptr(h_col, "i32", nnz, "h_col", host=True),
                                     _ptr(h_val, "f64", nnz, "h_val", host=True), _stream(stream)), "wq_form_host")


def wq_export_rules(plan, dir: int, p: int) -> dict:
    info = wq_plan_info(plan)
    n, nq, mq = info["n_dof"][dir], info["n_qp"][dir], info["max_q"][dir]
    out = dict(points=np.empty(nq), qlo=np.empty(n, np.int32), qlen=np.empty(n, np.int32),
               w=np.empty((n, 4, mq)), basis=np.empty((nq, 3, p + 1)), span=np.empty(nq, np.int32))
    _chk(load_library().wq_export_rules(plan, dir, *[out[k].ctypes.data for k in ("points", "qlo", "qlen", "w",
                                                                                  "basis", "span")]),
         "wq_export_rules")
    return out


def wq_export_coef(plan):
    lib = load_library()
    nv, nc, qb = C.c_int64(), C.c_int32(), C.c_int64()
    _chk(lib.wq_export_coef(plan, None, C.byref(nv), C.byref(nc), C.byref(qb)), "wq_export_coef")
    out = np.empty(nv.value)
    _chk(lib.wq_export_coef(plan, out.ctypes.data, C.byref(nv), C.byref(nc), C.byref(qb)), "wq_export_coef")
    return out.reshape(nc.value, -1), qb.value


def wq_version() -> str:
    return load_library().wq_version().decode()


def wq_launch_count() -> int:
    return int(load_library().wq_launch_count())


# ---------------------------------------------------------------- convenience
class Plan:
    """RAII wrapper: one plan (one GPU, one slab) + torch-allocated buffers.  Passing `ctrl` (host
    control net) validates the geometry at creation (WQ_EGEOMETRY) and builds its coefficient
    field; otherwise call setup(d_ctrl) before assembling."""

    def __init__(self, p, knots, ctrl=None, kappa=None, gamma=None, slab=(0, -1), need_mass=True,
                 need_stiffness=True, device=0, bpts=WQ_BPTS_INTERIOR):
        self.p = int(p)
        self.d = len(knots)
        self.device = device
        self.h = wq_plan_create(p, knots, ctrl, kappa, gamma, slab, need_mass, need_stiffness, device, bpts)
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

    def setup(self, d_ctrl, stream=None, d_kappa=None, d_gamma=None):
        wq_build_rules(self.h, stream)
        wq_build_coef(self.h, d_ctrl, d_kappa, d_gamma, stream)

    def form(self, matrix, d_ctrl=None, nnz_base=0, out=None, stream=None, kernel=WQ_KERNEL_AUTO, check=True,
             d_kappa=None, d_gamma=None):
        """Whole hot path on device: rules, coefficients (if d_ctrl is given; else the geometry
        passed at creation), pattern, values."""
        rp, col, val = out if out is not None else self.alloc_csr()
        if d_ctrl is not None:
            self.setup(d_ctrl, stream, d_kappa, d_gamma)
        wq_pattern(self.h, nnz_base, rp, None, stream)
        wq_assemble(self.h, matrix, val, col, stream, kernel)
        if check:
            wq_check(self.h, stream)
        return rp, col, val
