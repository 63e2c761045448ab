"""CPU-side checks of the C-ABI boundary (no GPU): the library loads, exports
every symbol include/wq.h declares, and rejects invalid input in
wq_plan_create before touching the device (P:463-478 knot rules)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1605_01238_b200 as wq
from wqinputs import uniform_open_knots

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "wq.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]*?\b(wq_\w+)\s*\(", txt, re.M)))


def test_header_symbols_exported():
    lib = wq.load_library()
    syms = header_symbols()
    assert len(syms) >= 14, syms
    for s in syms:
        assert hasattr(lib, s), f"libwq.so does not export {s}"
    assert set(syms) == set(wq.EXPORTED)


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", wq.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings():
    lib = wq.load_library()
    for s in range(8):
        assert lib.wq_status_string(s).decode().startswith("WQ_")
    assert b"sm_100a" in lib.wq_version()


@pytest.mark.parametrize("knots,p,status", [
    ([0, 0, 0, 0.5, 0.5, 1, 1, 1], 2, wq.WQ_EKNOTS),      # repeated interior knot
    ([0, 0, 0.5, 1, 1, 1], 2, wq.WQ_EKNOTS),              # not open at the left
    ([0, 0, 0, 0.7, 0.3, 1, 1, 1], 2, wq.WQ_EKNOTS),      # decreasing
    ([0, 0, 1, 1], 2, wq.WQ_EKNOTS),                      # too few knots
    ([0, 0, 0, np.nan, 1, 1, 1], 2, wq.WQ_EKNOTS),        # non-finite
    ([0, 0, 0.5, 1, 1], 0, wq.WQ_EKNOTS),                 # p < 1
    ([0] * 12 + [1] * 12, 11, wq.WQ_EINVAL),              # p > WQ_MAX_DEGREE
])
def test_plan_create_rejects(knots, p, status):
    with pytest.raises(wq.WQError) as e:
        wq.wq_plan_create(p, [np.array(knots, float)])
    assert e.value.status == status


def test_plan_create_bad_slab_and_d():
    k = uniform_open_knots(2, 4)
    with pytest.raises(wq.WQError) as e:
        wq.wq_plan_create(2, [k, k], slab=(3, 2))
    assert e.value.status == wq.WQ_EINVAL
    with pytest.raises(wq.WQError) as e:
        wq.wq_plan_create(2, [k] * 4)
    assert e.value.status == wq.WQ_EINVAL
    with pytest.raises(wq.WQError) as e:
        wq.wq_plan_create(2, [k], need_mass=False, need_stiffness=False)
    assert e.value.status == wq.WQ_EINVAL


def test_bpts_endpoints_rejected():
    """Reading R1: the endpoints-included boundary points leave #Q_0 = p-1 < #I_0 = p+1, which Eq.
    numb_nodes forbids; wq_plan_create reports WQ_ESINGULAR naming row 0."""
    for p in (1, 2, 5):
        with pytest.raises(wq.WQError) as e:
            wq.wq_plan_create(p, [uniform_open_knots(p, 6)], bpts=wq.WQ_BPTS_ENDPOINTS)
        assert e.value.status == wq.WQ_ESINGULAR and "row 0" in e.value.detail


def test_coefficients_need_geometry():
    k = uniform_open_knots(2, 4)
    with pytest.raises(wq.WQError) as e:
        wq.wq_plan_create(2, [k], kappa=np.ones(6))
    assert e.value.status == wq.WQ_EINVAL
    with pytest.raises(wq.WQError) as e:
        wq.wq_plan_create(2, [k], bpts=7)
    assert e.value.status == wq.WQ_EINVAL


def test_binding_checks_buffers():
    """The binding refuses buffers the C side would misuse (ADVICE: dtype, memory space, size)."""
    import torch
    with pytest.raises(wq.WQError):
        wq._ptr(torch.zeros(4, dtype=torch.float32), "f64", 4, "val")
    with pytest.raises(wq.WQError):
        wq._ptr(torch.zeros(4, dtype=torch.float64), "f64", 4, "val")  # host tensor, device expected
    with pytest.raises(wq.WQError):
        wq._ptr(np.zeros(3), "f64", 4, "h_val", host=True)  # too short
    with pytest.raises(wq.WQError):
        wq._ptr(np.zeros((4, 4))[:, 0], "f64", 4, "h_val", host=True)  # not contiguous
    assert wq._ptr(np.zeros(4), "f64", 4, "h_val", host=True) != 0


def test_null_plan_calls():
    lib = wq.load_library()
    assert lib.wq_build_rules(None, None) == wq.WQ_EINVAL
    assert lib.wq_assemble(None, 0, None, None, None) == wq.WQ_EINVAL
    assert lib.wq_check(None, None) == wq.WQ_EINVAL
    assert lib.wq_plan_destroy(None) == wq.WQ_OK


def test_no_cpu_fallback_in_binding():
    """The product binding never imports the oracle or computes values itself."""
    src = open(wq.__file__).read()
    assert "import oracle" not in src and "from oracle" not in src
    for f in os.listdir(os.path.join(ROOT, "paper_1605_01238_b200", "csrc")):
        txt = open(os.path.join(ROOT, "paper_1605_01238_b200", "csrc", f)).read()
        assert "oracle" not in txt.replace("Shares nothing with oracle/", "").replace("shares nothing with oracle", "")
