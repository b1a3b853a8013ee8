"""The C-ABI library (CPU-side checks: no kernel is launched here).

* libvalve.so loads and exports every function declared in include/valve_cuda.h;
* the reference-facing calls fail loudly (CudaError) without a GPU -- there is no CPU path;
* the product package never references the checkers under oracle/.
"""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT
from paper_2604_07874_b200 import api as A

HEADER = os.path.join(ROOT, "include", "valve_cuda.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(valve_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("valve_pool_create", "valve_pool_apply_reclaim", "valve_select", "valve_pool_reclaim",
                 "valve_pool_reclaim_copy", "valve_gate_raise", "valve_gate_wait_quiesced",
                 "valve_channel_note_busy", "valve_resctl_window_tick", "valve_offline_launch"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(A.LIBVALVE)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_no_cpu_fallback_without_gpu(has_cuda):
    if has_cuda:
        pytest.skip("GPU present")
    with pytest.raises(A.CudaError):
        A.MemoryPool(4, 4, 16)
    with pytest.raises(A.CudaError):
        A.selective_reclaim(A.ReclaimInstance([A.ReclaimHandle(1, 0, [1])], {1: 1}), 1)
    with pytest.raises(A.CudaError):
        A.Gate(0)


def test_argument_errors_precede_device_work():
    # validation that the reference performs before touching state maps to the same types
    with pytest.raises(A.InvalidArgument):
        A.selective_reclaim(A.ReclaimInstance(), -1)
    with pytest.raises(A.InvalidArgument):
        A.oracle_reclaim(A.ReclaimInstance([A.ReclaimHandle(h, 0, []) for h in range(21)], {}), 1)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2604_07874_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "valve_oracle" not in src, f


def test_host_controllers_need_no_gpu():
    """ReservationController / ChannelController are the host control plane (north star (c))."""
    ctl = A.ReservationController()
    assert ctl.grow_target(10, 100) == 15
    ch = A.ChannelController(1000, 600)
    assert ch.ensure_disabled(100) == 1100
