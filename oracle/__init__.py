"""CPU checkers for the hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg / --impl reference) may
import this package.  It loads
  oracle/_build/libvalve_oracle.so  -- the C restatement (valve_oracle.c)
  oracle/_ref/libcolosim_ref.so     -- the reference's own sources compiled in place (ref_shim.cpp)
and exposes them through the product's Python API wrapper so a test can run the same call
sequence against the device and the checker.
"""
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
C_LIB = os.path.join(_HERE, "_build", "libvalve_oracle.so")
REF_LIB = os.path.join(_HERE, "_ref", "libcolosim_ref.so")

_cache = {}


def _backend(path, name):
    from paper_2604_07874_b200.api import Backend

    if name not in _cache:
        _cache[name] = Backend(path, "vo_", False, name)
        _declare_extras(_cache[name].lib)
    return _cache[name]


def c_backend():
    """The C restatement (always buildable: gcc only)."""
    return _backend(C_LIB, "oracle-c")


def ref_available():
    return os.path.exists(REF_LIB)


def ref_backend():
    """The reference implementation itself (only where it was built from /root/reference)."""
    return _backend(REF_LIB, "oracle-ref")


def _declare_extras(L):
    import ctypes as C

    L.vo_page_word.restype = C.c_uint64
    L.vo_page_word.argtypes = [C.c_int64, C.c_int32, C.c_int64]
    L.vo_gather_images.restype = None
    L.vo_gather_images.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.c_void_p]
    L.vo_gather_memcpy.restype = None
    L.vo_gather_memcpy.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int,
                                   C.c_void_p, C.c_int]


def build(quiet=True):
    """Compile the C restatement (and oracle/_ref when /root/reference is present)."""
    import subprocess

    subprocess.run(["make", "-C", _HERE], check=True, capture_output=quiet)
