"""The reference's own test suites and simulator, run against the drop-in.

oracle/_ref/ holds binaries built (oracle/Makefile) from /root/reference/proj sources compiled
in place:
  ref_<suite>    the reference doctest suite linked against the reference implementation
  valve_<suite>  the SAME suite source compiled against include/colosim (the C++ drop-in headers)
                 and linked against libvalve.so -- the reference's tests exercising the GPU path
  ref_des / valve_des   the reference simulator with either backend (DES link-swap)

CPU tests check the checkers are alive (the reference suites pass under the doctest shim, the
committed DES digests reproduce); GPU tests run the valve_* binaries and require the
simulator's event logs to be byte-identical to the reference's on every scenario x preset.
"""
import hashlib
import json
import os
import subprocess

import pytest

import des_cases

SUITES = ["test_memory", "test_reclaim", "test_channel", "test_sim", "test_baselines", "acceptance"]
GOLDEN = os.path.join(des_cases.ROOT, "tests", "golden", "des_sha256.json")


def _bin(name):
    path = os.path.join(des_cases.REF_DIR, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (needs /root/reference when oracle/ was built)")
    return path


def _run_suite(binary, timeout):
    r = subprocess.run([binary], capture_output=True, text=True, timeout=timeout)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0 and "SUCCESS" in r.stdout, tail
    return r.stdout


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_reference(suite):
    """The reference suites pass on the reference itself under the doctest shim (pins the shim)."""
    out = _run_suite(_bin("ref_" + suite), 300)
    if suite == "acceptance":
        assert out.count("[PASS]") == 8, out


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_device(suite):
    """The reference's own suites, compiled against include/colosim, on the sm_100a path."""
    out = _run_suite(_bin("valve_" + suite), 1200)
    if suite == "acceptance":
        assert out.count("[PASS]") == 8, out


def _des(binary, scen, preset, tmp_path):
    path = os.path.join(str(tmp_path), f"{binary}_{scen}_{preset}.jsonl".replace("+", "_"))
    subprocess.run([_bin(binary), os.path.join(des_cases.SCEN, scen + ".json"), path, preset],
                   check=True, capture_output=True, timeout=1200)
    return open(path, "rb").read()


@pytest.mark.parametrize("scen,preset", [("pair_06", "valve"), ("pair_09", "channel+uvm"),
                                         ("pair_01", "channel+static")])
def test_reference_des_matches_committed_digest(scen, preset, tmp_path):
    """ref_des reproduces the digests committed in tests/golden/des_sha256.json."""
    golden = json.load(open(GOLDEN))[f"{scen}/{preset}"]
    data = _des("ref_des", scen, preset, tmp_path)
    assert hashlib.sha256(data).hexdigest() == golden["sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("scen,preset", des_cases.cases())
def test_des_link_swap_byte_identical(scen, preset, tmp_path):
    """The reference simulator driven by the GPU pool/selection/channel emits the same event log,
    byte for byte, as with the reference implementation."""
    golden = json.load(open(GOLDEN))[f"{scen}/{preset}"]
    data = _des("valve_des", scen, preset, tmp_path)
    assert data.count(b"\n") == golden["records"]
    assert hashlib.sha256(data).hexdigest() == golden["sha256"], f"{scen}/{preset} diverged"
