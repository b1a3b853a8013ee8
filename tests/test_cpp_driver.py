"""The C++ driver on the reference's runtime API (tools/cpp/colosim_ops.cpp), compiled against the
reference (oracle/_ref/ref_ops, CPU) and against the include/colosim drop-in over libvalve.so
(tools/_bin/valve_ops, B200): both builds run the same population and must agree on what the
reclaims did; the valve build's e2e leg moves the reported bytes."""
import json
import os
import subprocess

import pytest

from conftest import ROOT

REF_OPS = os.path.join(ROOT, "oracle", "_ref", "ref_ops")
VALVE_OPS = os.path.join(ROOT, "tools", "_bin", "valve_ops")


def _run(exe, *args, env=None, timeout=600):
    try:
        r = subprocess.run([exe, *args], capture_output=True, text=True, timeout=timeout, env=env)
    except subprocess.TimeoutExpired as e:  # show how far the driver got (VALVE_OPS_TRACE)
        err = e.stderr.decode() if isinstance(e.stderr, bytes) else (e.stderr or "")
        raise AssertionError(f"{exe} {' '.join(args)} timed out after {timeout} s; stderr tail:\n{err[-3000:]}")
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.skipif(not os.path.exists(REF_OPS), reason="reference not built here")
def test_reference_build_table_cpu():
    d = _run(REF_OPS, "table", "128", "1,4")
    assert d["build"] == "reference" and d["handles"] == 128 and d["live_requests"] > 0
    assert [x["k"] for x in d["reclaim"]] == [1, 4] and all(x["pages"] > 0 for x in d["reclaim"])


def test_valve_build_exists_and_links():
    assert os.path.exists(VALVE_OPS), "build() compiles tools/_bin/valve_ops"
    out = subprocess.run(["ldd", VALVE_OPS], capture_output=True, text=True).stdout
    assert "libvalve.so" in out and "not found" not in out.split("libvalve.so")[1].split("\n")[0]


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(REF_OPS), reason="reference not built here")
def test_table_same_reclaims_as_reference():
    """Same seeded population through both builds: identical live-request counts and identical
    invalidated page counts per k (the drop-in reproduces the reference's decisions)."""
    ref = _run(REF_OPS, "table", "256", "1,4,15")
    dev = _run(VALVE_OPS, "table", "256", "1,4,15")
    assert dev["live_requests"] == ref["live_requests"]
    assert [x["pages_all_reps"] for x in dev["reclaim"]] == [x["pages_all_reps"] for x in ref["reclaim"]]
    assert all(x["fused_us"] > 0 for x in dev["reclaim"])


@pytest.mark.gpu
def test_e2e_leg_moves_the_reported_bytes():
    d = _run(VALVE_OPS, "e2e", "128", "8", "3", "1", env=dict(os.environ, VALVE_OPS_TRACE="1"), timeout=180)
    assert d["steps"] == 3 and d["bytes"] > 0 and d["gbs"] > 1.0
    assert d["d2h_bytes_per_step"] >= d["bytes"] // 3
