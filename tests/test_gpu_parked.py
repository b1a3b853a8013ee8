"""Host-side pool / selection calls while a gated offline launch is parked behind a closed gate
(tests/parked_tenant_probe.py, in a subprocess so a deadlock fails the test instead of hanging the
suite): growth paths use stream-ordered allocation, so nothing waits for the parked stream."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT


@pytest.mark.gpu
def test_pool_ops_never_wait_for_a_parked_tenant():
    probe = os.path.join(ROOT, "tests", "parked_tenant_probe.py")
    try:
        r = subprocess.run([sys.executable, probe], capture_output=True, text=True, timeout=240)
    except subprocess.TimeoutExpired as e:
        out = e.stdout.decode() if isinstance(e.stdout, bytes) else (e.stdout or "")
        raise AssertionError(f"deadlock with the tenant parked; probe got as far as:\n{out}")
    assert r.returncode == 0, r.stderr[-2000:]
    for step in ("parked", "table grown", "selection grown", "fused reclaim True", "released"):
        assert step in r.stdout, r.stdout
