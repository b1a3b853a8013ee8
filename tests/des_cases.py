"""Scenario x preset cases for the DES link-swap (reference simulator, two pool backends)."""
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCEN = os.path.join(ROOT, "tests", "golden", "scenarios")
REF_DIR = os.path.join(ROOT, "oracle", "_ref")
# valve = channel + our_mem (Algorithm 1 + apply_reclaim); channel+uvm = FIFO selection +
# apply; channel+static = FIFO + kill; channel+prism never reclaims (control)
PRESETS = ["valve", "channel+uvm", "channel+static", "channel+prism"]


def scenarios():
    return sorted(f[:-5] for f in os.listdir(SCEN) if f.endswith(".json"))


def cases():
    return [(s, p) for s in scenarios() for p in PRESETS]
