"""The real-time harness's TTFT/TPOT deltas recomputed by the reference's own report code.

realtime.py writes every run's events in the reference's events.jsonl schema (log.hpp:13-59);
oracle/_ref/ref_metrics is the reference's build_report + ttft_increase / tpot_increase
(metrics.cpp:85-241, compiled unmodified).  The paired increases the harness reports must equal
what the reference computes from the same logs ("compute the deltas with
build_report + ttft_increase/tpot_increase").

CPU tests: a synthetic schedule written through EventLog, and the logs of a measured B200 run
committed under tests/golden/realtime/ (bench.py wrote them; see the README there).
GPU test: a short live run of the harness on a 2-layer model, logs checked the same way.
"""
import glob
import json
import os
import random
import subprocess

import pytest

from paper_2604_07874_b200.realtime import EventLog, paired_increase

HERE = os.path.dirname(os.path.abspath(__file__))
REF_METRICS = os.path.join(HERE, "..", "oracle", "_ref", "ref_metrics")
GOLDEN = os.path.join(HERE, "golden", "realtime")

need_ref = pytest.mark.skipif(not os.path.exists(REF_METRICS), reason="oracle/_ref/ref_metrics not built")


def ref_metrics(solo, colo):
    out = subprocess.run([REF_METRICS, solo, colo], capture_output=True, text=True, check=True)
    return json.loads(out.stdout)


def deltas_from_log(path):
    """(ttft_by_req, tpot_by_req) from a log, as build_report defines them (metrics.cpp:189-201)."""
    arrival, ttft, tpot = {}, {}, {}
    for line in open(path):
        r = json.loads(line)
        if r["kind"] == "arrival" and r["class"] == "online":
            arrival[r["request_id"]] = r["time_us"]
        elif r["kind"] == "done" and r["class"] == "online":
            rid, n = r["request_id"], r["tokens"]
            if n >= 1:
                ttft[rid] = float(r["first_token_us"] - arrival[rid])
            if n >= 2:
                tpot[rid] = (r["last_token_us"] - r["first_token_us"]) / (n - 1)
    return ttft, tpot


def _synthetic_run(path, trace, rng, colocated):
    log = EventLog()
    log.add(0, "run_meta", scenario="synthetic", preset="valve" if colocated else "standalone", seed=0,
            gpus=1, horizon_us=10_000_000, online_fingerprint="0x00000000000000ab",
            offline_fingerprint="0x0000000000000000")
    ttft, tpot = {}, {}
    for rid, arr, prompt, out in trace:
        log.add(arr, "arrival", **{"class": "online"}, request_id=rid, gpu=0, prompt_tokens=prompt,
                output_tokens=out)
        first = arr + rng.randint(40_000, 90_000) + (rng.randint(0, 50) if colocated else 0)
        step = rng.randint(9_000, 21_000)
        last = first + step * (out - 1)
        if colocated and rng.random() < 0.3:
            log.add(arr, "disable_issued", effective_us=arr, cause="busy")
            log.add(arr + 5, "preempt_wait", gpu=0, request_id=rid, delay_us=12)
        log.add(first, "first_token", **{"class": "online"}, request_id=rid, gpu=0)
        log.add(last, "done", **{"class": "online"}, request_id=rid, gpu=0, tokens=out, first_token_us=first,
                last_token_us=last, digest="0x0000000000000000")
        ttft[rid] = float(first - arr)
        tpot[rid] = (last - first) / (out - 1)
    if colocated:
        log.add(5_000, "reclaim_request", gpu=0, handles=2, op=0, purpose="shortfall")
        log.add(5_000, "reclaim_done", gpu=0, op=0, latency_us=150, handle_ids=[3, 7])
        log.add(5_000, "evicted", request_id=900, gpu=0, recompute_tokens=3000)
    log.write_jsonl(path)
    return ttft, tpot


@need_ref
def test_eventlog_schema_and_deltas_match_reference_metrics(tmp_path):
    rng = random.Random(4)
    trace = [(i, i * 170_000 + rng.randint(0, 9_000), rng.randint(2500, 3500), rng.randint(8, 12))
             for i in range(25)]
    solo = str(tmp_path / "solo.jsonl")
    colo = str(tmp_path / "colo.jsonl")
    s_ttft, s_tpot = _synthetic_run(solo, trace, random.Random(1), False)
    c_ttft, c_tpot = _synthetic_run(colo, trace, random.Random(2), True)
    ref = ref_metrics(solo, colo)
    ours_t, ours_p = paired_increase(s_ttft, c_ttft), paired_increase(s_tpot, c_tpot)
    assert ref["pairs"] == ours_t["pairs"] == 25
    assert ref["ttft_mean_pct"] == pytest.approx(ours_t["mean_pct"], rel=1e-12, abs=1e-12)
    assert ref["ttft_max_pct"] == pytest.approx(ours_t["max_pct"], rel=1e-12, abs=1e-12)
    assert ref["tpot_mean_pct"] == pytest.approx(ours_p["mean_pct"], rel=1e-12, abs=1e-12)
    assert ref["tpot_max_pct"] == pytest.approx(ours_p["max_pct"], rel=1e-12, abs=1e-12)
    assert ref["reclaim_ops"] == 1 and ref["evictions"] == 1 and ref["online_completed"] == 25
    # the logs parse back to the dicts the harness computed
    assert deltas_from_log(colo) == (c_ttft, c_tpot)


def _golden_pairs():
    for colo in sorted(glob.glob(os.path.join(GOLDEN, "colo*.jsonl"))):
        i = os.path.basename(colo)[4:-6]
        solo = os.path.join(GOLDEN, f"solo{i}.jsonl")
        if os.path.exists(solo):
            yield solo, colo


@need_ref
@pytest.mark.skipif(not list(_golden_pairs()), reason="no committed B200 realtime logs")
@pytest.mark.parametrize("solo,colo", list(_golden_pairs()) or [("", "")])
def test_measured_b200_run_deltas_match_reference_metrics(solo, colo):
    ref = ref_metrics(solo, colo)
    (s_ttft, s_tpot), (c_ttft, c_tpot) = deltas_from_log(solo), deltas_from_log(colo)
    t, p = paired_increase(s_ttft, c_ttft), paired_increase(s_tpot, c_tpot)
    assert ref["pairs"] == t["pairs"] > 0
    assert ref["ttft_mean_pct"] == pytest.approx(t["mean_pct"], rel=1e-12, abs=1e-12)
    assert ref["tpot_mean_pct"] == pytest.approx(p["mean_pct"], rel=1e-12, abs=1e-12)
    assert ref["disables_issued"] >= 1  # the colocated run really gated the offline tenant


SMALL = dict(horizon=4.0, base=1.0, spike=6.0, period=4.0, width=1.0, handles=16, layers=2, output=(4, 6),
             prompt=(600, 900), tail_s=4.0)


@pytest.mark.gpu
@need_ref
def test_live_harness_logs_match_reference_metrics(tmp_path):
    """The live loop's events.jsonl (online KV in pool slots, decode-pass + GEMM-chain tenant)
    pair through the reference's own build_report / ttft_increase / tpot_increase."""
    from paper_2604_07874_b200 import realtime as RT

    cfg = RT.RtConfig(gemm_tokens=256, gemm_layers=2, gemm_ctas=16)
    out = RT.measure(repeats=1, policies=(), cfg=cfg, log_dir=str(tmp_path), **SMALL)
    assert out["valve"]["pairs"] > 0
    solo, colo = str(tmp_path / "solo0.jsonl"), str(tmp_path / "colo0.jsonl")
    ref = ref_metrics(solo, colo)
    (s_ttft, s_tpot), (c_ttft, c_tpot) = deltas_from_log(solo), deltas_from_log(colo)
    assert ref["pairs"] == paired_increase(s_ttft, c_ttft)["pairs"] > 0
    assert ref["ttft_mean_pct"] == pytest.approx(paired_increase(s_ttft, c_ttft)["mean_pct"], rel=1e-12, abs=1e-12)
    assert ref["tpot_mean_pct"] == pytest.approx(paired_increase(s_tpot, c_tpot)["mean_pct"], rel=1e-12, abs=1e-12)
    assert ref["disables_issued"] >= 1


@pytest.mark.gpu
def test_live_harness_policies_on_the_same_kernels():
    """Every policy arm runs on the same kernels and replays the standalone plan exactly; the
    offline engine completes requests (harvest > 0) and the static arm kills instead of evicting."""
    from paper_2604_07874_b200 import realtime as RT

    cfg = RT.RtConfig(gemm_tokens=256, gemm_layers=2, gemm_ctas=16)
    out = RT.measure(repeats=1, policies=("valve-fifo", "channel+static", "channel+prism"), cfg=cfg, **SMALL)
    for pol in ("valve", "valve-fifo", "channel+static", "channel+prism"):
        assert out[pol]["plan_deviations"] == [0] * len(out[pol]["plan_deviations"]), pol
        assert out[pol]["pairs"] > 0, pol
        assert out[pol]["offline_forwards_per_s"] > 0, pol
    assert out["channel+static"]["evictions"] == 0
    assert out["channel+prism"]["reclaims"] == 0
