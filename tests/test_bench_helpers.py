"""Host logic of bench.py (no GPU): the stage-overlap summary and the k_push
per-role / per-launch reduction of sp_debug_plan_profile snapshots."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _k(**us):
    return {k: {"avg_us": v} for k, v in us.items()}


def test_overlap_efficiency_bounds(bench):
    k = _k(plan=30.0, transfer=40.0, forward=10.0, surrogate=10.0, backward=20.0)
    # fully overlapped: the step costs the slowest stream (compute, 40 = transfer)
    assert bench._overlap(k, 40.0)["efficiency"] == 1.0
    # back to back: the step costs the sum of the streams
    full = bench._overlap(k, 110.0)
    assert full["efficiency"] == 0.0 and full["serial_sum_us"] == 110.0
    half = bench._overlap(k, 75.0)
    assert half["efficiency"] == 0.5
    assert half["stream_us"] == {"plan": 30.0, "transfer": 40.0, "compute": 40.0}


def test_plan_roles_window_means_and_percentiles(bench):
    T = 3
    p0 = {"launches": [10, 10], "plan_us": [5.0, 6.0, 7.0], "dedup_us": [4.0, 4.0, 4.0],
          "plan_phase_us": [[1.0] * 8] * T, "dedup_phase_us": [[0.5] * 8] * T}
    # 10 more launches; table 1's plan CTA averaged 16 us over the window
    p1 = {"launches": [20, 20], "plan_us": [5.0, 11.0, 7.0], "dedup_us": [4.0, 4.0, 6.0],
          "plan_phase_us": [[1.0] * 8] * T, "dedup_phase_us": [[0.5] * 8] * T,
          "per_launch": {"span_us": [10.0, 20.0, 30.0], "plan_cta_max_us": [9.0, 19.0, 29.0],
                         "dedup_cta_max_us": [8.0, 8.0, 8.0]}}
    r = bench._plan_roles(p0, p1)
    assert r["plan"]["argmax_table"] == 1
    assert r["plan"]["max_table_us"] == pytest.approx(16.0)
    assert r["dedup"]["max_table_us"] == pytest.approx(8.0)
    assert len(r["plan"]["phases_us_of_argmax"]) == 6 and len(r["dedup"]["phases_us_of_argmax"]) == 5
    pl = r["per_launch_p50_p90_p99_us"]
    assert pl["launches"] == 3 and pl["kernel_span"][0] == pytest.approx(20.0)
