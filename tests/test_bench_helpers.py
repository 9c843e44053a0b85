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


def test_union_of_stage_intervals(bench):
    # overlapping intervals count once; disjoint ones add
    assert bench._union_us([(0.0, 0.010), (0.005, 0.020), (0.030, 0.040)]) == pytest.approx(30.0)
    assert bench._union_us([]) == 0.0


def test_stream_busy_and_overlap_verdict(bench):
    import numpy as np
    ev = np.full((16, 8), np.nan)
    # 4 steps of 100 us: plan 0-30, compute 40-100 (fwd 40-60, surr 60-70, bwd 70-100),
    # transfers of 50 us each (disjoint here: the union is their sum)
    for r in range(4):
        t0 = r * 0.1
        ev[r, :6] = [t0, t0 + 0.03, t0 + 0.04, t0 + 0.06, t0 + 0.07, t0 + 0.1]
        ev[r, 6:8] = [t0 + 0.02, t0 + 0.07]
    busy = bench._stream_busy(ev)
    assert busy["plan"] == pytest.approx(30.0) and busy["compute"] == pytest.approx(60.0)
    assert busy["transfer"] == pytest.approx(50.0) and busy["steps"] == 4
    assert busy["step_us"] == pytest.approx(100.0)
    # the verdict compares against the timing pass's own step (100 us here),
    # not the timed region's (62 us)
    ov = bench._overlap({}, 62.0, busy)
    assert ov["busiest_stream"] == "compute" and ov["full_overlap"] is False
    assert ov["timing_pass_step_us"] == pytest.approx(100.0)
    assert ov["step_over_busiest"] == pytest.approx(100.0 / 60.0, rel=1e-3)
    # stages packed back to back: step 62 us, compute busy 60 us -> full overlap
    ev2 = np.full((16, 8), np.nan)
    for r in range(4):
        t0 = r * 0.062
        ev2[r, :6] = [t0, t0 + 0.03, t0 + 0.002, t0 + 0.02, t0 + 0.03, t0 + 0.062]
        ev2[r, 6:8] = [t0, t0 + 0.05]
    ov2 = bench._overlap({}, 62.0, bench._stream_busy(ev2))
    assert ov2["full_overlap"] is True and ov2["busiest_over_step"] <= 1.0
    assert bench._overlap({}, 62.0, None) is None


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


def test_span_summary_durations_busy_and_step(bench):
    import numpy as np
    sp = np.full((5, 16, 2), np.nan)
    # 4 steps of 50 us: plan 0-20, transfer 10-60 (overlapping the next step's),
    # fwd 20-30, surrogate 30-35, backward 35-50
    for r in range(4):
        t0 = r * 0.05
        sp[0, r] = [t0, t0 + 0.02]
        sp[1, r] = [t0 + 0.01, t0 + 0.06]
        sp[2, r] = [t0 + 0.02, t0 + 0.03]
        sp[3, r] = [t0 + 0.03, t0 + 0.035]
        sp[4, r] = [t0 + 0.035, t0 + 0.05]
    s = bench._span_summary(sp)
    assert s["duration_us"]["backward"] == pytest.approx(15.0)
    assert s["duration_us"]["transfer"] == pytest.approx(50.0)
    assert s["step_us"] == pytest.approx(50.0)
    assert s["stream_busy_us_per_step"]["compute"] == pytest.approx(30.0)
    # transfers back to back (each 50 us, one per step): busy the whole step
    assert s["stream_busy_us_per_step"]["transfer"] == pytest.approx(50.0)
