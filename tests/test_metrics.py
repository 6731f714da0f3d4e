"""Metrics (test_metrics.cpp:39-120; acceptance.cpp criterion 7) through the
native make_report."""
import pytest

import paper_1805_02755_b200 as P


def trace_with_spans(spans):
    pk = []
    per = {}
    for i, s in enumerate(spans):
        pk.append({"seq": i, "device_index": i, "device_id": f"dev{i}", "offset_wg": i, "size_wg": 1,
                   "t_enqueue_ms": 0.0, "t_start_ms": 0.0, "t_end_ms": s})
        per[f"dev{i}"] = s
    raw = {"schema": 1, "program": {"kernel": "synthetic:constant", "global_work_size": len(spans),
                                    "local_work_size": 1, "total_work_groups": len(spans),
                                    "out_pattern": {"out_indices": 1, "work_items": 1}},
           "devices": [], "scheduler": "dynamic(packages=1)", "clock_mode": "virtual", "seed": 0, "init_ms": 0.0,
           "init_in_total": True, "packages": pk, "t_total_ms": max(spans), "per_device_time_ms": per}
    return P.ExecutionTrace(raw)


def test_balance_equal_spans():
    assert P.balance(trace_with_spans([7.5, 7.5, 7.5])) == 1.0
    assert P.balance(trace_with_spans([42.0])) == 1.0


def test_balance_first_over_last():
    assert P.balance(trace_with_spans([5.0, 10.0])) == 0.5
    assert P.balance(trace_with_spans([10.0, 5.0])) == 0.5
    assert P.balance(trace_with_spans([2.0, 8.0, 4.0])) == 0.25


def test_balance_requires_packages():
    t = trace_with_spans([1.0])
    t.raw["packages"] = []
    with pytest.raises(P.Error) as e:
        P.make_report(t, [1.0])
    assert e.value.code == P.ErrorCode.EmptyTrace


def test_s_max_and_speedup():
    t = trace_with_spans([6.0, 6.0])
    r = P.make_report(t, [10.0, 30.0, 60.0])
    assert abs(r.s_max - 100.0 / 60.0) < 1e-15
    assert abs(r.speedup - 10.0 / 6.0) < 1e-15
    assert r.efficiency == r.speedup / r.s_max


def test_s_max_rejects_non_positive():
    with pytest.raises(P.Error) as e:
        P.make_report(trace_with_spans([1.0]), [10.0, 0.0])
    assert e.value.code == P.ErrorCode.NonPositiveTime


def test_missing_baseline():
    with pytest.raises(P.Error) as e:
        P.make_report(trace_with_spans([1.0]), [])
    assert e.value.code == P.ErrorCode.MissingBaseline


def test_overhead_formula():
    assert abs(P.overhead_pct(102.8, 100.0) - 2.8) < 1e-12
    assert P.overhead_pct(100.0, 100.0) == 0.0 and P.overhead_pct(99.0, 100.0) == -1.0
    with pytest.raises(P.Error):
        P.overhead_pct(1.0, 0.0)


def test_report_identities():
    t = trace_with_spans([10.5, 11.0])
    r = P.make_report(t, [15.0, 40.0], 14.0)
    assert r.efficiency == r.speedup / r.s_max
    assert abs(sum(r.work_share.values()) - 1.0) < 1e-9
    assert r.overhead_pct == P.overhead_pct(t.t_total_ms, 14.0)
    assert r.notes == []


def test_report_anomaly_note():
    t = trace_with_spans([1.0, 1.0])
    r = P.make_report(t, [10.0, 10.0])  # speedup 10 over s_max 2
    assert r.notes and "anomaly" in r.notes[0]


def test_trace_csv_columns():
    csv = trace_with_spans([1.5, 2.0]).to_csv().splitlines()
    assert csv[0] == "seq,device_id,offset_wg,size_wg,t_enqueue_ms,t_start_ms,t_end_ms"
    assert csv[1] == "0,dev0,0,1,0,0,1.5"
