"""Property-based differential tests (hypothesis) of the scheduler subsystem
against the reference compiled in place (oracle/_ref): random device sets,
powers, minimum packages, totals and scheduler parameters — Static with
proportions and delivery orders, Dynamic, HGuided with and without the
device count and explicit powers (schedulers.hpp:87-315) — must produce the
reference's package sequence exactly, or fail where the reference fails.
Every accepted drain tiles the work-group range exactly (core.hpp:188-198)."""
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import paper_1805_02755_b200 as P
from tests.test_schedulers import drain, tiles

SETTINGS = settings(max_examples=150, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])


@st.composite
def cases(draw):
    n = draw(st.integers(1, 8))
    powers = [draw(st.floats(0.05, 200.0, allow_nan=False)) for _ in range(n)]
    min_wg = [draw(st.integers(1, 64)) for _ in range(n)]
    total = draw(st.integers(1, 250_000))
    kind = draw(st.sampled_from(["static", "dynamic", "hguided"]))
    if kind == "static":
        props = [draw(st.floats(0.01, 10.0, allow_nan=False)) for _ in range(n)] if draw(st.booleans()) else []
        order = draw(st.permutations([f"d{i}" for i in range(n)])) if draw(st.booleans()) else []
        cfg = P.StaticConfig(props, list(order))
    elif kind == "dynamic":
        cfg = P.DynamicConfig(draw(st.integers(1, 4000)))
    else:
        hp = [draw(st.floats(0.05, 50.0, allow_nan=False)) for _ in range(n)] if draw(st.booleans()) else []
        cfg = P.HGuidedConfig(draw(st.floats(0.25, 8.0, allow_nan=False)), hp, draw(st.booleans()))
    devs = [P.simulated_device(f"d{i}", powers[i], min_wg=min_wg[i]) for i in range(n)]
    return cfg, devs, total


@SETTINGS
@given(cases())
def test_scheduler_drains_match_reference(ref, case):
    cfg, devs, total = case
    try:
        exp = ref.drain(cfg.to_json(), [d.to_json() for d in devs], total)
    except RuntimeError:
        with pytest.raises(P.Error):
            drain(P.Scheduler(cfg, total, devs), len(devs))
        return
    got = drain(P.Scheduler(cfg, total, devs), len(devs))
    assert got == exp
    assert tiles(got, total)


@SETTINGS
@given(st.integers(1, 8), st.integers(1, 10_000_000), st.floats(0.25, 8.0, allow_nan=False), st.booleans())
def test_hguided_sizes_never_grow_for_equal_devices(n, total, k, with_n):
    # equal powers, minimum 1: G_r only shrinks, so does floor(G_r P/(k n ΣP))
    devs = [P.simulated_device(f"d{i}", 1.0) for i in range(n)]
    if total < n:
        return
    pk = drain(P.Scheduler(P.HGuidedConfig(k, [], with_n), total, devs), n)
    sizes = [p[2] for p in pk]
    assert all(a >= b for a, b in zip(sizes, sizes[1:]))
    assert tiles(pk, total)


@st.composite
def programs(draw):
    lws = draw(st.integers(1, 512))
    wgs = draw(st.integers(1, 4096))
    gws = lws * wgs + (draw(st.integers(1, lws - 1)) if lws > 1 and draw(st.integers(0, 9)) == 0 else 0)
    oi, wi = draw(st.integers(1, 8)), draw(st.sampled_from([1, 2, 3, 4, lws, 2 * lws]))
    exact = gws * oi // wi if (gws * oi) % wi == 0 else gws
    count = exact if draw(st.integers(0, 9)) else draw(st.integers(1, 2 * gws))
    spec = P.ProgramSpec(gws, lws, [], [P.BufferDesc("out", 4, count)], P.OutPattern(oi, wi), "synthetic", [])
    o = draw(st.integers(0, wgs))
    n = draw(st.integers(0, wgs + 1 - o))
    return spec, o, n


@SETTINGS
@given(programs())
def test_validate_and_out_range_match_reference(ref, case):
    # validate_program (core.hpp:107-143) then out_range_for (core.hpp:172-185):
    # same range, or the same ErrorCode, as the reference on random shapes,
    # out patterns, ragged sizes and packages (including empty and
    # out-of-range ones)
    import ctypes
    import json
    spec, o, n = case
    lib = ref.lib
    lib.ref_out_range.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_uint64,
                                  ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]
    a, b = ctypes.c_uint64(), ctypes.c_uint64()
    rc = lib.ref_out_range(json.dumps(spec.to_json()).encode(), o, n, ctypes.byref(a), ctypes.byref(b))
    assert rc >= 0, ref.lib.ref_last_error()

    def ours():
        return P.out_range_for(P.Package(offset_wg=o, size_wg=n), P.validate_program(spec))

    if rc == 0:
        r = ours()
        assert (r.offset, r.count) == (a.value, b.value)
    else:
        with pytest.raises(P.Error) as e:
            ours()
        assert e.value.code.value == rc - 1


@st.composite
def traces(draw):
    n = draw(st.integers(1, 6))
    ids = [f"dev{i}" for i in range(n)]
    times = st.floats(0.001, 1e5, allow_nan=False)
    packages, off = [], 0
    for seq in range(draw(st.integers(1, 24))):
        d = draw(st.integers(0, n - 1))
        size = draw(st.integers(1, 5000))
        t0 = draw(times)
        t1 = t0 + draw(times)
        packages.append({"seq": seq, "device_index": d, "device_id": ids[d], "offset_wg": off, "size_wg": size,
                         "t_enqueue_ms": t0, "t_start_ms": t0, "t_end_ms": t1})
        off += size
    used = sorted({p["device_index"] for p in packages})
    per_dev = {ids[d]: draw(times) for d in used}
    raw = {"schema": 1, "clock_mode": "wall", "seed": 0, "init_ms": 0.0, "init_in_total": True,
           "scheduler": "dynamic(n=1)", "t_total_ms": max(per_dev.values()) * draw(st.floats(1.0, 1.5)),
           "per_device_time_ms": per_dev, "packages": packages,
           "program": {"global_work_size": off, "local_work_size": 1, "total_work_groups": off, "kernel": "synthetic",
                       "out_pattern": {"out_indices": 1, "work_items": 1}},
           "devices": [{"id": i, "name": i, "computing_power": 1.0, "launch_overhead_ms": 0.0,
                        "bandwidth_bytes_per_ms": 1.0, "min_package_work_groups": 1,
                        "backend": {"kind": "simulated"}} for i in ids]}
    solo = [draw(times) for _ in range(draw(st.integers(1, n)))]
    ref_ms = draw(st.one_of(st.none(), times))
    return raw, solo, ref_ms


@SETTINGS
@given(traces())
def test_metrics_report_matches_reference(ref, case):
    # make_report (metrics.hpp:23-117) on random traces: balance, speedup,
    # s_max, efficiency, overhead and work shares equal the reference's
    import ctypes
    import json
    raw, solo, ref_ms = case
    lib = ref.lib
    lib.ref_report_json.restype = ctypes.c_int64
    lib.ref_report_json.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double), ctypes.c_uint32,
                                    ctypes.c_double, ctypes.c_char_p, ctypes.c_uint64]
    arr = (ctypes.c_double * len(solo))(*solo)
    buf = ctypes.create_string_buffer(1 << 16)
    n = lib.ref_report_json(json.dumps(raw).encode(), arr, len(solo), -1.0 if ref_ms is None else ref_ms, buf,
                            1 << 16)
    if n < 0:
        with pytest.raises(P.Error):
            P.make_report(P.ExecutionTrace(raw), solo, ref_ms)
        return
    exp = json.loads(buf.value.decode())
    got = P.make_report(P.ExecutionTrace(raw), solo, ref_ms)
    assert got.balance == exp["balance"]
    assert got.speedup == exp["speedup"]
    assert got.s_max == exp["s_max"]
    assert got.efficiency == exp["efficiency"]
    assert got.overhead_pct == exp.get("overhead_pct")
    assert got.work_share == exp["work_share"]
