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
