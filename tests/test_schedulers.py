"""Scheduler parity: the reference's golden cases (test_schedulers.cpp) and a
differential check against package sequences the reference itself produced
(tests/golden/scheduler_drains.json, made by tests/golden/make_golden.py
from oracle/_ref)."""
import json
import os

import pytest

import paper_1805_02755_b200 as P

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def devs(*powers):
    return [P.simulated_device(f"d{i}", p) for i, p in enumerate(powers)]


def drain(s, n):
    """Coordinator emulator of test_schedulers.cpp:27-49."""
    out, granted = [], True
    while granted:
        granted = False
        for d in range(n):
            r = s.next(d)
            if r is not None:
                out.append((d, r.offset_wg, r.size_wg))
                granted = True
    return out


def sizes(pk):
    return [p[2] for p in pk]


def tiles(pk, total):
    return P.tiles_exactly([P.Package(i, d, f"d{d}", o, s) for i, (d, o, s) in enumerate(pk)], total)


# ---- Static (test_schedulers.cpp:53-128) ------------------------------------

def test_static_exact_proportions():
    d = devs(1, 1)
    pk = P.static_partition(1000, P.resolve_static(P.StaticConfig([0.25, 0.75]), d), d)
    assert [p.size_wg for p in pk] == [250, 750] and pk[1].offset_wg == 250


def test_static_three_proportions():
    d = devs(1, 1, 1)
    pk = P.static_partition(1000, P.resolve_static(P.StaticConfig([0.08, 0.30, 0.62]), d), d)
    assert [p.size_wg for p in pk] == [80, 300, 620]


def test_static_remainder_to_last():
    d = devs(1, 1, 1)
    pk = P.static_partition(10, P.resolve_static(P.StaticConfig([1 / 3, 1 / 3, 1 / 3]), d), d)
    assert [p.size_wg for p in pk] == [3, 3, 4]


def test_static_n_minus_one_rule():
    r = P.resolve_static(P.StaticConfig([0.08, 0.3]), devs(1, 1, 1))
    assert len(r.proportions) == 3 and abs(r.proportions[2] - 0.62) < 1e-12


def test_static_normalized():
    assert P.resolve_static(P.StaticConfig([2.0, 2.0]), devs(1, 1)).proportions == [0.5, 0.5]


def test_static_power_shares():
    r = P.resolve_static(P.StaticConfig(), devs(6, 2))
    assert abs(r.proportions[0] - 0.75) < 1e-12 and abs(r.proportions[1] - 0.25) < 1e-12


def test_static_delivery_order():
    d = devs(1, 1, 1)
    fwd = P.static_partition(100, P.resolve_static(P.StaticConfig([0.2, 0.3, 0.5], ["d0", "d1", "d2"]), d), d)
    rev = P.static_partition(100, P.resolve_static(P.StaticConfig([0.2, 0.3, 0.5], ["d2", "d1", "d0"]), d), d)
    assert fwd[0].device_id == "d0" and rev[0].device_id == "d2"
    assert [p.size_wg for p in fwd] == [p.size_wg for p in rev] and fwd[0].size_wg == 20
    assert rev[0].offset_wg == 0
    assert P.tiles_exactly(fwd, 100) and P.tiles_exactly(rev, 100)


def test_static_needs_one_wg_per_device():
    with pytest.raises(P.Error) as e:
        P.Scheduler(P.StaticConfig(), 2, devs(1, 1, 1))
    assert e.value.code == P.ErrorCode.TooFewWorkGroups


def test_static_rejects_bad_order():
    for order in (["d0", "d0"], ["d0", "nope"]):
        with pytest.raises(P.Error) as e:
            P.resolve_static(P.StaticConfig([0.5, 0.5], order), devs(1, 1))
        assert e.value.code == P.ErrorCode.BadSchedulerConfig


# ---- Dynamic (test_schedulers.cpp:130-184) ----------------------------------

def test_dynamic_equal_packages():
    pk = drain(P.Scheduler(P.DynamicConfig(50), 1000, devs(1, 1)), 2)
    assert len(pk) == 50 and set(sizes(pk)) == {20} and tiles(pk, 1000)


def test_dynamic_short_final_package():
    pk = drain(P.Scheduler(P.DynamicConfig(150), 1000, devs(1, 1)), 2)
    assert len(pk) == 143 and set(sizes(pk)[:-1]) == {7} and pk[-1][2] == 6 and tiles(pk, 1000)


def test_dynamic_clamps_to_one():
    pk = drain(P.Scheduler(P.DynamicConfig(50), 20, devs(1)), 1)
    assert len(pk) == 20 and set(sizes(pk)) == {1}


def test_dynamic_needs_package_per_device():
    with pytest.raises(P.Error) as e:
        P.Scheduler(P.DynamicConfig(2), 1000, devs(1, 1, 1))
    assert e.value.code == P.ErrorCode.BadSchedulerConfig


# ---- HGuided (test_schedulers.cpp:186-289) ----------------------------------

def test_hguided_equation_187():
    d = devs(3, 1)
    for x in d:
        x.min_package_work_groups = 16
    s = P.Scheduler(P.HGuidedConfig(2.0), 1000, d)
    assert s.unclamped_size(1000, 0) == 187
    assert s.next(0).size_wg == 187 and s.remaining_work_groups() == 813


def test_hguided_upper_clamp():
    d = devs(3, 1)
    d[0].min_package_work_groups = 16
    s = P.Scheduler(P.HGuidedConfig(2.0), 10, d)
    assert s.next(0).size_wg == 10 and s.remaining_work_groups() == 0


def test_hguided_exhaustion():
    assert P.Scheduler(P.HGuidedConfig(2.0), 0, devs(3, 1)).next(0) is None


def test_hguided_lower_clamp():
    d = devs(3, 1)
    d[0].min_package_work_groups = 50
    s = P.Scheduler(P.HGuidedConfig(16.0), 1000, d)
    assert s.unclamped_size(1000, 0) == 23 and s.next(0).size_wg == 50


def test_hguided_powers_override():
    assert P.Scheduler(P.HGuidedConfig(2.0, [3.0, 1.0]), 1000, devs(1, 1)).unclamped_size(1000, 0) == 187


def test_hguided_no_n_toggle():
    d = devs(3, 1)
    assert P.Scheduler(P.HGuidedConfig(2.0), 1000, d).unclamped_size(1000, 0) == 187
    assert P.Scheduler(P.HGuidedConfig(2.0, [], False), 1000, d).unclamped_size(1000, 0) == 375


def test_hguided_first_package_grows_as_k_shrinks():
    firsts = [P.Scheduler(P.HGuidedConfig(k), 4096, devs(8, 3, 1)).next(0).size_wg for k in (1.0, 2.0, 4.0)]
    assert firsts[0] > firsts[1] > firsts[2]


def test_hguided_rejects_bad_parameters():
    for cfg in (P.HGuidedConfig(0.0), P.HGuidedConfig(2.0, [1.0]), P.HGuidedConfig(2.0, [1.0, -1.0])):
        with pytest.raises(P.Error):
            P.Scheduler(cfg, 10, devs(3, 1))


def test_hguided_unclamped_never_increases():
    import random
    rng = random.Random(31)
    for _ in range(30):
        d = devs(*[1 + rng.random() * 7 for _ in range(3)])
        s = P.Scheduler(P.HGuidedConfig(0.5 + rng.random() * 4), 500 + rng.randrange(5000), d)
        last = [1 << 63] * 3
        granted = True
        while granted:
            granted = False
            for i in range(3):
                raw = s.unclamped_size(s.remaining_work_groups(), i)
                if s.next(i) is not None:
                    assert raw <= last[i]
                    last[i] = raw
                    granted = True


def test_hguided_adaptive_follows_measured_rate():
    d = devs(1, 1)
    s = P.Scheduler(P.HGuidedConfig(2.0, adaptive=True, ema_alpha=1.0), 100000, d)
    first = s.unclamped_size(100000, 0)
    s.observe(0, 3000, 1.0)  # device 0 measured 3000 items/ms
    s.observe(1, 1000, 1.0)  # device 1 measured 1000 items/ms
    assert s.unclamped_size(100000, 0) == 100000 * 3000 // (2 * 4000 * 2)
    assert s.unclamped_size(100000, 0) > first > s.unclamped_size(100000, 1)


def test_every_scheduler_tiles_exactly():
    import random
    rng = random.Random(43)
    for _ in range(40):
        n = 1 + rng.randrange(4)
        d = devs(*[1 + rng.random() * 9 for _ in range(n)])
        total = n + rng.randrange(4000)
        for cfg in (P.StaticConfig(), P.DynamicConfig(n + rng.randrange(64)), P.HGuidedConfig(0.5 + rng.random() * 4)):
            s = P.Scheduler(cfg, total, d)
            pk = drain(s, n)
            assert tiles(pk, total) and all(x[2] > 0 for x in pk) and s.remaining_work_groups() == 0


def test_descriptions():
    assert P.describe(P.DynamicConfig(150)) == "dynamic(packages=150)"
    assert P.describe(P.HGuidedConfig()) == "hguided(k=2)"
    assert P.describe(P.HGuidedConfig(2.0, [], False)) == "hguided(k=2;no-n)"
    assert P.describe(P.StaticConfig([0.25, 0.75], ["a", "b"])) == "static(props=0.25,0.75;order=a,b)"
    assert P.describe(P.StaticConfig()) == "static(props=power)"


def test_default_min_package_heuristic():
    d = [P.simulated_device("gpu", 8), P.simulated_device("phi", 3), P.simulated_device("cpu", 1)]
    for x in d:
        x.min_package_work_groups = 0
    d[1].min_package_work_groups = 7
    P.apply_default_min_package(d)
    assert [x.min_package_work_groups for x in d] == [8, 7, 1]


# ---- differential against the reference's own drains ------------------------

def _golden_drains():
    with open(os.path.join(GOLDEN, "scheduler_drains.json")) as f:
        return json.load(f)


def _cfg(j):
    t = j["type"]
    if t == "static":
        return P.StaticConfig(j.get("proportions", []), j.get("device_order", []))
    if t == "dynamic":
        return P.DynamicConfig(j["num_packages"])
    return P.HGuidedConfig(j.get("k", 2.0), j.get("powers", []), j.get("include_device_count", True))


@pytest.mark.parametrize("case", range(122))
def test_drain_matches_reference(case):
    c = _golden_drains()[case]
    d = [P.DeviceProfile.from_json(x) for x in c["devices"]]
    s = P.Scheduler(_cfg(c["scheduler"]), c["total_work_groups"], d)
    got = drain(s, len(d))
    assert [list(x) for x in got] == c["packages"]


def test_paper_scale_hguided_package_counts():
    # 8 equal GPUs, 1,048,576 WGs, k=2: first package 8192,
    # 1350 packages with min 1 and 375 with min 1184.
    cases = _golden_drains()[-2:]
    assert [len(c["packages"]) for c in cases] == [1350, 375]
    assert cases[0]["packages"][0][2] == 8192


def test_drains_against_live_reference(ref):
    import random
    rng = random.Random(5)
    for _ in range(20):
        n = 1 + rng.randrange(6)
        d = [P.simulated_device(f"d{i}", 1 + rng.random() * 5, min_wg=1 + rng.randrange(4)) for i in range(n)]
        total = n + rng.randrange(30000)
        for cfg in (P.StaticConfig(), P.DynamicConfig(n + rng.randrange(500)), P.HGuidedConfig(0.5 + rng.random() * 3)):
            exp = ref.drain(cfg.to_json(), [x.to_json() for x in d], total)
            assert drain(P.Scheduler(cfg, total, d), n) == exp


def test_hguided_adaptive_first_report_keeps_units_consistent():
    """Seeds are relative (computing_power = 1.0) and a report is in
    work-items/ms (~7e6 for a B200 on Mandelbrot): until every device has
    reported, the unmeasured devices' seeds are scaled by the measured
    rate/seed ratio, so one early report cannot take ~all of sum(P)."""
    n, total = 8, 1 << 20
    s = P.Scheduler(P.HGuidedConfig(2.0, adaptive=True, ema_alpha=0.5), total, devs(*[1.0] * n))
    before = [s.unclamped_size(total, i) for i in range(n)]
    s.observe(0, 1_000_000, 0.14)  # ~7.1e6 items/ms
    after = [s.unclamped_size(total, i) for i in range(n)]
    assert after == before  # equal devices, equal shares, whatever the unit
    s.observe(1, 1_000_000, 0.28)  # device 1 measured at half the rate
    sizes = [s.unclamped_size(total, i) for i in range(n)]
    assert sizes[0] == pytest.approx(2 * sizes[1], rel=1e-6)
    # devices 2..7 are seeded at the measured mean rate/seed
    assert all(x == sizes[2] for x in sizes[2:]) and sizes[1] < sizes[2] < sizes[0]


def test_hguided_adaptive_seed_powers_in_rates_are_unchanged_by_scaling():
    # seeds already in items/ms (e.g. learned by a previous run): scaling by
    # the measured rate/seed ratio leaves them as they are
    d = devs(4000.0, 2000.0)
    s = P.Scheduler(P.HGuidedConfig(2.0, adaptive=True, ema_alpha=1.0), 100000, d)
    s.observe(0, 4000, 1.0)
    assert s.unclamped_size(100000, 1) == 100000 * 2000 // (2 * 6000 * 2)


def test_hguided_adaptive_weighs_reports_by_busy_time():
    """The guided tail's tiny packages (busy time mostly launch latency) must
    not outvote the large packages: forgetting is by busy time."""
    s = P.Scheduler(P.HGuidedConfig(2.0, adaptive=True, ema_alpha=0.5), 1 << 20, devs(1.0, 1.0))
    s.observe(0, 1_000_000, 100.0)  # 1e4 items/ms
    s.observe(1, 1_000_000, 100.0)
    for _ in range(20):
        s.observe(0, 256, 0.01)  # 2.56e4 items/ms each, 0.2 ms in total
    a, b = s.unclamped_size(1 << 20, 0), s.unclamped_size(1 << 20, 1)
    assert abs(a / b - 1.0) < 0.01
    # a report as long as the history halves it (alpha 0.5): the rate becomes
    # the busy-weighted mean (50 ms at 1e4, 100 ms at 2e4) = 1.667e4
    s.observe(0, 2_000_000, 100.0)
    assert s.unclamped_size(1 << 20, 0) / s.unclamped_size(1 << 20, 1) == pytest.approx(5 / 3, rel=0.01)
