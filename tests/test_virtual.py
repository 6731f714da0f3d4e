"""Virtual-clock engine vs the reference's own traces.

tests/golden/virtual_traces.json holds traces the reference engine produced
(drive_virtual, engine.hpp:306-338) for experiments/mandelbrot-{batel,remo}
(made by tests/golden/make_golden.py from oracle/_ref).  Our engine replays
the same schedulers with per-item costs = the oracle's Mandelbrot counts
(the reference cost model, workloads.hpp:243-246) and must produce the
identical trace: same packages, same virtual timestamps, same totals.
"""
import json
import os

import numpy as np
import pytest

import paper_1805_02755_b200 as P
from paper_1805_02755_b200 import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
REF_OUT = "/root/reference/proj/out/mandelbrot-batel"


def load():
    with open(os.path.join(GOLDEN, "virtual_traces.json")) as f:
        return json.load(f)


def engine_for(cfg):
    devs = [P.DeviceProfile.from_json(d) for d in cfg["devices"]]
    P.apply_default_min_package(devs)
    s = cfg["scheduler"]
    if s["type"] == "static":
        sched = P.StaticConfig(s.get("proportions", []), s.get("device_order", []))
    elif s["type"] == "dynamic":
        sched = P.DynamicConfig(s["num_packages"])
    else:
        sched = P.HGuidedConfig(s.get("k", 2.0))
    pj = cfg["program"]
    args = pj["args"]
    prog = P.validate_program(W.mandelbrot_spec(args[0], args[1], args[2], lws=pj["local_work_size"],
                                                viewport=tuple(args[3:7])))
    return P.Engine(P.EngineConfig(devs, sched, P.ClockMode.Virtual, cfg["seed"]), prog), args


@pytest.mark.parametrize("key", sorted(load().keys()))
def test_virtual_trace_matches_reference(key, oracle):
    g = load()[key]
    eng, args = engine_for(g["config"])
    costs = oracle.mandelbrot(args[0], args[1], args[2], tuple(args[3:7])).astype(np.float64)
    t = eng.run_virtual(costs)
    assert t.raw == g["trace"]


def test_batel_traces_equal_committed_reference_outputs(oracle):
    """The reference repo's own proj/out traces (present in this container)."""
    if not os.path.isdir(REF_OUT):
        pytest.skip("reference tree absent")
    for i, name in enumerate(["s0-static", "s1-static", "s2-dynamic", "s3-dynamic", "s4-hguided"]):
        with open(os.path.join(REF_OUT, f"{name}-rep0.trace.json")) as f:
            ref_trace = json.load(f)
        g = load()[f"mandelbrot-batel/s{i}"]
        mine = dict(g["trace"])
        # load_experiment resolves static proportions before the run (config.hpp:192)
        assert {k: v for k, v in mine.items() if k != "scheduler"} == \
               {k: v for k, v in ref_trace.items() if k != "scheduler"}


def test_virtual_analytic_costs_vecscale_and_synthetic():
    devs = [P.simulated_device("a", 64.0, 0.25), P.simulated_device("b", 16.0, 0.5)]
    prog = P.validate_program(W.synthetic_spec(4000, 10))
    e = P.Engine(P.EngineConfig(devs, P.DynamicConfig(4), P.ClockMode.Virtual), prog)
    t = e.run_virtual(None)
    assert P.tiles_exactly(t.packages, 400)


def test_virtual_tie_break_lower_device_first():
    # test_engine.cpp:155-167
    devs = [P.simulated_device("d0", 10.0, 0.0, 1e30), P.simulated_device("d1", 10.0, 0.0, 1e30)]
    prog = P.validate_program(W.synthetic_spec(4000, 10))
    t = P.Engine(P.EngineConfig(devs, P.DynamicConfig(4), P.ClockMode.Virtual), prog).run_virtual(None)
    assert [p.device_id for p in t.packages] == ["d0", "d1", "d0", "d1"]


def test_virtual_overhead_plus_compute():
    # test_engine.cpp:82-92: 1 ms overhead + 100 items / 50 per ms = 3.0
    devs = [P.simulated_device("d", 50.0, 1.0, 1e30)]
    prog = P.validate_program(W.synthetic_spec(100, 10))
    t = P.Engine(P.EngineConfig(devs, P.StaticConfig(), P.ClockMode.Virtual), prog).run_virtual(None)
    assert t.t_total_ms == 3.0


def test_virtual_static_balances_regular_kernel():
    devs = [P.simulated_device("s", 1.0, 0.0, 1e18), P.simulated_device("m", 2.0, 0.0, 1e18),
            P.simulated_device("f", 5.0, 0.0, 1e18)]
    prog = P.validate_program(W.synthetic_spec(8000, 10))
    t = P.Engine(P.EngineConfig(devs, P.StaticConfig(), P.ClockMode.Virtual), prog).run_virtual(None)
    assert len(t.packages) == 3 and P.balance(t) >= 0.999


def test_virtual_requires_simulated_devices():
    prog = P.validate_program(W.synthetic_spec(100, 10))
    with pytest.raises(P.Error) as e:
        P.Engine(P.EngineConfig([P.cuda_device("g")], P.StaticConfig(), P.ClockMode.Virtual), prog)
    assert e.value.code == P.ErrorCode.ConfigError


def test_virtual_mandelbrot_needs_costs():
    devs = [P.simulated_device("a", 1.0)]
    prog = P.validate_program(W.mandelbrot_spec(16, 16, 8, lws=16))
    e = P.Engine(P.EngineConfig(devs, P.StaticConfig(), P.ClockMode.Virtual), prog)
    with pytest.raises(P.Error) as ei:
        e.run_virtual(None)
    assert ei.value.code == P.ErrorCode.BadKernelArgs


def test_virtual_runs_are_deterministic(oracle):
    devs = [P.simulated_device("a", 64.0, 0.25), P.simulated_device("b", 16.0, 0.5)]
    prog = P.validate_program(W.mandelbrot_spec(64, 64, 100, lws=64))
    costs = oracle.mandelbrot(64, 64, 100).astype(np.float64)
    e = P.Engine(P.EngineConfig(devs, P.HGuidedConfig(), P.ClockMode.Virtual, 5), prog)
    assert e.run_virtual(costs).raw == e.run_virtual(costs).raw


def test_virtual_adaptive_hguided_recovers_from_wrong_seeds():
    """Seeds claim four equal devices; one is 8x faster and every package
    costs 0.5 ms of launch overhead.  HGuided balances either way (it is
    self-scheduling), but measured-throughput HGuided sizes packages from the
    learned rates: fewer packages, less overhead, closer to the ideal."""
    devs = [P.simulated_device("fast", 8.0, 0.5, 1e30)] + \
        [P.simulated_device(f"slow{i}", 1.0, 0.5, 1e30) for i in range(3)]
    prog = P.validate_program(W.synthetic_spec(400000, 100))
    t = {}
    for adaptive in (False, True):
        cfg = P.HGuidedConfig(2.0, [1.0] * 4, adaptive=adaptive, ema_alpha=0.5)
        t[adaptive] = P.Engine(P.EngineConfig(devs, cfg, P.ClockMode.Virtual), prog).run_virtual(None)
        assert P.tiles_exactly(t[adaptive].packages, prog.total_work_groups())
    assert t[True].t_total_ms < t[False].t_total_ms
    assert len(t[True].packages) < len(t[False].packages)
    assert t[True].t_total_ms < 1.002 * 400000 / 11.0  # ideal: 11 work-items/ms in total
