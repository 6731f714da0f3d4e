"""One process per GPU: the shared-memory decision log (coexec/shared.hpp)
driven by several real processes (torch.distributed gloo on 127.0.0.1 for
the rendezvous, world size 2 and 3, CPU only).

Each rank drains the shared scheduler for its own device index; the ranks'
packages together must tile the index space exactly once, match the order a
single coordinator would grant (the log replay keeps every rank's scheduler
instance in lockstep), and survive the measured-throughput feedback of
adaptive HGuided.
"""
import ctypes
import json
import os
import socket
import uuid

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1805_02755_b200 as P
from paper_1805_02755_b200 import _native as N

N.lib.ecl_shared_open.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
N.lib.ecl_shared_open.restype = ctypes.c_int
N.lib.ecl_shared_close.argtypes = [ctypes.c_void_p]
N.lib.ecl_shared_begin.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)]
N.lib.ecl_shared_next.argtypes = [ctypes.c_void_p, ctypes.c_uint32] + [ctypes.POINTER(ctypes.c_uint64)] * 3
N.lib.ecl_shared_observe.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double]
N.lib.ecl_shared_complete.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64,
                                      ctypes.c_uint64, ctypes.c_double, ctypes.c_double]
N.lib.ecl_shared_fail.argtypes = [ctypes.c_void_p]
N.lib.ecl_shared_end.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64), ctypes.c_uint64,
                                 ctypes.POINTER(ctypes.c_int)]
N.lib.ecl_shared_end.restype = ctypes.c_int64


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def worker(rank, world, port, name, doc, runs, fail_rank, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = dict(doc, name=name, rank=rank, world=world, local_devices=[rank])
        h = ctypes.c_void_p()
        if rank == 0:
            rc = N.lib.ecl_shared_open(json.dumps(cfg).encode(), ctypes.byref(h))
            dist.barrier()
        else:
            dist.barrier()  # rank 0 created the segment
            rc = N.lib.ecl_shared_open(json.dumps(cfg).encode(), ctypes.byref(h))
        assert rc == 0, N.last_error()
        results = []
        for run in range(runs):
            ep = ctypes.c_double()
            assert N.lib.ecl_shared_begin(h, ctypes.byref(ep)) == 0, N.last_error()
            off, size, seq = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
            mine = 0
            while True:
                if run == 1 and rank == fail_rank and mine == 2:
                    N.lib.ecl_shared_fail(h)  # fault injection: this rank's device faults
                    break
                g = N.lib.ecl_shared_next(h, rank, ctypes.byref(off), ctypes.byref(size), ctypes.byref(seq))
                assert g >= 0, N.last_error()
                if g == 0:
                    break
                mine += 1
                # pretend the device ran it: faster ranks report higher throughput
                N.lib.ecl_shared_observe(h, rank, size.value * 64, size.value / (1.0 + rank))
                N.lib.ecl_shared_complete(h, seq.value, rank, off.value, size.value, 0.0, 1.0)
            cap = 4 * 100000
            buf = (ctypes.c_uint64 * cap)()
            failed = ctypes.c_int()
            n = N.lib.ecl_shared_end(h, buf, cap, ctypes.byref(failed))
            assert n >= 0, N.last_error()
            quads = [tuple(buf[4 * i:4 * i + 4]) for i in range(n)]
            results.append({"packages": quads, "mine": mine, "peer_failed": failed.value})
        N.lib.ecl_shared_close(h)
        q.put((rank, results))
    finally:
        dist.destroy_process_group()


def run_world(world, doc, runs=2, fail_rank=-1):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = "/ecl_test_" + uuid.uuid4().hex[:12]
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, name, doc, runs, fail_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def devices(world, powers=None):
    return [P.simulated_device(f"gpu{i}", powers[i] if powers else 1.0).to_json() for i in range(world)]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("sched", [{"type": "hguided", "k": 2.0}, {"type": "dynamic", "num_packages": 37},
                                   {"type": "static"},
                                   {"type": "hguided", "k": 2.0, "adaptive": True, "ema_alpha": 0.5}],
                         ids=["hguided", "dynamic", "static", "hguided-adaptive"])
def test_ranks_tile_exactly_once(world, sched):
    total = 20000
    doc = {"scheduler": sched, "devices": devices(world), "total_work_groups": total}
    out = run_world(world, doc)
    for run in range(2):
        views = [out[r][run]["packages"] for r in range(world)]
        assert all(v == views[0] for v in views), "every rank assembles the same run"
        pk = views[0]
        assert [p[0] for p in pk] == list(range(len(pk))), "seqs are dense"
        assert P.tiles_exactly([P.Package(s, d, f"gpu{d}", o, z) for s, d, o, z in pk], total)
        assert sum(out[r][run]["mine"] for r in range(world)) == len(pk)
        for r in range(world):
            assert sum(1 for p in pk if p[1] == r) == out[r][run]["mine"]


def test_grants_follow_the_single_coordinator_schedule():
    # Replaying the log keeps every rank's scheduler in lockstep: the package
    # sizes granted in seq order equal what one scheduler hands out to the
    # same sequence of requesting devices.
    world, total = 3, 12000
    sched = {"type": "hguided", "k": 2.0}
    doc = {"scheduler": sched, "devices": devices(world, [1.0, 2.0, 4.0]), "total_work_groups": total}
    pk = run_world(world, doc, runs=1)[0][0]["packages"]
    s = P.Scheduler(P.HGuidedConfig(2.0), total, [P.simulated_device(f"gpu{i}", p) for i, p in
                                                  enumerate([1.0, 2.0, 4.0])])
    for seq, dev, off, size in pk:
        r = s.next(dev)
        assert (r.offset_wg, r.size_wg) == (off, size)
    assert s.remaining_work_groups() == 0


def test_peer_failure_stops_every_rank():
    world = 2
    doc = {"scheduler": {"type": "dynamic", "num_packages": 400}, "devices": devices(world),
           "total_work_groups": 40000}
    out = run_world(world, doc, runs=2, fail_rank=1)
    assert out[0][1]["peer_failed"] == 1 and out[1][1]["peer_failed"] == 1
    assert out[0][0]["peer_failed"] == 0  # the clean run before the fault
