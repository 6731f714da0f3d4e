"""One process per GPU through the real engine: two processes (gloo
rendezvous on 127.0.0.1) co-execute one Mandelbrot image with a shared
HGuided schedule, each on its own CUDA device context.  On a one-GPU box both
logical devices map to cuda:0 — independent kernels in two processes, nothing
waits on the other GPU-side."""
import json
import os
import socket
import uuid

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def worker(rank, world, port, name, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1805_02755_b200 as P
    from paper_1805_02755_b200 import workloads as W
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ng = P.gpu_count()
        devs = [P.cuda_device(f"gpu{i}", ordinal=i % ng) for i in range(world)]
        prog = P.validate_program(W.mandelbrot_spec(512, 384, 400))
        shared = {"name": name, "rank": rank, "world": world, "local_devices": [rank]}
        if rank != 0:
            dist.barrier()
        eng = P.Engine(P.EngineConfig(devs, P.HGuidedConfig(), shared=shared, tally=True), prog)
        if rank == 0:
            dist.barrier()
        traces, outs = [], []
        for _ in range(2):
            out = eng.allocate_outputs()
            t = eng.run_into([], out)
            traces.append(t.raw)
            outs.append(out[0].view(np.uint32).copy())
        eng.close()
        q.put((rank, traces, outs))
    finally:
        dist.destroy_process_group()


def test_two_processes_share_one_schedule(gpu_available, oracle):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = "/ecl_gpu_" + uuid.uuid4().hex[:12]
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, traces, outs = q.get(timeout=300)
        res[r] = (traces, outs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    exp = np.repeat(oracle.mandelbrot(512, 384, 400), 4)
    import paper_1805_02755_b200 as P
    for run in range(2):
        t0, t1 = res[0][0][run], res[1][0][run]
        assert t0["packages"] == t1["packages"], "both ranks assemble the same trace"
        pk = [P.Package(p["seq"], p["device_index"], p["device_id"], p["offset_wg"], p["size_wg"])
              for p in t0["packages"]]
        assert P.tiles_exactly(pk, 512 * 384 // 256)
        assert {p.device_index for p in pk} == {0, 1}, "both processes executed packages"
        merged = np.zeros_like(exp)
        for p in pk:
            lo, hi = p.offset_wg * 256 * 4, (p.offset_wg + p.size_wg) * 256 * 4
            merged[lo:hi] = res[p.device_index][1][run][lo:hi]
        assert np.array_equal(merged, exp)


def nbody_worker(rank, world, port, name, steps, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1805_02755_b200 as P
    from paper_1805_02755_b200 import workloads as W
    from tests._oracle import Oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ng = P.gpu_count()
        n = 3072
        pos, vel = Oracle().nbody_init(21, n)
        devs = [P.cuda_device(f"gpu{i}", ordinal=i % ng) for i in range(world)]
        prog = P.validate_program(W.nbody_spec(n))
        shared = {"name": name, "rank": rank, "world": world, "local_devices": [rank]}
        if rank != 0:
            dist.barrier()
        eng = P.Engine(P.EngineConfig(devs, P.DynamicConfig(5), shared=shared), prog)
        if rank == 0:
            dist.barrier()
        out = [np.zeros((n, 4), np.float32), np.zeros((n, 4), np.float32)]
        t = eng.run_steps([pos, vel], out, steps, [(0, 0), (1, 1)])
        eng.close()
        q.put((rank, t.raw, out[0], out[1]))
    finally:
        dist.destroy_process_group()


def test_two_processes_iterate_nbody_with_ipc_exchange(gpu_available, oracle):
    """Iterative program across processes: after every step each process
    pulls the position/velocity slices its peer owns through CUDA IPC
    (engine.cpp PeerBuffers) before swapping state — the multi-process form
    of the per-step allgatherv.  The merged result matches the oracle's
    multi-step integration."""
    world, steps, n = 2, 4, 3072
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = "/ecl_nb_" + uuid.uuid4().hex[:12]
    port = free_port()
    procs = [ctx.Process(target=nbody_worker, args=(r, world, port, name, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, raw, npos, nvel = q.get(timeout=300)
        res[r] = (raw, npos, nvel)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    raw = res[0][0]
    assert raw["packages"] == res[1][0]["packages"], "both ranks assemble the same trace"
    assert {p["device_index"] for p in raw["packages"]} == {0, 1}, "both processes executed packages"
    # final state: each rank wrote the slices of its own last-step packages
    npos, nvel = np.zeros((n, 4), np.float32), np.zeros((n, 4), np.float32)
    for r in (0, 1):
        mask = np.any(res[r][1] != 0, axis=1)
        npos[mask] = res[r][1][mask]
        nvel[mask] = res[r][2][mask]
    ep, ev = oracle.nbody_init(21, n)
    for _ in range(steps):
        ep, ev = oracle.nbody_step(ep, ev, 0.005, 500.0)
    assert np.all(np.abs(npos - ep) <= 1e-4 * np.abs(ep) + 1e-6)
    scale = float(np.abs(ev[:, :3]).max())
    assert float(np.abs(nvel[:, :3] - ev[:, :3]).max()) <= 2e-4 * scale
