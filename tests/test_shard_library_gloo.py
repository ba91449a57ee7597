"""Two processes drive the time-sharded protocol through the library (map_shard_phase,
include/pmap.h) on one GPU, with the chunk payloads exchanged by gloo all-gathers over
host copies (D2H -> gloo -> H2D): the multi-process counterpart of test_virtual_time_shards.
Each rank's kernels complete on their own (the exchange is host-driven), so no kernel of
one process waits on another's.  The concatenated trajectory must match the CPU oracle."""
import os
import socket

import numpy as np
import pytest

import oracle
import workloads as wl

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spec():
    spec = wl.wiener_velocity()
    spec.c = np.array([0.3, -0.2, 0.1, 0.05])
    spec.r = np.array([0.5, -0.25])
    return spec


def _worker(rank, world, port, T, out):
    import sys
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2512_13319_b200 as pm
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    spec = _spec()
    _, y = wl.simulate_linear(spec, T, seed=23)
    a, b = pm.shard_range(rank, world, T)
    plan = pm.Plan(T=T, t0=spec.t0, tf=spec.tf, F=spec.F, c=spec.c, L=spec.L, W=spec.W, H=spec.H, r=spec.r,
                   R=spec.R, m0=spec.m0, P0=spec.P0, rank=rank, world=world)
    yd = torch.tensor(np.ascontiguousarray(y[None, a:b]), device="cuda")

    def gather(payload):  # device payload -> host -> gloo all-gather -> device, rank order
        h = payload.cpu()
        parts = [torch.zeros_like(h) for _ in range(world)]
        dist.all_gather(parts, h)
        return torch.cat(parts).cuda()

    g1 = gather(plan.shard_phase(1, yd))
    g2 = gather(plan.shard_phase(2, yd, g1))
    x = plan.shard_phase(3, gathered=g2)
    plan.sync()
    out[rank] = (a, b, x[0].cpu().numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shard_phases_two_processes(world):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    T = 50_001
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), T, out), nprocs=world, join=True)
    spec = _spec()
    _, y = wl.simulate_linear(spec, T, seed=23)
    xo = oracle.kf_rts(oracle.LinearModel(spec.F, spec.L, spec.W, spec.H, spec.R, spec.m0, spec.P0, c=spec.c,
                                          r=spec.r), y, T, spec.t0, spec.tf)
    x = np.concatenate([out[r][2] for r in range(world)])
    assert sum(out[r][1] - out[r][0] for r in range(world)) == T + 1
    assert np.abs(x - xo).max() / np.abs(xo).max() < 1e-9
