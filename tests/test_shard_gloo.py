"""Multi-process (gloo, world_size 2 and 3, CPU) check of the time-sharding protocol's
host-side logic: node ranges (shard_range), payload order of the all-gathers, the fold
of preceding-rank pass-1 aggregates into the carry and of following-rank pass-2
aggregates onto x*_T.  The per-rank arithmetic is the NumPy
transcription of the method in test_method_numpy.py (the CUDA phases are covered by
test_parity_gpu.py::test_virtual_time_shards)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_13319_b200.binding import shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, T, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_method_numpy import combine, node_elements
    import workloads as wl
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = wl.wiener_velocity()
    spec.c = np.array([0.3, -0.2, 0.1, 0.05])
    spec.r = np.array([0.5, -0.25])
    _, y = wl.simulate_linear(spec, T, seed=11)
    E = node_elements(spec, y, T)
    n = spec.nx
    a, b = shard_range(rank, world, T)
    # phase 1: chunk aggregate Agg_r = E_{b-1} (x) ... (x) E_a  (R-FLIP)
    acc = E[a]
    for i in range(a + 1, b):
        acc = combine(E[i], acc)
    flat = np.concatenate([acc[0].ravel(), acc[1], acc[2].ravel(), acc[3], acc[4].ravel()])
    g1 = [torch.zeros(flat.size, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(g1, torch.from_numpy(flat))

    def unflat(v):
        v = v.numpy()
        return (v[:n * n].reshape(n, n), v[n * n:n * n + n], v[n * n + n:2 * n * n + n].reshape(n, n),
                v[2 * n * n + n:2 * n * n + 2 * n], v[2 * n * n + 2 * n:].reshape(n, n))
    # carry = Agg_{r-1} (x) ... (x) Agg_0 applied to (0, 0): (S, v) of node a-1
    S, v = np.zeros((n, n)), np.zeros(n)
    for q in range(rank):
        Aq = unflat(g1[q])
        M = np.linalg.inv(np.eye(n) + Aq[2] @ S)
        S, v = Aq[0].T @ S @ M @ Aq[0] + Aq[4], Aq[0].T @ np.linalg.inv(np.eye(n) + S @ Aq[2]) @ (v - S @ Aq[1]) + Aq[3]
    S_prev, v_prev = S, v  # (S, v) of node a-1: the carry (no halo exchange)
    # local pass 1 and the chunk's pass-2 aggregate (x_{b-1} -> x_{a-1})
    Ss, vs = [], []
    P, q = np.eye(n), np.zeros(n)
    for i in range(a, b):
        Ai, bi, Ci, hi, Ji = E[i]
        if i == 0:
            S, v = Ji, hi
        else:
            M = np.linalg.inv(np.eye(n) + Ci @ S)
            Phi, beta = M @ Ai, M @ (bi + Ci @ v)
            P, q = P @ Phi, P @ beta + q
            S, v = Ai.T @ S @ M @ Ai + Ji, Ai.T @ np.linalg.inv(np.eye(n) + S @ Ci) @ (v - S @ bi) + hi
        Ss.append(S)
        vs.append(v)
    last = rank == world - 1
    xT = np.linalg.solve(Ss[-1], vs[-1]) if last else np.zeros(n)
    g2 = [torch.zeros(n * n + 2 * n, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(g2, torch.from_numpy(np.concatenate([P.ravel(), q, xT])))
    # x at this rank's last node = Agg_{r+1} o ... o Agg_{G-1} (x*_T)
    x = g2[world - 1].numpy()[n * n + n:]
    for qq in range(world - 1, rank, -1):
        w = g2[qq].numpy()
        x = w[:n * n].reshape(n, n) @ x + w[n * n:n * n + n]
    xs = np.zeros((b - a, n))
    for i in range(b - 1, a - 1, -1):
        xs[i - a] = x
        if i > 0:
            Ai, bi, Ci = E[i][:3]
            Sp, vp = (Ss[i - a - 1], vs[i - a - 1]) if i > a else (S_prev, v_prev)
            x = np.linalg.solve(np.eye(n) + Ci @ Sp, Ai @ x + bi + Ci @ vp)
    out[rank] = (a, b, xs)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_time_shard_protocol(world):
    import oracle
    import workloads as wl
    T = 240
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, T, out), nprocs=world, join=True)
    spec = wl.wiener_velocity()
    spec.c = np.array([0.3, -0.2, 0.1, 0.05])
    spec.r = np.array([0.5, -0.25])
    _, y = wl.simulate_linear(spec, T, seed=11)
    xo = oracle.kf_rts(oracle.LinearModel(spec.F, spec.L, spec.W, spec.H, spec.R, spec.m0, spec.P0, c=spec.c,
                                          r=spec.r), y, T, spec.t0, spec.tf)
    x = np.concatenate([out[r][2] for r in range(world)])
    assert sum(out[r][1] - out[r][0] for r in range(world)) == T + 1
    assert np.abs(x - xo).max() / np.abs(xo).max() < 1e-12
