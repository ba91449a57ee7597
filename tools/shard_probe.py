"""Per-GPU cost of one rank of a time-sharded C3 solve, measured on one GPU (tools only).

Runs the local part of rank r of a G-way shard (T/G nodes) through the NCCL path on a
1-rank communicator (PMAP_FORCE_SHARD=1) and through the plain path, and prints the
per-kernel event table.  The collective then moves G x payload on one GPU only, so the
all-gather cost is a lower bound; the local kernels are exactly what each rank runs."""
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_13319_b200 as pm  # noqa: E402
import workloads as wl  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 8
T = 10_000_000 // G
torch.cuda.set_device(0)
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
comm = dist.group.WORLD._get_backend(torch.device("cuda", 0))._comm_ptr()
spec = wl.wiener_velocity()
_, y = wl.simulate_linear(spec, T, seed=0)
yd = torch.tensor(y[None], device="cuda")
out = {}
for mode in ("plain", "nccl"):
    if mode == "nccl":
        os.environ["PMAP_FORCE_SHARD"] = "1"
    plan = pm.Plan(T=T, t0=spec.t0, tf=5.0 / G, F=spec.F, L=spec.L, W=spec.W, H=spec.H, R=spec.R, m0=spec.m0,
                   P0=spec.P0, nccl_comm=comm if mode == "nccl" else None)
    x = torch.empty((1, T + 1, 4), dtype=torch.float64, device="cuda")
    for _ in range(5):
        plan.solve_linear(yd, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 200
    for _ in range(n):
        plan.solve_linear(yd, x)
    e1.record()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        plan.solve_linear(yd, x)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / n * 1e3
    plan.profile(True)
    for _ in range(50):
        plan.solve_linear(yd, x)
    prof = {k: round(v[0] / 50, 4) for k, v in plan.profile_read().items()}
    plan.profile(False)
    out[mode] = {"ms_per_solve": e0.elapsed_time(e1) / n, "wall_ms": wall, "launches": plan.launches,
                 "kernels": prof}
print(json.dumps({"G": G, "T_local": T, **out}))
dist.destroy_process_group()
