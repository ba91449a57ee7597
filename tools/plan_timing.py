"""Plan-creation time breakdown (PMAP_PLAN_TIMING=1): map_plan phases for a workload."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PMAP_PLAN_TIMING"] = "1"

if __name__ == "__main__":
    import torch
    import workloads as wl
    import paper_2512_13319_b200 as pm
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
    spec = wl.wiener_velocity()
    torch.cuda.synchronize()
    for k in range(2):
        t = time.perf_counter()
        plan = pm.Plan(T=T, t0=spec.t0, tf=spec.tf, F=spec.F, L=spec.L, W=spec.W, H=spec.H, R=spec.R, m0=spec.m0,
                       P0=spec.P0)
        print(f"plan {k}: {1e3 * (time.perf_counter() - t):.1f} ms (workspace {plan.workspace_bytes / 1e6:.0f} MB)",
              file=sys.stderr, flush=True)
        plan.close()
