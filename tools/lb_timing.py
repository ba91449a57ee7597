"""Phase timeline of the two look-back kernels (PMAP_LB_TIMING=1 diagnostics).

Runs C3 (or --T), records per-tile %globaltimer stamps at the phase boundaries and prints
the median / p90 of each phase and the kernel span, so the look-back waits can be told
apart from the per-tile work.  Usage: python tools/lb_timing.py [--T N]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PMAP_LB_TIMING"] = "1"

# stamp slots in the order they are taken (pmap_lb.cuh LB_STAMP)
PHASES = {
    0: [(0, 1, "1a: y staged"), (1, 2, "1a: fold + tile reduce"), (2, 3, "1a: scan + run maps"),
        (4, 5, "1b: look-back"), (5, 6, "1b: run values, offsets")],
    1: [(0, 1, "look-back"), (1, 2, "y staged"), (2, 3, "node loop")],
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=10_000_000)
    a = ap.parse_args()
    import torch
    import workloads as wl
    import paper_2512_13319_b200 as pm
    spec = wl.wiener_velocity()
    _, y = wl.simulate_linear(spec, a.T, seed=0)
    plan = pm.Plan(T=a.T, t0=spec.t0, tf=spec.tf, F=spec.F, L=spec.L, W=spec.W, H=spec.H, R=spec.R, m0=spec.m0,
                   P0=spec.P0)
    yd = torch.tensor(y[None], device="cuda")
    for _ in range(3):
        plan.solve_linear(yd)
    torch.cuda.synchronize()
    t = plan.lb_timing().astype(np.int64)
    for ps in (0, 1):
        tt = t[ps]
        tt = tt[tt[:, 0] > 0]
        t0 = tt[:, 0].min()
        last = max(k for k in range(8) if np.any(tt[:, k] > 0))
        print(f"pass {ps + 1}: {len(tt)} tiles, span {(tt.max() - t0) / 1e3:.1f} us")
        for k0, k1, nm in PHASES[ps]:
            ok = (tt[:, k0] > 0) & (tt[:, k1] > 0)
            d = (tt[ok, k1] - tt[ok, k0]) / 1e3
            if len(d):
                print(f"  {nm:22s} median {np.median(d):7.2f} us  p90 {np.percentile(d, 90):7.2f}  max {d.max():7.2f}"
                      f"  (n={ok.sum()})")
        for s0, s1 in ((0, 3), (4, 6)) if ps == 0 else ((0, 3),):
            ok = (tt[:, s0] > 0) & (tt[:, s1] > 0)
            if ok.any():
                life = (tt[ok, s1] - tt[ok, s0]) / 1e3
                span = (tt[ok, s1].max() - tt[ok, s0].min()) / 1e3
                print(f"  stamps {s0}..{s1}: lifetime median {np.median(life):.2f} us, p90 {np.percentile(life, 90):.2f};"
                      f" span {span:.1f} us")


if __name__ == "__main__":
    main()
