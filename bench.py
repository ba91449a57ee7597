#!/usr/bin/env python
"""bench.py -- smoothed time steps/s of the parallel MAP scan (arXiv 2512.13319) on B200.

Metric (BASELINE.json): smoothed time steps/s = batch * T / t_solve (fp64 parallel
MAP scan), one "step" = one complete solve (pass 1 + pass 2 over all nodes) of the
workload.  Default workload at N = 1: BASELINE config 3, the Wiener-velocity model
of P:519-548 (nx = 4, ny = 2) at T = 1e7 grid steps, one trajectory.  With
--gpus N > 1 (launched by torchrun) the same T = 1e7 problem is time-sharded over
the ranks with an NCCL all-gather of chunk carries (strong scaling).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl pmap|reference]

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle (the
reference arm of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
# FP64 (DFMA) peak derived from unit counts and clock: 148 SM x 64 FP64 FMA/clk x 2 flop x 1.965 GHz,
# and the figure a DFMA microbenchmark measured on this pool (tools/fp64_peak.cu,
# profiles/r01_fp64_peak_probe.log); the roofline uses the measured one.
FP64_PEAK_TFLOPS_DERIVED = 148 * 64 * 2 * 1.965e9 / 1e12
FP64_PEAK_TFLOPS_MEASURED = 34.2
FALLBACK_HBM_GBS = 6650.0


# ----------------------------------------------------------- algorithmic counts
def alg_counts(nx: int, ny: int, K: int = 32, lti: bool = True, nw: int = 0, zero_b: bool = False,
               euler_n: int = 0, amask=None, umask=None):
    """Algorithmic FP64 flops (FMA = 2) and HBM bytes per node of each kernel class
    (DESIGN.md section 6): the arithmetic each kernel's per-node recurrence performs
    in this decomposition, excluding the intra-tile scan overheads (Kogge-Stone
    rounds, carries), which are implementation cost.  nw > 0: low-rank diffusion
    (R-LOWRANK node update, R-P2REC pass-2 records of nw (nx + 1) values).  euler_n > 0:
    Euler blocks (R-EULER): y rows of euler_n * ny values, element data parts b, eta built
    from them (2 * nx * euler_n * ny FMA per build: reduce, down; nx * euler_n * ny in pass 2).
    amask / umask (bool arrays, R-MASK): structural non-zeros of A (nx x nx) and U (nx x nw)
    the specialised kernels exploit -- terms with a structurally zero factor are not counted."""
    N = nx
    lu = sum((N - k - 1) + (N - k - 1) ** 2 for k in range(N))
    solve = N * N
    combine = N ** 3 + lu + 2 * N * solve + (N * N + solve) * 2 + N ** 3 + N * N + (N ** 3 + N * N * (N + 1) // 2) * 2 + N * N
    vapply = N ** 3 + lu + N * solve + (N * N + solve) + N ** 3 + N * N * (N + 1) // 2 + N * N
    vapply_tr = vapply + (N * N + solve)
    trans = N ** 3 + lu + 2 * N * N + solve
    ns = N * (N + 1) // 2
    esz = N * N + 2 * N + 2 * ns
    vsz = ns + N
    asz = N * N + N
    d = 8
    reduce_fl = 2 * N * ny if lti else combine  # LTI: impulse-response fold (y_m -> (b, eta))
    vsz2 = vsz  # per-node values pass 1 stores for pass 2
    vapply_dense = vapply
    vapply_node = vapply
    if nw > 0:  # R-LOWRANK node update (vapply_lowrank), R-P2REC records when smaller than (S, v)
        r = nw
        am = np.ones((N, N), bool) if amask is None else np.asarray(amask, bool)
        um = np.ones((N, r), bool) if umask is None else np.asarray(umask, bool)
        nA, nU = int(am.sum()), int(um.sum())
        gram = sum((a + 1) * int(um[:, a].sum()) for a in range(r))
        chol = gram + r * (r - 1) // 2 * (r + 1) + r
        ata = sum(int(am[:, i].sum()) * (N - i) for i in range(N))  # A^T (B A), upper triangle
        # S U, Gram + LDL, Y = L^-1 (S U)^T and D^-1 Y, B = S - Ys^T Y, w = v - S b (skipped
        # when b == 0), q = G^-1 U^T w, w - S U q, B A, A^T (B A) + J, A^T w + eta
        vapply = (N * nU + chol + r * (r - 1) // 2 * N + r * N + ns * r + (0 if zero_b else N * N)
                  + nU + r * r + N * r + N * nA + ata + nA)
        vapply_node = vapply  # the plain node update (no pass-2 record written)
        gram_d = sum((a + 1) * N for a in range(r))
        chol_d = gram_d + r * (r - 1) // 2 * (r + 1) + r
        vapply_dense = (N * N * r + chol_d + r * (r - 1) // 2 * N + r * N + ns * r + (0 if zero_b else N * N)
                        + N * r + r * r + N * r + N * N * N + ns * N + N * N)
        compact = (N == 4 and r == 2 and umask is not None and np.array_equal(
            um, np.array([[0, 0], [0, 0], [1, 0], [0, 1]], bool)))  # CompactRec (pmap_algebra.cuh)
        if r * (N + 1) < vsz:
            vsz2 = r * (N + 1)
            vapply += nU  # U^T v
            trans = nA + nU + chol + r * N + r * r + nU
        if compact:  # the record holds S[:, 2:4] (7 values) and v[2:4]; pass 2 forms S U, U^T v
            vsz2 = 9
            vapply -= nU
            trans += (N * r + r) // 2
    if euler_n > 0:
        ny_row = euler_n * ny
        build = 2 * N * ny_row
        return {
            "k_p1_reduce": (2 * (combine + build), d * (ny_row + esz / K)),
            "k_p1_down": (2 * (vapply + build + vapply_tr / K), d * (ny_row + esz / K + vsz + asz / K)),
            "k_p2_down": (2 * (trans + build // 2), d * (ny_row + vsz + nx + asz / K)),
            "solve": (2 * (combine + 2 * build + vapply + vapply_tr / K + trans + build // 2),
                      d * (3 * ny_row + 2 * vsz + nx)),
        }
    # two-filter pass B epilogue (k_tf_down): mirrored node update (the mirrored diffusion
    # factor is dense) + LDL^T solve of (S + Lam - J^m) x = v + xi - eta^m; reads y, the
    # stored (S, v) and the run prefix, writes x
    ldl = N ** 3 // 6 + N * N + 2 * N * N
    vap_m = vapply_dense if nw > 0 else vapply
    tf_down = (2 * (vap_m + ldl + 2 * N + ns), d * (ny + esz / K + vsz + nx))
    L = 64 * K  # nodes per tile
    # LTI data recurrence of the boundary-tile reduce (lti_fold_data): per node eta = K y + h0,
    # b += Wb eta + cb, eta' = We eta + ... (2 N^2 + N ny FMA); it covers <= 2 tiles per trajectory
    edge = (2 * (2 * N * N + N * ny), d * (ny + esz / K))
    # look-back path (pmap_lb.cuh, R-FWD): pass 1 = the LTI fold (2 N ny FMA) + per run four
    # N x N mat-vecs with the plan's run tables (S pb, Gp u, C_R v, Wr t); reads y and the run
    # tables (Gp, Wr, Phi: 3 N^2 per run), writes v entering each run (N) and the run suffix
    # maps (N^2 + N).  Pass 2 = per node the forward recovery of x (R-FWD: U^T (S x - v), U u,
    # A^-1 z on the structural non-zeros) + the value-function update (the same Woodbury /
    # general update as k_p1_down) + eta = K y; reads y, the run's S (plan table), v and
    # suffix map, writes x.
    if nw > 0:
        xstep = nU * (N + 1) + nU + nA + (0 if zero_b else N)
    else:
        xstep = 3 * N * N + N
    # pass 1a writes v_{s-1} (N) and only the offset (N) of each run's suffix map: its matrix
    # is a plan table (LbRunTab::PS) that pass 2 reads instead (counted there as asz / K)
    lb1 = (2 * (2 * N * ny + 4 * N * N / K), d * (ny + 3 * N * N / K + N / K + N / K))
    # pass 1b: per run v_{s-1} = GP v_in + c and the map offset q += QB v_in (reads GP, QB, c, q;
    # writes c, q): 2 N^2 FMA and 2 N^2 + 4 N values per run
    lb1b = (2 * (2 * N * N / K), d * ((2 * N * N + 4 * N) / K))
    lb2 = (2 * (vapply_node + xstep + N * ny), d * (ny + nx + ns / K + N / K + asz / K))
    return {
        "k_p1_reduce": (2 * combine, d * (ny + esz / K)),          # general models: one combine per node
        "k_p1_reduce_lti": (2 * 2 * N * ny, d * (ny + esz / K)),   # LTI: impulse-response fold
        "k_p1_reduce_lti_edge": edge + ("edge",),
        "k_tf_reduce": (2 * reduce_fl, d * (ny + esz / K)),
        "k_tf_reduce_lti_edge": edge + ("edge",),
        "k_tf_down": tf_down,
        "k_p1_down": (2 * (vapply + vapply_tr / K), d * (ny + esz / K + vsz2 + asz / K)),
        "k_p2_down": (2 * trans, d * (vsz2 + nx + asz / K)),
        # tile / group scans: one combine per tile (per group), amortised per node
        "k_p1_tiles": (2 * combine / L, d * 2 * esz / L), "k_p1_groups": (2 * combine / (L * 128), d * esz / L),
        "k_p2_tiles": (2 * N ** 3 / L, d * 2 * asz / L), "k_p2_groups": (2 * N ** 3 / (L * 128), d * asz / L),
        "k_tf_tiles": (2 * combine / L, d * 2 * esz / L), "k_tf_groups": (2 * combine / (L * 128), d * esz / L),
        "k_lb_pass1a": lb1,
        "k_lb_pass1b": lb1b,
        "k_lb_pass2": lb2,
        "solve": (2 * (reduce_fl + vapply + vapply_tr / K + trans), d * (ny + 2 * vsz + nx)),
        "solve_lb": (lb1[0] + lb1b[0] + lb2[0], lb1[1] + lb1b[1] + lb2[1]),
    }


def structural_masks(spec, T):
    """Structural non-zeros of A = I - dt F and U = sqrt(dt) L chol(W) the library's
    specialised kernels use (R-MASK; the compiled Wiener-velocity masks), else dense."""
    dt = (spec.tf - spec.t0) / T
    A = np.eye(spec.nx) - dt * spec.F
    U = np.sqrt(dt) * spec.L @ np.linalg.cholesky(spec.W)
    wa = np.zeros((4, 4), bool)
    for i, j in ((0, 0), (0, 2), (1, 1), (1, 3), (2, 2), (3, 3)):
        wa[i, j] = True
    wu = np.zeros((4, 2), bool)
    wu[2, 0] = wu[3, 1] = True
    if A.shape == (4, 4) and U.shape == (4, 2) and not np.any((A != 0) & ~wa) and not np.any((U != 0) & ~wu):
        return wa, wu
    return None, None


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None
        time.sleep(0.3)

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.count(",") >= 7]
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[4 + k].strip() == "Active"})
        load = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": float(np.median(load)) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- workloads
def build_inputs(config: str, rank: int, world: int):
    """This rank's inputs: batch workloads (C5) shard the trajectories (MAP_FLAG_BATCH_SHARD,
    no exchange), single trajectories shard time."""
    import workloads as wl
    from paper_2512_13319_b200.binding import batch_range, shard_range
    spec, y, T, B = wl.make_workload(config, seed=0)
    if y.ndim == 2:
        y = y[None]
    if B > 1 and world > 1:
        b0, b1 = batch_range(rank, world, B)
        return spec, np.ascontiguousarray(y[b0:b1]), T, B
    a0, a1 = shard_range(rank, world, T)
    return spec, np.ascontiguousarray(y[:, a0:a1]), T, B


def make_plan(pm, spec, T, B, rank, world, comm, substeps=1, mixed=False):
    import workloads as wl
    if isinstance(spec, wl.LinearSpec):
        return pm.Plan(T=T, t0=spec.t0, tf=spec.tf, F=spec.F, c=spec.c, L=spec.L, W=spec.W, H=spec.H,
                       r=spec.r, R=spec.R, m0=spec.m0, P0=spec.P0, batch=B, rank=rank, world=world,
                       nccl_comm=comm, substeps=substeps, mixed=mixed, shard="batch" if B > 1 else "time")
    return pm.Plan(T=T, t0=spec.t0, tf=spec.tf, L=spec.L, W=spec.W, R=spec.R, m0=spec.m0, P0=spec.P0,
                   nl_kind=spec.kind, params=spec.params, batch=B, rank=rank, world=world, nccl_comm=comm,
                   shard="batch" if B > 1 else "time")


def solve_fn(plan, config):
    from workloads.models import CONFIGS
    method = CONFIGS[config]["method"]
    if method == "rts":
        return lambda y, x: plan.solve_linear(y, x)
    if method == "two_filter":
        return lambda y, x: plan.two_filter(y, x)
    passes = CONFIGS[config].get("passes", 10)
    return lambda y, x: plan.solve_nonlinear(y, passes=passes, x_map=x)


def workload_name(config, T, B):
    from workloads.models import CONFIGS
    c = CONFIGS[config]
    return (f"{config}: {c['model']} {c['method']} T={T} batch={B}" + (f" passes={c['passes']}" if "passes" in c else "")
            + (f" euler_substeps={c['substeps']} (T blocks, n*T fine steps)" if "substeps" in c else ""))


# ---------------------------------------------------------------- CPU oracle
def oracle_sample(config: str, budget_s: float = 12.0):
    """Time the CPU oracle as it stands on a bounded sample of the workload."""
    import oracle
    import workloads as wl
    from workloads.models import CONFIGS
    c = CONFIGS[config]
    if c["method"] == "ieks":
        T = 20_000
        s = wl.coordinated_turn()
        _, y = wl.simulate_nonlinear(s, T, seed=0)
        t = time.perf_counter()
        oracle.ieks(1, None, s.L, s.W, s.R, s.m0, s.P0, y, T, s.t0, s.tf, passes=c["passes"])
        dt = time.perf_counter() - t
        return T / dt, 1, f"coordinated turn T={T}, {c['passes']} passes, 1 thread (full run is T={c['T']})"
    spec = wl.wiener_velocity() if c["model"] == "wiener_velocity" else wl.ornstein_uhlenbeck()
    md = oracle.LinearModel(spec.F, spec.L, spec.W, spec.H, spec.R, spec.m0, spec.P0)
    if "substeps" in c:
        n, T = c["substeps"], c["T"]
        _, yf = wl.simulate_linear(spec, n * T, seed=0)
        t = time.perf_counter()
        oracle.euler_rts(md, yf, T, n, spec.t0, spec.tf)
        dt = time.perf_counter() - t
        return T / dt, 1, f"Euler blocks T={T} x n={n} (full workload), sequential, 1 thread"
    if c["method"] == "two_filter":
        B, T = 64, c["T"]
        _, y = wl.simulate_linear(spec, T, seed=0, batch=B)
        t = time.perf_counter()
        oracle.batch(md, y, T, spec.t0, spec.tf, mode=1)
        dt = time.perf_counter() - t
        return B * T / dt, oracle.num_threads(), f"{B} of {c['batch']} trajectories x T={T}, OpenMP"
    T = min(c["T"], 2_000_000)
    _, y = wl.simulate_linear(spec, T, seed=0)
    t = time.perf_counter()
    oracle.kf_rts(md, y, T, spec.t0, spec.tf)
    dt = time.perf_counter() - t
    return T / dt, 1, f"{c['model']} T={T} (of {c['T']}), sequential KF+RTS, 1 thread"


def run_reference(args):
    """Reference arm of this tier: the CPU oracle timed on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    import workloads as wl
    from workloads.models import CONFIGS
    c = CONFIGS[args.config]
    spec = wl.wiener_velocity() if c["model"] == "wiener_velocity" else wl.ornstein_uhlenbeck()
    if c["method"] == "ieks":
        spec = wl.coordinated_turn()
        T = 5_000
        _, y = wl.simulate_nonlinear(spec, T, seed=0)
        step = lambda: oracle.ieks(1, None, spec.L, spec.W, spec.R, spec.m0, spec.P0, y, T, spec.t0, spec.tf,
                                   passes=c["passes"])
        units, cores, sample = T, 1, f"coordinated turn T={T} x {c['passes']} passes per step"
    elif "substeps" in c:
        n, T = c["substeps"], c["T"]
        md = oracle.LinearModel(spec.F, spec.L, spec.W, spec.H, spec.R, spec.m0, spec.P0)
        _, yf = wl.simulate_linear(spec, n * T, seed=0)
        step = lambda: oracle.euler_rts(md, yf, T, n, spec.t0, spec.tf)
        units, cores, sample = T, 1, f"Euler blocks T={T} x n={n} per step (full workload), sequential"
    elif c["method"] == "two_filter":
        B, T = 32, c["T"]
        md = oracle.LinearModel(spec.F, spec.L, spec.W, spec.H, spec.R, spec.m0, spec.P0)
        _, y = wl.simulate_linear(spec, T, seed=0, batch=B)
        step = lambda: oracle.batch(md, y, T, spec.t0, spec.tf, mode=1)
        units, cores, sample = B * T, oracle.num_threads(), f"{B} trajectories x T={T} per step, OpenMP"
    else:
        T = min(c["T"], 300_000)
        md = oracle.LinearModel(spec.F, spec.L, spec.W, spec.H, spec.R, spec.m0, spec.P0)
        _, y = wl.simulate_linear(spec, T, seed=0)
        step = lambda: oracle.kf_rts(md, y, T, spec.t0, spec.tf)
        units, cores, sample = T, 1, f"{c['model']} T={T} per step (of {c['T']}), sequential KF+RTS"
    for _ in range(args.warmup):
        step()
    t = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = (time.perf_counter() - t) / args.steps
    v = units / el
    out = {"metric": "smoothed time steps/s (fp64 parallel MAP scan)", "value": v, "unit": "steps/s",
           "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": el * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic (seeded Euler-Maruyama simulation of the paper's SDE)",
           "config": {"workload": workload_name(args.config, c["T"], c["batch"]), "sample": sample},
           "cpu_baseline": {"value": v, "unit": "steps/s", "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": v, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------- sequential GPU baseline (f1)
def sequential_gpu(plan, config, yd, xd, ms_parallel, torch, stream):
    """The paper's comparison: the same smoother run sequentially
    on the same B200 (map_solve_sequential, one thread per trajectory), full workload,
    timed with CUDA events (after one untimed run unless the run is long)."""
    from workloads.models import CONFIGS
    c = CONFIGS[config]
    method = 1 if c["method"] == "two_filter" else 0
    passes = c.get("passes", 1)
    run = lambda: plan.solve_sequential(yd, method=method, passes=passes, x_map=xd)
    if plan.batch * plan.T * passes < 2_000_000:  # long runs (C3: ~19 s) are timed cold: load cost is noise
        run()
        plan.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    run()
    e1.record(stream)
    torch.cuda.synchronize()
    plan.sync()
    ms = e0.elapsed_time(e1)
    B, T = plan.batch, plan.T
    return {"value": B * T / (ms * 1e-3), "unit": "steps/s", "ms_per_solve": ms,
            "method": ("two-filter" if method else "RTS") + (f", {passes} IEKS passes" if "passes" in c else ""),
            "threads": B, "parallel_speedup": ms / ms_parallel,
            "what": "map_solve_sequential: one GPU thread per trajectory, same element build and fp64 algebra"}


# ---------------------------------------------------------------- launcher
def self_launch(args):
    """`python bench.py --gpus N` without torchrun: re-exec under torch.distributed.run with
    N ranks (one per GPU, rendezvous on 127.0.0.1); fails loudly if N GPUs are not present."""
    import socket
    if args.impl != "reference":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} requested but only {have} CUDA devices are visible")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    rc = subprocess.call(cmd)
    if rc != 0:
        raise SystemExit(rc)


# ---------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C3", choices=["C1", "C2", "C3", "C4", "C5", "C2E"])
    ap.add_argument("--impl", default="pmap", choices=["pmap", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-seq", action="store_true", help="skip the sequential on-device baseline (SURVEY f1)")
    ap.add_argument("--mixed", action="store_true",
                    help="MAP_FLAG_MIXED: fp32 node recursion in pass 2 from fp64 carries (SURVEY f4; not the headline)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: the N ranks were not formed")
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist.barrier()
        be = dist.group.WORLD._get_backend(torch.device("cuda", local))
        comm = be._comm_ptr()
    import paper_2512_13319_b200 as pm

    from workloads.models import CONFIGS
    substeps = CONFIGS[args.config].get("substeps", 1)
    spec, y_host, T, B = build_inputs(args.config, rank, world)
    torch.cuda.synchronize()
    tp = time.perf_counter()
    plan = make_plan(pm, spec, T, B, rank, world, comm, substeps, mixed=args.mixed)
    plan_ms = (time.perf_counter() - tp) * 1e3  # map_plan: model preprocessing, LTI / look-back tables, workspace
    # the first plan of a process also pays the lazy loading of its kernels' modules: time a
    # second identical plan (created and destroyed) for the steady-state plan cost
    tp = time.perf_counter()
    make_plan(pm, spec, T, B, rank, world, comm, substeps, mixed=args.mixed).close()
    torch.cuda.synchronize()
    plan_ms_warm = (time.perf_counter() - tp) * 1e3
    solve = solve_fn(plan, args.config)
    dev = torch.device("cuda", local)
    yd = torch.from_numpy(y_host).to(dev)
    xd = torch.empty((B, plan.n_local, plan.nx), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        solve(yd, xd)
    plan.sync()
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        solve(yd, xd)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    plan.sync()
    ms = e0.elapsed_time(e1) / args.steps
    launches_per_step = plan.launches
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = B * T / (ms * 1e-3)

    # per-kernel CUDA-event timing on the launching stream (separate region)
    plan.profile(True)
    for _ in range(min(args.steps, 50)):
        solve(yd, xd)
    prof = plan.profile_read()
    plan.profile(False)

    # end to end through the C ABI with host (pinned) buffers, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        from workloads.models import CONFIGS
        yh = torch.from_numpy(y_host).pin_memory()
        xh = torch.empty((B, plan.n_local, plan.nx), dtype=torch.float64).pin_memory()
        pipelined = CONFIGS[args.config]["method"] == "rts" and substeps == 1

        def e2e_time(pipe):
            run = (lambda: plan.solve_linear_pipelined(yh, xh)) if pipe else (lambda: solve(yh, xh))
            run()
            run()
            plan.sync()
            barrier()
            t0 = time.perf_counter()
            for _ in range(args.e2e_steps):
                run()
            plan.sync()  # every solve's x is in host memory
            torch.cuda.synchronize()
            el = torch.tensor([(time.perf_counter() - t0) / args.e2e_steps], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(el, op=dist.ReduceOp.MAX)
            return float(el.item())
        el_sync = e2e_time(False)
        el = e2e_time(True) if pipelined else el_sync
        e2e = {"value": B * T / el, "unit": "steps/s",
               "h2d_bytes_per_step": int(yh.numel() * 8 * world), "d2h_bytes_per_step": int(xh.numel() * 8 * world),
               "api": ("map_solve_linear_pipelined: host buffers, each solve's copies overlap the neighbouring "
                       "solves' copies in the other direction" if pipelined else "map_solve_linear, host buffers"),
               "sync_call_value": B * T / el_sync}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # roofline of the dominant kernel (FP64-ALU bound)
    import workloads as wl
    lowrank = 0
    if (isinstance(spec, wl.LinearSpec) and spec.L.shape[1] < spec.nx and os.environ.get("PMAP_NO_LOWRANK") != "1"
            and os.environ.get("PMAP_GENERAL") != "1"):
        lowrank = spec.L.shape[1]
    zero_b = isinstance(spec, wl.LinearSpec) and (spec.c is None or not np.any(spec.c))
    amask = umask = None
    if lowrank and os.environ.get("PMAP_NO_MASK") != "1":
        amask, umask = structural_masks(spec, T)
    if substeps > 1:  # Euler blocks: general kernels, element build from n*ny measurements
        counts = alg_counts(plan.nx, plan.ny, lti=False, euler_n=substeps)
    else:
        kk = 32 if B * -(-plan.n_local // 2048) >= 4 * 148 else 8  # the library's run length (choose_run_length)
        counts = alg_counts(plan.nx, plan.ny, K=kk, lti=isinstance(spec, wl.LinearSpec) and np.ndim(spec.F) == 2,
                            nw=lowrank, zero_b=zero_b, amask=amask, umask=umask)
    dom = max(prof.items(), key=lambda kv: kv[1][0])
    dname, (dms, dl) = dom
    per_launch_ms = dms / dl
    rec = counts.get(dname)
    Bl = plan.batch  # this rank's trajectories (batch-sharded plans hold a slice of B)
    tile_nodes = 64 * (32 if Bl * -(-plan.n_local // 2048) >= 4 * 148 else 8)
    if rec is not None:
        fl, by = rec[0], rec[1]
        # units one launch processes: every node, or the <= 2 boundary tiles per trajectory
        nodes_per_launch = Bl * plan.n_local if len(rec) < 3 else Bl * min(plan.n_local, 2 * tile_nodes)
    traffic = None  # dram__bytes_read.sum + dram__bytes_write.sum per launch, from a committed ncu capture
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        trk = tr.get("kernels", {}).get(dname)
        if trk and tr.get("nodes") in (B * plan.n_local, B * (plan.n_local - 1)):
            traffic = trk["dram_bytes_per_launch"]
    except Exception:
        traffic = None
    try:
        peaks = json.load(open(PEAKS_PATH))
        hbm = float(peaks["hbm_gbs"])
        hbm_src = "measured"
    except Exception:
        hbm, hbm_src = FALLBACK_HBM_GBS, "fallback"
    fp64 = FP64_PEAK_TFLOPS_MEASURED
    alu_src = ("measured: DFMA microbenchmark 34.2 TF/s on this pool (tools/fp64_peak.cu, "
               "profiles/r01_fp64_peak_probe.log); MEASURED_PEAKS.json has no FP64 figure; derived 148 SM x 64 "
               "DFMA/clk x 2 x 1.965 GHz = %.1f TF/s" % FP64_PEAK_TFLOPS_DERIVED)
    hbm_desc = f"{hbm_src}: MEASURED_PEAKS.json hbm_gbs" if hbm_src == "measured" else "fallback (B200_PROFILING.md)"
    if rec is None:
        roofline = {"bound": None, "kernel": dname, "achieved": None, "peak": None, "unit": None, "frac": None,
                    "traffic": traffic, "why": f"no algorithmic count for {dname}"}
    else:
        achieved_tflops = fl * nodes_per_launch / (per_launch_ms * 1e-3) / 1e12
        achieved_gbs = by * nodes_per_launch / (per_launch_ms * 1e-3) / 1e9
        # the binding roof of the dominant kernel: FP64 ALU (DFMA pipe) or HBM, whichever
        # fraction is larger; the other is reported alongside
        alu_frac = achieved_tflops / fp64
        hbm_frac = achieved_gbs / hbm
        if hbm_frac >= alu_frac:
            roofline = {"bound": "hbm", "kernel": dname, "achieved": achieved_gbs, "peak": hbm, "unit": "GB/s",
                        "frac": hbm_frac, "peak_source": hbm_desc,
                        "other_roof": {"bound": "alu", "achieved": achieved_tflops, "peak": fp64,
                                       "unit": "TFLOP/s", "frac": alu_frac, "peak_source": alu_src}}
        else:
            roofline = {"bound": "alu", "kernel": dname, "achieved": achieved_tflops, "peak": fp64,
                        "unit": "TFLOP/s", "frac": alu_frac, "peak_source": alu_src,
                        "other_roof": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm, "unit": "GB/s",
                                       "frac": hbm_frac, "peak_source": hbm_desc}}
        roofline.update({"traffic": traffic,
                         "traffic_source": "profiles/ncu_traffic.json (ncu --set full, same workload)" if traffic else None,
                         "alg_flops_per_node": fl, "alg_bytes_per_node": by, "nodes_per_launch": nodes_per_launch,
                         "kernel_ms_per_launch": per_launch_ms,
                         "kernel_share_of_step": dms / max(1e-9, sum(v[0] for v in prof.values()))})
    lb = "k_lb_pass2" in prof
    sfl, sby = counts["solve_lb" if lb else "solve"]
    cfl, cby = counts["solve"]
    npg = B * T / world  # nodes per GPU per solve (per-GPU rooflines)
    solve_hbm = {"schedule": "look-back (3 kernels, R-FWD)" if lb else "scan hierarchy", "per": "GPU",
                 "alg_bytes_per_node": sby, "achieved_gbs": sby * npg / (ms * 1e-3) / 1e9, "peak_gbs": hbm,
                 "peak_source": hbm_src, "frac_of_hbm_roofline": sby * npg / (ms * 1e-3) / 1e9 / hbm,
                 "alg_tflops": sfl * npg / (ms * 1e-3) / 1e12, "frac_of_fp64_peak": sfl * npg / (ms * 1e-3) / 1e12 / fp64,
                 "canonical_bytes_per_node": cby,
                 "canonical_frac_of_hbm_roofline": cby * npg / (ms * 1e-3) / 1e9 / hbm}

    seq = None
    if world == 1 and not args.no_seq:
        seq = sequential_gpu(plan, args.config, yd, xd, ms, torch, stream)

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, cores, sample = oracle_sample(args.config)
        cpu = {"value": v, "unit": "steps/s", "cores": cores, "kind": "oracle", "sample": sample}

    out = {
        "metric": "smoothed time steps/s (fp64 parallel MAP scan)",
        "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64 (pass-2 node recursion f32, MAP_FLAG_MIXED)" if args.mixed else "f64",
        "data": "synthetic (seeded Euler-Maruyama simulation of the paper's SDE, NumPy PCG64 seed 0)",
        "config": {"workload": workload_name(args.config, T, B), "T": T, "batch": B, "nx": plan.nx, "ny": plan.ny,
                   "parallelism": (f"batch-shard x{world} (MAP_FLAG_BATCH_SHARD, no exchange)" if world > 1 and B > 1
                                   else f"time-shard x{world}" if world > 1 else "single GPU"),
                   "l2": "inputs larger than L2 (y %.0f MB, workspace %.0f MB per GPU)" % (
                       y_host.nbytes / 1e6, plan.workspace_bytes / 1e6)},
        "roofline": roofline,
        "solve_roofline": solve_hbm,
        "kernels_ms_per_step": {k: v[0] / max(1, min(args.steps, 50)) for k, v in prof.items()},
        "cpu_baseline": cpu,
        "sequential_gpu": seq,
        "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps,
        "launches_per_solve": launches_per_step,
        "plan_ms": plan_ms,
        "plan_ms_warm": plan_ms_warm,
        "clocks": clk,
    }
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
