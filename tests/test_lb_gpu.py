"""GPU parity of the single-pass decoupled look-back path (pmap_lb.cuh).

LTI single-GPU solves run k_lb_pass1a + k_lb_pass1b + k_lb_pass2 (three launches).  These tests cover
it against the CPU oracle (<= 1e-9 relative in fp64, G23, plus the per-component
scaled error) and against the multi-kernel scan hierarchy (PMAP_NO_LB=1, <= 1e-12),
at sizes that span one tile, several tiles, several look-back groups (32 tiles) and
several warp windows of groups, with ragged tails; batches; filter outputs; both run
lengths; fp32; and a stress mode that injects pseudo-random delays before every
look-back publication (PMAP_LB_STRESS=1) so that the look-back walks through
aggregates, group aggregates and prefixes in every combination.
"""
import numpy as np
import pytest

import oracle
import workloads as wl
from test_parity_gpu import TOL32, TOL64, gpu_plan, ora_model, random_lti, rel, rel_comp, to_dev, torch_cuda  # noqa: F401

pytestmark = pytest.mark.gpu

TILE = 64 * 32  # nodes per tile at K = 32 (group = 32 tiles = 65536 nodes)
LB_LAUNCHES = 3  # k_lb_pass1a, k_lb_pass1b, k_lb_pass2


def _wiener_offsets():
    spec = wl.wiener_velocity()
    spec.c = np.array([0.3, -0.2, 0.1, 0.05])
    spec.r = np.array([0.5, -0.25])
    return spec


@pytest.mark.parametrize("T", [1, 2, 33, TILE, TILE + 1, 3 * TILE + 17, 32 * TILE, 32 * TILE + 1, 33 * TILE + 5,
                               40 * 32 * TILE + 999])
def test_lb_matches_oracle(torch_cuda, T):
    torch = torch_cuda
    spec = _wiener_offsets()
    _, y = wl.simulate_linear(spec, T, seed=T % 997)
    plan = gpu_plan(spec, T)
    x = plan.solve_linear(to_dev(torch, y[None]))
    plan.sync()
    if T >= TILE:  # dt <= 2.4e-3: the forward-recovery bound admits the look-back path (R-FWD)
        assert plan.launches == LB_LAUNCHES
    xo = oracle.kf_rts(ora_model(spec), y, T, spec.t0, spec.tf)
    xg = x[0].cpu().numpy()
    assert rel(xg, xo) < TOL64
    assert rel_comp(xg, xo) < 1e-8


@pytest.mark.parametrize("T,B", [(9_001, 3), (200_003, 2), (1_000, 64)])
def test_lb_batch_and_hierarchy(torch_cuda, T, B, monkeypatch):
    """Batches (tickets run trajectory-major across the whole grid) against the oracle and
    against the multi-kernel scan hierarchy of round 1 (PMAP_NO_LB=1)."""
    torch = torch_cuda
    spec = _wiener_offsets()
    _, y = wl.simulate_linear(spec, T, seed=T % 1000, batch=B)
    y = y.reshape(B, T + 1, 2)
    yd = to_dev(torch, y)
    x_lb = gpu_plan(spec, T, batch=B).solve_linear(yd).cpu().numpy()
    monkeypatch.setenv("PMAP_NO_LB", "1")
    plan_h = gpu_plan(spec, T, batch=B)
    x_h = plan_h.solve_linear(yd).cpu().numpy()
    assert plan_h.launches > LB_LAUNCHES
    xo = oracle.batch(ora_model(spec), y, T, spec.t0, spec.tf, mode=0)
    for b in range(B):
        assert rel(x_lb[b], x_h[b]) < 1e-12
        assert rel(x_lb[b], xo[b]) < TOL64


@pytest.mark.parametrize("T", [5_000, 70 * TILE + 3])
def test_lb_stress_delays(torch_cuda, T, monkeypatch):
    """Look-back under injected delays (up to ~16 us before each publication): results
    stay within rounding of the undisturbed run and of the oracle, and repeated solves
    (flags and tickets recycled without a memset) stay correct."""
    torch = torch_cuda
    spec = _wiener_offsets()
    _, y = wl.simulate_linear(spec, T, seed=4)
    yd = to_dev(torch, y[None])
    x0 = gpu_plan(spec, T).solve_linear(yd).cpu().numpy()
    monkeypatch.setenv("PMAP_LB_STRESS", "1")
    plan = gpu_plan(spec, T)
    xo = oracle.kf_rts(ora_model(spec), y, T, spec.t0, spec.tf)
    for _ in range(3):
        x = plan.solve_linear(yd)
        plan.sync()
        xs = x.cpu().numpy()
        assert rel(xs[0], x0[0]) < 1e-12
        assert rel(xs[0], xo) < TOL64


def test_lb_filter_outputs(torch_cuda):
    torch = torch_cuda
    spec = _wiener_offsets()
    T = 3 * TILE + 11
    _, y = wl.simulate_linear(spec, T, seed=3)
    xo, fm, fP = oracle.kf_rts(ora_model(spec), y, T, spec.t0, spec.tf, want_filter=True)
    plan = gpu_plan(spec, T)
    nx = spec.nx
    m = torch.empty((1, T + 1, nx), dtype=torch.float64, device="cuda")
    P = torch.empty((1, T + 1, nx * (nx + 1) // 2), dtype=torch.float64, device="cuda")
    x = plan.solve_linear(to_dev(torch, y[None]), filt_m=m, filt_P=P)
    plan.sync()
    assert plan.launches == LB_LAUNCHES
    iu = np.triu_indices(nx)
    assert rel(x[0].cpu().numpy(), xo) < TOL64
    assert rel(m[0].cpu().numpy(), fm) < TOL64
    assert rel(P[0].cpu().numpy(), fP[:, iu[0], iu[1]]) < TOL64
    # either output alone (the other NULL)
    m2 = torch.zeros_like(m)
    P2 = torch.zeros_like(P)
    plan.solve_linear(to_dev(torch, y[None]), filt_m=m2)
    plan.solve_linear(to_dev(torch, y[None]), filt_P=P2)
    plan.sync()
    assert rel(m2[0].cpu().numpy(), fm) < TOL64
    assert rel(P2[0].cpu().numpy(), fP[:, iu[0], iu[1]]) < TOL64


@pytest.mark.parametrize("K", ["8", "32"])
@pytest.mark.parametrize("shape", [(1, 1), (2, 1), (3, 2), (4, 2), (5, 2)])
def test_lb_random_lti_shapes(torch_cuda, K, shape, monkeypatch):
    """Every compiled LTI shape (full-rank and low-rank diffusion, c, r != 0) at both run
    lengths, multi-tile with a ragged tail."""
    torch = torch_cuda
    monkeypatch.setenv("PMAP_K", K)
    nx, ny = shape
    spec = random_lti(nx, ny, seed=nx * 10 + ny)
    T = 60_001
    y = np.random.default_rng(nx + ny).standard_normal((T + 1, ny))
    plan = gpu_plan(spec, T)
    x = plan.solve_linear(to_dev(torch, y[None]))
    plan.sync()
    xo = oracle.kf_rts(ora_model(spec), y, T, spec.t0, spec.tf)
    assert rel(x[0].cpu().numpy(), xo) < TOL64


def test_lb_fp32(torch_cuda):
    torch = torch_cuda
    spec = wl.wiener_velocity()
    T = 200_000
    _, y = wl.simulate_linear(spec, T, seed=8)
    plan = gpu_plan(spec, T, dtype="f32")
    x = plan.solve_linear(to_dev(torch, y[None], dtype=torch.float32))
    plan.sync()
    assert plan.launches == LB_LAUNCHES
    xo = oracle.kf_rts(ora_model(spec), y, T, spec.t0, spec.tf)
    assert rel(x[0].cpu().numpy(), xo) < TOL32


@pytest.mark.parametrize("T,B", [(3 * TILE + 11, 1), (40 * 32 * TILE + 999, 1), (9_001, 3)])
def test_lb_smoother_covariance(torch_cuda, T, B):
    """Parallel RTS smoother covariances (map_solve_linear_cov): the plan's
    covariance chain over the tiles plus the forward recursion inside each run, against
    the oracle's textbook RTS covariance recursion (P1-cov pins it to dense conditioning)."""
    torch = torch_cuda
    spec = _wiener_offsets()
    _, y = wl.simulate_linear(spec, T, seed=T % 101, batch=B)
    y = y.reshape(B, T + 1, 2)
    plan = gpu_plan(spec, T, batch=B)
    x, P = plan.solve_linear_cov(to_dev(torch, y))
    plan.sync()
    assert plan.launches == LB_LAUNCHES
    iu = np.triu_indices(spec.nx)
    for b in range(B):
        xo, Po = oracle.kf_rts_cov(ora_model(spec), y[b], T, spec.t0, spec.tf)
        assert rel(x[b].cpu().numpy(), xo) < TOL64
        Pp = Po[:, iu[0], iu[1]]
        assert rel(P[b].cpu().numpy(), Pp) < TOL64
        assert rel_comp(P[b].cpu().numpy(), Pp) < 1e-8


def test_lb_smoother_covariance_unsupported(torch_cuda, monkeypatch):
    """Plans off the look-back path refuse map_solve_linear_cov with MAP_E_UNSUPPORTED."""
    import paper_2512_13319_b200 as pm
    torch = torch_cuda
    monkeypatch.setenv("PMAP_NO_LB", "1")
    spec = wl.wiener_velocity()
    T = 5_000
    _, y = wl.simulate_linear(spec, T, seed=1)
    with pytest.raises(pm.MapError) as ei:
        gpu_plan(spec, T).solve_linear_cov(to_dev(torch, y[None]))
    assert ei.value.status == 2


@pytest.mark.parametrize("T", [100_000, 10_000_000])
def test_lb_mixed_precision(torch_cuda, T):
    """Mixed-precision pass 2 (MAP_FLAG_MIXED): the per-node recursion in fp32
    from fp64 run carries; pass 1, the look-backs, the plan tables and all I/O fp64.
    Rounding does not accumulate across runs, so the error stays near fp32 epsilon times
    the run length (measured value in DESIGN.md), far below the fp32 variant's."""
    import paper_2512_13319_b200 as pm
    torch = torch_cuda
    spec = wl.wiener_velocity()
    _, y = wl.simulate_linear(spec, T, seed=2)
    plan = pm.Plan(T=T, t0=spec.t0, tf=spec.tf, F=spec.F, L=spec.L, W=spec.W, H=spec.H, R=spec.R, m0=spec.m0,
                   P0=spec.P0, mixed=True)
    x = plan.solve_linear(to_dev(torch, y[None]))
    plan.sync()
    assert plan.launches == LB_LAUNCHES
    xo = oracle.kf_rts(ora_model(spec), y, T, spec.t0, spec.tf)
    e = rel(x[0].cpu().numpy(), xo)
    print(f"mixed precision T={T}: relative error {e:.3e}")
    assert e < 1e-5


@pytest.mark.parametrize("T", [3 * TILE + 17, 200_003])
def test_lb_s_mask(torch_cuda, T, monkeypatch):
    """R-SMASK: for the Wiener-velocity model the two axes decouple, so S keeps exact zeros
    between them and the pass-2 node recursion skips those entries.  Against the same plan
    without the S mask (PMAP_NO_SMASK=1) the result agrees to rounding (the look-back's
    association varies run to run, R-LBDET), and both match the oracle."""
    torch = torch_cuda
    spec = wl.wiener_velocity()
    _, y = wl.simulate_linear(spec, T, seed=21)
    yd = to_dev(torch, y[None])
    x_sm = gpu_plan(spec, T).solve_linear(yd).cpu().numpy()
    monkeypatch.setenv("PMAP_NO_SMASK", "1")
    x_full = gpu_plan(spec, T).solve_linear(yd).cpu().numpy()
    xo = oracle.kf_rts(ora_model(spec), y, T, spec.t0, spec.tf)
    assert rel(x_sm[0], x_full[0]) < 1e-13
    assert rel(x_sm[0], xo) < TOL64
    assert rel_comp(x_sm[0], xo) < 1e-8


def test_lb_s_mask_not_eligible(torch_cuda):
    """A prior that couples the axes (P0 with an x-y cross term) puts non-zeros into J0
    outside the S mask: the plan must take the unmasked S path and still match the oracle."""
    torch = torch_cuda
    spec = wl.wiener_velocity()
    spec.P0 = spec.P0.copy()
    spec.P0[0, 1] = spec.P0[1, 0] = 4e-3
    T = 3 * TILE + 5
    _, y = wl.simulate_linear(spec, T, seed=22)
    plan = gpu_plan(spec, T)
    x = plan.solve_linear(to_dev(torch, y[None]))
    plan.sync()
    assert plan.launches == LB_LAUNCHES
    xo = oracle.kf_rts(ora_model(spec), y, T, spec.t0, spec.tf)
    assert rel(x[0].cpu().numpy(), xo) < TOL64


@pytest.mark.parametrize("T", [TILE + 5, 300_001])
def test_pipelined_host_solves(torch_cuda, T):
    """map_solve_linear_pipelined: five host-buffer solves in flight (distinct inputs and
    outputs, staging slots reused every second call), then one map_sync: each equals the
    oracle; a device buffer is refused."""
    import paper_2512_13319_b200 as pm
    torch = torch_cuda
    spec = _wiener_offsets()
    plan = gpu_plan(spec, T)
    ys, xs = [], []
    for k in range(5):
        _, y = wl.simulate_linear(spec, T, seed=100 + k)
        ys.append(torch.from_numpy(np.ascontiguousarray(y[None])).pin_memory())
        xs.append(torch.zeros((1, T + 1, 4), dtype=torch.float64).pin_memory())
    for k in range(5):
        plan.solve_linear_pipelined(ys[k], xs[k])
    plan.sync()
    for k in range(5):
        xo = oracle.kf_rts(ora_model(spec), ys[k][0].numpy(), T, spec.t0, spec.tf)
        assert rel(xs[k][0].numpy(), xo) < TOL64
    with pytest.raises(pm.MapError):
        plan.solve_linear_pipelined(to_dev(torch, ys[0].numpy()), xs[0])
