"""GPU parity of the SURVEY §8(f) rows built after (a)-(e):

f1  sequential on-device baselines (map_solve_sequential: RTS and two-filter, one
    thread per trajectory; sequential IEKS for nonlinear plans) vs the CPU oracle;
f4  smoother covariances (parallel two-filter combine, sequential RTS covariance
    recursion, sequential two-filter) vs the oracle's textbook RTS covariance
    recursion (itself pinned to dense Gaussian conditioning, test_oracle_pins P1-cov).

Tolerance as in test_parity_gpu.py: <= 1e-9 relative (inf-norm, per trajectory) in fp64.
"""
import numpy as np
import pytest

import oracle
import workloads as wl
from test_parity_gpu import TOL64, TOL32, gpu_plan, ora_model, random_lti, rel, rel_comp, to_dev, torch_cuda, tv_spec  # noqa: F401

pytestmark = pytest.mark.gpu


def packed(P):
    """[N, nx, nx] -> [N, nx(nx+1)/2] upper triangle, row-major (include/pmap.h layout)."""
    nx = P.shape[-1]
    iu = np.triu_indices(nx)
    return P[..., iu[0], iu[1]]


@pytest.mark.parametrize("method", [0, 1])
@pytest.mark.parametrize("case", ["wiener", "ou", "tv", "random52"])
def test_sequential_matches_oracle(torch_cuda, case, method):
    torch = torch_cuda
    T = 3001
    if case == "wiener":
        spec = wl.wiener_velocity()
        _, y = wl.simulate_linear(spec, T, seed=4)
    elif case == "ou":
        spec = wl.ornstein_uhlenbeck()
        _, y = wl.simulate_linear(spec, T, seed=5)
    elif case == "tv":
        spec = tv_spec(T)
        y = np.random.default_rng(2).standard_normal((T + 1, spec.ny))
    else:
        spec = random_lti(5, 2, seed=52)
        y = np.random.default_rng(3).standard_normal((T + 1, 2))
    xo, Po = oracle.kf_rts_cov(ora_model(spec), y, T, spec.t0, spec.tf)
    plan = gpu_plan(spec, T)
    nx = spec.nx
    Pd = torch.empty((1, T + 1, nx * (nx + 1) // 2), dtype=torch.float64, device="cuda")
    x = plan.solve_sequential(to_dev(torch, y[None]), method=method, smooth_P=Pd)
    plan.sync()
    assert rel(x[0].cpu().numpy(), xo) < TOL64
    assert rel(Pd[0].cpu().numpy(), packed(Po)) < TOL64


def test_sequential_batch_matches_parallel(torch_cuda):
    """Batched sequential baseline (one thread per trajectory, C5-shaped) = oracle, both methods."""
    torch = torch_cuda
    spec = wl.wiener_velocity()
    spec.c = np.array([0.3, -0.2, 0.1, 0.05])
    T, B = 2000, 40
    _, y = wl.simulate_linear(spec, T, seed=12, batch=B)
    xo = oracle.batch(ora_model(spec), y, T, spec.t0, spec.tf, mode=0)
    plan = gpu_plan(spec, T, batch=B)
    yd = to_dev(torch, y)
    for method in (0, 1):
        x = plan.solve_sequential(yd, method=method).cpu().numpy()
        for b in range(B):
            assert rel(x[b], xo[b]) < TOL64


@pytest.mark.parametrize("case", ["wiener", "tv", "c5_small_batch"])
def test_parallel_two_filter_smoother_covariance(torch_cuda, case):
    torch = torch_cuda
    if case == "c5_small_batch":
        spec = wl.wiener_velocity()
        T, B = 10_000, 3
        _, y = wl.simulate_linear(spec, T, seed=21, batch=B)
    else:
        T, B = 5000, 1
        if case == "wiener":
            spec = wl.wiener_velocity()
            _, y = wl.simulate_linear(spec, T, seed=7)
        else:
            spec = tv_spec(T)
            y = np.random.default_rng(8).standard_normal((T + 1, spec.ny))
        y = y[None]
    nx = spec.nx
    plan = gpu_plan(spec, T, batch=B)
    Pd = torch.empty((B, T + 1, nx * (nx + 1) // 2), dtype=torch.float64, device="cuda")
    x = plan.two_filter(to_dev(torch, y), smooth_P=Pd)
    plan.sync()
    for b in range(B):
        xo, Po = oracle.kf_rts_cov(ora_model(spec), y[b], T, spec.t0, spec.tf)
        assert rel(x[b].cpu().numpy(), xo) < TOL64
        assert rel(Pd[b].cpu().numpy(), packed(Po)) < TOL64


def test_sequential_fp32(torch_cuda):
    torch = torch_cuda
    spec = wl.wiener_velocity()
    T = 4000
    _, y = wl.simulate_linear(spec, T, seed=31)
    xo = oracle.kf_rts(ora_model(spec), y, T, spec.t0, spec.tf)
    plan = gpu_plan(spec, T, dtype="f32")
    for method in (0, 1):
        x = plan.solve_sequential(to_dev(torch, y[None], torch.float32), method=method)
        assert rel(x[0].cpu().numpy(), xo) < TOL32


@pytest.mark.parametrize("kind", [1, 2])
def test_sequential_ieks(torch_cuda, kind):
    """Sequential on-device IEKS (f1, the paper's nonlinear comparison P:625) = oracle per iterate."""
    import paper_2512_13319_b200 as pm
    torch = torch_cuda
    T = 2500
    s = wl.coordinated_turn() if kind == 1 else wl.van_der_pol()
    _, y = wl.simulate_nonlinear(s, T, seed=3)
    plan = pm.Plan(T=T, t0=s.t0, tf=s.tf, L=s.L, W=s.W, R=s.R, m0=s.m0, P0=s.P0, nl_kind=kind,
                   params=s.params)
    yd = to_dev(torch, y[None])
    for passes in (1, 4):
        xo, _ = oracle.ieks(kind, s.params, s.L, s.W, s.R, s.m0, s.P0, y, T, s.t0, s.tf, passes=passes)
        x = plan.solve_sequential(yd, method=0, passes=passes)
        assert rel(x[0].cpu().numpy(), xo) < TOL64
        xp, _ = plan.solve_nonlinear(yd, passes=passes)
        assert rel(xp[0].cpu().numpy(), x[0].cpu().numpy()) < TOL64


def test_sequential_errors(torch_cuda):
    import paper_2512_13319_b200 as pm
    torch = torch_cuda
    s = wl.coordinated_turn()
    T = 100
    _, y = wl.simulate_nonlinear(s, T, seed=1)
    plan = pm.Plan(T=T, t0=s.t0, tf=s.tf, L=s.L, W=s.W, R=s.R, m0=s.m0, P0=s.P0, nl_kind=1)
    with pytest.raises(pm.MapError):  # no sequential two-filter for nonlinear plans
        plan.solve_sequential(to_dev(torch, y[None]), method=1)
    spec = wl.wiener_velocity()
    lp = gpu_plan(spec, T)
    with pytest.raises(pm.MapError):
        lp.solve_sequential(to_dev(torch, np.zeros((1, T + 1, 2))), method=2)


@pytest.mark.parametrize("T", [3000, 100_000])
def test_vdp_om_divergence(torch_cuda, T):
    """f3: Van der Pol with the OM divergence term (params = [mu, 1]) = oracle per iterate
    (parallel and sequential); the term changes the answer (it is not silently dropped)."""
    import paper_2512_13319_b200 as pm
    torch = torch_cuda
    s = wl.van_der_pol(mu=1.5)
    _, y = wl.simulate_nonlinear(s, T, seed=17)
    yd = to_dev(torch, y[None])
    plan = pm.Plan(T=T, t0=s.t0, tf=s.tf, L=s.L, W=s.W, R=s.R, m0=s.m0, P0=s.P0, nl_kind=2,
                   params=np.array([1.5, 1.0]))
    plan0 = pm.Plan(T=T, t0=s.t0, tf=s.tf, L=s.L, W=s.W, R=s.R, m0=s.m0, P0=s.P0, nl_kind=2,
                    params=np.array([1.5]))
    for passes in (2, 10):
        xo, _ = oracle.ieks(2, [1.5, 1.0], s.L, s.W, s.R, s.m0, s.P0, y, T, s.t0, s.tf, passes=passes)
        x, _ = plan.solve_nonlinear(yd, passes=passes)
        assert rel(x[0].cpu().numpy(), xo) < TOL64
        xs = plan.solve_sequential(yd, method=0, passes=passes)
        assert rel(xs[0].cpu().numpy(), xo) < TOL64
    x0, _ = plan0.solve_nonlinear(yd, passes=10)
    assert rel(x0[0].cpu().numpy(), xo) > 1e-6


@pytest.mark.parametrize("case,T,B", [("wiener", 3000, 1), ("wiener", 100_000, 1), ("wiener_c", 20_000, 3),
                                       ("ou", 4097, 2)])
def test_euler_blocks(torch_cuda, case, T, B):
    """f2: the paper's Euler blocks (n = 10 substeps per grid interval) on the GPU
    (parallel scan and sequential baseline) = the step-by-step Euler-block oracle."""
    import paper_2512_13319_b200 as pm
    torch = torch_cuda
    n = 10
    if case.startswith("wiener"):
        spec = wl.wiener_velocity()
        if case == "wiener_c":
            spec.c = np.array([0.3, -0.2, 0.1, 0.05])
            spec.r = np.array([0.5, -0.25])
    else:
        spec = wl.ornstein_uhlenbeck()
    _, yf = wl.simulate_linear(spec, n * T, seed=T, batch=B)
    yf = yf.reshape(B, n * T + 1, spec.ny)
    plan = pm.Plan(T=T, t0=spec.t0, tf=spec.tf, F=spec.F, c=spec.c, L=spec.L, W=spec.W, H=spec.H, r=spec.r,
                   R=spec.R, m0=spec.m0, P0=spec.P0, batch=B, substeps=n)
    yd = to_dev(torch, pm.binding.euler_rows(yf, n))
    x = plan.solve_linear(yd).cpu().numpy()
    xs = plan.solve_sequential(yd, method=0).cpu().numpy()
    for b in range(B):
        xo = oracle.euler_rts(ora_model(spec), yf[b], T, n, spec.t0, spec.tf)
        assert rel(x[b], xo) < TOL64
        assert rel(xs[b], xo) < TOL64


@pytest.mark.parametrize("case,T,B", [("wiener_c", 1, 1), ("wiener_c", 3000, 1), ("wiener", 100_000, 1),
                                       ("wiener_c", 20_000, 3), ("ou", 4097, 2)])
def test_euler_refinement(torch_cuda, case, T, B):
    """f2 remainder: x* at every fine point (map_solve_linear_fine, R-REFINE) =
    the oracle's step-by-step refinement (pins P15-P17), per component, host and device
    buffers; block boundaries = the block solve."""
    import paper_2512_13319_b200 as pm
    torch = torch_cuda
    n = 10
    if case.startswith("wiener"):
        spec = wl.wiener_velocity()
        if case == "wiener_c":
            spec.c = np.array([0.3, -0.2, 0.1, 0.05])
            spec.r = np.array([0.5, -0.25])
        if T < 10:  # explicit Euler blocks need short blocks (delta H^T R^-1 H << 1): shorten the span
            spec.tf = spec.t0 + 0.01 * T
    else:
        spec = wl.ornstein_uhlenbeck()
    _, yf = wl.simulate_linear(spec, n * T, seed=T + 7, batch=B)
    yf = yf.reshape(B, n * T + 1, spec.ny)
    plan = pm.Plan(T=T, t0=spec.t0, tf=spec.tf, F=spec.F, c=spec.c, L=spec.L, W=spec.W, H=spec.H, r=spec.r,
                   R=spec.R, m0=spec.m0, P0=spec.P0, batch=B, substeps=n)
    rows = pm.binding.euler_rows(yf, n)
    yd = to_dev(torch, rows)
    xf = plan.solve_linear_fine(yd)
    plan.sync()
    xf = xf.cpu().numpy()
    xh = plan.solve_linear_fine(torch.from_numpy(np.ascontiguousarray(rows)))  # host buffers
    xb = plan.solve_linear(yd).cpu().numpy()
    for b in range(B):
        xo = oracle.euler_refine(ora_model(spec), yf[b], T, n, spec.t0, spec.tf)
        assert xf[b].shape == (n * T + 1, spec.nx)
        assert rel(xf[b], xo) < TOL64
        assert rel_comp(xf[b], xo) < 1e-8
        assert rel(xf[b][::n], xb[b]) < 1e-12
        assert rel(xh[b].numpy(), xo) < TOL64


def test_euler_refinement_unsupported(torch_cuda):
    """map_solve_linear_fine on a plan without Euler blocks: MAP_E_UNSUPPORTED."""
    import paper_2512_13319_b200 as pm
    torch = torch_cuda
    spec = wl.wiener_velocity()
    T = 100
    _, y = wl.simulate_linear(spec, T, seed=1)
    plan = gpu_plan(spec, T)
    with pytest.raises(pm.MapError) as ei:
        pm.map_solve_linear_fine(plan.handle, to_dev(torch, y[None]),
                                 torch.empty((1, T + 1, 4), dtype=torch.float64, device="cuda"))
    assert ei.value.status == 2


def test_euler_blocks_errors(torch_cuda):
    import paper_2512_13319_b200 as pm
    torch = torch_cuda
    spec = wl.wiener_velocity()
    T = 100
    plan = pm.Plan(T=T, t0=spec.t0, tf=spec.tf, F=spec.F, L=spec.L, W=spec.W, H=spec.H, R=spec.R, m0=spec.m0,
                   P0=spec.P0, substeps=10)
    with pytest.raises(pm.MapError):  # two-filter needs separable measurements
        plan.two_filter(to_dev(torch, np.zeros((1, T + 1, 20))))
    with pytest.raises(pm.MapError):  # only n = 10 is compiled
        pm.Plan(T=T, t0=spec.t0, tf=spec.tf, F=spec.F, L=spec.L, W=spec.W, H=spec.H, R=spec.R, m0=spec.m0,
                P0=spec.P0, substeps=7)
    # Euler blocks are LTI-only: a time-varying model with substeps > 1 must be refused
    # (it used to fall through to the time-varying path and read y wrongly)
    Ftv = np.repeat(spec.F[None], T + 1, axis=0)
    with pytest.raises(pm.MapError) as ei:
        pm.Plan(T=T, t0=spec.t0, tf=spec.tf, F=Ftv, L=spec.L, W=spec.W, H=spec.H, R=spec.R, m0=spec.m0,
                P0=spec.P0, substeps=10)
    assert ei.value.status == 2  # MAP_E_UNSUPPORTED


def test_binding_rejects_bad_buffers(torch_cuda):
    """The C ABI cannot check sizes: the binding validates dtype, contiguity, element
    count and model shapes before any pointer crosses it."""
    import paper_2512_13319_b200 as pm
    torch = torch_cuda
    spec = wl.wiener_velocity()
    T = 1000
    plan = gpu_plan(spec, T)
    good = torch.zeros((1, T + 1, 2), dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):  # fp32 buffer on an f64 plan
        plan.solve_linear(good.float())
    with pytest.raises(ValueError):  # too short
        plan.solve_linear(good[:, :T])
    with pytest.raises(ValueError):  # non-contiguous view
        plan.solve_linear(torch.zeros((1, T + 1, 4), dtype=torch.float64, device="cuda")[:, :, :2])
    with pytest.raises(ValueError):  # x_map of the wrong size
        plan.solve_linear(good, x_map=torch.empty((1, T + 1, 3), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):  # H of the wrong shape
        pm.Plan(T=T, t0=spec.t0, tf=spec.tf, F=spec.F, L=spec.L, W=spec.W, H=spec.H[:, :3], R=spec.R, m0=spec.m0,
                P0=spec.P0)
    plan.solve_linear(good)  # the valid call still works


def test_nonlinear_diverged_status(torch_cuda):
    """tol > 0 that is not reached within `passes` returns MAP_E_DIVERGED with the last
    iterate in x_map; the device-side stop reports the pass count."""
    import paper_2512_13319_b200 as pm
    torch = torch_cuda
    s = wl.van_der_pol()
    T = 2000
    _, y = wl.simulate_nonlinear(s, T, seed=3)
    plan = pm.Plan(T=T, t0=s.t0, tf=s.tf, L=s.L, W=s.W, R=s.R, m0=s.m0, P0=s.P0, nl_kind=2, params=s.params)
    yd = to_dev(torch, y[None])
    x = torch.empty((1, T + 1, 2), dtype=torch.float64, device="cuda")
    with pytest.raises(pm.MapError) as ei:
        plan.solve_nonlinear(yd, passes=1, tol=1e-300, x_map=x)
    assert ei.value.status == 6  # MAP_E_DIVERGED
    xo, _ = oracle.ieks(2, s.params, s.L, s.W, s.R, s.m0, s.P0, y, T, s.t0, s.tf, passes=1)
    assert rel(x[0].cpu().numpy(), xo) < TOL64  # the last (only) iterate was returned


@pytest.mark.parametrize("T", [5000, 300_001])
def test_structural_zero_masks_bit_identical(torch_cuda, T, monkeypatch):
    """R-MASK: the Wiener-velocity kernels specialised on the structural zeros of A and U
    skip only terms whose factor is exactly 0, so they match the dense kernels bit for
    bit (and the oracle to 1e-9)."""
    torch = torch_cuda
    spec = wl.wiener_velocity()
    _, y = wl.simulate_linear(spec, T, seed=77)
    yd = to_dev(torch, y[None])
    x_lb_mask = gpu_plan(spec, T).solve_linear(yd).cpu().numpy()
    monkeypatch.setenv("PMAP_NO_LB", "1")  # the scan hierarchy is deterministic: bit for bit
    x_mask = gpu_plan(spec, T).solve_linear(yd).cpu().numpy()
    monkeypatch.setenv("PMAP_NO_MASK", "1")
    x_dense = gpu_plan(spec, T).solve_linear(yd).cpu().numpy()
    assert np.array_equal(x_mask, x_dense)
    assert rel(x_mask[0], oracle.kf_rts(ora_model(spec), y, T, spec.t0, spec.tf)) < TOL64
    # the look-back path (masked node step and forward recovery) agrees to rounding: its
    # look-back depth, hence the association of a few sums, varies run to run
    monkeypatch.delenv("PMAP_NO_LB")
    x_lb_dense = gpu_plan(spec, T).solve_linear(yd).cpu().numpy()
    assert rel(x_lb_mask[0], x_lb_dense[0]) < 1e-13
    assert rel(x_lb_mask[0], x_mask[0]) < 1e-12


@pytest.mark.parametrize("method", ["rts", "tf", "shard_nccl"])
def test_graph_replay_matches_eager(torch_cuda, method, monkeypatch):
    """Repeated solves on the same device buffers are captured into a CUDA graph (second
    call) and replayed (third call on); every call must equal the eager launches exactly."""
    import paper_2512_13319_b200 as pm
    torch = torch_cuda
    spec = wl.wiener_velocity()
    T = 70_001
    _, y = wl.simulate_linear(spec, T, seed=5)
    yd = to_dev(torch, y[None])
    comm = None
    created = False
    if method == "shard_nccl":
        import os
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29561")
        if not dist.is_initialized():
            dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
            created = True
        comm = dist.group.WORLD._get_backend(torch.device("cuda", 0))._comm_ptr()
        monkeypatch.setenv("PMAP_FORCE_SHARD", "1")
    try:
        _graph_replay_body(torch, pm, spec, T, y, yd, comm, method)
    finally:
        if created:
            import torch.distributed as dist
            dist.destroy_process_group()


def _graph_replay_body(torch, pm, spec, T, y, yd, comm, method):
    plan = pm.Plan(T=T, t0=spec.t0, tf=spec.tf, F=spec.F, L=spec.L, W=spec.W, H=spec.H, R=spec.R, m0=spec.m0,
                   P0=spec.P0, nccl_comm=comm)
    x = torch.empty((1, T + 1, 4), dtype=torch.float64, device="cuda")
    run = (lambda: plan.two_filter(yd, x)) if method == "tf" else (lambda: plan.solve_linear(yd, x))
    outs = []
    for _ in range(4):
        x.zero_()
        run()
        plan.sync()
        outs.append(x.cpu().numpy().copy())
    for o in outs[1:]:
        if method in ("rts", "shard_nccl"):  # look-back paths: reproducible to rounding (R-LBDET)
            assert rel(o[0], outs[0][0]) < 1e-13
        else:
            assert np.array_equal(o, outs[0])
    xo = oracle.kf_rts(ora_model(spec), y, T, spec.t0, spec.tf)
    assert rel(outs[-1][0], xo) < TOL64


@pytest.mark.parametrize("case,T,B", [("rts", 300_001, 1), ("rts", 10_000_000, 1), ("tf", 40_000, 3),
                                       ("rts_k8", 9_000, 2), ("rts", 2_048 * 128 * 3, 1), ("rts", 2_048 * 3 - 1, 1)])
def test_lti_data_only_scans_match_general(torch_cuda, case, T, B, monkeypatch):
    """The data-only LTI tile / group scans (pmap_lti_scan.cuh) agree with the general
    combine-based scans to rounding (<= 1e-12 relative) and with the oracle (1e-9)."""
    torch = torch_cuda
    monkeypatch.setenv("PMAP_NO_LB", "1")  # the scan hierarchy (the look-back path has its own tests)
    spec = wl.wiener_velocity()
    spec.c = np.array([0.3, -0.2, 0.1, 0.05])
    if case == "rts_k8":
        monkeypatch.setenv("PMAP_K", "8")
    _, y = wl.simulate_linear(spec, T, seed=T % 1000, batch=B)
    y = y.reshape(B, T + 1, 2)
    yd = to_dev(torch, y)
    run = (lambda pl: pl.two_filter(yd)) if case == "tf" else (lambda pl: pl.solve_linear(yd))
    x_scan = run(gpu_plan(spec, T, batch=B)).cpu().numpy()
    monkeypatch.setenv("PMAP_NO_LTI_SCAN", "1")
    x_gen = run(gpu_plan(spec, T, batch=B)).cpu().numpy()
    for b in range(B):
        assert rel(x_scan[b], x_gen[b]) < 1e-12
        if T <= 400_000:
            assert rel(x_scan[b], oracle.kf_rts(ora_model(spec), y[b], T, spec.t0, spec.tf)) < TOL64
