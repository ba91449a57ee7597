"""Pins of the CPU oracle against what the paper and the mathematics fix (CPU only).

Each test names the pin id of DESIGN.md "Oracle pins" (P1..P12) and the passage
it follows.  None of these re-types the oracle's own recursion: they use dense
Gaussian conditioning, a direct solve of the discretised objective, closed forms
of the continuous problem, Moebius/linear-fractional identities, a cross-method
identity, finite differences and autograd.
"""
import json
import os

import numpy as np
import pytest

import oracle
import workloads as wl

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rel_inf(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / np.abs(np.asarray(b)).max()


def tv_model(T, nx=4, ny=2, nw=2, seed=3, full_rank_q=False, with_offsets=True):
    """A random time-varying linear-affine model with node arrays."""
    rng = np.random.default_rng(seed)
    N = T + 1
    F = 0.5 * rng.standard_normal((N, nx, nx)) + np.linspace(0, 1, N)[:, None, None] * np.eye(nx)
    nw_ = nx if full_rank_q else nw
    L = rng.standard_normal((N, nx, nw_))
    if full_rank_q:  # well-conditioned diffusion so the dense reference solve is accurate
        L = np.eye(nx)[None] + 0.3 * L
    W = np.stack([np.eye(nw_) * (1 + 0.5 * np.sin(k)) for k in range(N)])
    H = rng.standard_normal((N, ny, nx))
    a = rng.standard_normal((ny, ny))
    R = np.stack([a @ a.T + np.eye(ny) * (1 + 0.1 * k / N) for k in range(N)])
    c = rng.standard_normal((N, nx)) if with_offsets else None
    r = rng.standard_normal((N, ny)) if with_offsets else None
    m0 = rng.standard_normal(nx)
    b = rng.standard_normal((nx, nx))
    P0 = b @ b.T + np.eye(nx)
    return oracle.LinearModel(F, L, W, H, R, m0, P0, c=c, r=r)


def node(a, i, nd):
    return a if a.ndim == nd else a[i]


def dense_conditioning(md, y, T, t0, tf):
    """P1: E[x_{0..T} | y_{0..T}] by joint-Gaussian conditioning of the discrete model.

    x_0 = m0 + z_0, x_i = Phi_i (x_{i-1} + dt c_i + w_i) with Phi_i = (I - dt F_i)^{-1},
    w_i ~ N(0, dt Q_i); y_i = H_i x_i + r_i + nu_i, nu_i ~ N(0, R_i / dt)."""
    nx, ny, N = md.nx, md.ny, T + 1
    dt = (tf - t0) / T
    mu = np.zeros((N, nx))
    G = np.zeros((N * nx, N * nx))          # x = mu + G z
    Sz = np.zeros((N * nx, N * nx))
    mu[0] = md.m0
    G[:nx, :nx] = np.eye(nx)
    Sz[:nx, :nx] = md.P0
    for i in range(1, N):
        Phi = np.linalg.inv(np.eye(nx) - dt * node(md.F, i, 2))
        c = np.zeros(nx) if md.c is None else node(md.c, i, 1)
        mu[i] = Phi @ (mu[i - 1] + dt * c)
        G[i * nx:(i + 1) * nx] = Phi @ G[(i - 1) * nx:i * nx]
        G[i * nx:(i + 1) * nx, i * nx:(i + 1) * nx] += Phi
        L, W = node(md.L, i, 2), node(md.W, i, 2)
        Sz[i * nx:(i + 1) * nx, i * nx:(i + 1) * nx] = dt * L @ W @ L.T
    SX = G @ Sz @ G.T
    Hb = np.zeros((N * ny, N * nx))
    SR = np.zeros((N * ny, N * ny))
    my = np.zeros(N * ny)
    for i in range(N):
        Hi = node(md.H, i, 2)
        Hb[i * ny:(i + 1) * ny, i * nx:(i + 1) * nx] = Hi
        SR[i * ny:(i + 1) * ny, i * ny:(i + 1) * ny] = node(md.R, i, 2) / dt
        r = np.zeros(ny) if md.r is None else node(md.r, i, 1)
        my[i * ny:(i + 1) * ny] = Hi @ mu[i] + r
    SY = Hb @ SX @ Hb.T + SR
    return SX, Hb, SY, mu, my


@pytest.mark.parametrize("case", ["wiener", "tv_offsets", "ou"])
def test_P1_dense_conditioning(case):
    """P1 -- oracle x_map (and filter means/covariances) = exact Gaussian conditioning."""
    T, t0, tf = 40, 0.0, 2.0
    if case == "wiener":
        s = wl.wiener_velocity()
        md = oracle.LinearModel(s.F, s.L, s.W, s.H, s.R, s.m0, s.P0)
        _, y = wl.simulate_linear(s, T, seed=1)
    elif case == "ou":
        s = wl.ornstein_uhlenbeck()
        md = oracle.LinearModel(s.F, s.L, s.W, s.H, s.R, s.m0, s.P0)
        _, y = wl.simulate_linear(s, T, seed=2)
    else:
        md = tv_model(T)
        y = np.random.default_rng(5).standard_normal((T + 1, md.ny))
    x, fm, fP = oracle.kf_rts(md, y, T, t0, tf, want_filter=True)
    SX, Hb, SY, mu, my = dense_conditioning(md, y, T, t0, tf)
    post = mu.reshape(-1) + SX @ Hb.T @ np.linalg.solve(SY, y.reshape(-1) - my)
    assert rel_inf(x.reshape(-1), post) < 1e-12
    # filter at node i = conditioning on y_0..y_i only
    nx, ny = md.nx, md.ny
    for i in (0, 1, T // 2, T):
        k = (i + 1) * ny
        Sxy = SX[i * nx:(i + 1) * nx] @ Hb[:k].T
        gain = np.linalg.solve(SY[:k, :k], Sxy.T).T
        m_i = mu[i] + gain @ (y.reshape(-1)[:k] - my[:k])
        P_i = SX[i * nx:(i + 1) * nx, i * nx:(i + 1) * nx] - gain @ Sxy.T
        assert rel_inf(fm[i], m_i) < 1e-11
        assert rel_inf(fP[i], P_i) < 1e-10


@pytest.mark.parametrize("case", ["wiener", "tv_offsets", "ou"])
def test_P1_smoother_covariance_dense(case):
    """P1-cov -- oracle RTS smoother covariances = the exact posterior
    covariance Cov[x_i | y_0..y_T] of the discrete model by dense conditioning."""
    T, t0, tf = 40, 0.0, 2.0
    if case == "wiener":
        s = wl.wiener_velocity()
        md = oracle.LinearModel(s.F, s.L, s.W, s.H, s.R, s.m0, s.P0)
        _, y = wl.simulate_linear(s, T, seed=1)
    elif case == "ou":
        s = wl.ornstein_uhlenbeck()
        md = oracle.LinearModel(s.F, s.L, s.W, s.H, s.R, s.m0, s.P0)
        _, y = wl.simulate_linear(s, T, seed=2)
    else:
        md = tv_model(T)
        y = np.random.default_rng(5).standard_normal((T + 1, md.ny))
    x, Ps = oracle.kf_rts_cov(md, y, T, t0, tf)
    assert rel_inf(x, oracle.kf_rts(md, y, T, t0, tf)) == 0.0
    SX, Hb, SY, mu, my = dense_conditioning(md, y, T, t0, tf)
    post_cov = SX - SX @ Hb.T @ np.linalg.solve(SY, Hb @ SX)
    nx = md.nx
    for i in range(T + 1):
        blk = post_cov[i * nx:(i + 1) * nx, i * nx:(i + 1) * nx]
        assert np.abs(Ps[i] - blk).max() <= 1e-11 * np.abs(blk).max(), i
        assert np.array_equal(Ps[i], Ps[i].T)
        assert np.linalg.eigvalsh(Ps[i]).min() > 0


def test_P2_discretised_objective_minimiser():
    """P2 -- x_map minimises the discretised OM/LQT objective
    J(x) = 1/2|x0-m0|^2_{P0^-1} + sum_i 1/2|x_{i-1} - A_i x_i - b_i|^2_{(dt Q_i)^-1}
           + sum_i dt/2 |y_i - H_i x_i - r_i|^2_{R_i^-1},  A_i = I - dt F_i, b_i = -dt c_i.
    Solved directly as one dense (block-tridiagonal) normal-equation system."""
    T, t0, tf = 60, 0.0, 1.5
    md = tv_model(T, nx=3, ny=2, full_rank_q=True, seed=11)
    y = np.random.default_rng(4).standard_normal((T + 1, md.ny))
    nx, N, dt = md.nx, T + 1, (tf - t0) / T
    Hs = np.zeros((N * nx, N * nx))
    g = np.zeros(N * nx)
    P0i = np.linalg.inv(md.P0)
    Hs[:nx, :nx] += P0i
    g[:nx] += P0i @ md.m0
    for i in range(1, N):
        A = np.eye(nx) - dt * md.F[i]
        b = -dt * md.c[i]
        Qi = np.linalg.inv(dt * md.L[i] @ md.W[i] @ md.L[i].T)
        D = np.zeros((nx, N * nx))           # residual = D x - b
        D[:, (i - 1) * nx:i * nx] = np.eye(nx)
        D[:, i * nx:(i + 1) * nx] = -A
        Hs += D.T @ Qi @ D
        g += D.T @ Qi @ b
    for i in range(N):
        Ri = dt * np.linalg.inv(md.R[i])
        sl = slice(i * nx, (i + 1) * nx)
        Hs[sl, sl] += md.H[i].T @ Ri @ md.H[i]
        g[sl] += md.H[i].T @ Ri @ (y[i] - md.r[i])
    xd = np.linalg.solve(Hs, g)
    x = oracle.kf_rts(md, y, T, t0, tf)
    assert rel_inf(x.reshape(-1), xd) < 1e-11


def ou_closed_form(theta, q, R, m0, P0, yc, tf, t):
    """Continuous OU MAP with constant y (Euler--Lagrange of P:80-97):
    x'' = lam^2 x - (q/R) y, x' + theta x = 0 at tf, (x' + theta x)/q = (x - m0)/P0 at 0."""
    lam = np.sqrt(theta ** 2 + q / R)
    xp = (q / R) * yc / lam ** 2
    # x = xp + A e^{lam (t - tf)} + B e^{-lam t}   (scaled exponentials)
    e = np.exp(-lam * tf)
    M = np.array([
        [lam + theta, (-lam + theta) * e],                           # at tf
        [(lam + theta - q / P0) * e, -lam + theta - q / P0],         # at 0
    ])
    rhs = np.array([-theta * xp, -(theta - q / P0) * xp - q / P0 * m0])
    A, B = np.linalg.solve(M, rhs)
    return xp + A * np.exp(lam * (t - tf)) + B * np.exp(-lam * t)


def ou_kb_variance(theta, q, R, P0, t):
    """Kalman--Bucy variance of the scalar OU: Riccati with constant coefficients."""
    lam = np.sqrt(theta ** 2 + q / R)
    Pp, Pm = R * (-theta + lam), R * (-theta - lam)
    K = (P0 - Pp) / (P0 - Pm)
    E = K * np.exp(-2 * lam * t)
    return (Pp - Pm * E) / (1 - E)


def test_P3_ou_continuous_limit_first_order():
    """P3 -- discrete MAP and filter variance converge at first order to the continuous
    OU closed forms: error ratio in [1.9, 2.1] per halving of dt."""
    s = wl.ornstein_uhlenbeck()
    th, q, R, m0, P0, yc, tf = 1.0, 2.0, 0.1, 1.0, 1.0, 0.7, 5.0
    md = oracle.LinearModel(s.F, s.L, s.W, s.H, s.R, s.m0, s.P0)
    errs, perrs = [], []
    for T in (1600, 3200, 6400, 12800):
        t = np.linspace(0, tf, T + 1)
        x, _, fP = oracle.kf_rts(md, np.full((T + 1, 1), yc), T, 0.0, tf, want_filter=True)
        errs.append(np.abs(x[:, 0] - ou_closed_form(th, q, R, m0, P0, yc, tf, t)).max())
        perrs.append(np.abs(fP[:, 0, 0] - ou_kb_variance(th, q, R, P0, t)).max())
    for e in (errs, perrs):
        ratios = np.array(e[:-1]) / np.array(e[1:])
        assert np.all((ratios > 1.9) & (ratios < 2.1)), (e, ratios)
    assert errs[-1] < 5e-4



def test_P13_euler_blocks():
    """P13 -- the paper-faithful Euler-block oracle (T blocks of n
    Euler substeps of P:416-427): (a) n = 1 is the exact discrete model (= the
    covariance-form KF/RTS, <= 1e-12); (b) at fixed T the block-boundary MAP converges at
    first order in the substep (ratio in [1.9, 2.1] per doubling of n) to the continuous
    OU Euler--Lagrange closed form; (c) with the printed sign of dA/ds it does
    not converge, so the pin detects that error."""
    s = wl.wiener_velocity()
    md = oracle.LinearModel(s.F, s.L, s.W, s.H, s.R, s.m0, s.P0, c=np.array([0.3, -0.2, 0.1, 0.05]))
    T = 300
    _, y = wl.simulate_linear(s, T, seed=1)
    assert rel_inf(oracle.euler_rts(md, y, T, 1, 0.0, 5.0), oracle.kf_rts(md, y, T, 0.0, 5.0)) < 1e-12
    o = wl.ornstein_uhlenbeck()
    mo = oracle.LinearModel(o.F, o.L, o.W, o.H, o.R, o.m0, o.P0)
    th, q, R, m0, P0, yc, tf = 1.0, 2.0, 0.1, 1.0, 1.0, 0.7, 5.0
    T = 100
    xc = ou_closed_form(th, q, R, m0, P0, yc, tf, np.linspace(0, tf, T + 1))
    for printed in (False, True):
        errs = np.array([np.abs(oracle.euler_rts(mo, np.full((n * T + 1, 1), yc), T, n, 0.0, tf,
                                                 g6_printed=printed)[:, 0] - xc).max() for n in (4, 8, 16, 32, 64)])
        ratios = errs[:-1] / errs[1:]
        if printed:
            assert errs[-1] > 0.05 and np.all(ratios < 1.5), (errs, ratios)
        else:
            assert np.all((ratios > 1.9) & (ratios < 2.1)) and errs[-1] < 1e-3, (errs, ratios)

def test_P4_scalar_moebius_closed_form():
    """P4 -- scalar discrete filter variance = linear-fractional (Moebius) power:
    P_i = M^i (P_{0|0}, 1), M = [[R_d Phi^2, R_d Q_d], [Phi^2, Q_d + R_d]],
    Phi = 1/(1 + theta dt), Q_d = Phi^2 dt q, R_d = R/dt."""
    th, q, R, m0, P0, T, tf = 1.0, 2.0, 0.1, 1.0, 1.0, 200, 5.0
    s = wl.ornstein_uhlenbeck(th, q, R, m0, P0, tf)
    md = oracle.LinearModel(s.F, s.L, s.W, s.H, s.R, s.m0, s.P0)
    y = np.random.default_rng(0).standard_normal((T + 1, 1))
    _, _, fP = oracle.kf_rts(md, y, T, 0.0, tf, want_filter=True)
    dt = tf / T
    Phi = 1 / (1 + th * dt)
    Qd, Rd = Phi ** 2 * dt * q, R / dt
    M = np.array([[Rd * Phi ** 2, Rd * Qd], [Phi ** 2, Qd + Rd]])
    P00 = P0 * Rd / (P0 + Rd)
    for i in (0, 1, 7, 50, T):
        v = np.linalg.matrix_power(M, i) @ np.array([P00, 1.0])
        assert abs(fP[i, 0, 0] - v[0] / v[1]) < 1e-14
    # G30: F = 0, Q = H = R = P0 = 1 -> P_{0|0} = 1/(1+dt), P_inf = (-dt + sqrt(dt^2+4))/2
    for dt_, T_ in ((0.1, 400), (0.01, 4000)):
        md1 = oracle.LinearModel([[0.0]], [[1.0]], [[1.0]], [[1.0]], [[1.0]], [0.0], [[1.0]])
        _, _, fP1 = oracle.kf_rts(md1, np.zeros((T_ + 1, 1)), T_, 0.0, dt_ * T_, want_filter=True)
        assert abs(fP1[0, 0, 0] - 1 / (1 + dt_)) < 1e-15
        assert abs(fP1[-1, 0, 0] - (-dt_ + np.sqrt(dt_ ** 2 + 4)) / 2) < 1e-12


@pytest.mark.parametrize("case", ["wiener", "tv_offsets"])
def test_P5_two_filter_equals_rts(case):
    """P5 -- two-filter smoother = RTS smoother."""
    if case == "wiener":
        s = wl.wiener_velocity()
        T = 20_000
        md = oracle.LinearModel(s.F, s.L, s.W, s.H, s.R, s.m0, s.P0)
        _, y = wl.simulate_linear(s, T, seed=7)
        t0, tf = 0.0, 5.0
    else:
        T, t0, tf = 300, 0.0, 3.0
        md = tv_model(T, seed=9)
        y = np.random.default_rng(1).standard_normal((T + 1, md.ny))
    x = oracle.kf_rts(md, y, T, t0, tf)
    x2 = oracle.two_filter(md, y, T, t0, tf)
    assert rel_inf(x2, x) < 1e-12


def test_P5b_batch_equals_single():
    s = wl.wiener_velocity()
    T, B = 500, 6
    md = oracle.LinearModel(s.F, s.L, s.W, s.H, s.R, s.m0, s.P0)
    _, y = wl.simulate_linear(s, T, seed=2, batch=B)
    xb = oracle.batch(md, y, T, 0.0, 5.0, mode=0)
    xt = oracle.batch(md, y, T, 0.0, 5.0, mode=1)
    for b in range(B):
        assert np.array_equal(xb[b], oracle.kf_rts(md, y[b], T, 0.0, 5.0))
        assert rel_inf(xt[b], xb[b]) < 1e-12


def test_P6_wiener_continuous_riccati_first_order():
    """P6 -- Wiener-velocity filter covariance converges at first order to the
    Kalman--Bucy Riccati ODE, integrated by scipy at tight tolerance."""
    from scipy.integrate import solve_ivp
    s = wl.wiener_velocity()
    Q = s.L @ s.W @ s.L.T
    Ri = np.linalg.inv(s.R)

    def rhs(t, p):
        P = p.reshape(4, 4)
        return (s.F @ P + P @ s.F.T + Q - P @ s.H.T @ Ri @ s.H @ P).reshape(-1)

    tf = 1.0
    sol = solve_ivp(rhs, (0, tf), s.P0.reshape(-1), rtol=1e-12, atol=1e-14, dense_output=True)
    md = oracle.LinearModel(s.F, s.L, s.W, s.H, s.R, s.m0, s.P0)
    errs = []
    for T in (500, 1000, 2000):
        _, _, fP = oracle.kf_rts(md, np.zeros((T + 1, 2)), T, 0.0, tf, want_filter=True)
        t = np.linspace(0, tf, T + 1)
        ref = sol.sol(t).T.reshape(-1, 4, 4)
        errs.append(np.abs(fP - ref).max())
    ratios = np.array(errs[:-1]) / np.array(errs[1:])
    assert np.all((ratios > 1.85) & (ratios < 2.15)), (errs, ratios)


def test_P7_covariances_spd():
    """P7 -- filter covariances symmetric positive definite at every node."""
    s = wl.wiener_velocity()
    T = 10_000
    md = oracle.LinearModel(s.F, s.L, s.W, s.H, s.R, s.m0, s.P0)
    _, y = wl.simulate_linear(s, T, seed=3)
    _, _, fP = oracle.kf_rts(md, y, T, 0.0, 5.0, want_filter=True)
    assert np.array_equal(fP, np.transpose(fP, (0, 2, 1)))
    assert np.linalg.eigvalsh(fP).min() > 0


def test_P8_linear_model_through_ieks():
    """P8 -- Van der Pol with mu = 0 is linear (harmonic oscillator): pass 1 of the
    iterated linearisation equals the linear MAP; pass 2 is a fixed point."""
    s = wl.van_der_pol(mu=0.0)
    T = 2000
    _, y = wl.simulate_nonlinear(s, T, seed=4)
    x, delta = oracle.ieks(2, [0.0], s.L, s.W, s.R, s.m0, s.P0, y, T, 0.0, 5.0, passes=2)
    md = oracle.LinearModel([[0.0, 1.0], [-1.0, 0.0]], s.L, s.W, [[1.0, 0.0]], s.R, s.m0, s.P0)
    xl = oracle.kf_rts(md, y, T, 0.0, 5.0)
    assert rel_inf(x, xl) < 1e-12
    assert delta[1] < 1e-12 * np.abs(x).max()


def test_P9_nonlinear_model_functions():
    """P9 -- CT drift/measurement Jacobians vs central differences; h(3,4,..)."""
    g = json.load(open(os.path.join(GOLD, "coordinated_turn_P588-623.json")))
    assert np.allclose(oracle.ct_h(g["h_at_3_4"]["x"]), g["h_at_3_4"]["h"], rtol=0, atol=1e-15)
    rng = np.random.default_rng(0)
    for _ in range(20):
        x = rng.standard_normal(5) + np.array([5, 5, 0, 0.3, 0])
        for fn, jac, m in ((oracle.ct_f, oracle.ct_dfdx, 5), (oracle.ct_h, oracle.ct_dhdx, 2)):
            Jn = np.zeros((m, 5))
            for k in range(5):
                e = np.zeros(5)
                e[k] = 1e-6 * (1 + abs(x[k]))
                Jn[:, k] = (fn(x + e) - fn(x - e)) / (2 * e[k])
            assert np.allclose(jac(x), Jn, atol=1e-8)
        mu = 1.3
        xv = rng.standard_normal(2)
        Jn = np.zeros((2, 2))
        for k in range(2):
            e = np.zeros(2)
            e[k] = 1e-6
            Jn[:, k] = (oracle.vdp_f(mu, xv + e) - oracle.vdp_f(mu, xv - e)) / 2e-6
        assert np.allclose(oracle.vdp_dfdx(mu, xv), Jn, atol=1e-8)
    assert np.allclose(oracle.ct_f([1, 2, 3, 4, 5]), [3, 4, -20, 15, 0])


def test_P10_long_double_self_error():
    """P10 -- the fp64 oracle's own rounding floor at long horizons, measured against
    the same recursion in long double (80-bit): must stay far below the 1e-9 budget."""
    s = wl.wiener_velocity()
    T = int(os.environ.get("PMAP_P10_T", "200000"))
    md = oracle.LinearModel(s.F, s.L, s.W, s.H, s.R, s.m0, s.P0)
    _, y = wl.simulate_linear(s, T, seed=0)
    x = oracle.kf_rts(md, y, T, 0.0, 5.0)
    xl = oracle.kf_rts(md, y, T, 0.0, 5.0, long_double=True)
    assert rel_inf(x, xl) < 1e-11


def test_P11_ieks_fixed_point_is_stationary():
    """P11 -- the iterated-linearisation fixed point (Gauss--Newton) is a stationary
    point of the nonlinear discretised objective; checked by torch autograd on a
    coordinated-turn variant with full-rank diffusion (so the objective is unconstrained)."""
    import torch
    s = wl.coordinated_turn()
    L = np.diag([0.05, 0.05, 0.2, 0.2, 0.05])
    T, tf = 150, 1.5
    _, y = wl.simulate_nonlinear(wl.models.NonlinearSpec("ct", 1, 5, 2, L, np.eye(5), s.R, s.m0, s.P0,
                                                         tf=tf), T, seed=5)
    x, delta = oracle.ieks(1, None, L, np.eye(5), s.R, s.m0, s.P0, y, T, 0.0, tf, passes=30)
    assert delta[-1] < 1e-11
    dt = tf / T
    X = torch.tensor(x, requires_grad=True)
    Y = torch.tensor(y)
    Qi = torch.tensor(np.linalg.inv(dt * L @ L.T))
    Ri = torch.tensor(dt * np.linalg.inv(s.R))
    P0i = torch.tensor(np.linalg.inv(s.P0))
    m0 = torch.tensor(s.m0)
    f = torch.stack([X[:, 2], X[:, 3], -X[:, 4] * X[:, 3], X[:, 4] * X[:, 2], torch.zeros(T + 1, dtype=X.dtype)], 1)
    e = X[:-1] - X[1:] + dt * f[1:]                        # x_{i-1} - (x_i - dt f(x_i))
    h = torch.stack([torch.sqrt(X[:, 0] ** 2 + X[:, 1] ** 2), torch.atan2(X[:, 1], X[:, 0])], 1)
    res = Y - h
    res = torch.stack([res[:, 0], torch.remainder(res[:, 1] + np.pi, 2 * np.pi) - np.pi], 1)
    d0 = X[0] - m0
    J = 0.5 * d0 @ P0i @ d0 + 0.5 * torch.einsum("ia,ab,ib->", e, Qi, e) + 0.5 * torch.einsum("ia,ab,ib->", res, Ri, res)
    (g,) = torch.autograd.grad(J, X)
    scale = np.abs(np.linalg.inv(dt * L @ L.T)).max() * np.abs(x).max()
    assert g.abs().max().item() < 1e-9 * scale


@pytest.mark.parametrize("om_div", [0.0, 1.0])
def test_P12_om_divergence_fixed_point_is_stationary(om_div):
    """P12 -- with params = [mu, 1] the iterated-linearisation fixed point is a
    stationary point of the discretised Onsager--Machlup functional INCLUDING the
    divergence term 1/2 int div f dt, sum_{i>=1} dt/2 mu (1 - x_{i,0}^2) for Van der
    Pol; with params = [mu, 0] it is stationary for the functional without it (IEKS),
    and each is NOT stationary for the other (so a dropped term or a sign error fails).
    Full-rank diffusion so the objective is unconstrained; torch autograd."""
    import torch
    s = wl.van_der_pol()
    mu = 1.5
    L = np.diag([0.3, 1.0])
    W = np.array([[0.5]])[0, 0] * np.eye(2)
    T, tf = 200, 2.0
    spec = wl.models.NonlinearSpec("vdp", 2, 2, 1, L, W, s.R, s.m0, s.P0, params=np.array([mu]), tf=tf)
    _, y = wl.simulate_nonlinear(spec, T, seed=9)
    x, delta = oracle.ieks(2, [mu, om_div], L, W, s.R, s.m0, s.P0, y, T, 0.0, tf, passes=40)
    assert delta[-1] < 1e-11
    dt = tf / T
    X = torch.tensor(x, requires_grad=True)
    Y = torch.tensor(y).reshape(T + 1, 1)
    Qi = torch.tensor(np.linalg.inv(dt * L @ W @ L.T))
    Ri = torch.tensor(dt * np.linalg.inv(s.R))
    P0i = torch.tensor(np.linalg.inv(s.P0))
    m0 = torch.tensor(s.m0)
    f = torch.stack([X[:, 1], mu * (1 - X[:, 0] ** 2) * X[:, 1] - X[:, 0]], 1)
    e = X[:-1] - X[1:] + dt * f[1:]
    res = Y - X[:, :1]
    d0 = X[0] - m0
    J = 0.5 * d0 @ P0i @ d0 + 0.5 * torch.einsum("ia,ab,ib->", e, Qi, e) + 0.5 * torch.einsum("ia,ab,ib->", res, Ri, res)
    div = 0.5 * dt * torch.sum(mu * (1 - X[1:, 0] ** 2))
    scale = np.abs(Qi.numpy()).max() * np.abs(x).max()
    (g_with,) = torch.autograd.grad(J + div, X, retain_graph=True)
    (g_without,) = torch.autograd.grad(J, X)
    g_ok, g_other = (g_with, g_without) if om_div else (g_without, g_with)
    assert g_ok.abs().max().item() < 1e-9 * scale
    assert g_other.abs().max().item() > 1e-6 * scale

def test_golden_model_parameters():
    """The workload generator uses the paper's printed parameters."""
    g = json.load(open(os.path.join(GOLD, "wiener_velocity_P519-548.json")))
    s = wl.wiener_velocity()
    for k in ("F", "H", "L", "W", "R", "m0"):
        assert np.array_equal(getattr(s, k), np.array(g[k], dtype=float)), k
    assert np.array_equal(np.diag(s.P0), g["P0_diag"])
    g = json.load(open(os.path.join(GOLD, "coordinated_turn_P588-623.json")))
    s = wl.coordinated_turn()
    assert np.array_equal(s.L, np.array(g["L"]))
    assert np.array_equal(np.diag(s.R), g["R_diag"])
    assert np.array_equal(s.m0, g["m0"])
    assert np.array_equal(np.diag(s.P0), g["P0_diag"])


# ---------------------------------------------------------------- P14: Euler blocks, nx > 1
def _euler_block_reference(F, c, Q, H, R, r, ys, length):
    """The block as the composition of n exact one-substep elements of the discrete
    model (R-ELEM, length delta = length / n, measurement weight delta at each substep end),
    later substeps on the left (R-FLIP), by the combination rule P:395-407
    (test_method_numpy.combine).  Independent of the oracle's ODE integration."""
    from test_method_numpy import combine
    n = len(ys)
    d = length / n
    Ri = np.linalg.inv(R)
    acc = None
    for k in range(n):
        e = (np.eye(F.shape[0]) - d * F, -d * c, d * Q, d * H.T @ Ri @ (ys[k] - r), d * H.T @ Ri @ H)
        acc = e if acc is None else combine(e, acc)
    return acc


P14_MODELS = {
    # Wiener velocity with drift and measurement offsets c, r != 0
    "wiener": lambda: (wl.wiener_velocity().F, np.array([0.3, -0.2, 0.1, 0.05]), wl.wiener_velocity().L,
                       wl.wiener_velocity().W, wl.wiener_velocity().H, wl.wiener_velocity().R, np.array([0.1, -0.3])),
    # a dense random nx = 4 model: no product in the ODEs commutes by structure
    "dense": lambda: (lambda g: (g.normal(size=(4, 4)), g.normal(size=4), g.normal(size=(4, 4)), np.eye(4),
                                 g.normal(size=(2, 4)), np.diag([0.5, 0.2]), g.normal(size=2)))(np.random.default_rng(5)),
}


def _p14_ratios(model, lib=None, ns=(64, 128, 256, 512), length=0.05):
    """Per-field error of the oracle's Euler block element against the exact composition,
    and the error ratios per doubling of n (first order: -> 2)."""
    F, c, L, W, H, R, r = model
    Q = L @ W @ L.T
    md = oracle.LinearModel(F, L, W, H, R, np.zeros(4), np.eye(4), c=c, r=r)
    errs = []
    for n in ns:
        t = length * np.arange(1, n + 1) / n
        ys = np.stack([np.sin(3 * t) + 0.5, np.cos(2 * t) - 0.2], 1)  # smooth measurement signal
        eu = oracle.euler_block(md, ys, n, length, lib=lib)
        rf = _euler_block_reference(F, c, Q, H, R, r, ys, length)
        errs.append([np.abs(a - b).max() / np.abs(b).max() for a, b in zip(eu, rf)])
    errs = np.array(errs)
    return errs, errs[:-1] / errs[1:]


@pytest.mark.parametrize("name", sorted(P14_MODELS))
def test_P14_euler_block_element_nx4(name):
    """P14 -- the oracle's n-substep Euler block element (A, b, C,
    eta, J) at nx = 4 converges at first order (error ratio in [1.9, 2.1] per doubling of
    n, for every field) to the same limit as the exact composition of n one-substep
    elements.  Unlike P13 (n = 1 and the scalar OU case) this exercises every
    non-commuting product of the ODEs (A Q~ J, J Q~ eta, J Q~ J, F~^T J)."""
    errs, ratios = _p14_ratios(P14_MODELS[name]())
    assert np.all((ratios > 1.9) & (ratios < 2.1)), (errs, ratios)
    assert errs[-1].max() < 1e-3


MUTATIONS = {
    # d(eta)/ds and dJ/ds with Q~ J instead of J Q~
    "JQ->QJ": ("mm_(nx, J, nm->Q, JQ);", "mm_(nx, nm->Q, J, JQ);"),
    # dA/ds with Q~ A J instead of A Q~ J
    "AQJ->QAJ": ("mm_(nx, AQ, g6_printed ? JT : J, t1);",
                 "{ REAL QA_[MAXN * MAXN]; mm_(nx, nm->Q, A, QA_); mm_(nx, QA_, g6_printed ? JT : J, t1); }"),
    # dC/ds with A^T Q~ A
    "AQAt->AtQA": ("mat_mul_bt(nx, nx, nx, AQ, A, dC);",
                   "{ REAL At_[MAXN * MAXN], t3_[MAXN * MAXN]; for (int a = 0; a < nx; ++a) for (int q = 0; q < nx; ++q) "
                   "At_[a * nx + q] = A[q * nx + a]; mm_(nx, At_, nm->Q, t3_); mm_(nx, t3_, A, dC); }"),
}


@pytest.mark.parametrize("mut", sorted(MUTATIONS))
def test_P14_detects_mutations(mut, tmp_path):
    """The P14 pin is sensitive: an oracle build with a transposed product in the ODEs
    fails it (the mutated element converges to another limit, so the ratios fall to ~1)."""
    import subprocess
    src = open(os.path.join(os.path.dirname(oracle.__file__), "oracle.c")).read()
    old, new = MUTATIONS[mut]
    assert src.count(old) == 1
    path = tmp_path / "oracle_mut.c"
    path.write_text(src.replace(old, new))
    so = tmp_path / "liboracle_mut.so"
    subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", str(so), str(path), "-lm"])
    lib = oracle.load_variant(str(so))
    failed = False
    for name in sorted(P14_MODELS):
        errs, ratios = _p14_ratios(P14_MODELS[name](), lib=lib)
        failed |= not (np.all((ratios > 1.9) & (ratios < 2.1)) and errs[-1].max() < 1e-3)
    assert failed, f"mutation {mut} not detected by P14"


# ------------------------------------------------ P15-P17: intra-block refinement (f2)
def _refine_spec():
    spec = wl.wiener_velocity()
    spec.c = np.array([0.3, -0.2, 0.1, 0.05])
    spec.r = np.array([0.5, -0.25])
    spec.tf = 1.0
    return spec


def _smooth_y(t):
    return np.stack([5 + np.sin(3 * t) + 0.3 * t, 5 + np.cos(2 * t)], -1)


def _ora(spec):
    return oracle.LinearModel(spec.F, spec.L, spec.W, spec.H, spec.R, spec.m0, spec.P0, c=spec.c, r=spec.r)


def _p15_ratios(lib=None, T=8, ns=(8, 16, 32)):
    """Error of the refined x* at the fine points inside the blocks against the MAP of the
    one-element-per-fine-node discrete model on the same fine grid (R-ELEM, oracle.kf_rts,
    itself pinned by P1-P3/P6); both converge to the continuous MAP at first order, so the
    per-component error ratio per doubling of n tends to 2."""
    spec = _refine_spec()
    md = _ora(spec)
    errs = []
    for n in ns:
        y = _smooth_y(np.linspace(spec.t0, spec.tf, n * T + 1))
        xr = oracle.euler_refine(md, y, T, n, spec.t0, spec.tf, lib=lib)
        xref = oracle.kf_rts(md, y, n * T, spec.t0, spec.tf)
        inner = np.ones(n * T + 1, bool)
        inner[::n] = False
        errs.append(np.abs(xr - xref)[inner].max(axis=0))
    errs = np.array(errs)
    return errs, errs[:-1] / errs[1:]


def test_P15_refinement_first_order():
    """P15 -- x* at the sub-block points of the Euler-block
    method (value function of the first k substeps, forward-HJB element of the remaining
    n - k, transition P:456-459) converges to the continuous MAP at first order: against
    the fine-grid discrete MAP the error ratio per doubling of n lies in [1.5, 2.5] for
    every state component; the block boundaries are euler_rts's x exactly."""
    errs, ratios = _p15_ratios()
    assert np.all((ratios > 1.5) & (ratios < 2.5)), (errs, ratios)
    spec = _refine_spec()
    n, T = 5, 6
    y = _smooth_y(np.linspace(spec.t0, spec.tf, n * T + 1))
    xr = oracle.euler_refine(_ora(spec), y, T, n, spec.t0, spec.tf)
    assert np.array_equal(xr[::n], oracle.euler_rts(_ora(spec), y, T, n, spec.t0, spec.tf))


P16_MODELS = {"wiener": lambda: P14_MODELS["wiener"](), "dense": lambda: P14_MODELS["dense"]()}


def _p16_ratios(model, lib=None, ns=(64, 128, 256, 512), length=0.2):
    """Per-field error of the forward-HJB element (A, b, C) of P:490-505 over one interval
    against the exact composition of n one-substep elements (as P14), and the ratios."""
    F, c, L, W, H, R, r = model
    Q = L @ W @ L.T
    md = oracle.LinearModel(F, L, W, H, R, np.zeros(4), np.eye(4), c=c, r=r)
    errs = []
    for n in ns:
        t = length * np.arange(1, n + 1) / n
        ys = np.stack([np.sin(3 * t) + 0.5, np.cos(2 * t) - 0.2], 1)
        hj = oracle.hjb_element(md, ys, n, length, lib=lib)
        rf = _euler_block_reference(F, c, Q, H, R, r, ys, length)[:3]
        errs.append([np.abs(a - b).max() / np.abs(b).max() for a, b in zip(hj, rf)])
    errs = np.array(errs)
    return errs, errs[:-1] / errs[1:]


@pytest.mark.parametrize("name", sorted(P16_MODELS))
def test_P16_forward_hjb_element(name):
    """P16 -- the forward-HJB element (A, b, C) integrated in reversed time by
    explicit Euler converges at first order (ratio in [1.9, 2.1] per doubling, every field)
    to the element of the same interval as an exact composition of one-substep elements:
    the same conditional value function reached from its other end (cf. P14)."""
    errs, ratios = _p16_ratios(P16_MODELS[name]())
    assert np.all((ratios > 1.9) & (ratios < 2.1)), (errs, ratios)
    assert errs[-1].max() < 5e-3


def _p17_err(lib=None):
    """Largest relative difference between the refined fine midpoint (n = 2, one block) and
    the textbook RTS step (see test_P17), over three random drift matrices."""
    worst = 0.0
    for seed in range(3):
        spec = _refine_spec()
        rng = np.random.default_rng(seed)
        spec.F = spec.F + 0.3 * rng.standard_normal((4, 4))
        spec.tf = 0.3
        y = 5 + rng.standard_normal((3, 2))
        md = _ora(spec)
        xr = oracle.euler_refine(md, y, 1, 2, spec.t0, spec.tf, lib=lib)
        _, fm, fP = oracle.kf_rts(md, y, 2, spec.t0, spec.tf, want_filter=True)
        d = (spec.tf - spec.t0) / 2
        Phi = np.linalg.inv(np.eye(4) - d * spec.F)
        Q = spec.L @ spec.W @ spec.L.T
        mp = Phi @ (fm[1] + d * spec.c)
        Pp = Phi @ (fP[1] + d * Q) @ Phi.T
        G = fP[1] @ Phi.T @ np.linalg.inv(Pp)
        x1 = fm[1] + G @ (xr[2] - mp)
        worst = max(worst, rel_inf(xr[1], x1))
    return worst


def test_P17_refinement_two_substeps_is_textbook_rts():
    """P17 -- with n = 2 substeps and one block, the refinement at the fine midpoint reduces
    to the textbook RTS step: the one-substep prefix is the exact discrete element of the
    first fine step (so V_1 is the fine-grid Kalman filter at t_1) and the one-step forward-
    HJB element is the exact (A, b, C) of the second; so x*(t_1) = m_1 + G (x*(t_2) - m_2^-),
    G = P_1 Phi^T (P_2^-)^-1, Phi = (I - d F)^-1, m_2^- = Phi (m_1 + d c), P_2^- = Phi (P_1 + d Q) Phi^T,
    with (m_1, P_1) the fine-grid filter (oracle.kf_rts, P1-pinned) and x*(t_2) the block end."""
    assert _p17_err() < 1e-11


REFINE_MUTATIONS = {
    "CMA-sign": ("for (int a = 0; a < nx * nx; ++a) dA[a] = -t1[a] + t2[a];",
                 "for (int a = 0; a < nx * nx; ++a) dA[a] = t1[a] + t2[a];"),
    "FtA-sign": ("for (int a = 0; a < nx * nx; ++a) dA[a] = -t1[a] + t2[a];",
                 "for (int a = 0; a < nx * nx; ++a) dA[a] = -t1[a] - t2[a];"),
    "drop-ct": ("for (int a = 0; a < nx; ++a) db[a] += t3[a] + ct[a];", "for (int a = 0; a < nx; ++a) db[a] += t3[a];"),
    "drop-CMb": ("    for (int a = 0; a < nx; ++a) db[a] -= t3[a];\n    mm_(nx, CM, C, t1);", "    mm_(nx, CM, C, t1);"),
    "CFt^T->Ft^TC": ("mat_mul_bt(nx, nx, nx, C, Ft, dC);                       /* C F~^T */",
                     "for (int a = 0; a < nx; ++a) for (int c = 0; c < nx; ++c) { REAL s_ = 0; "
                     "for (int l = 0; l < nx; ++l) s_ += Ft[l * nx + a] * C[l * nx + c]; dC[a * nx + c] = s_; }"),
    "y-order": ("const double* yk = y_blk + (long)(nsub - 1 - j) * ny;", "const double* yk = y_blk + (long)j * ny;"),
    "prefix-k+1": ("euler_block(nx, ny, k, de, &nm, Ft, ct, HRi, HRH, y_blk, 0, A, b, C, eta, J);   /* first k substeps */",
                   "euler_block(nx, ny, k + 1, de, &nm, Ft, ct, HRi, HRH, y_blk, 0, A, b, C, eta, J);"),
}


@pytest.mark.parametrize("mut", sorted(REFINE_MUTATIONS))
def test_P15_P17_detect_mutations(mut, tmp_path):
    """Every listed slip in the refinement (a sign, a dropped term, a transposed product,
    the measurement order, an off-by-one prefix) fails P15, P16 or P17."""
    import subprocess
    src = open(os.path.join(os.path.dirname(oracle.__file__), "oracle.c")).read()
    old, new = REFINE_MUTATIONS[mut]
    assert src.count(old) == 1
    path = tmp_path / "oracle_mut.c"
    path.write_text(src.replace(old, new))
    so = tmp_path / "liboracle_mut.so"
    subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", str(so), str(path), "-lm"])
    lib = oracle.load_variant(str(so))
    failed = False
    try:
        _, r15 = _p15_ratios(lib=lib)
        failed |= not np.all((r15 > 1.5) & (r15 < 2.5))
        for name in sorted(P16_MODELS):
            e16, r16 = _p16_ratios(P16_MODELS[name](), lib=lib)
            failed |= not (np.all((r16 > 1.9) & (r16 < 2.1)) and e16[-1].max() < 5e-3)
        failed |= _p17_err(lib) > 1e-11
    except FloatingPointError:
        failed = True
    assert failed, f"mutation {mut} not detected by P15-P17"
