"""Seeded Euler--Maruyama simulation of the paper's SDEs (data generation only).

Measurement noise nu_k ~ N(0, R / dt) is the white-noise discretisation of
P:57 (reading G29).  Generator: NumPy PCG64 ``default_rng(seed)``.
"""
from __future__ import annotations

import numpy as np

from .models import LinearSpec, NonlinearSpec, wiener_velocity, ornstein_uhlenbeck, coordinated_turn, van_der_pol


def _chol(a):
    a = np.asarray(a, dtype=np.float64)
    w, v = np.linalg.eigh(a)
    return v * np.sqrt(np.clip(w, 0, None))


def simulate_linear(spec: LinearSpec, T: int, seed: int = 0, batch: int | None = None):
    """Simulate x (truth) and y on the grid t_k = t0 + k dt, k = 0..T.

    Returns (x, y) of shapes [T+1, nx], [T+1, ny] (or with a leading batch axis)."""
    rng = np.random.default_rng(seed)
    B = 1 if batch is None else batch
    nx, ny = spec.nx, spec.ny
    dt = (spec.tf - spec.t0) / T
    c = np.zeros(nx) if spec.c is None else spec.c
    r = np.zeros(ny) if spec.r is None else spec.r
    x0 = spec.m0 + rng.standard_normal((B, nx)) @ _chol(spec.P0).T
    Lq = spec.L @ _chol(spec.W)
    wv = spec.name == "wiener_velocity" and spec.c is None
    if wv:
        # F = [[0, I], [0, 0]]: velocity is a random walk, position its integral.
        dv = np.sqrt(dt) * rng.standard_normal((B, T, Lq.shape[1])) @ Lq[2:].T
        v = np.concatenate([x0[:, None, 2:], x0[:, None, 2:] + np.cumsum(dv, axis=1)], axis=1)
        p = np.concatenate([x0[:, None, :2], x0[:, None, :2] + dt * np.cumsum(v[:, :-1], axis=1)], axis=1)
        x = np.concatenate([p, v], axis=2)
    else:
        x = np.empty((B, T + 1, nx))
        x[:, 0] = x0
        F = spec.F
        for k in range(T):
            xi = rng.standard_normal((B, Lq.shape[1]))
            x[:, k + 1] = x[:, k] + (x[:, k] @ F.T + c) * dt + np.sqrt(dt) * xi @ Lq.T
    nu = rng.standard_normal((B, T + 1, ny)) @ _chol(spec.R / dt).T
    y = x @ spec.H.T + r + nu
    if batch is None:
        return x[0], y[0]
    return x, y


def _f(spec: NonlinearSpec, x):
    if spec.kind == 1:
        return np.stack([x[..., 2], x[..., 3], -x[..., 4] * x[..., 3], x[..., 4] * x[..., 2],
                         np.zeros_like(x[..., 0])], axis=-1)
    mu = spec.params[0]
    return np.stack([x[..., 1], mu * (1 - x[..., 0] ** 2) * x[..., 1] - x[..., 0]], axis=-1)


def _h(spec: NonlinearSpec, x):
    if spec.kind == 1:
        return np.stack([np.hypot(x[..., 0], x[..., 1]), np.arctan2(x[..., 1], x[..., 0])], axis=-1)
    return x[..., :1]


def simulate_nonlinear(spec: NonlinearSpec, T: int, seed: int = 0):
    """Euler--Maruyama simulation of P:590-595; returns (x [T+1, nx], y [T+1, ny])."""
    rng = np.random.default_rng(seed)
    dt = (spec.tf - spec.t0) / T
    Lq = spec.L @ _chol(spec.W)
    x = np.empty((T + 1, spec.nx))
    x[0] = spec.m0 + _chol(spec.P0) @ rng.standard_normal(spec.nx)
    noise = np.sqrt(dt) * rng.standard_normal((T, Lq.shape[1])) @ Lq.T
    for k in range(T):
        x[k + 1] = x[k] + _f(spec, x[k]) * dt + noise[k]
    nu = rng.standard_normal((T + 1, spec.ny)) @ _chol(spec.R / dt).T
    y = _h(spec, x) + nu
    if spec.kind == 1:
        y[:, 1] = (y[:, 1] + np.pi) % (2 * np.pi) - np.pi
    return x, y


def make_workload(config: str, seed: int = 0, T: int | None = None, batch: int | None = None):
    """Build (spec, y, T, batch) for a BASELINE.json config id ("C1".."C5")."""
    from .models import CONFIGS
    cfg = dict(CONFIGS[config])
    T = cfg["T"] if T is None else T
    B = cfg["batch"] if batch is None else batch
    name = cfg["model"]
    if name == "wiener_velocity":
        spec = wiener_velocity()
    elif name == "ornstein_uhlenbeck":
        spec = ornstein_uhlenbeck()
    elif name == "coordinated_turn":
        spec = coordinated_turn()
    else:
        spec = van_der_pol()
    n = cfg.get("substeps", 1)
    if isinstance(spec, LinearSpec) and n > 1:
        # Euler blocks: simulate on the fine grid of n*T steps, then lay the rows out as
        # include/pmap.h expects ([T+1][n*ny], row 0 = y(t_0) in its last sub-slot)
        _, yf = simulate_linear(spec, n * T, seed=seed, batch=(B if B > 1 else None))
        yf = yf.reshape(B, n * T + 1, spec.ny)
        y = np.zeros((B, T + 1, n, spec.ny))
        y[:, 0, n - 1] = yf[:, 0]
        y[:, 1:] = yf[:, 1:].reshape(B, T, n, spec.ny)
        y = y.reshape(B, T + 1, n * spec.ny)
        if B == 1:
            y = y[0]
    elif isinstance(spec, LinearSpec):
        _, y = simulate_linear(spec, T, seed=seed, batch=(B if B > 1 else None))
    else:
        _, y = simulate_nonlinear(spec, T, seed=seed)
    return spec, y, T, B
