"""CPU check of the paper's element algebra and of this build's readings (DESIGN.md R-*).

A deliberately naive NumPy transcription of the *parallel method* (not of the
oracle): node elements E_i, the combination rule of P:395-407, the flipped
prefix scan (R-FLIP), the transition elements (Phi, beta) of P:441-459 and the
mirrored information-form two-filter elements (R-TF).  Scans are evaluated in
several bracketings (sequential and a random tree) to exercise associativity.
Results are compared with the independent CPU oracle.  This validates the
readings the CUDA kernels implement; it is not used by the product.
"""
import json
import os

import numpy as np
import pytest

import oracle
import workloads as wl

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def combine(e1, e2):
    """(A, b, C, eta, J) of V(.,s;.,t) = V(.,s;.,gamma) (x) V(.,gamma;.,t)."""
    A1, b1, C1, h1, J1 = e1
    A2, b2, C2, h2, J2 = e2
    n = A1.shape[0]
    I = np.eye(n)
    M = np.linalg.inv(I + C1 @ J2)
    Mt = np.linalg.inv(I + J2 @ C1)
    A = A2 @ M @ A1
    b = A2 @ M @ (b1 + C1 @ h2) + b2
    C = A2 @ M @ C1 @ A2.T + C2
    h = A1.T @ Mt @ (h2 - J2 @ b1) + h1
    J = A1.T @ Mt @ J2 @ A1 + J1
    return (A, b, C, h, J)


def ident(n):
    return (np.eye(n), np.zeros(n), np.zeros((n, n)), np.zeros(n), np.zeros((n, n)))


def node_elements(spec, y, T):
    """E_0 = (0, 0, 0, P0^-1 m0 + dt K0 (y0 - r0), P0^-1 + dt H^T R^-1 H) and
    E_i = (I - dt F, -dt c, dt Q, dt H^T R^-1 (y_i - r), dt H^T R^-1 H) (R-ELEM)."""
    n = spec.nx
    dt = (spec.tf - spec.t0) / T
    Q = spec.L @ spec.W @ spec.L.T
    Ri = np.linalg.inv(spec.R)
    c = np.zeros(n) if spec.c is None else spec.c
    r = np.zeros(spec.ny) if spec.r is None else spec.r
    Jm = dt * spec.H.T @ Ri @ spec.H
    out = []
    for i in range(T + 1):
        hm = dt * spec.H.T @ Ri @ (y[i] - r)
        if i == 0:
            P0i = np.linalg.inv(spec.P0)
            out.append((np.zeros((n, n)), np.zeros(n), np.zeros((n, n)), P0i @ spec.m0 + hm, P0i + Jm))
        else:
            out.append((np.eye(n) - dt * spec.F, -dt * c, dt * Q, hm, Jm))
    return out


def tree_reduce(elems, rng):
    """Fold a list with the (flipped) operator in a random bracketing."""
    elems = list(elems)
    while len(elems) > 1:
        k = rng.integers(0, len(elems) - 1)
        elems[k:k + 2] = [combine(elems[k + 1], elems[k])]   # flipped: later element on the left
    return elems[0]


def method_rts(spec, y, T, rng=None):
    E = node_elements(spec, y, T)
    n = spec.nx
    # pass 1: acc_i = E_i (x) acc_{i-1}  (R-FLIP), (S_i, v_i) = (J, eta) of acc_i
    S, v = [], []
    acc = None
    for i in range(T + 1):
        if rng is not None and i in (T // 3, T):
            acc_i = tree_reduce(E[:i + 1], rng)
        else:
            acc_i = E[0] if acc is None else combine(E[i], acc)
        acc = acc_i
        assert np.abs(acc[0]).max() == 0 and np.abs(acc[2]).max() == 0
        S.append(acc[4])
        v.append(acc[3])
    # pass 2: x_{i-1} = Phi_i x_i + beta_i, Phi_i = (I + C_i S_{i-1})^-1 A_i, beta_i = (I + C_i S_{i-1})^-1 (b_i + C_i v_{i-1})
    x = np.zeros((T + 1, n))
    x[T] = np.linalg.solve(S[T], v[T])
    for i in range(T, 0, -1):
        A, b, C = E[i][0], E[i][1], E[i][2]
        M = np.linalg.inv(np.eye(n) + C @ S[i - 1])
        x[i - 1] = M @ A @ x[i] + M @ (b + C @ v[i - 1])
    return x, S, v


def method_two_filter(spec, y, T):
    """R-TF: mirrored elements M_i = (A', b', C', eta_i^m, J_i^m), A' = (I - dt F)^-1,
    b' = A' dt c, C' = A' dt Q A'^T; suffix scan acc_i = M_i (x) acc_{i+1};
    x_i = (S_i + Lam_i - J_i^m)^-1 (v_i + xi_i - eta_i^m)."""
    _, S, v = method_rts(spec, y, T)
    E = node_elements(spec, y, T)
    n = spec.nx
    dt = (spec.tf - spec.t0) / T
    Ap = np.linalg.inv(np.eye(n) - dt * spec.F)
    c = np.zeros(n) if spec.c is None else spec.c
    bp = Ap @ (dt * c)
    Cp = Ap @ (dt * spec.L @ spec.W @ spec.L.T) @ Ap.T
    Ri = np.linalg.inv(spec.R)
    r = np.zeros(spec.ny) if spec.r is None else spec.r
    Jm = dt * spec.H.T @ Ri @ spec.H
    x = np.zeros((T + 1, n))
    acc = None
    for i in range(T, -1, -1):
        hm = dt * spec.H.T @ Ri @ (y[i] - r)
        Mi = (np.zeros((n, n)), np.zeros(n), np.zeros((n, n)), hm, Jm) if i == T else (Ap, bp, Cp, hm, Jm)
        acc = Mi if acc is None else combine(Mi, acc)
        Lam, xi = acc[4], acc[3]
        x[i] = np.linalg.solve(S[i] + Lam - Jm, v[i] + xi - hm)
    return x


def test_associativity_identity_singular():
    """A1 -- (x) is associative; (I,0,0,0,0) is an exact two-sided identity;
    singular C and J are fine (reading G14)."""
    rng = np.random.default_rng(0)

    def rand_el(n, singular=False):
        A = rng.standard_normal((n, n))
        b = rng.standard_normal(n)
        a = rng.standard_normal((n, 2 if singular else n))
        c = rng.standard_normal((n, 2 if singular else n))
        return (A, b, a @ a.T, rng.standard_normal(n), c @ c.T)

    worst = 0.0
    for k in range(300):
        a, b, c = (rand_el(4, singular=(k % 2 == 0)) for _ in range(3))
        l = combine(combine(a, b), c)
        r = combine(a, combine(b, c))
        for u, w in zip(l, r):
            worst = max(worst, np.abs(u - w).max() / max(1.0, np.abs(w).max()))
        e = ident(4)
        for u, w in zip(combine(e, a), a):
            assert np.array_equal(u, w)
        for u, w in zip(combine(a, e), a):
            assert np.array_equal(u, w)
    assert worst < 1e-10


def test_spec_hand_values():
    """SPEC S:255, S:264, S:442 hand values (golden)."""
    g = json.load(open(os.path.join(GOLD, "spec_hand_values.json")))
    t = g["terminal_element"]
    one = np.ones((1, 1))
    e = (0 * one, np.zeros(1), 0 * one, np.array([t["m0"] / t["P0"]]), one / t["P0"])
    assert e[3][0] == t["eta"] and e[4][0, 0] == t["J"]
    d = g["pure_diffusion"]
    c = combine((one, np.zeros(1), d["d1"] * one, np.zeros(1), 0 * one),
                (one, np.zeros(1), d["d2"] * one, np.zeros(1), 0 * one))
    assert c[2][0, 0] == d["C"] and c[0][0, 0] == 1
    a = g["affine_composition"]
    (p1, q1), (p2, q2) = a["first"], a["second"]
    assert [p2 * p1, p2 * q1 + q2] == a["combined"]
    assert a["combined"][0] * a["phi0"] + a["combined"][1] == a["phi"]


@pytest.mark.parametrize("name", ["wiener", "ou", "wiener_offsets"])
def test_method_equals_oracle(name):
    """A2 -- the scan of node elements (pass 1 + pass 2) reproduces the oracle's
    discrete KF + RTS, and S_i^-1 v_i its filter means."""
    T = 60
    if name == "ou":
        spec = wl.ornstein_uhlenbeck()
    else:
        spec = wl.wiener_velocity()
        if name == "wiener_offsets":
            spec.c = np.array([0.3, -0.2, 0.1, 0.05])
            spec.r = np.array([0.5, -0.25])
    _, y = wl.simulate_linear(spec, T, seed=3)
    x, S, v = method_rts(spec, y, T, rng=np.random.default_rng(1))
    md = oracle.LinearModel(spec.F, spec.L, spec.W, spec.H, spec.R, spec.m0, spec.P0, c=spec.c, r=spec.r)
    xo, fm, _ = oracle.kf_rts(md, y, T, spec.t0, spec.tf, want_filter=True)
    assert np.abs(x - xo).max() / np.abs(xo).max() < 1e-12
    m = np.stack([np.linalg.solve(S[i], v[i]) for i in range(T + 1)])
    assert np.abs(m - fm).max() / np.abs(fm).max() < 1e-12
    xt = method_two_filter(spec, y, T)
    assert np.abs(xt - xo).max() / np.abs(xo).max() < 1e-12
