"""Model parameter sets of arXiv 2512.13319 (P:n = PAPER.md line n) and BASELINE.json configs."""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class LinearSpec:
    """Linear-affine SDE dx = (F x + c) dt + L dbeta, y = H x + r + nu."""
    name: str
    F: np.ndarray
    L: np.ndarray
    W: np.ndarray
    H: np.ndarray
    R: np.ndarray
    m0: np.ndarray
    P0: np.ndarray
    c: np.ndarray | None = None
    r: np.ndarray | None = None
    t0: float = 0.0
    tf: float = 5.0

    @property
    def nx(self) -> int:
        return self.F.shape[-1]

    @property
    def ny(self) -> int:
        return self.H.shape[-2]

    @property
    def nw(self) -> int:
        return self.L.shape[-1]


@dataclass
class NonlinearSpec:
    """Nonlinear SDE dx = f(x) dt + L dbeta, y = h(x) + nu."""
    name: str
    kind: int            # 1 = coordinated turn, 2 = Van der Pol (DESIGN.md R-VDP)
    nx: int
    ny: int
    L: np.ndarray
    W: np.ndarray
    R: np.ndarray
    m0: np.ndarray
    P0: np.ndarray
    params: np.ndarray = field(default_factory=lambda: np.zeros(1))
    t0: float = 0.0
    tf: float = 5.0

    @property
    def nw(self) -> int:
        return self.L.shape[1]


def wiener_velocity() -> LinearSpec:
    """Partially observed 2-D Wiener velocity model, P:519-548 (P0 = 1e-2 I_4, reading G11)."""
    Z, I = np.zeros((2, 2)), np.eye(2)
    return LinearSpec(
        name="wiener_velocity",
        F=np.block([[Z, I], [Z, Z]]),
        L=np.vstack([Z, I]),
        W=4.0 * I,
        H=np.hstack([I, Z]),
        R=1e-2 * I,
        m0=np.array([5.0, 5.0, 0.0, 0.0]),
        P0=1e-2 * np.eye(4),
        t0=0.0, tf=5.0)


def ornstein_uhlenbeck(theta=1.0, q=2.0, R=0.1, m0=1.0, P0=1.0, tf=5.0) -> LinearSpec:
    """Scalar OU (BASELINE.json config 1; not in the paper): dx = -theta x dt + dbeta, E dbeta^2 = q dt."""
    return LinearSpec(name="ornstein_uhlenbeck", F=np.array([[-theta]]), L=np.array([[1.0]]),
                      W=np.array([[q]]), H=np.array([[1.0]]), R=np.array([[R]]),
                      m0=np.array([m0]), P0=np.array([[P0]]), t0=0.0, tf=tf)


def coordinated_turn() -> NonlinearSpec:
    """Coordinated-turn model, P:588-623 (time span [0, 5], reading G12)."""
    sv, sw = 5e-4, 0.02
    L = np.zeros((5, 3))
    L[2, 0], L[3, 1], L[4, 2] = sv, sv, sw
    return NonlinearSpec(name="coordinated_turn", kind=1, nx=5, ny=2, L=L, W=np.eye(3),
                         R=np.diag([5e-3, 1e-3]), m0=np.array([5.0, 5.0, 0.0, 0.3, 0.0]),
                         P0=np.diag([0.01, 0.01, 0.01, 0.01, 0.04]), t0=0.0, tf=5.0)


def van_der_pol(mu=1.0, q=0.1, R=1e-2) -> NonlinearSpec:
    """Van der Pol oscillator (reading R-VDP; not in the paper)."""
    return NonlinearSpec(name="van_der_pol", kind=2, nx=2, ny=1, L=np.array([[0.0], [1.0]]),
                         W=np.array([[q]]), R=np.array([[R]]), m0=np.array([2.0, 0.0]),
                         P0=0.01 * np.eye(2), params=np.array([mu]), t0=0.0, tf=5.0)


# BASELINE.json "configs", in order (C1..C5).
CONFIGS = {
    "C1": dict(model="ornstein_uhlenbeck", T=1_000, batch=1, method="rts"),
    "C2": dict(model="wiener_velocity", T=100_000, batch=1, method="rts"),
    "C3": dict(model="wiener_velocity", T=10_000_000, batch=1, method="rts"),
    "C4": dict(model="coordinated_turn", T=100_000, batch=1, method="ieks", passes=10),
    "C5": dict(model="wiener_velocity", T=10_000, batch=1024, method="two_filter"),
    # not a BASELINE config: the paper's own discretisation of its linear experiment
    # (T blocks of n = 10 Euler substeps, a measurement at every substep), SURVEY f2
    "C2E": dict(model="wiener_velocity", T=100_000, batch=1, method="rts", substeps=10),
}
