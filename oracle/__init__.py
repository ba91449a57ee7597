"""oracle -- TEST INFRASTRUCTURE ONLY (arXiv 2512.13319).

A plain, slow, sequential CPU fp64 reference (``oracle.c``: discrete Kalman
filter + RTS smoother, backward-information two-filter smoother, iterated
linearisation) and its ctypes binding.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` leg may import this package.  It shares no code with the CUDA
product path in ``paper_2512_13319_b200/`` and never imports it.

Every function cites the PAPER.md passage it follows ("P:n" = line n).
Pins: see tests/test_oracle_pins.py and DESIGN.md section "Oracle pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIBS = {False: os.path.join(_HERE, "liboracle.so"), True: os.path.join(_HERE, "liboracle_ld.so")}


def build(force: bool = False) -> None:
    """Compile oracle.c (plain C, -O2, no fast-math) into the two shared objects."""
    for ld, path in _LIBS.items():
        if not force and os.path.exists(path) and os.path.getmtime(path) >= os.path.getmtime(_SRC):
            continue
        cmd = ["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-o", path, _SRC, "-lm"]
        if ld:
            cmd.insert(1, "-DORA_LONG_DOUBLE")
        subprocess.check_call(cmd)


class OraModel(ctypes.Structure):
    _fields_ = [
        ("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nw", ctypes.c_int),
        ("T", ctypes.c_long), ("t0", ctypes.c_double), ("tf", ctypes.c_double),
    ] + [(n, ctypes.c_void_p) for n in ("F", "c", "L", "W", "H", "r", "R")] + [
        (n, ctypes.c_long) for n in ("sF", "sc", "sL", "sW", "sH", "sr", "sR")
    ] + [("m0", ctypes.c_void_p), ("P0", ctypes.c_void_p), ("g", ctypes.c_void_p)]


_loaded: dict = {}


def _lib(long_double: bool = False):
    if long_double not in _loaded:
        build()
        lib = ctypes.CDLL(_LIBS[long_double])
        P = ctypes.c_void_p
        lib.ora_kf_rts.argtypes = [ctypes.POINTER(OraModel), P, P, P, P]
        lib.ora_two_filter.argtypes = [ctypes.POINTER(OraModel), P, P]
        lib.ora_kf_rts_cov.argtypes = [ctypes.POINTER(OraModel), P, P, P]
        lib.ora_euler_rts.argtypes = [ctypes.POINTER(OraModel), ctypes.c_int, P, P, ctypes.c_int]
        lib.ora_euler_block.argtypes = [ctypes.POINTER(OraModel), ctypes.c_int, P, P, P, P, P, P, ctypes.c_int]
        lib.ora_euler_refine.argtypes = [ctypes.POINTER(OraModel), ctypes.c_int, P, P]
        lib.ora_hjb_element.argtypes = [ctypes.POINTER(OraModel), ctypes.c_int, P, P, P, P]
        lib.ora_batch.argtypes = [ctypes.POINTER(OraModel), ctypes.c_long, P, P, ctypes.c_int]
        lib.ora_ieks.argtypes = [ctypes.c_int, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long,
                                 ctypes.c_double, ctypes.c_double, P, P, P, P, P, P, ctypes.c_int, P, P, P]
        for n in ("ora_ct_f", "ora_ct_dfdx", "ora_ct_h", "ora_ct_dhdx"):
            getattr(lib, n).argtypes = [P, P]
        lib.ora_vdp_f.argtypes = [ctypes.c_double, P, P]
        lib.ora_vdp_dfdx.argtypes = [ctypes.c_double, P, P]
        lib.ora_num_threads.restype = ctypes.c_int
        _loaded[long_double] = lib
    return _loaded[long_double]


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a) -> int | None:
    return None if a is None else a.ctypes.data


class LinearModel:
    """Linear-affine model of P:134-140 sampled on the grid.

    Each of F, c, L, W, H, r, R is either one matrix (constant in time) or an
    array with a leading node axis of length T+1 (time-varying)."""

    def __init__(self, F, L, W, H, R, m0, P0, c=None, r=None):
        self.F, self.L, self.W, self.H, self.R = map(_f64, (F, L, W, H, R))
        self.c = None if c is None else _f64(c)
        self.r = None if r is None else _f64(r)
        self.m0, self.P0 = _f64(m0), _f64(P0)

    @property
    def nx(self) -> int:
        return self.m0.shape[-1]

    @property
    def ny(self) -> int:
        return self.H.shape[-2]

    @property
    def nw(self) -> int:
        return self.L.shape[-1]

    def _struct(self, T: int, t0: float, tf: float) -> OraModel:
        def stride(a, base_ndim):
            if a is None:
                return 0
            if a.ndim == base_ndim:
                return 0
            assert a.shape[0] == T + 1, "time-varying arrays need T+1 node entries"
            return int(np.prod(a.shape[1:]))

        s = OraModel()
        s.nx, s.ny, s.nw, s.T, s.t0, s.tf = self.nx, self.ny, self.nw, T, t0, tf
        for name, nd in (("F", 2), ("c", 1), ("L", 2), ("W", 2), ("H", 2), ("r", 1), ("R", 2)):
            a = getattr(self, name)
            setattr(s, name, _ptr(a))
            setattr(s, "s" + name, stride(a, nd))
        s.m0, s.P0 = _ptr(self.m0), _ptr(self.P0)
        s.g = None
        return s


def kf_rts(model: LinearModel, y, T: int, t0: float, tf: float, long_double: bool = False,
           want_filter: bool = False):
    """Discrete KF + RTS MAP (P:200-226 discretised).

    Returns x_map [T+1, nx] (and filter means [T+1, nx], covariances
    [T+1, nx, nx] when want_filter)."""
    y = _f64(y).reshape(T + 1, model.ny)
    N, nx = T + 1, model.nx
    x = np.empty((N, nx))
    fm = np.empty((N, nx)) if want_filter else None
    fP = np.empty((N, nx, nx)) if want_filter else None
    s = model._struct(T, t0, tf)
    rc = _lib(long_double).ora_kf_rts(ctypes.byref(s), _ptr(y), _ptr(x), _ptr(fm), _ptr(fP))
    if rc:
        raise FloatingPointError(f"oracle kf_rts failed rc={rc}")
    return (x, fm, fP) if want_filter else x


def kf_rts_cov(model: LinearModel, y, T: int, t0: float, tf: float, long_double: bool = False):
    """Discrete KF + RTS MAP and smoother covariances (textbook RTS covariance recursion,
    SURVEY f4).  Returns (x_map [T+1, nx], smooth_P [T+1, nx, nx])."""
    y = _f64(y).reshape(T + 1, model.ny)
    N, nx = T + 1, model.nx
    x = np.empty((N, nx))
    P = np.empty((N, nx, nx))
    s = model._struct(T, t0, tf)
    rc = _lib(long_double).ora_kf_rts_cov(ctypes.byref(s), _ptr(y), _ptr(x), _ptr(P))
    if rc:
        raise FloatingPointError(f"oracle kf_rts_cov failed rc={rc}")
    return x, P


def euler_rts(model: LinearModel, y_fine, T: int, nsub: int, t0: float, tf: float, g6_printed: bool = False,
              long_double: bool = False):
    """Paper-faithful Euler blocks: T blocks of nsub explicit Euler
    substeps of the element ODEs P:416-427, sequential value-function fold and RTS
    transitions.  y_fine [nsub*T+1, ny]; returns x_map [T+1, nx] at the block boundaries.
    g6_printed: use the printed dA/ds = -A Q J^T - A F -- pins only."""
    y = _f64(y_fine).reshape(nsub * T + 1, model.ny)
    x = np.empty((T + 1, model.nx))
    s = model._struct(T, t0, tf)
    rc = _lib(long_double).ora_euler_rts(ctypes.byref(s), nsub, _ptr(y), _ptr(x), 1 if g6_printed else 0)
    if rc:
        raise FloatingPointError(f"oracle euler_rts failed rc={rc}")
    return x


def euler_refine(model: LinearModel, y_fine, T: int, nsub: int, t0: float, tf: float, long_double: bool = False,
                 lib=None):
    """Euler blocks plus the intra-block refinement of P:485-507 (DESIGN.md
    R-REFINE): x* at every fine point, the n - 1 inside each block from the value function
    of the block's first k substeps, the forward-HJB element (first three
    equations) of the remaining n - k and the transition P:456-459.  y_fine [nsub*T+1, ny];
    returns x_fine [nsub*T+1, nx].  `lib`: another build of oracle.c (pin mutation checks)."""
    y = _f64(y_fine).reshape(nsub * T + 1, model.ny)
    x = np.empty((nsub * T + 1, model.nx))
    s = model._struct(T, t0, tf)
    L = lib or _lib(long_double)
    rc = L.ora_euler_refine(ctypes.byref(s), nsub, _ptr(y), _ptr(x))
    if rc:
        raise FloatingPointError(f"oracle euler_refine failed rc={rc}")
    return x


def hjb_element(model: LinearModel, y_sub, m: int, length: float, lib=None):
    """The forward-HJB element (A, b, C) of P:490-505 (first three equations) over one
    interval of the given length: m explicit Euler steps in reversed time from the boundary
    (I, 0, 0); y_sub [m, ny] in forward-time order (y_sub[k] at t_start + (k+1) length/m).
    Step 2 of euler_refine's suffix, alone (pin P16)."""
    nx = model.nx
    y = _f64(y_sub).reshape(m, model.ny)
    A, C = np.empty((nx, nx)), np.empty((nx, nx))
    b = np.empty(nx)
    s = model._struct(1, 0.0, length)
    rc = (lib or _lib()).ora_hjb_element(ctypes.byref(s), m, _ptr(y), _ptr(A), _ptr(b), _ptr(C))
    if rc:
        raise FloatingPointError(f"oracle hjb_element failed rc={rc}")
    return A, b, C


def euler_block(model: LinearModel, y_sub, nsub: int, length: float, g6_printed: bool = False, lib=None):
    """One Euler block element alone (step 1 of euler_rts; P:416-427 from the boundary of
    P:427): nsub explicit Euler substeps of length length/nsub, substep k reading y_sub[k].
    Returns (A, b, C, eta, J).  `lib`: another build of oracle.c (mutation checks of the pins)."""
    nx = model.nx
    y = _f64(y_sub).reshape(nsub, model.ny)
    A, C, J = (np.empty((nx, nx)) for _ in range(3))
    b, eta = np.empty(nx), np.empty(nx)
    s = model._struct(1, 0.0, length)
    rc = (lib or _lib()).ora_euler_block(ctypes.byref(s), nsub, _ptr(y), _ptr(A), _ptr(b), _ptr(C), _ptr(eta),
                                         _ptr(J), 1 if g6_printed else 0)
    if rc:
        raise FloatingPointError(f"oracle euler_block failed rc={rc}")
    return A, b, C, eta, J


def load_variant(path: str):
    """ctypes handle of another build of oracle.c (pin mutation checks only)."""
    lib = ctypes.CDLL(path)
    lib.ora_euler_block.argtypes = [ctypes.POINTER(OraModel), ctypes.c_int] + [ctypes.c_void_p] * 6 + [ctypes.c_int]
    lib.ora_euler_refine.argtypes = [ctypes.POINTER(OraModel), ctypes.c_int] + [ctypes.c_void_p] * 2
    lib.ora_hjb_element.argtypes = [ctypes.POINTER(OraModel), ctypes.c_int] + [ctypes.c_void_p] * 4
    return lib


def two_filter(model: LinearModel, y, T: int, t0: float, tf: float, long_double: bool = False):
    """Two-filter MAP via the textbook backward information filter."""
    y = _f64(y).reshape(T + 1, model.ny)
    x = np.empty((T + 1, model.nx))
    s = model._struct(T, t0, tf)
    rc = _lib(long_double).ora_two_filter(ctypes.byref(s), _ptr(y), _ptr(x))
    if rc:
        raise FloatingPointError(f"oracle two_filter failed rc={rc}")
    return x


def batch(model: LinearModel, y, T: int, t0: float, tf: float, mode: int = 0):
    """Batched linear MAP over independent trajectories (OpenMP); y [B, T+1, ny]."""
    y = _f64(y)
    B = y.shape[0]
    x = np.empty((B, T + 1, model.nx))
    s = model._struct(T, t0, tf)
    rc = _lib().ora_batch(ctypes.byref(s), B, _ptr(y), _ptr(x), mode)
    if rc:
        raise FloatingPointError(f"oracle batch failed rc={rc}")
    return x


def ieks(kind: int, params, L, W, R, m0, P0, y, T: int, t0: float, tf: float, passes: int,
         x_init=None):
    """Iterated linearisation MAP (5 passes in P:625). kind 1 = CT, 2 = VdP
    (params = [mu] or [mu, om_div]; om_div != 0 keeps the OM divergence term of P:66).

    Returns (x_map [T+1, nx], per-pass max |dx|)."""
    L, W, R, m0, P0 = map(_f64, (L, W, R, m0, P0))
    nx, nw, ny = L.shape[0], L.shape[1], R.shape[0]
    y = _f64(y).reshape(T + 1, ny)
    params = _f64(params if params is not None else [0.0])
    params = np.concatenate([params, np.zeros(max(0, 2 - params.size))])  # C reads params[0..1]
    xi = None if x_init is None else _f64(x_init)
    x = np.empty((T + 1, nx))
    delta = np.empty(max(passes, 1))
    rc = _lib().ora_ieks(kind, _ptr(params), nx, ny, nw, T, t0, tf, _ptr(L), _ptr(W), _ptr(R),
                         _ptr(m0), _ptr(P0), _ptr(y), passes, _ptr(xi), _ptr(x), _ptr(delta))
    if rc:
        raise FloatingPointError(f"oracle ieks failed rc={rc}")
    return x, delta[:passes]


def ct_f(x):
    x, out = _f64(x), np.empty(5)
    _lib().ora_ct_f(_ptr(x), _ptr(out))
    return out


def ct_dfdx(x):
    x, out = _f64(x), np.empty((5, 5))
    _lib().ora_ct_dfdx(_ptr(x), _ptr(out))
    return out


def ct_h(x):
    x, out = _f64(x), np.empty(2)
    _lib().ora_ct_h(_ptr(x), _ptr(out))
    return out


def ct_dhdx(x):
    x, out = _f64(x), np.empty((2, 5))
    _lib().ora_ct_dhdx(_ptr(x), _ptr(out))
    return out


def vdp_f(mu, x):
    x, out = _f64(x), np.empty(2)
    _lib().ora_vdp_f(mu, _ptr(x), _ptr(out))
    return out


def vdp_dfdx(mu, x):
    x, out = _f64(x), np.empty((2, 2))
    _lib().ora_vdp_dfdx(mu, _ptr(x), _ptr(out))
    return out


def num_threads() -> int:
    return int(_lib().ora_num_threads())
