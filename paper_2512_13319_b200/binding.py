"""ctypes binding of include/pmap.h (argument marshalling only; every step runs in libpmap.so).

The functions ``map_plan``, ``map_solve_linear``, ``map_two_filter``,
``map_solve_nonlinear``, ``map_sync``, ``map_last_error`` and
``map_plan_destroy`` mirror the C entry points one to one.  ``Plan`` is a small
convenience wrapper that accepts torch tensors (device or host) or NumPy arrays
and borrows torch's current CUDA stream.  There is no CPU fallback: if the
shared library is missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

LIB_PATH = os.environ.get("PMAP_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpmap.so")

MAP_F64, MAP_F32 = 0, 1
MAP_FLAG_MIXED = 1  # mixed-precision pass 2 (include/pmap.h)
MAP_FLAG_BATCH_SHARD = 2  # world > 1 shards the batch instead of time (include/pmap.h)
MAP_NL_COORD_TURN, MAP_NL_VAN_DER_POL = 1, 2
STATUS = {0: "MAP_OK", 1: "MAP_E_ARG", 2: "MAP_E_UNSUPPORTED", 3: "MAP_E_CUDA", 4: "MAP_E_NCCL",
          5: "MAP_E_NUMERIC", 6: "MAP_E_DIVERGED"}

# every symbol include/pmap.h declares
EXPORTS = ["map_plan", "map_plan_destroy", "map_solve_linear", "map_two_filter", "map_solve_nonlinear",
           "map_sync", "map_last_error", "map_status_string", "map_workspace_bytes", "map_last_launch_count",
           "map_profile_enable", "map_profile_read", "map_shard_payload_bytes", "map_shard_phase",
           "map_version", "map_solve_sequential", "map_debug_lb_timing", "map_solve_linear_cov",
           "map_solve_linear_fine", "map_solve_linear_pipelined"]


class MapError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}: {msg}")


class PlanDesc(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nw", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("T", ctypes.c_int64), ("batch", ctypes.c_int64), ("t0", ctypes.c_double), ("tf", ctypes.c_double),
                ("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("substeps", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("nccl_comm", ctypes.c_void_p), ("stream", ctypes.c_void_p)]


class LinearModel(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("F", "c", "L", "W", "H", "r", "R", "m0", "P0")] + \
               [(n, ctypes.c_int64) for n in ("sF", "sc", "sL", "sW", "sH", "sr", "sR")]


class NlModel(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("nparams", ctypes.c_int32), ("params", ctypes.c_void_p),
                ("L", ctypes.c_void_p), ("W", ctypes.c_void_p), ("R", ctypes.c_void_p), ("m0", ctypes.c_void_p),
                ("P0", ctypes.c_void_p)]


_lib = None


def load_library():
    """Load libpmap.so (raises if it was not built: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -m paper_2512_13319_b200.build`")
        lib = ctypes.CDLL(LIB_PATH)
        P, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        lib.map_plan.argtypes = [ctypes.POINTER(PlanDesc), ctypes.POINTER(LinearModel), ctypes.POINTER(NlModel),
                                 ctypes.POINTER(P)]
        lib.map_plan.restype = ctypes.c_int
        lib.map_plan_destroy.argtypes = [P]
        lib.map_plan_destroy.restype = None
        lib.map_solve_linear.argtypes = [P, P, P, P, P]
        lib.map_solve_linear.restype = ctypes.c_int
        lib.map_two_filter.argtypes = [P, P, P, P]
        lib.map_solve_linear_cov.argtypes = [P, P, P, P]
        lib.map_solve_linear_cov.restype = ctypes.c_int
        lib.map_solve_linear_fine.argtypes = [P, P, P]
        lib.map_solve_linear_fine.restype = ctypes.c_int
        lib.map_solve_linear_pipelined.argtypes = [P, P, P]
        lib.map_solve_linear_pipelined.restype = ctypes.c_int
        lib.map_two_filter.restype = ctypes.c_int
        lib.map_solve_sequential.argtypes = [P, I32, P, I32, P, P]
        lib.map_solve_sequential.restype = ctypes.c_int
        lib.map_solve_nonlinear.argtypes = [P, P, I32, D, P, P, ctypes.POINTER(I32)]
        lib.map_solve_nonlinear.restype = ctypes.c_int
        lib.map_sync.argtypes = [P]
        lib.map_sync.restype = ctypes.c_int
        lib.map_last_error.argtypes = [P]
        lib.map_last_error.restype = ctypes.c_char_p
        lib.map_status_string.argtypes = [ctypes.c_int]
        lib.map_status_string.restype = ctypes.c_char_p
        lib.map_workspace_bytes.argtypes = [P]
        lib.map_workspace_bytes.restype = I64
        lib.map_last_launch_count.argtypes = [P]
        lib.map_last_launch_count.restype = I64
        lib.map_version.restype = ctypes.c_char_p
        lib.map_profile_enable.argtypes = [P, I32]
        lib.map_profile_enable.restype = ctypes.c_int
        lib.map_profile_read.argtypes = [P, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(D),
                                         ctypes.POINTER(I64), I32]
        lib.map_profile_read.restype = I32
        lib.map_shard_payload_bytes.argtypes = [P, I32]
        lib.map_shard_payload_bytes.restype = I64
        lib.map_shard_phase.argtypes = [P, I32, P, P, P, P, P, P]
        lib.map_shard_phase.restype = ctypes.c_int
        lib.map_debug_lb_timing.argtypes = [P, P, I64]
        lib.map_debug_lb_timing.restype = I64
        _lib = lib
    return _lib


def _check(st: int, plan=None):
    if st != 0:
        msg = ""
        if plan:
            msg = load_library().map_last_error(plan).decode()
        raise MapError(st, msg)


def _ptr(a) -> int | None:
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("NumPy buffers passed to the C ABI must be C-contiguous")
        return a.ctypes.data
    return a.data_ptr()  # torch.Tensor (device or host)


def _check_buf(name: str, a, dtype: str, numel: int) -> None:
    """The C ABI takes plain pointers and cannot check sizes: validate a caller buffer
    (dtype == the plan dtype, contiguous, exactly `numel` elements, CUDA or host memory)."""
    if a is None:
        return
    want = np.float64 if dtype == "f64" else np.float32
    if isinstance(a, np.ndarray):
        ok_dtype, contig, n, dev = a.dtype == want, a.flags.c_contiguous, a.size, "cpu"
    else:
        import torch
        if not isinstance(a, torch.Tensor):
            raise ValueError(f"{name}: expected a torch.Tensor or numpy.ndarray, got {type(a).__name__}")
        ok_dtype = a.dtype == (torch.float64 if dtype == "f64" else torch.float32)
        contig, n, dev = a.is_contiguous(), a.numel(), a.device.type
    if not ok_dtype:
        raise ValueError(f"{name}: dtype must match the plan dtype ({dtype})")
    if not contig:
        raise ValueError(f"{name}: buffer must be contiguous")
    if n != numel:
        raise ValueError(f"{name}: expected {numel} elements, got {n}")
    if dev not in ("cuda", "cpu"):
        raise ValueError(f"{name}: buffer must live in CUDA device memory or host memory")


def batch_range(rank: int, world: int, batch: int) -> tuple[int, int]:
    """Trajectories [a, b) owned by `rank` of a batch-sharded plan (MAP_FLAG_BATCH_SHARD)."""
    return rank * batch // world, (rank + 1) * batch // world


def shard_range(rank: int, world: int, T: int) -> tuple[int, int]:
    """Nodes [a, b) owned by `rank` of a time-sharded plan (include/pmap.h: a_r = floor(r (T+1) / world))."""
    N = T + 1
    return rank * N // world, (rank + 1) * N // world


# ------------------------------------------------------------ raw C entry points
def map_plan(desc: PlanDesc, lin: LinearModel | None = None, nl: NlModel | None = None) -> int:
    lib = load_library()
    h = ctypes.c_void_p()
    st = lib.map_plan(ctypes.byref(desc), ctypes.byref(lin) if lin is not None else None,
                      ctypes.byref(nl) if nl is not None else None, ctypes.byref(h))
    _check(st)
    return h.value


def map_plan_destroy(plan: int) -> None:
    load_library().map_plan_destroy(plan)


def map_solve_linear(plan: int, y, x_map, filt_m=None, filt_P=None) -> None:
    _check(load_library().map_solve_linear(plan, _ptr(y), _ptr(x_map), _ptr(filt_m), _ptr(filt_P)), plan)


def map_solve_linear_pipelined(plan: int, y_host, x_host) -> None:
    _check(load_library().map_solve_linear_pipelined(plan, _ptr(y_host), _ptr(x_host)), plan)


def map_solve_linear_fine(plan: int, y, x_fine) -> None:
    _check(load_library().map_solve_linear_fine(plan, _ptr(y), _ptr(x_fine)), plan)


def map_solve_linear_cov(plan: int, y, x_map, smooth_P) -> None:
    _check(load_library().map_solve_linear_cov(plan, _ptr(y), _ptr(x_map), _ptr(smooth_P)), plan)


def map_two_filter(plan: int, y, x_map, smooth_P=None) -> None:
    _check(load_library().map_two_filter(plan, _ptr(y), _ptr(x_map), _ptr(smooth_P)), plan)


def map_solve_sequential(plan: int, method: int, y, passes: int, x_map, smooth_P=None) -> None:
    _check(load_library().map_solve_sequential(plan, method, _ptr(y), passes, _ptr(x_map), _ptr(smooth_P)), plan)


def map_solve_nonlinear(plan: int, y, passes: int, tol: float, x_init, x_map) -> int:
    run = ctypes.c_int32(0)
    _check(load_library().map_solve_nonlinear(plan, _ptr(y), passes, tol, _ptr(x_init), _ptr(x_map),
                                              ctypes.byref(run)), plan)
    return run.value


def map_shard_payload_bytes(plan: int, phase: int) -> int:
    return int(load_library().map_shard_payload_bytes(plan, phase))


def map_shard_phase(plan: int, phase: int, y=None, gathered=None, payload=None, x_map=None, filt_m=None,
                    filt_P=None) -> None:
    _check(load_library().map_shard_phase(plan, phase, _ptr(y), _ptr(gathered), _ptr(payload), _ptr(x_map),
                                          _ptr(filt_m), _ptr(filt_P)), plan)


def map_sync(plan: int) -> None:
    _check(load_library().map_sync(plan), plan)


def map_last_error(plan: int) -> str:
    return load_library().map_last_error(plan).decode()


def map_version() -> str:
    return load_library().map_version().decode()


# ------------------------------------------------------------------ convenience
def euler_rows(y_fine: np.ndarray, n: int) -> np.ndarray:
    """Lay out fine-grid measurements [..., n*T+1, ny] as the Euler-block rows
    [..., T+1, n*ny] of include/pmap.h (row 0: y(t_0) in its last sub-slot).  Layout only."""
    y_fine = np.asarray(y_fine)
    *lead, nf, ny = y_fine.shape
    T = (nf - 1) // n
    assert nf == n * T + 1, "fine grid must have n*T+1 points"
    out = np.zeros((*lead, T + 1, n, ny), dtype=y_fine.dtype)
    out[..., 0, n - 1, :] = y_fine[..., 0, :]
    out[..., 1:, :, :] = y_fine[..., 1:, :].reshape(*lead, T, n, ny)
    return out.reshape(*lead, T + 1, n * ny)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class Plan:
    """A solver plan for one model, grid and batch size (wraps map_plan / map_plan_destroy).

    linear model: pass F, L, W, H, R, m0, P0 (and optionally c, r); each array is
    either constant or carries a leading node axis of length T+1 (time-varying).
    nonlinear model: pass nl_kind (1 = coordinated turn, 2 = Van der Pol), L, W, R,
    m0, P0 and params.  substeps = n > 1: the paper's Euler blocks (include/pmap.h), y
    as [batch][T+1][n*ny] (see euler_rows)."""

    def __init__(self, *, T: int, t0: float, tf: float, m0, P0, L, W, R, F=None, H=None, c=None, r=None,
                 batch: int = 1, dtype: str = "f64", nl_kind: int | None = None, params=None,
                 rank: int = 0, world: int = 1, nccl_comm: int | None = None, stream: int | None = None,
                 substeps: int = 1, mixed: bool = False, shard: str = "time"):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2512_13319_b200 needs a CUDA device (no CPU fallback)")
        self._keep = []
        L, W, R, m0, P0 = map(_f64, (L, W, R, m0, P0))
        nx, nw = L.shape[-2], L.shape[-1]
        ny = R.shape[-1]
        self.nx, self.ny, self.nw, self.T, self.batch = nx, ny, nw, T, batch
        self.dtype = dtype
        self.torch_dtype = torch.float64 if dtype == "f64" else torch.float32
        d = PlanDesc()
        d.nx, d.ny, d.nw, d.dtype = nx, ny, nw, MAP_F64 if dtype == "f64" else MAP_F32
        d.T, d.batch, d.t0, d.tf = T, batch, t0, tf
        d.rank, d.world = rank, world
        d.substeps = substeps
        if shard not in ("time", "batch"):
            raise ValueError("shard: 'time' or 'batch'")
        d.flags = (MAP_FLAG_MIXED if mixed else 0) | (MAP_FLAG_BATCH_SHARD if shard == "batch" else 0)
        self.substeps = substeps
        d.nccl_comm = nccl_comm
        self.stream = torch.cuda.current_stream().cuda_stream if stream is None else stream
        d.stream = self.stream
        self.rank, self.world = rank, world
        self.shard = shard
        if shard == "batch" and world > 1:  # the rank's trajectories, every node
            self.batch0, b1 = batch_range(rank, world, batch)
            self.batch = b1 - self.batch0
            self.node0, self.n_local = 0, T + 1  # an independent single-GPU plan over them
        else:
            self.batch0 = 0
            self.node0, a1 = shard_range(rank, world, T)
            self.n_local = a1 - self.node0
        self.ny_row = ny * max(1, substeps)
        lin = nl = None

        def shape_ok(name, a, base):  # constant (base) or time-varying ((T+1,) + base)
            a = np.asarray(a)
            if a.shape != base and a.shape != (T + 1,) + base:
                raise ValueError(f"{name}: shape {a.shape}, expected {base} or {(T + 1,) + base}")
        for name, a, base in (("L", L, (nx, nw)), ("W", W, (nw, nw)), ("R", R, (ny, ny))):
            shape_ok(name, a, base)
        if m0.shape != (nx,) or P0.shape != (nx, nx):
            raise ValueError(f"m0/P0: shapes {m0.shape}/{P0.shape}, expected ({nx},)/({nx}, {nx})")
        if nl_kind is None:
            if F is None or H is None:
                raise ValueError("linear plans need F and H")
            shape_ok("F", F, (nx, nx))
            shape_ok("H", H, (ny, nx))
            if c is not None:
                shape_ok("c", c, (nx,))
            if r is not None:
                shape_ok("r", r, (ny,))
            lin = LinearModel()
            arrs = dict(F=(F, 2), c=(c, 1), L=(L, 2), W=(W, 2), H=(H, 2), r=(r, 1), R=(R, 2))
            for k, (a, nd) in arrs.items():
                if a is None:
                    setattr(lin, k, None)
                    setattr(lin, "s" + k, 0)
                    continue
                a = _f64(a)
                self._keep.append(a)
                setattr(lin, k, a.ctypes.data)
                setattr(lin, "s" + k, 0 if a.ndim == nd else int(np.prod(a.shape[1:])))
            lin.m0, lin.P0 = m0.ctypes.data, P0.ctypes.data
            self._keep += [m0, P0]
        else:
            nl = NlModel()
            params = _f64(params if params is not None else [0.0])
            self._keep += [params, L, W, R, m0, P0]
            nl.kind, nl.nparams, nl.params = nl_kind, params.size, params.ctypes.data
            nl.L, nl.W, nl.R, nl.m0, nl.P0 = (x.ctypes.data for x in (L, W, R, m0, P0))
        self.handle = map_plan(d, lin, nl)
        self.nonlinear = nl_kind is not None

    def close(self):
        if getattr(self, "handle", None):
            map_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _out(self, like, *shape):
        import torch
        dev = like.device if hasattr(like, "device") else "cpu"
        return torch.empty(shape, dtype=self.torch_dtype, device=dev)

    def _check_io(self, y=None, **outs):
        nodes = self.batch * self.n_local
        ns = self.nx * (self.nx + 1) // 2
        _check_buf("y", y, self.dtype, nodes * self.ny_row)
        rows = dict(x_map=self.nx, x_init=self.nx, filt_m=self.nx, filt_P=ns, smooth_P=ns)
        for k, a in outs.items():
            _check_buf(k, a, self.dtype, nodes * rows[k])

    def solve_linear(self, y, x_map=None, filt_m=None, filt_P=None):
        """Parallel RTS MAP (pass 1 + pass 2).  y: [batch][n_local][ny] (torch, device or host)."""
        if x_map is None:
            x_map = self._out(y, self.batch, self.n_local, self.nx)
        self._check_io(y, x_map=x_map, filt_m=filt_m, filt_P=filt_P)
        map_solve_linear(self.handle, y, x_map, filt_m, filt_P)
        return x_map

    def solve_linear_cov(self, y, x_map=None, smooth_P=None):
        """Parallel RTS MAP and the smoother covariances (map_solve_linear_cov); returns
        (x_map, smooth_P [batch][n_local][nx(nx+1)/2])."""
        if x_map is None:
            x_map = self._out(y, self.batch, self.n_local, self.nx)
        if smooth_P is None:
            smooth_P = self._out(y, self.batch, self.n_local, self.nx * (self.nx + 1) // 2)
        self._check_io(y, x_map=x_map, smooth_P=smooth_P)
        map_solve_linear_cov(self.handle, y, x_map, smooth_P)
        return x_map, smooth_P

    def solve_linear_pipelined(self, y_host, x_host):
        """map_solve_linear_pipelined: host (pinned) buffers, returns at once; consecutive
        calls overlap their copies; call sync() before reading x_host."""
        self._check_io(y_host, x_map=x_host)
        map_solve_linear_pipelined(self.handle, y_host, x_host)

    def solve_linear_fine(self, y, x_fine=None):
        """Euler-block plans: x* at every fine point (map_solve_linear_fine, R-REFINE);
        y as solve_linear (Euler rows), returns x_fine [batch][substeps*T+1][nx]."""
        nf = self.substeps * self.T + 1
        if x_fine is None:
            x_fine = self._out(y, self.batch, nf, self.nx)
        _check_buf("y", y, self.dtype, self.batch * (self.T + 1) * self.ny_row)
        _check_buf("x_fine", x_fine, self.dtype, self.batch * nf * self.nx)
        map_solve_linear_fine(self.handle, y, x_fine)
        return x_fine

    def two_filter(self, y, x_map=None, smooth_P=None):
        """Parallel two-filter MAP; smooth_P (optional, [batch][T+1][nx(nx+1)/2]) receives
        the smoother covariances."""
        if x_map is None:
            x_map = self._out(y, self.batch, self.n_local, self.nx)
        self._check_io(y, x_map=x_map, smooth_P=smooth_P)
        map_two_filter(self.handle, y, x_map, smooth_P)
        return x_map

    def solve_sequential(self, y, method: int = 0, passes: int = 1, x_map=None, smooth_P=None):
        """Sequential on-device baseline (map_solve_sequential): method 0 = RTS, 1 = two-filter."""
        if x_map is None:
            x_map = self._out(y, self.batch, self.n_local, self.nx)
        self._check_io(y, x_map=x_map, smooth_P=smooth_P)
        map_solve_sequential(self.handle, method, y, passes, x_map, smooth_P)
        return x_map

    def solve_nonlinear(self, y, passes: int = 10, tol: float = 0.0, x_init=None, x_map=None):
        if x_map is None:
            x_map = self._out(y, self.batch, self.n_local, self.nx)
        self._check_io(y, x_map=x_map, x_init=x_init)
        run = map_solve_nonlinear(self.handle, y, passes, tol, x_init, x_map)
        return x_map, run

    def sync(self):
        map_sync(self.handle)

    def shard_phase(self, phase: int, y=None, gathered=None, x_map=None, filt_m=None, filt_P=None):
        """One phase of a caller-driven time-sharded solve (map_shard_phase); returns the
        phase's payload tensor (phases 1, 2) or x_map (phase 3).  Filter outputs are
        written at phase 3 and must be passed at phase 2 too (full (S, v) storage)."""
        import torch
        if phase in (1, 2):
            self._check_io(y, filt_m=filt_m, filt_P=filt_P)
        else:
            self._check_io(y, x_map=x_map, filt_m=filt_m, filt_P=filt_P)
        if gathered is not None:
            per = {2: map_shard_payload_bytes(self.handle, 1), 3: map_shard_payload_bytes(self.handle, 2)}[phase]
            _check_buf("gathered", gathered, self.dtype, self.world * per // (8 if self.dtype == "f64" else 4))
        if phase in (1, 2):
            n = map_shard_payload_bytes(self.handle, phase) // (8 if self.dtype == "f64" else 4)
            payload = torch.empty(n, dtype=self.torch_dtype, device="cuda")
            map_shard_phase(self.handle, phase, y, gathered, payload, None, filt_m, filt_P)
            return payload
        if x_map is None:
            x_map = torch.empty((self.batch, self.n_local, self.nx), dtype=self.torch_dtype, device="cuda")
        map_shard_phase(self.handle, 3, y, gathered, None, x_map, filt_m, filt_P)  # y: optional at phase 3
        return x_map

    def profile(self, enable: bool = True) -> None:
        """Per-kernel CUDA-event timing of subsequent solves (map_profile_enable)."""
        _check(load_library().map_profile_enable(self.handle, 1 if enable else 0), self.handle)

    def profile_read(self) -> dict:
        """{kernel class: (total ms, launches)} since the last read (map_profile_read)."""
        n = 32
        names = (ctypes.c_char_p * n)()
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_int64 * n)()
        k = load_library().map_profile_read(self.handle, names, ms, cnt, n)
        if k < 0:
            raise MapError(3, map_last_error(self.handle))
        return {names[i].decode(): (ms[i], cnt[i]) for i in range(k)}

    def lb_timing(self):
        """Per-tile %globaltimer stamps of the last look-back solve ([2][tiles][8] uint64 ns),
        recorded only by plans created with PMAP_LB_TIMING=1 (diagnostics); None otherwise."""
        lib = load_library()
        n = int(lib.map_debug_lb_timing(self.handle, None, 0))
        if n <= 0:
            return None
        out = np.zeros(n, dtype=np.uint64)
        lib.map_debug_lb_timing(self.handle, out.ctypes.data, n)
        return out.reshape(2, -1, 8)

    @property
    def launches(self) -> int:
        return int(load_library().map_last_launch_count(self.handle))

    @property
    def workspace_bytes(self) -> int:
        return int(load_library().map_workspace_bytes(self.handle))
