"""CPU-side checks of the C ABI library: it loads, exports every symbol include/pmap.h
declares, and the product path refuses to run without a CUDA device (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "pmap.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(map_[a-z_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    import paper_2512_13319_b200 as pm
    if not os.path.exists(pm.LIB_PATH):
        from paper_2512_13319_b200 import build
        build.build()
    return ctypes.CDLL(pm.LIB_PATH)


def test_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    from paper_2512_13319_b200.binding import EXPORTS
    assert sorted(EXPORTS) == syms


def test_version_and_status_strings(lib):
    lib.map_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.map_version()
    lib.map_status_string.restype = ctypes.c_char_p
    lib.map_status_string.argtypes = [ctypes.c_int]
    assert lib.map_status_string(5) == b"numeric failure"


def test_null_arguments_rejected(lib):
    lib.map_plan.restype = ctypes.c_int
    assert lib.map_plan(None, None, None, None) == 1          # MAP_E_ARG
    lib.map_solve_linear.restype = ctypes.c_int
    assert lib.map_solve_linear(None, None, None, None, None) == 1


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_2512_13319_b200 as pm
    with pytest.raises(RuntimeError):
        pm.Plan(T=10, t0=0.0, tf=1.0, F=[[0.0]], L=[[1.0]], W=[[1.0]], H=[[1.0]], R=[[1.0]], m0=[0.0], P0=[[1.0]])


def test_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2512_13319_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.c" not in txt, f


def test_nccl_symbol_lookup_strategy():
    """libpmap resolves ncclAllGather from the NCCL that torch already loaded (dlsym on
    RTLD_DEFAULT, else dlopen("libnccl.so.2", RTLD_NOLOAD)); check that lookup works in a
    torch process (no GPU needed)."""
    import torch  # noqa: F401  (loads libtorch_cuda -> libnccl.so.2)
    import torch.distributed as dist
    if not dist.is_nccl_available():
        pytest.skip("torch built without NCCL")
    RTLD_NOLOAD = 4
    h = ctypes.CDLL("libnccl.so.2", mode=RTLD_NOLOAD)
    assert hasattr(h, "ncclAllGather")


def test_batch_range_partition():
    """batch_range / shard_range partition [0, n) in rank order (MAP_FLAG_BATCH_SHARD, time shards)."""
    from paper_2512_13319_b200.binding import batch_range, shard_range
    for n, w in [(7, 3), (1024, 8), (4, 4), (10_001, 8)]:
        for f, m in ((batch_range, n), (shard_range, n - 1)):
            parts = [f(r, w, m) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[r][1] == parts[r + 1][0] for r in range(w - 1))
