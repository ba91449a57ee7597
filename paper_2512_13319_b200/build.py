"""Build libpmap.so (sm_100a) in-tree: one nvcc invocation per instantiation unit, in parallel.

Usage: python -m paper_2512_13319_b200.build [-j N] [--f64-only]
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.environ.get("PMAP_OBJ_DIR", "/tmp/pmap_build")  # object files live outside the repo
LIB = os.path.join(HERE, "libpmap.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-diag-suppress", "128"] + ARCH + \
    [f for f in os.environ.get("PMAP_NVCC_EXTRA", "").split() if f]

SHAPES = [(1, 1), (2, 1), (2, 2), (3, 1), (3, 2), (4, 2), (5, 2)]


EULER_SHAPES = [(1, 1), (4, 2)]  # OU (C1) and Wiener velocity
EULER_NSUB = 10                  # substeps per block

RUN_LENGTHS = (32, 8)  # nodes per run (tile = 64 runs): large / small problems
NL_TINY_K = 4          # nonlinear plans on modest grids (general combines: shorter chains)


def units(f64_only: bool = False):
    out = []
    for R in (("double",) if f64_only else ("double", "float")):
        tag = "f64" if R == "double" else "f32"
        for K in RUN_LENGTHS:
            base = ["-DPM_R=" + R, f"-DPM_K={K}"]
            for kind in (0, 1):
                for nx, ny in SHAPES:
                    out.append((f"inst_{tag}_K{K}_k{kind}_{nx}{ny}",
                                base + [f"-DPM_NX={nx}", f"-DPM_NY={ny}", f"-DPM_KIND={kind}"], "inst.cu"))
            out.append((f"inst_{tag}_K{K}_ct", base + ["-DPM_NX=5", "-DPM_NY=2", "-DPM_KIND=2"], "inst.cu"))
            out.append((f"inst_{tag}_K{K}_vdp", base + ["-DPM_NX=2", "-DPM_NY=1", "-DPM_KIND=3"], "inst.cu"))
            for nx, ny in EULER_SHAPES:  # paper-faithful Euler blocks
                out.append((f"inst_{tag}_K{K}_eu{nx}{ny}", base + [f"-DPM_NX={nx}", f"-DPM_NY={ny}", "-DPM_KIND=4",
                                                                   f"-DPM_NSUB={EULER_NSUB}"], "inst.cu"))
        # nonlinear models also get the tiny run length (pmap_abi.cu choose_run_length)
        tb = ["-DPM_R=" + R, f"-DPM_K={NL_TINY_K}"]
        out.append((f"inst_{tag}_K{NL_TINY_K}_ct", tb + ["-DPM_NX=5", "-DPM_NY=2", "-DPM_KIND=2"], "inst.cu"))
        out.append((f"inst_{tag}_K{NL_TINY_K}_vdp", tb + ["-DPM_NX=2", "-DPM_NY=1", "-DPM_KIND=3"], "inst.cu"))
    out.append(("pmap_abi", [], "pmap_abi.cu"))
    return out


def _deps_mtime() -> float:
    paths = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "pmap.h")]
    return max(os.path.getmtime(p) for p in paths)


def _compile(u, verbose=False):
    name, defs, src = u
    obj = os.path.join(OBJ, name + ".o")
    cmd = [NVCC] + FLAGS + defs + ["-c", os.path.join(CSRC, src), "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {name}:\n{r.stderr}")
    return obj, r.stderr


def build(jobs: int | None = None, f64_only: bool = False, force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    us = units(f64_only)
    dep = _deps_mtime()
    todo = [u for u in us if force or not os.path.exists(os.path.join(OBJ, u[0] + ".o"))
            or os.path.getmtime(os.path.join(OBJ, u[0] + ".o")) < dep]
    logs = []
    if todo:
        with ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
            for obj, log in ex.map(lambda u: _compile(u, verbose), todo):
                logs.append(log)
    objs = [os.path.join(OBJ, u[0] + ".o") for u in us]
    if todo or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        tmp = LIB + ".tmp"
        subprocess.check_call([NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl"])
        os.replace(tmp, LIB)
    if verbose:
        sys.stderr.write("".join(logs))
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("--f64-only", action="store_true")
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    a = ap.parse_args()
    print(build(a.j, a.f64_only, a.force, a.v))
