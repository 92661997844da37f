"""Build libhcnn_b200.so in-tree for sm_100a (nvcc; one object per ring degree).

    python -m paper_1811_00778_b200.build [--force] [-j N]
"""

from __future__ import annotations

import argparse
import concurrent.futures
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(os.path.dirname(PKG), "build", "hcnn")
LIB = os.path.join(PKG, "libhcnn_b200.so")
LOGNS = list(range(2, 16))
KS = list(range(1, 17))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
]


def _sources():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(os.path.dirname(PKG), "include", "hcnn_b200.h")
    ]


def _newest_source() -> float:
    return max(os.path.getmtime(p) for p in _sources())


def _deps(src: str, seen=None) -> set:
    """src plus every file it #includes with quotes, transitively."""
    import re

    seen = set() if seen is None else seen
    src = os.path.normpath(src)
    if src in seen or not os.path.exists(src):
        return seen
    seen.add(src)
    with open(src) as fh:
        for inc in re.findall(r'^\s*#\s*include\s+"([^"]+)"', fh.read(), re.M):
            _deps(os.path.join(os.path.dirname(src), inc), seen)
    return seen


def _compile(args):
    src, obj, defs = args
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in _deps(src)) \
            and os.path.getmtime(obj) >= os.path.getmtime(__file__):
        return obj  # up to date
    cmd = [NVCC, *FLAGS, *defs, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {os.path.basename(obj)}:\n{r.stderr[-4000:]}")
    return obj


def build(force: bool = False, jobs: int | None = None, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest_source():
        if not os.path.exists(EXAMPLE) or os.path.getmtime(EXAMPLE) < os.path.getmtime(EXAMPLE + ".c"):
            build_example()
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    units = [(os.path.join(CSRC, "hcnn.cu"), os.path.join(BUILD, "hcnn.o"), [])]
    for L in LOGNS:
        units.append((os.path.join(CSRC, "ntt_inst.cu"), os.path.join(BUILD, f"ntt_{L}.o"),
                      [f"-DHCNN_LOGN={L}"]))
    for K in KS:
        units.append((os.path.join(CSRC, "conv_inst.cu"), os.path.join(BUILD, f"conv_{K}.o"),
                      [f"-DHCNN_K={K}"]))
    # biggest units first
    units.sort(key=lambda u: -int(u[2][0].split("=")[1]) if u[2] else -99)
    for stale in os.listdir(BUILD):
        if stale.endswith(".o") and os.path.join(BUILD, stale) not in [u[1] for u in units]:
            os.remove(os.path.join(BUILD, stale))
    jobs = jobs or os.cpu_count() or 4
    with concurrent.futures.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(_compile, units))
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    build_example()
    if verbose:
        print(f"built {LIB}")
    return LIB


EXAMPLE = os.path.join(os.path.dirname(PKG), "examples", "capi_hsquare")


def build_example() -> str:
    """examples/capi_hsquare: a plain C program calling the C ABI (gcc, linked
    against the in-tree library with an $ORIGIN-relative rpath)."""
    src = EXAMPLE + ".c"
    cmd = ["gcc", "-O2", "-std=c11", "-I", os.path.join(os.path.dirname(PKG), "include"), src, "-o", EXAMPLE,
           "-L", PKG, "-lhcnn_b200", "-Wl,-rpath,$ORIGIN/../paper_1811_00778_b200"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"gcc failed for {src}:\n{r.stderr[-4000:]}")
    return EXAMPLE


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    a = ap.parse_args()
    build(force=a.force, jobs=a.j, verbose=True)
    sys.exit(0)
