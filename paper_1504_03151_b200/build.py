"""Build libb200rt.so (the C-ABI library of include/rt.h) for sm_100a with nvcc, in-tree."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libb200rt.so")
SRCS = [os.path.join(HERE, "csrc", f) for f in ("rt_api.cu", "rt_kernels.cu", "rt_scene_io.cpp")]
DEPS = [os.path.join(HERE, "csrc", f) for f in sorted(os.listdir(os.path.join(HERE, "csrc")))] + \
    [os.path.join(ROOT, "include", "rt.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    newest = max(os.path.getmtime(p) for p in DEPS)
    if not force and os.path.exists(out) and os.path.getmtime(out) >= newest:
        return out
    tmp = out + f".tmp{os.getpid()}"
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "-Xptxas", "-v", "-I", os.path.join(ROOT, "include"), *[f"-D{d}" for d in defines], "-o", tmp, *SRCS]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stdout.write(res.stderr)
    os.replace(tmp, out)
    return out


CHECKED_LIB = os.path.join(HERE, "libb200rt_checked.so")


def build_checked(force: bool = False) -> str:
    """The checked build (-DRT_CHECKS=1): every kernel checks its queue / list / slot indices and
    capacities and records the first failure (rt_check_status). Test support (compute-sanitizer
    is not available on this pool)."""
    return build(force=force, out=CHECKED_LIB, defines=("RT_CHECKS=1",))


FFMA2_PEAK_SRC = os.path.join(ROOT, "tools", "micro", "ffma2_peak.cu")
FFMA2_PEAK_BIN = os.path.join(ROOT, "tools", "micro", "ffma2_peak")


def build_peak_tool(force: bool = False) -> str:
    """The FFMA2 peak microbenchmark bench.py runs before timing (a measurement tool, not part of
    the library)."""
    if not force and os.path.exists(FFMA2_PEAK_BIN) and os.path.getmtime(FFMA2_PEAK_BIN) >= os.path.getmtime(FFMA2_PEAK_SRC):
        return FFMA2_PEAK_BIN
    tmp = FFMA2_PEAK_BIN + f".tmp{os.getpid()}"
    subprocess.check_call([nvcc(), *ARCH, "-O3", "-lineinfo", "-o", tmp, FFMA2_PEAK_SRC])
    os.replace(tmp, FFMA2_PEAK_BIN)
    return FFMA2_PEAK_BIN


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--out", default=LIB)
    ap.add_argument("-D", dest="defines", action="append", default=[])
    a = ap.parse_args()
    print(build(force=a.force, verbose=True, out=a.out, defines=a.defines))
