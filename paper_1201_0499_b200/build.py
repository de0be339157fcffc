"""In-tree build of libpolyjac_b200.so (sm_100a) — nvcc cross-compiles without a GPU.

    python -m paper_1201_0499_b200.build [--force]

The .so lands next to this file (git-ignored, shipped to the GPU box by gpurun).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
SO = os.path.join(HERE, "libpolyjac_b200.so")
CLI = os.path.join(HERE, "polyjac_b200")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU = ["eval_kernels.cu", "eval_fast.cu", "eval_fast_ws.cu", "eval_fastd.cu", "newton.cu", "fp64_probe.cu"]
CPP = ["capi.cpp", "sysio.cpp"]
HEADERS = ["dd.cuh", "eval_kernels.h", "fast_common.cuh"]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd))
    return r


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "polyjac_b200.h")]
    objs = []
    for f in CU:
        src = os.path.join(CSRC, f)
        obj = os.path.join(BUILD, f + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
               "-fmad=false", "-Xptxas", "-v", "-c", src, "-o", obj]
        ks = os.environ.get("PJB_FAST_KS")  # developer shortcut: e.g. "8,16" (default: 2..16)
        if ks and f in ("eval_fast.cu", "eval_fast_ws.cu"):
            mac = "PJB_FAST_KS" if f == "eval_fast.cu" else "PJB_WS_KS"
            cmd.insert(-4, f"-D{mac}(X)=" + " ".join(f"X({k})" for k in ks.split(",") if f == "eval_fast.cu" or int(k) <= 12))
        stamp = obj + ".cmd"
        old = open(stamp).read() if os.path.exists(stamp) else ""
        if force or old != " ".join(cmd) or _newer(obj, [src] + hdrs):
            r = _run(cmd)
            with open(stamp, "w") as fh:
                fh.write(" ".join(cmd))
            if verbose:
                sys.stderr.write(r.stderr)
        objs.append(obj)
    for f in CPP:
        src = os.path.join(CSRC, f)
        obj = os.path.join(BUILD, f + ".o")
        if force or _newer(obj, [src] + hdrs):
            _run(["g++", "-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-fvisibility=hidden",
                  "-I/usr/local/cuda/include", "-c", src, "-o", obj])
        objs.append(obj)
    vs = os.path.join(BUILD, "exports.map")
    with open(vs, "w") as fh:
        fh.write("{ global: pj_*; local: *; };\n")
    if force or _newer(SO, objs):
        _run([NVCC, *ARCH, "-shared", "-o", SO, *objs, "-Xlinker", "--version-script=" + vs])
    # command-line front end (f3): links the library with an $ORIGIN rpath
    cli_src = os.path.join(CSRC, "cli.cpp")
    cli_obj = os.path.join(BUILD, "cli.cpp.o")
    if force or _newer(cli_obj, [cli_src] + hdrs):
        _run(["g++", "-std=c++17", "-O2", "-I/usr/local/cuda/include", "-c", cli_src, "-o", cli_obj])
    if force or _newer(CLI, [cli_obj, SO]):
        _run([NVCC, *ARCH, "-o", CLI, cli_obj, "-L" + HERE, "-lpolyjac_b200", "-Xlinker", "-rpath,$ORIGIN"])
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
