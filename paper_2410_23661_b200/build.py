"""Build libpicker.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

    python -m paper_2410_23661_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libpicker.so")
BUILD = os.path.join(HERE, "..", "build", "picker")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++17", "-O3", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall"]
CUFLAGS = ARCH + COMMON + ["-lineinfo", "--expt-relaxed-constexpr", "-Xptxas", "-v"]

CU = ["k_generic.cu", "k_exact.cu", "k_jit_host.cu"]
CPP = ["loader.cpp", "picker.cpp", "dispatch.cpp", "jit.cpp"]


def _sources():
    cu = [f for f in CU if os.path.exists(os.path.join(CSRC, f))]
    cpp = [f for f in CPP if os.path.exists(os.path.join(CSRC, f))]
    return cu, cpp


def _newer(src_files, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(f) > t for f in src_files)


def build(verbose=False, force=False):
    os.makedirs(BUILD, exist_ok=True)
    cu, cpp = _sources()
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh", ".h"))]
    headers.append(os.path.join(HERE, "..", "include", "picker.h"))
    jobs = []
    objs = []
    for f in cu + cpp:
        src = os.path.join(CSRC, f)
        obj = os.path.join(BUILD, f + ".o")
        objs.append(obj)
        if force or _newer([src] + headers, obj):
            cmd = [NVCC] + (CUFLAGS if f.endswith(".cu") else ARCH + COMMON) + ["-c", src, "-o", obj]
            jobs.append((f, cmd))

    def run(job):
        name, cmd = job
        p = subprocess.run(cmd, capture_output=True, text=True)
        return name, cmd, p

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for name, cmd, p in ex.map(run, jobs):
            if p.returncode != 0:
                sys.stderr.write(p.stdout + p.stderr)
                raise RuntimeError(f"nvcc failed on {name}")
            if verbose:
                sys.stderr.write(f"[build] {name}\n{p.stderr}")
    if force or jobs or not os.path.exists(OUT):
        cmd = [NVCC] + ARCH + ["-shared", "-o", OUT] + objs + [
            "-cudart", "static", f"-L{CUDA}/lib64", "-lnvrtc", f"-Xlinker", f"-rpath={CUDA}/lib64",
        ]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            sys.stderr.write(p.stdout + p.stderr)
            raise RuntimeError("link failed")
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
