"""Build libbiot_pit.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2310_10430_b200.build [--force]

Writes paper_2310_10430_b200/libbiot_pit.so and the ptxas resource report
paper_2310_10430_b200/build/ptxas.txt (registers / spills per kernel).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libbiot_pit.so")
BUILD = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["host_assembly.cpp", "sweep_kernels.cu", "march_kernels.cu", "tile2d_kernels.cu", "tile3d_kernels.cu", "gmres_kernels.cu", "cheb_kernels.cu", "biot_api.cu"]
HEADERS = ["host_assembly.h", "sweep_kernels.cuh", "node_update.cuh", "tma_util.cuh"]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "biot_pit.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """out / defines: an experimental variant (-D flags) built beside the product library
    (tools/build_variant.py; loaded through BIOT_LIB_OVERRIDE for A/B timing)."""
    variant = out is not None
    out = out or OUT
    if not variant and not force and not _stale():
        return OUT
    bdir = BUILD if not variant else os.path.join(BUILD, "variant_" + os.path.splitext(os.path.basename(out))[0])
    os.makedirs(bdir, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]
    def compile_one(src):
        path = os.path.join(CSRC, src)
        obj = os.path.join(bdir, src + ".o")
        if src.endswith(".cu"):
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *dflags,
                   "-Xptxas", "-v", "--expt-relaxed-constexpr", "-c", path, "-o", obj]
        else:
            cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-fopenmp", "-Wall", "-c", path, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, cmd, r

    # translation units compile in parallel (the tile kernels dominate the build time)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(SOURCES), os.cpu_count() or 1))) as ex:
        results = list(ex.map(compile_one, SOURCES))
    objs = []
    report = []
    for src, obj, cmd, r in results:
        report.append(f"$ {' '.join(cmd)}\n{r.stdout}{r.stderr}")
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"compile failed: {src}")
        objs.append(obj)
    tmp = out + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs,
           "-Xcompiler", "-fopenmp", "-lgomp", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    report.append(f"$ {' '.join(cmd)}\n{r.stdout}{r.stderr}")
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, out)
    with open(os.path.join(bdir, "ptxas.txt"), "w") as f:
        f.write("\n".join(report))
    if verbose:
        print("\n".join(report))
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
