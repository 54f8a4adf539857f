"""Build libsupra_bf.so in-tree: sm_100a kernels (nvcc) + binary64 host library
(g++ -ffp-contract=off).  ``python -m paper_1711_06127_b200.build``."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsupra_bf.so")
BUILD = os.path.join(HERE, "_build")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU = (["das.cu", "das_warp.cu"] + [f"das_warp_inst{i}.cu" for i in range(3)] +
      ["epilogue.cu", "scanconv.cu", "stage.cu"])
CPP = ["host.cpp"]
HDRS = ["internal.h", "epilogue.cuh", "das_common.cuh", "das_kernel.cuh", "das_warp_kernel.cuh"]


def das_instances() -> int:
    """Rows of kDasInst in csrc/das_inst.cu (one DAS kernel per translation unit)."""
    import re
    src = open(os.path.join(CSRC, "das_inst.cu")).read()
    table = src[src.index("kDasInst[][4] = {"):src.index("};", src.index("kDasInst[][4] = {"))]
    return len(re.findall(r"\{\s*\d+,\s*\d+,\s*[01],\s*\d+\s*\}", table))


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False, variant: str = "",
          defines=()) -> str:
    """Build the library; ``variant``/``defines`` build an A/B variant into
    _variants/<variant>/libsupra_bf.so (dev aid, loaded with binding.use_library)."""
    global BUILD, OUT
    if variant:
        BUILD = os.path.join(ROOT, "_variants", variant, "_build")
        OUT = os.path.join(ROOT, "_variants", variant, "libsupra_bf.so")
    os.makedirs(BUILD, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    hdr_deps = [os.path.join(CSRC, h) for h in HDRS] + [os.path.join(ROOT, "include", "supra_bf.h")]
    objs = []
    cmds = []
    units = [(f, f + ".o", []) for f in CU]
    units += [("das_inst.cu", f"das_inst.{i}.o", [f"-DDAS_INST={i}"]) for i in range(das_instances())]
    for f, o, udefs in units:
        src = os.path.join(CSRC, f)
        obj = os.path.join(BUILD, o)
        objs.append(obj)
        if force or _stale(obj, [src] + hdr_deps):
            cmd = [os.path.join(CUDA, "bin", "nvcc"), *ARCH, *dflags, *udefs, "-O3", "-lineinfo", "-std=c++17",
                   "--expt-relaxed-constexpr", "-Xfatbin=-compress-all", "-Xcompiler", "-fPIC", *inc, "-c", src, "-o", obj]
            if ptxas_v:
                cmd.insert(1, "-Xptxas=-v")
            cmds.append(cmd)
    # translation units compile in parallel (one DAS batch variant per unit;
    # the warp-split variants are split over das_warp_inst*.cu)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        list(ex.map(lambda c: _run(c, verbose), cmds))
    for f in CPP:
        src = os.path.join(CSRC, f)
        obj = os.path.join(BUILD, f + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + hdr_deps):
            _run(["g++", *dflags, "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                  "-Wall", "-I", os.path.join(CUDA, "include"), *inc, "-c", src, "-o", obj], verbose)
    if force or _stale(OUT, objs):
        _run([os.path.join(CUDA, "bin", "nvcc"), *ARCH, "-shared", "-o", OUT, *objs,
              "-Xcompiler", "-fPIC", "-cudart", "static", "-Xlinker", "--no-undefined"], verbose)
    return OUT


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), "")
    defs = [a[2:] for a in sys.argv if a.startswith("-D")]
    build(force="--force" in sys.argv, verbose=True, ptxas_v="-v" in sys.argv, variant=var, defines=defs)
    print(OUT)
