"""Build libmxmoe.so (in-tree) with nvcc for sm_100a."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmxmoe.so")
SOURCES = ["api.cu", "quant.cu", "route.cu", "plan.cu", "gemm.cu", "ep.cu", "gptq.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-warn-spills",
]


def _nccl_dir() -> str:
    """NCCL 2.28 of the torch wheel (nvidia-nccl-cu12): headers + libnccl.so.2 (the EP C ABI's collectives)."""
    import nvidia.nccl
    return list(nvidia.nccl.__path__)[0]


NCCL = _nccl_dir()
FLAGS += ["-I" + os.path.join(NCCL, "include"), "-L" + os.path.join(NCCL, "lib"), "-l:libnccl.so.2",
          "-Xlinker", "-rpath=" + os.path.join(NCCL, "lib")]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "mxmoe.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every source to an object in parallel (gemm.cu dominates), then link libmxmoe.so."""
    if not force and not _stale():
        return LIB
    import tempfile
    tmp = tempfile.mkdtemp(prefix="mxmoe_build_")
    compile_flags = [f for f in FLAGS if f not in ("-shared", "-l:libnccl.so.2", "-Xlinker")
                     and not f.startswith("-rpath") and not f.startswith("-L")]
    procs = []
    for src in SOURCES:
        obj = os.path.join(tmp, src.replace(".cu", ".o"))
        cmd = [NVCC, *compile_flags, "-c", "-o", obj, os.path.join(CSRC, src)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    objs = []
    for obj, pr in procs:
        out, err = pr.communicate()
        if pr.returncode != 0:
            sys.stderr.write(out + err)
            raise RuntimeError("nvcc failed compiling " + os.path.basename(obj))
        if verbose:
            sys.stderr.write(err)
        objs.append(obj)
    link = [NVCC, *FLAGS, "-o", LIB + ".tmp", *objs]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libmxmoe.so")
    os.replace(LIB + ".tmp", LIB)
    return LIB


def build_variant(out: str, defines) -> str:
    """Build an experiment variant of the library (extra -D flags) at `out` (in-tree, for A/B timing)."""
    cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-o", out, *[os.path.join(CSRC, s) for s in SOURCES]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building " + out)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
