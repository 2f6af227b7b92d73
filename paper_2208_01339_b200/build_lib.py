"""Build libnpc.so in-tree with nvcc for sm_100a (no GPU needed; nvcc cross-compiles).

    python -m paper_2208_01339_b200.build_lib [--force]

Each csrc/*.cu is compiled to an object (-gencode arch=compute_100a,code=sm_100a -lineinfo
-O3) and linked into paper_2208_01339_b200/libnpc.so against the NCCL that torch loads
(pip package nvidia-nccl, soname libnccl.so.2; SURVEY finding 9).
"""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libnpc.so")
OBJDIR = os.path.join(PKG, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia-nccl (the NCCL torch loads) not found")
    base = list(spec.submodule_search_locations)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _flags():
    inc, _ = nccl_dirs()
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-I", INCLUDE,
                   "-I", CSRC, "-I", inc, "--expt-relaxed-constexpr", "-Xptxas", "-v"] + \
        (["-DNPC_DEBUG"] if os.environ.get("NPC_DEBUG") else []) + \
        os.environ.get("NPC_EXTRA_FLAGS", "").split()


def build_variant(name: str, defines: list[str]) -> str:
    """Build an A/B variant of the library (tuning experiments only) to
    paper_2208_01339_b200/variants/libnpc_<name>.so; load it with NPC_LIB_PATH=<path>."""
    global LIB, OBJDIR
    saved = (LIB, OBJDIR, os.environ.get("NPC_EXTRA_FLAGS"))
    vdir = os.path.join(PKG, "variants")
    os.makedirs(vdir, exist_ok=True)
    LIB = os.path.join(vdir, f"libnpc_{name}.so")
    OBJDIR = os.path.join(PKG, "build", f"variant_{name}")
    os.environ["NPC_EXTRA_FLAGS"] = " ".join(defines)
    try:
        return build()
    finally:
        LIB, OBJDIR = saved[0], saved[1]
        if saved[2] is None:
            os.environ.pop("NPC_EXTRA_FLAGS", None)
        else:
            os.environ["NPC_EXTRA_FLAGS"] = saved[2]


def _digest(paths, flags):
    h = hashlib.sha256(" ".join(flags).encode())
    for p in sorted(paths):
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(INCLUDE, "npc.h")]
    flags = _flags()
    stamp = os.path.join(OBJDIR, "digest")
    dig = _digest(srcs + hdrs, flags)
    if not force and os.path.exists(LIB) and os.path.exists(stamp) and open(stamp).read() == dig:
        return LIB
    os.makedirs(OBJDIR, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(OBJDIR, os.path.basename(src) + ".o")
        cmd = [NVCC, *flags, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        with open(obj + ".ptxas.txt", "w") as f:
            f.write(r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, srcs))
    _, libdir = nccl_dirs()
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-L", libdir, "-l:libnccl.so.2",
           f"-Xlinker=-rpath,{libdir}", "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    with open(stamp, "w") as f:
        f.write(dig)
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
