"""In-tree build of libpsn_b200.so for sm_100a (nvcc, no JIT cache).

The shared library is written to ``paper_2501_14490_b200/_lib/`` so it travels
with the repo snapshot to the GPU box.  A stamp of the source hashes and flags
skips rebuilding when nothing changed.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(OUT_DIR, "libpsn_b200.so")
SOURCES = ["psn_layer.cu", "psn_engines.cu", "psn_stream.cu", "psn_stream_f32_fwd.cu", "psn_stream_f32_bwd.cu",
           "psn_stream_bf16_fwd.cu", "psn_stream_bf16_bwd.cu", "psn_readout.cu", "psn_optim.cu"]
HEADERS = ["psn_common.cuh", "psn_stream.cuh", "psn_stream_inst.cuh", "psn_stream_dispatch.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-cudart=static",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the PSN CUDA library cannot be built")


def _stamp() -> str:
    h = hashlib.sha256()
    for name in SOURCES + HEADERS:
        with open(os.path.join(CSRC, name), "rb") as f:
            h.update(f.read())
    with open(os.path.join(ROOT, "include", "psn_b200.h"), "rb") as f:
        h.update(f.read())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False, trace: bool = False, variant: str = "",
          defines: tuple = ()) -> str:
    """Compile every CUDA source for sm_100a and link libpsn_b200.so.

    ``trace=True`` builds the per-CTA wait/compute tracing variant
    (-DPSN_TRACE_BUILD=1) into ``_lib_trace/``; ``variant``/``defines`` build
    an experiment variant (extra -D flags) into ``_lib_<variant>/``.  Load
    either with PSN_B200_LIB (profiling and A/B tooling only).
    """
    if trace:
        variant, defines = "trace", tuple(defines) + ("PSN_TRACE_BUILD=1",)
    out_dir = OUT_DIR + (f"_{variant}" if variant else "")
    lib_path = os.path.join(out_dir, "libpsn_b200.so")
    extra = [f"-D{d}" for d in defines]
    os.makedirs(out_dir, exist_ok=True)
    stamp_path = os.path.join(out_dir, "build.stamp")
    stamp = _stamp() + " " + " ".join(extra)
    if not force and os.path.exists(lib_path) and os.path.exists(stamp_path):
        if open(stamp_path).read().strip() == stamp:
            return lib_path
    nvcc = _nvcc()
    objs = []

    def compile_one(src):
        obj = os.path.join(out_dir, src.replace(".cu", ".o"))
        cmd = [nvcc, *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-c",
               os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = lib_path + ".tmp"
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart=static",
           "-Xcompiler", "-fPIC", *objs, "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib_path)
    for o in objs:
        os.remove(o)
    with open(stamp_path, "w") as f:
        f.write(stamp + "\n")
    return lib_path


if __name__ == "__main__":
    # python -m paper_2501_14490_b200._build [--force] [--trace] [--variant NAME -DX=1 ...]
    args = sys.argv[1:]
    var = args[args.index("--variant") + 1] if "--variant" in args else ""
    defs = tuple(a[2:] for a in args if a.startswith("-D"))
    print(build(force="--force" in args, verbose=True, trace="--trace" in args, variant=var, defines=defs))
