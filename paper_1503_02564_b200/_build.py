"""Build libswr.so (the C-ABI library) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SO = os.path.join(PKG, "libswr.so")
SOURCES = ["swr_march.cu", "swr_march_stream.cu", "swr_linalg.cu", "swr_pinv.cu", "swr_api.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
         "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"), "-I", CSRC]


STAMP = os.path.join(PKG, "build", "flags.txt")


def _extra_flags() -> list:
    # SWR_TRACE_BUILD=1: compile the march phase-trace points in (tools/march_trace.sh)
    return ["-DSWR_MARCH_TRACE=1"] if os.environ.get("SWR_TRACE_BUILD") == "1" else []


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    try:
        if open(STAMP).read() != " ".join(_extra_flags()):
            return True
    except OSError:
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "swr.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return SO
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)

    def comp(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *_extra_flags(), "-Xptxas", "-v" if verbose else "-O3", "-c", os.path.join(CSRC, src),
               "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return obj, r.stderr

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        res = list(ex.map(comp, SOURCES))
    if verbose:
        for _, err in res:
            sys.stderr.write(err)
    objs = [o for o, _ in res]
    tmp = SO + ".tmp"
    subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs,
                           "-ldl"])
    os.replace(tmp, SO)
    with open(STAMP, "w") as f:
        f.write(" ".join(_extra_flags()))
    return SO


def build_variant(tag: str, defines: list, force: bool = False) -> str:
    """A libswr build with extra nvcc defines at ROOT/build_variants/libswr_<tag>.so
    (race-stress tests: -DSWR_RACE_STRESS=1; kernel-shape experiments).  Not
    the product library; never loaded by the package unless passed explicitly."""
    out = os.path.join(ROOT, "build_variants")
    os.makedirs(out, exist_ok=True)
    so = os.path.join(out, f"libswr_{tag}.so")
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "swr.h")]
    if not force and os.path.exists(so) and all(os.path.getmtime(d) <= os.path.getmtime(so) for d in deps):
        return so

    def comp(src):
        obj = os.path.join(out, f"{tag}_{src.replace('.cu', '.o')}")
        r = subprocess.run([NVCC, *FLAGS, *defines, "-Xptxas", "-O3", "-c", os.path.join(CSRC, src), "-o", obj],
                           capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(comp, SOURCES))
    subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", so + ".tmp", *objs,
                           "-ldl"])
    os.replace(so + ".tmp", so)
    for o in objs:
        os.remove(o)
    return so


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
