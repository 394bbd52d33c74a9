"""Build libmoe_dts.so (all CUDA kernels + the C ABI) in-tree for sm_100a.

    python -m paper_2112_14397_b200.build [--force] [--verbose]

nvcc cross-compiles for `-gencode arch=compute_100a,code=sm_100a` without a GPU.
Objects are rebuilt when their source or any header is newer.  The shared object is
written to paper_2112_14397_b200/lib/libmoe_dts.so (git-ignored, shipped by gpurun).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# Experiment builds: MOE_NVCC_EXTRA="-DFOO" MOE_LIB_OUT=.../libx.so (separate object dir)
EXTRA = os.environ.get("MOE_NVCC_EXTRA", "").split()
_tag = ("_" + "".join(c if c.isalnum() else "_" for c in "".join(EXTRA))) if EXTRA else ""
BUILD = os.path.join(PKG, "build" + _tag)
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.environ.get("MOE_LIB_OUT", os.path.join(LIB_DIR, "libmoe_dts.so"))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str | None:
    try:
        import nvidia.nccl  # type: ignore
        d = os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
    except Exception:
        d = os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl")
    return d if os.path.isdir(os.path.join(d, "include")) else None


def _flags(extra_inc):
    f = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
                "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC]
    for i in extra_inc:
        f += ["-I", i]
    if os.environ.get("MOE_PTXAS_VERBOSE"):
        f += ["-Xptxas", "-v"]
    return f


def _newest_header() -> float:
    hs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    return max((os.path.getmtime(h) for h in hs), default=0.0)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    nd = nccl_dir()
    inc = [os.path.join(nd, "include")] if nd else []
    defs = ["-DMOE_HAVE_NCCL=1"] if nd else []
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdr_t = _newest_header()
    jobs = []
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s)[:-3] + ".o")
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), hdr_t):
            jobs.append((s, o))

    def comp(so):
        s, o = so
        cmd = [NVCC] + _flags(inc) + defs + EXTRA + ["-c", s, "-o", o]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {s}:\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stderr.strip() or r.stdout.strip()):
            print(r.stdout + r.stderr, flush=True)
        return o

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        list(ex.map(comp, jobs))
    objs = [os.path.join(BUILD, os.path.basename(s)[:-3] + ".o") for s in srcs]
    if force or jobs or not os.path.exists(LIB) or \
            os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        link = [NVCC] + ARCH + ["-shared", "-o", LIB + ".tmp"] + objs + ["-lcudart"]
        if nd:
            link += ["-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
                     "-Xlinker", "-rpath=" + os.path.join(nd, "lib")]
        if verbose:
            print(" ".join(link), flush=True)
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(LIB + ".tmp", LIB)
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args(argv)
    print(build(force=a.force, verbose=a.verbose))


if __name__ == "__main__":
    sys.exit(main())
