"""Build libls.so in-tree with nvcc for sm_100a (called by __graft_entry__.build()).

Every translation unit is compiled separately (in parallel) with
    nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -Xcompiler -fPIC -c
and linked with nvcc -shared.  rd_inst.cu is compiled once per k-step bucket of
the register-direct FD mode kernel (-DLS_RD_KS=<KS>).  Links the torch-bundled
NCCL 2.28 (one libnccl.so.2 per process).
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libls.so")
OBJ = os.path.join(HERE, "build")
SOURCES = ["api.cu", "comm.cu", "setup_host.cpp", "mv2.cu", "mv3.cu", "mv4.cu", "mv5.cu", "geo.cu", "geo_host.cpp", "err.cu", "ft.cu", "pl.cu", "mv6.cu"]
RD_BUCKETS = [2, 4, 5, 8, 9, 12, 13, 16, 17, 18, 24, 25, 26, 30, 33, 34]  # = LS_RD_BUCKETS


def _nccl_dir():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in spec.submodule_search_locations:
        d = os.path.join(base, "nccl")
        if os.path.isdir(os.path.join(d, "include")):
            return d
    raise RuntimeError("torch-bundled NCCL not found")


def _newest_source_mtime():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    files.append(os.path.join(ROOT, "include", "ls_api.h"))
    files.append(os.path.abspath(__file__))
    return max(os.path.getmtime(f) for f in files)


def _deps(src, seen=None):
    """src plus every local header it includes (recursively): the rebuild trigger of a unit."""
    import re
    seen = set() if seen is None else seen
    if src in seen or not os.path.exists(src):
        return seen
    seen.add(src)
    for inc in re.findall(r'^#include "([^"]+)"', open(src).read(), re.M):
        for d in (CSRC, os.path.join(ROOT, "include")):
            f = os.path.join(d, inc)
            if os.path.exists(f):
                _deps(f, seen)
                break
    return seen


def _stale(unit):
    src, obj, extra = unit
    if not os.path.exists(obj):
        return True
    flag = obj + ".flags"
    if not os.path.exists(flag) or open(flag).read() != " ".join(extra):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(f) > t for f in _deps(src) | {os.path.abspath(__file__)})


def _units():
    units = [(os.path.join(CSRC, s), os.path.join(OBJ, s + ".o"), []) for s in SOURCES]
    for k in RD_BUCKETS:
        units.append((os.path.join(CSRC, "rd_inst.cu"), os.path.join(OBJ, f"rd_ks{k}.o"), [f"-DLS_RD_KS={k}"]))
    return units


def build(force=False, verbose=False, jobs=None):
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest_source_mtime():
        return LIB
    nccl = _nccl_dir()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    os.makedirs(OBJ, exist_ok=True)
    common = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
              "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", os.path.join(nccl, "include")]

    def compile_unit(u):
        src, obj, extra = u
        res = subprocess.run(common + extra + ["-c", src, "-o", obj], capture_output=True, text=True)
        if res.returncode == 0:
            with open(obj + ".flags", "w") as f:
                f.write(" ".join(extra))
        return src, extra, res

    todo = [u for u in _units() if force or _stale(u)]
    jobs = jobs or max(1, min(len(todo) or 1, os.cpu_count() or 1))
    with ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(compile_unit, todo))
    failed = [r for r in results if r[2].returncode != 0]
    for src, extra, res in results:
        if verbose or res.returncode != 0:
            sys.stderr.write(f"== {os.path.basename(src)} {' '.join(extra)}\n{res.stdout}{res.stderr}")
    if failed:
        raise RuntimeError("nvcc failed building libls.so")
    link = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB + ".tmp"]
    link += [u[1] for u in _units()]
    link += ["-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nccl, "lib")]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link of libls.so failed")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
