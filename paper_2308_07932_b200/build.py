"""Build libbbf.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo
snapshot to the GPU box).

    python -m paper_2308_07932_b200.build [--force] [-v]
    python -m paper_2308_07932_b200.build --variant NAME -DFLAG ...   (diagnostic builds)

The default build takes no extra flags.  A variant (profiling counters, compile-time knobs) is
built in its own object directory `_build_NAME` into `_build_NAME/libbbf.so`, never over the
default library; load it with BBF_LIB=<path>.  Every object directory keeps a stamp of the
flags it was compiled with, and a flag change forces a rebuild of that directory."""
from __future__ import annotations

import json
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libbbf.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]
SOURCES = ["mem.cu", "graph_build.cu", "plan.cu", "count_sparse.cu", "dense_i8.cu", "estimate.cu", "base.cu", "hybrid.cu", "api.cu"]
HEADERS = ["bbf_internal.cuh"]


def _stale(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, variant: str | None = None,
          extra: list[str] | None = None) -> str:
    """Compile (if stale) and link.  Returns the library path: LIB for the default build,
    `_build_<variant>/libbbf.so` for a variant."""
    bdir = BUILD if not variant else os.path.join(HERE, f"_build_{variant}")
    lib = LIB if not variant else os.path.join(bdir, "libbbf.so")
    extra = list(extra or [])
    os.makedirs(bdir, exist_ok=True)
    stamp = os.path.join(bdir, "flags.json")
    want = {"nvcc": NVCC, "arch": ARCH, "flags": FLAGS, "extra": extra}
    try:
        have = json.load(open(stamp))
    except (OSError, ValueError):
        have = None
    if have != want:
        force = True
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "bbf.h")]
    jobs = []
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(bdir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append((s, o))

    def compile_one(job):
        s, o = job
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", s, "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log = os.path.join(bdir, os.path.basename(o) + ".log")
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {s}:\n{r.stderr[-6000:]}")
        return log

    if jobs and os.path.exists(stamp):
        os.remove(stamp)  # a failed compile must not leave a stamp that vouches for old objects
    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for log in ex.map(compile_one, jobs):
            if verbose:
                print(open(log).read())
    if force or jobs or not os.path.exists(lib) or _stale(lib, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-ldl", "-lpthread", "-lcublas"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    json.dump(want, open(stamp, "w"))
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    variant = None
    if "--variant" in args:
        i = args.index("--variant")
        variant = args[i + 1]
        del args[i:i + 2]
    extra = [a for a in args if a.startswith("-D") or a.startswith("-X")]
    if extra and not variant:
        sys.exit("extra flags need --variant NAME (the default library is always built without them)")
    print(build(force="--force" in args, verbose="-v" in args, variant=variant, extra=extra))
