"""Build the in-tree CUDA library libzkl.so for sm_100a (and the C oracle, test infrastructure).

    python -m paper_2404_16109_b200.build        # or __graft_entry__.build()
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libzkl.so")
SOURCES = ["api.cu", "mm_api.cu", "hx_api.cu"]   # compiled in parallel, linked into one .so
DEPS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".h")))   # every source and header
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
def _nccl_include() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        inc = os.path.join(base, "nccl", "include")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    raise RuntimeError("nccl.h not found (nvidia-nccl wheel)")


FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include")]


def _includes(path, seen=None):
    """path and every file it includes with #include "..." (transitively)."""
    import re
    seen = set() if seen is None else seen
    path = os.path.normpath(path)
    if path in seen or not os.path.exists(path):
        return seen
    seen.add(path)
    for m in re.finditer(r'^#include "([^"]+)"', open(path).read(), re.M):
        _includes(os.path.join(os.path.dirname(path), m.group(1)), seen)
    return seen


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in DEPS] + [os.path.join(ROOT, "include", "zkl.h")]
    return any(os.path.getmtime(f) > t for f in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    import concurrent.futures as cf
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I", _nccl_include()]
    cflags = [f for f in FLAGS if f != "-shared"]

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *cflags, *inc, "-c", "-o", obj, os.path.join(CSRC, src)]
        if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(
                os.path.getmtime(f) for f in _includes(os.path.join(CSRC, src))):
            return src, obj, cmd, subprocess.CompletedProcess(cmd, 0, "", "(up to date)\n")
        r = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, cmd, r

    with cf.ThreadPoolExecutor(len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        for src, obj, cmd, r in results:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    for src, obj, cmd, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stderr[-8000:])
            raise RuntimeError(f"nvcc failed on {src} (see {log})")
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB] + [o for _, o, _, _ in results] + ["-ldl"]
    r = subprocess.run(link, capture_output=True, text=True)
    with open(log, "a") as f:
        f.write(" ".join(link) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stderr[-8000:])
        raise RuntimeError(f"link failed (see {log})")
    if verbose:
        for _, _, _, rr in results:
            sys.stderr.write(rr.stderr)
    return LIB


def build_check() -> str:
    """Debug variant libzkl_check.so: the tlookup translation unit compiled with -DZKL_CHECK (device asserts on every
    SoA access and table gather; tools/sanitize_cases.py --check).  Not used by the product path."""
    build()
    objdir = os.path.join(HERE, "build")
    out = os.path.join(HERE, "libzkl_check.so")
    obj = os.path.join(objdir, "api_check.o")
    cflags = [f for f in FLAGS if f != "-shared"]
    subprocess.run([NVCC, *cflags, "-I", _nccl_include(), "-DZKL_CHECK", "-c", "-o", obj, os.path.join(CSRC, "api.cu")],
                   check=True, capture_output=True)
    subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, obj,
                    os.path.join(objdir, "mm_api.o"), os.path.join(objdir, "hx_api.o"), "-ldl"], check=True,
                   capture_output=True)
    return out


def build_variant(name: str, defines) -> str:
    """Experiment variant build/exp_<name>.so: the tlookup translation unit compiled with extra -D flags (timing
    experiments through ZKL_LIB, tools only; never the product path)."""
    build()
    objdir = os.path.join(HERE, "build")
    out = os.path.join(objdir, f"exp_{name}.so")
    cflags = [f for f in FLAGS if f != "-shared"]
    objs = []
    for src in SOURCES:   # every translation unit with the extra flags
        obj = os.path.join(objdir, f"{src[:-3]}_{name}.o")
        subprocess.run([NVCC, *cflags, "-I", _nccl_include(), *defines, "-c", "-o", obj, os.path.join(CSRC, src)],
                       check=True, capture_output=True)
        objs.append(obj)
    subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs, "-ldl"],
                   check=True, capture_output=True)
    return out


if __name__ == "__main__":
    if "--variant" in sys.argv:   # python -m paper_2404_16109_b200.build --variant NAME -DFOO -DBAR=2
        i = sys.argv.index("--variant")
        print(build_variant(sys.argv[i + 1], sys.argv[i + 2:]))
        sys.exit(0)
    if "--check" in sys.argv:
        print(build_check())
        sys.exit(0)
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
