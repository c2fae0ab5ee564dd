"""Build libwq.so in-tree with nvcc for sm_100a (B200).  No JIT, no torch extension:
the C-ABI library is a plain shared object loaded through ctypes."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.environ.get("WQ_CSRC", os.path.join(HERE, "csrc"))    # experiment builds may point elsewhere
# Experiment builds: WQ_VARIANT=<name> WQ_NVCC_DEFS="-DX=1 ..." build and load lib/<name>/libwq.so
# (the same sources with extra defines); unset, the product library lib/libwq.so.
VARIANT = os.environ.get("WQ_VARIANT", "")
EXTRA_DEFS = os.environ.get("WQ_NVCC_DEFS", "").split()
LIBDIR = os.path.join(HERE, "lib", VARIANT) if VARIANT else os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libwq.so")
SOURCES = ["abi.cu", "scores.cu", "assign.cu", "search.cu", "quant.cu", "decode.cu", "decode_tc.cu", "dequant.cu", "unreordered.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-Xptxas", "-v,-warn-spills"]


def _build_id() -> str:
    try:
        return subprocess.check_output(["git", "-C", ROOT, "describe", "--always", "--dirty"],
                                       stderr=subprocess.DEVNULL, text=True).strip()
    except Exception:
        return "nogit"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "wq.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    objdir = os.path.join(LIBDIR, "obj")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, f'-DWQ_BUILD_ID="{_build_id()}"', *EXTRA_DEFS, "-I", os.path.join(ROOT, "include"),
               "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    logs = []
    for src, p in procs:
        out, _ = p.communicate()
        logs.append(f"== {src}\n{out}")
        if p.returncode != 0:
            sys.stderr.write(out)
            raise RuntimeError(f"nvcc failed on {src}")
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"])
    os.replace(tmp, LIB)
    with open(os.path.join(LIBDIR, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return LIB


def build_variant(name: str, defs: str, force: bool = False) -> str:
    """Build lib/<name>/libwq.so with extra nvcc defines (a separate process: the
    variant is chosen by the environment at import).  E.g. the checked build:
    build_variant("checked", "-DWQ_CHECKS=1") (tests/test_gpu_checked.py)."""
    env = dict(os.environ, WQ_VARIANT=name, WQ_NVCC_DEFS=defs)
    args = [sys.executable, "-m", "paper_2605_02262_b200.build"] + (["--force"] if force else [])
    out = subprocess.check_output(args, env=env, cwd=ROOT, text=True)
    return out.strip().splitlines()[-1]


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
