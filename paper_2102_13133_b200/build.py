"""Builds the sm_100a CUDA library in-tree: paper_2102_13133_b200/libpic_b200.so.

nvcc cross-compiles without a GPU.  Flags:
  -gencode arch=compute_100a,code=sm_100a   B200 only (no multi-arch fatbin)
  --fmad=false                              no FMA contraction: the parity path
                                            keeps the reference's IEEE operation
                                            sequence (proj/src/CMakeLists.txt:20
                                            builds with -ffp-contract=off)
  -lineinfo                                 ncu source mapping
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libpic_b200.so")
BUILD = os.path.join(ROOT, "build", "pic_b200")
# tools-only library with the measured advance_p / sort ablations and timing
# probes (-DPIC_ABLATIONS; PIC_LIB_PATH selects it); never built by the driver
OUT_ABLATE = os.path.join(HERE, "libpic_b200_ablate.so")
BUILD_ABLATE = os.path.join(ROOT, "build", "pic_b200_ablate")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "--fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
                "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-Xcompiler", "-Wall",
                "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _deps():
    return _sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.hpp")) + \
        [os.path.join(ROOT, "include", "pic_b200.h")]


def up_to_date(out: str = OUT) -> bool:
    if not os.path.exists(out):
        return False
    t = os.path.getmtime(out)
    return all(os.path.getmtime(p) <= t for p in _deps())


def build(verbose: bool = False, force: bool = False, ablate: bool = False, defines=(), tag: str = "") -> str:
    """tag + defines: an A/B build (e.g. tag "scalar", defines ["PIC_PACKED=0"])
    into libpic_b200_<tag>.so, selected at run time by PIC_LIB_PATH."""
    out, bdir = (OUT_ABLATE, BUILD_ABLATE) if ablate else (OUT, BUILD)
    if tag:
        out = os.path.join(HERE, f"libpic_b200_{tag}.so")
        bdir = os.path.join(ROOT, "build", f"pic_b200_{tag}")
    if not force and up_to_date(out):
        return out
    os.makedirs(bdir, exist_ok=True)
    srcs = _sources()
    extra = (["-DPIC_ABLATIONS"] if ablate else []) + ["-D" + d for d in defines]

    def compile_one(src):
        obj = os.path.join(bdir, os.path.basename(src) + ".o")
        cmd = [NVCC] + FLAGS + extra + (["-Xptxas", "-v"] if verbose else []) + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(compile_one, srcs))
    tmp = out + ".tmp"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    # python build.py [-v] [-f] [--ablate] [--tag NAME -DNAME=VALUE ...]
    tag = sys.argv[sys.argv.index("--tag") + 1] if "--tag" in sys.argv else ""
    defs = [a[2:] for a in sys.argv if a.startswith("-D")]
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, ablate="--ablate" in sys.argv,
                defines=defs, tag=tag))
