"""Build libwino.so (the C-ABI library) in-tree with nvcc for sm_100a.

Every CUDA translation unit under csrc/ is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo`` and linked into
``paper_1611_06565_b200/libwino.so`` (static cudart).  Rebuilds only what is
out of date (source or header newer than the object).
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
OBJ = PKG / "_obj"
LIB = PKG / "libwino.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=hidden", "-I", str(CSRC), "-I", str(INCLUDE)]
SOURCES = ["plan.cu", "xform_in.cu", "xform_in_const.cu", "xform_in_run.cu", "xform_in_run8.cu", "xform_out.cu", "xform_out_const.cu",
           "xform_out_run.cu", "xform_nd.cu", "xform_mixed.cu", "xform_tiny.cu", "xform_fold.cu", "xform_dfold.cu", "gemm_tc.cu", "gemm_ts2.cu", "gemm_fold.cu", "gemm_f16.cu",
           "gemm_ffma.cu"]


def _headers():
    return list(CSRC.glob("*.h")) + list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh")) + [INCLUDE / "wino.h"]


def build(verbose: bool = False, force: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    hdr_mtime = max(p.stat().st_mtime for p in _headers())
    procs = []
    objs = []
    for src in SOURCES:
        s = CSRC / src
        o = OBJ / (src + ".o")
        objs.append(o)
        if force or not o.exists() or o.stat().st_mtime < max(s.stat().st_mtime, hdr_mtime):
            cmd = [NVCC, *ARCH, *FLAGS, "-c", str(s), "-o", str(o)]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed.append((src, out.decode(errors="replace")))
        elif verbose and out:
            print(out.decode(errors="replace"), file=sys.stderr)
    if failed:
        msg = "\n".join("== %s ==\n%s" % f for f in failed)
        raise RuntimeError("nvcc failed:\n" + msg[-20000:])
    if force or procs or not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        tmp = LIB.with_suffix(".so.tmp%d" % os.getpid())
        cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-cudart", "static"]
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)
