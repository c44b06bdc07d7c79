"""Build libmlmc.so (sm_100a) in-tree with nvcc.  Used by __graft_entry__.build()."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
SO = os.path.join(HERE, "libmlmc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = (["-DMLMC_TUNING"] if os.environ.get("MLMC_TUNING") == "1" else []) + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-Wno-attributes", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills"]
SOURCES = ["host_kl.cpp", "capi.cu", "controller.cpp", "k_field.cu", "k_minres.cu", "k_minres_tile.cu", "k_minres_gm.cu", "k_minres_stream.cu", "k_mgcg.cu", "k_chol.cu",
           "k_reduce.cu", "k_dd.cu"]


def _needs(obj: str, deps) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Production build.  MLMC_TUNING=1 in the environment also compiles the measured-slower A/B kernel variants
    (env-selected tuning shapes, the global-memory K3 / K3m, the FFMA field kernel) -- tools only; that build
    writes the same libmlmc.so, so rebuild without it before tests or bench."""
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, "internal.h"), os.path.join(HERE, "..", "include", "mlmc.h")]
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _needs(o, [s] + headers):
            lang = [] if src.endswith(".cu") else ["-x", "cu"] if False else []
            jobs.append([NVCC, *ARCH, *FLAGS, *lang, "-c", s, "-o", o])
    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        return r.stdout + r.stderr
    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for out in ex.map(run, jobs):
            if verbose and out.strip():
                print(out)
    objs = [os.path.join(BUILD, s + ".o") for s in SOURCES]
    if force or jobs or not os.path.exists(SO) or _needs(SO, objs):
        run([NVCC, *ARCH, "-shared", "-o", SO, *objs, "-lcudart_static", "-lrt", "-lpthread", "-ldl"])
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
