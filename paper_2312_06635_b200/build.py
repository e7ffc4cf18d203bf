"""Build libgla.so (sm_100a) in-tree with nvcc.  Used by __graft_entry__.build() and the tests."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgla.so")
PROBE = os.path.join(HERE, "libgla_probe.so")   # tests only: tcgen05/TMA convention probe
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr",
         "-Xptxas", "-v"]
FLAGS_C = [f for f in FLAGS if f != "-shared"]
OBJ = os.path.join(HERE, "build")
RDC = {"simt.cu"}   # device-side (tail) launches of the exact fallback need relocatable device code


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "probe", "*.cu")) + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(HERE, "..", "include", "gla.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def _headers():
    return glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(HERE, "..", "include", "gla.h")]


def build(force: bool = False, verbose: bool = False) -> str:
    """One object per .cu (compiled in parallel, rebuilt when the source or any header is newer), then one
    shared-library link.  ptxas resource usage of every kernel goes to ptxas_info.txt."""
    if not force and not stale():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    hdr_t = max(os.path.getmtime(h) for h in _headers())
    jobs = []
    for src in sources():
        obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(src), hdr_t):
            rdc = ["-rdc=true"] if os.path.basename(src) in RDC else []
            cmd = [NVCC, *ARCH, *FLAGS_C, *rdc, "-I", os.path.join(HERE, "..", "include"), "-c", "-o", obj, src]
            jobs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    info = {}
    for src, pr in jobs:
        out, err = pr.communicate()
        if pr.returncode != 0:
            sys.stderr.write(out + err)
            raise RuntimeError(f"nvcc failed compiling {os.path.basename(src)}")
        info[src] = err
        with open(os.path.join(OBJ, os.path.basename(src)[:-3] + ".ptxas"), "w") as f:
            f.write(err)
    objs = [os.path.join(OBJ, os.path.basename(s)[:-3] + ".o") for s in sources()]
    res = subprocess.run([NVCC, *ARCH, "-shared", "-rdc=true", "-o", LIB, *objs, "-lcudadevrt"], capture_output=True,
                         text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libgla.so")
    with open(os.path.join(HERE, "ptxas_info.txt"), "w") as f:
        for s in sources():
            pf = os.path.join(OBJ, os.path.basename(s)[:-3] + ".ptxas")
            if os.path.exists(pf):
                f.write(open(pf).read())
    if verbose:
        sys.stderr.write("".join(info.values()))
    probe = [NVCC, *ARCH, *FLAGS, "-o", PROBE, os.path.join(CSRC, "probe", "tc_probe.cu")]
    res = subprocess.run(probe, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libgla_probe.so")
    return LIB


def build_timing() -> str:
    """libgla_timing.so: the same sources with -DGLA_PHASE_TIMING (kernels print per-chunk phase traces)."""
    out = os.path.join(HERE, "libgla_timing.so")
    cmd = [NVCC, *ARCH, *FLAGS, "-rdc=true", "-DGLA_PHASE_TIMING", "-I", os.path.join(HERE, "..", "include"), "-o",
           out, *sources(), "-lcudadevrt"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libgla_timing.so")
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
