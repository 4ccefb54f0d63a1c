"""Build the in-tree C-ABI library libvbddc.so for sm_100a with nvcc (no torch types involved)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libvbddc.so")
SOURCES = ["setup.cu", "dense.cu", "factor.cu", "solve.cu", "vem.cu", "adaptive.cu", "comm.cu", "exchange.cu", "abi.cu"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _defines():
    """Compile-time knobs (e.g. VB_NVCC_DEFINES="-DDOT_BLOCKS_CFG=592 -DGV_WARPS_CFG=8"): part of the
    object directory name, so a build with other knobs never reuses stale objects."""
    d = os.environ.get("VB_NVCC_DEFINES", "").split()
    for f in d:
        if not f.startswith("-D"):
            raise ValueError("VB_NVCC_DEFINES takes -DNAME=VALUE flags only: %r" % f)
    return d


def build(verbose=False, jobs=6):
    nvcc = os.environ.get("NVCC", "nvcc")
    defs = _defines()
    tag = "".join(c if c.isalnum() else "_" for c in "_".join(x[2:] for x in defs))
    objdir = os.path.join(HERE, "build" + ("_" + tag if tag else ""))
    os.makedirs(objdir, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(os.path.dirname(HERE), "include", "vbddc.h"))
    procs, objs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(o)
        if _newer(o, [s] + headers):
            cmd = [nvcc] + FLAGS + defs + ["-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd))
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        while len(procs) >= jobs:
            _wait(procs.pop(0))
    for p in procs:
        _wait(p)
    stamp = os.path.join(HERE, ".libvbddc.defines")
    old = open(stamp).read() if os.path.exists(stamp) else ""
    if _newer(OUT, objs) or old != " ".join(defs):
        cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", OUT] + objs
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
        with open(stamp, "w") as f:
            f.write(" ".join(defs))
    return OUT


def _wait(item):
    src, p = item
    out, _ = p.communicate()
    if p.returncode:
        raise RuntimeError("nvcc failed for %s:\n%s" % (src, out.decode()))
    text = out.decode().strip()
    if text:
        print(text, file=sys.stderr)


if __name__ == "__main__":
    print(build(verbose=True))
