"""Build libccnn.so (sm_100a) in-tree with nvcc.  Used by __graft_entry__.build()."""
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libccnn.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-ffp-contract=off",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
    "-I", os.path.join(ROOT, "include"),
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def build(force=False, verbose=False, variant=None, defines=()):
    """variant: build libccnn_<variant>.so with extra -D defines (experiments only)."""
    global LIB
    if variant:
        saved = LIB
        LIB = os.path.join(PKG, "libccnn_%s.so" % variant)
        try:
            return _build(True, verbose, ["-D" + d for d in defines], "build_" + variant)
        finally:
            LIB = saved
    return _build(force, verbose, [], "build")


def _build(force, verbose, extra, objname):
    srcs = sources()
    deps = srcs + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "ccnn.h"),
                                                          __file__]
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= max(map(os.path.getmtime, deps)):
        return LIB
    objdir = os.path.join(PKG, objname)
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        objs.append(o)
        cmd = [NVCC] + NVCC_FLAGS + extra + ["-c", s, "-o", o]
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    logs = []
    for s, p in procs:
        out = p.communicate()[0].decode()
        logs.append(out)
        if p.returncode != 0:
            sys.stderr.write(out)
            raise RuntimeError("nvcc failed on %s" % s)
    tmp = LIB + ".tmp"
    subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp]
                          + objs)
    os.replace(tmp, LIB)
    with open(os.path.join(objdir, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return LIB


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    if args:   # python build.py <variant> DEFINE1[,DEFINE2 ...] ...
        build(variant=args[0], defines=[d for a in args[1:] for d in a.split(",") if d])
    else:
        build(force="--force" in sys.argv, verbose=True)
