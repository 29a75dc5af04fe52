"""In-tree build of the product library (nvcc, sm_100a) and of the oracle (test infra).

``build_product()`` -> paper_2604_20503_b200/libfaser_b200.so
``build_oracle()``  -> oracle/_build/liboracle.so (+ oracle/_ref/libspecsim_ref.so when
                       /root/reference is present; the GPU box uses the prebuilt copy).
"""
import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libfaser_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _sources():
    csrc = os.path.join(PKG, "csrc")
    return sorted(glob.glob(os.path.join(csrc, "*.cu")) + glob.glob(os.path.join(csrc, "*.cpp")))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_product(force=False, verbose=False):
    srcs = _sources()
    deps = srcs + glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + glob.glob(os.path.join(PKG, "csrc", "*.inc")) + glob.glob(
        os.path.join(ROOT, "include", "faser", "*.h"))
    if not force and not _stale(LIB, deps):
        return LIB
    # one object per translation unit, compiled in parallel and rebuilt only when the unit or
    # any header changed (same flags as a single nvcc invocation; no device linking is needed)
    flags = [*ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
             "-I", os.path.join(ROOT, "include")]
    if verbose:
        flags.insert(0, "-Xptxas=-v")
    odir = os.path.join(ROOT, "build", "obj")
    os.makedirs(odir, exist_ok=True)
    headers = [d for d in deps if d not in srcs]
    objs, jobs = [], []
    for src in srcs:
        obj = os.path.join(odir, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            jobs.append(["nvcc", *flags, "-c", src, "-o", obj])
    procs = []
    for cmd in jobs:
        procs.append((cmd, subprocess.Popen(cmd)))
    failed = [cmd for cmd, p in procs if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, failed[0])
    subprocess.run(["nvcc", *ARCH, "-shared", "-cudart", "static", "-o", LIB + ".tmp", *objs], check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def build_oracle():
    odir = os.path.join(ROOT, "oracle")
    subprocess.run(["make", "-s", "-C", odir, "restated"], check=True)
    if os.path.isdir("/root/reference/proj/core"):
        subprocess.run(["make", "-s", "-C", odir, "ref"], check=True)


if __name__ == "__main__":
    build_oracle()
    print(build_product(force=True))
