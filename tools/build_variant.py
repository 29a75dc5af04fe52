"""Compile-time A/B variants of the product library: rebuild the named translation units with
extra -D flags, link them with the other units' objects, write build/variants/<name>.so. Load a
variant with FASER_LIB=<path> (engine.lib()). Usage:
  python tools/build_variant.py NAME TU[,TU...] -DMACRO=VALUE [...]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_20503_b200 import build  # noqa: E402


def main():
    name, tus, defs = sys.argv[1], sys.argv[2].split(","), sys.argv[3:]
    build.build_product()  # the base objects are current
    odir = os.path.join(ROOT, "build", "variants", name)
    os.makedirs(odir, exist_ok=True)
    flags = [*build.ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
             "-I", os.path.join(ROOT, "include"), *defs]
    objs = []
    for src in build._sources():
        base = os.path.basename(src)
        if base in tus:
            obj = os.path.join(odir, base + ".o")
            subprocess.run(["nvcc", *flags, "-c", src, "-o", obj], check=True)
        else:
            obj = os.path.join(ROOT, "build", "obj", base + ".o")
        objs.append(obj)
    out = os.path.join(ROOT, "build", "variants", name + ".so")
    subprocess.run(["nvcc", *build.ARCH, "-shared", "-cudart", "static", "-o", out, *objs], check=True)
    print(out)


if __name__ == "__main__":
    main()
