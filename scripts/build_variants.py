"""Build A/B variants of libtim.so that differ only in compile-time knobs of one source file
(e.g. correct.cu -DTIM_CORR_MINB=6): the other objects are compiled once and linked into every
variant.  Usage: python scripts/build_variants.py correct.cu name:-DFOO=1,-DBAR=2 name2:...
Outputs paper_2605_14220_b200/libtim_<name>.so (git-ignored; delete after the A/B)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_14220_b200 import build as B  # noqa: E402

OBJ = "/tmp/vb"


def cc(src, out, extra=()):
    cmd = [B.nvcc(), *B.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
           "-I", os.path.join(B.ROOT, "include"), *extra, "-c", os.path.join(B.CSRC, src), "-o", out]
    subprocess.run(cmd, check=True)


def main():
    target = sys.argv[1]
    os.makedirs(OBJ, exist_ok=True)
    others = []
    for s in B.SOURCES:
        if s == target:
            continue
        o = os.path.join(OBJ, s + ".o")
        cc(s, o)
        others.append(o)
    for spec in sys.argv[2:]:
        name, _, flags = spec.partition(":")
        extra = [f for f in flags.split(",") if f]
        o = os.path.join(OBJ, f"{target}.{name}.o")
        cc(target, o, extra)
        lib = os.path.join(B.HERE, f"libtim_{name}.so")
        subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", lib, *others, o, "-ldl"], check=True)
        print(lib)


if __name__ == "__main__":
    main()
